"""Per-CTA timeline of one batch-1 GEMV launch (QLRT_GEMV_TL build).
usage: QLRT_NVCC_EXTRA=-DQLRT_GEMV_TL QLRT_LIB_NAME=libqlrt_tl.so tools/build_lib.sh
       QLRT_LIB_PATH=paper_2305_14314_b200/_lib/libqlrt_tl.so python tools/gemv_tl.py [KxN ...]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from paper_2305_14314_b200 import _native  # noqa: E402

lib = _native.lib()
SMS = 148
buf = np.zeros(SMS * 16 + 2, dtype=np.uint64)
fetch = lambda: lib.qlrt_gemv_tl_fetch(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)))  # noqa: E731
STREAM = "--stream" in sys.argv  # 3 distinct weights back to back; the timeline of the last launch
for shp in [a for a in sys.argv[1:] if not a.startswith("--")] or ["8192x22016", "8192x8192"]:
    k, n = (int(v) for v in shp.split("x"))
    lins = [qb.QLinear(qb.quantize(torch.randn(k, n, device="cuda") * 0.02, qb.get_codebook("nf4"), 64,
                                   double_quant=True), []) for _ in range(3 if STREAM else 1)]
    x = torch.randn(1, k, device="cuda").bfloat16()
    for _ in range(2):
        for lin in lins:
            lin.forward(x)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()  # replayed like bench.py times it (no host gaps between launches)
    with torch.cuda.graph(g):
        for lin in lins:
            lin.forward(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rep in range(3):
        torch.cuda.synchronize()
        fetch()
        flush.fill_(rep)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        fetch()
    t = buf[:SMS * 16].reshape(SMS, 16).astype(np.int64)
    t = t[t[:, 0] > 0]  # CTAs of this launch (smaller grids leave rows unused)
    ps, pe = int(buf[SMS * 16]), int(buf[SMS * 16 + 1])
    t0 = min(t[:, 0].min(), ps) if ps > 0 else t[:, 0].min()
    rel = lambda v: (v - t0) / 1e3  # noqa: E731
    print(f"== {shp}: event {e0.elapsed_time(e1) * 1e3:.1f} us; prep {rel(ps):.1f}..{rel(pe):.1f} us")
    names = ["entry", "prologue_done", "first_stage", "loop_end", "exit", "wait_full_us", "producer_done"]
    names = list(enumerate(names)) + [(10, "init_synced"), (8, "table_built"), (13, "maxima_reduced"), (11, "ticket_done")]
    for i, nm in names:
        v = t[:, i] / 1e3 if nm == "wait_full_us" else rel(t[:, i])
        print(f"  {nm:14s} min {v.min():7.2f}  med {np.median(v):7.2f}  max {v.max():7.2f}")
    fin = t[:, 12] == 1
    print(f"  finalizers {fin.sum()}: loop_end med {np.median(rel(t[fin, 3])):.2f}, ticket med "
          f"{np.median(rel(t[fin, 11])):.2f}, exit med {np.median(rel(t[fin, 4])):.2f} max {rel(t[fin, 4]).max():.2f}")
    print(f"  units/CTA      min {t[:, 7].min()}  max {t[:, 7].max()}")
