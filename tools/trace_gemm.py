"""Where the fused NF4 GEMM's warp roles wait (QLRT_TRACE build, clock64 totals per CTA).
usage: QLRT_NVCC_EXTRA=-DQLRT_TRACE QLRT_LIB_NAME=libqlrt_trace.so tools/build_lib.sh
       QLRT_LIB_PATH=paper_2305_14314_b200/_lib/libqlrt_trace.so python tools/trace_gemm.py [KxN] [--m M]"""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from paper_2305_14314_b200 import _native  # noqa: E402

NAMES = ["mma_wait_tempty", "mma_wait_full(B)", "mma_wait_afull(deq)", "mma_total", "epi_wait_tfull",
         "epi_drain", "deq_wait_cfull(x8)", "deq_wait_empty(x8)", "deq_total(x8)", "tma_wait_empty",
         "cst_wait_cempty", "tiles", "mma_issue"]
ap = argparse.ArgumentParser()
ap.add_argument("shapes", nargs="*", default=["4096x11008"])
ap.add_argument("--m", type=int, default=2048)
a = ap.parse_args()
lib = _native.lib()
buf = np.zeros((296, 24), dtype=np.uint64)
fetch = lambda: lib.qlrt_trace_fetch(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)))  # noqa: E731
for shp in a.shapes:
    k, n = (int(v) for v in shp.split("x"))
    w = torch.randn(k, n, device="cuda") * 0.02
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    x = torch.randn(a.m, k, device="cuda").bfloat16()
    dy = torch.randn(a.m, n, device="cuda").bfloat16()
    lin = qb.QLinear(q, [])
    for name, fn in (("fwd", lambda: lin.forward(x)), ("bwd", lambda: lin.backward(dy, c))):
        _, c = lin.forward(x)
        fn()
        torch.cuda.synchronize()
        fetch()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        fetch()
        ms = ev[0].elapsed_time(ev[1])
        lead = buf[0::2].astype(np.float64)  # leader CTAs (MMA issuer lives there)
        allc = buf.astype(np.float64)
        tot = lead[:, 3].mean()
        print(f"== {shp} M={a.m} {name}: {ms * 1e3:.1f} us, leader mma_total {tot:.0f} cyc")
        for i, nm in enumerate(NAMES):
            src = lead if i <= 3 or i in (11, 12) else allc
            v = src[:, i]
            v = v[v > 0] if i != 11 else v
            if len(v) == 0:
                continue
            print(f"  {nm:22s} mean {v.mean():12.0f}  max {v.max():12.0f}  ({100 * v.mean() / tot:5.1f}% of mma_total)")
