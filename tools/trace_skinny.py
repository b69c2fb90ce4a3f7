"""Role-wait trace of the skinny LoRA GEMMs (QLRT_TRACE build; see tools/trace_gemm.py)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from paper_2305_14314_b200 import _native  # noqa: E402

lib = _native.lib()
buf = np.zeros((296, 24), dtype=np.uint64)
fetch = lambda: lib.qlrt_trace_fetch(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)))  # noqa: E731
m, k, n, r = 2048, 4096, 11008, 64
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
l1 = (torch.randn(k, r, device="cuda") / 8).bfloat16()
l2 = (torch.randn(r, n, device="cuda") * .01).bfloat16()
ts = torch.randn(m, 2 * r, device="cuda").bfloat16()
cases = {
    "Ts": lambda: qb.gemm_bf16(x, l1, out_dtype=torch.float32),
    "dT": lambda: qb.gemm_bf16(dy, l2, b_t=True, out_dtype=torch.float32),
    "dl2": lambda: qb.gemm_bf16(dy, ts, a_t=True, out_dtype=torch.float32),
    "dl1": lambda: qb.gemm_bf16(x, ts, a_t=True, out_dtype=torch.float32),
}
names = {0: "mma_wait_tempty", 1: "mma_wait_full", 3: "mma_total", 4: "epi_wait_tfull", 5: "epi_drain",
         9: "tma_wait_empty", 11: "tiles", 12: "mma_issue"}
for nm, fn in cases.items():
    fn()
    torch.cuda.synchronize()
    fetch()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    fn()
    ev[1].record()
    torch.cuda.synchronize()
    fetch()
    print(f"   ({ev[0].elapsed_time(ev[1]) * 1e3:.1f} us incl. reduce)")
    act = buf[buf[:, 3] > 0].astype(np.float64)
    print(f"== {nm}: {len(act)} CTAs")
    for i, s in names.items():
        print(f"  {s:16s} mean {act[:, i].mean():9.0f}  max {act[:, i].max():9.0f}")
