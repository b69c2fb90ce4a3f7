"""A/B the skinny LoRA GEMM shapes of one QLinear step (C2): env variants, per-launch time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402

m, k, n, r = 2048, 4096, 11008, 64
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
l1 = (torch.randn(k, r, device="cuda") / 8).bfloat16()
l2 = (torch.randn(r, n, device="cuda") * .01).bfloat16()
ts = torch.randn(m, 2 * r, device="cuda").bfloat16()
dy_gu = torch.randn(m, 2 * n, device="cuda").bfloat16()
l2_gu = (torch.randn(2 * r, 2 * n, device="cuda") * .01).bfloat16()
dy_o = torch.randn(m, k, device="cuda").bfloat16()
l2_o = (torch.randn(r, k, device="cuda") * .01).bfloat16()
cases = {
    "dT gu = dY l2^T (2048x128x22016)": lambda: qb.gemm_bf16(dy_gu, l2_gu, b_t=True, out_dtype=torch.float32),
    "dT o  = dY l2^T (2048x64x4096)": lambda: qb.gemm_bf16(dy_o, l2_o, b_t=True, out_dtype=torch.float32),
    "Ts = X l1      (2048x64x4096)": lambda: qb.gemm_bf16(x, l1, out_dtype=torch.float32),
    "dT = dY l2^T   (2048x64x11008)": lambda: qb.gemm_bf16(dy, l2, b_t=True, out_dtype=torch.float32),
    "dl2^T = dY^T Ts (11008x128x2048)": lambda: qb.gemm_bf16(dy, ts, a_t=True, out_dtype=torch.float32),
    "dl1 = X^T dT   (4096x128x2048)": lambda: qb.gemm_bf16(x, ts, a_t=True, out_dtype=torch.float32),
}
variants = sys.argv[1:] or ["QLRT_CSPLIT=0", "QLRT_CSPLIT=1"]
for name, fn in cases.items():
    ref = None
    row = []
    for v in variants:
        kk, vv = v.split("=")
        from paper_2305_14314_b200._native import set_policy
        set_policy(kk, int(vv))
        out = fn().clone()
        if ref is None:
            ref = out
        err = ((out - ref).abs().max() / ref.abs().max()).item()
        row.append((timed([fn] * 10, n=10) * 1e3 / 10, err))
    print(f"{name}: " + "   ".join(f"{v} {t:6.1f} us (rel {e:.1e})" for v, (t, e) in zip(variants, row)))
