"""Time the fused NF4 fwd GEMM and the plain bf16 engine (K-major B) alone."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402


def timed(fn, n=20):
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(n):
        flush.zero_()
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        tot += a.elapsed_time(b)
    return tot / n


m, k, n = 2048, 4096, 11008
w = torch.randn(k, n, device="cuda") * 0.02
q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
lin = qb.QLinear(q, [])
t = timed(lambda: lin.forward(x))
print(f"PAIR={os.environ.get('QLRT_PAIR')} fused fwd {2*m*k*n/t/1e9:.0f} TF/s ({t*1e3:.1f} us)")
_, c = lin.forward(x)
t = timed(lambda: lin.backward(dy, c))
print(f"PAIR={os.environ.get('QLRT_PAIR')} fused bwd {2*m*k*n/t/1e9:.0f} TF/s ({t*1e3:.1f} us)")
wt = w.t().contiguous().bfloat16()   # [N, K]: K-major B
o = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
t = timed(lambda: qb.gemm_bf16(x, wt, out=o, b_t=True))
print(f"PAIR={os.environ.get('QLRT_PAIR')} plain bf16 (K-major B) {2*m*k*n/t/1e9:.0f} TF/s ({t*1e3:.1f} us)")
w8 = torch.randn(8192, 8192, device="cuda").bfloat16()
x8 = torch.randn(8192, 8192, device="cuda").bfloat16()
o8 = torch.empty(8192, 8192, device="cuda", dtype=torch.bfloat16)
t = timed(lambda: qb.gemm_bf16(x8, w8, out=o8, b_t=True), n=10)
print(f"PAIR={os.environ.get('QLRT_PAIR')} plain bf16 8192^3 {2*8192**3/t/1e9:.0f} TF/s ({t*1e3:.1f} us)")
t = timed(lambda: torch.matmul(x8, w8.t(), out=o8), n=10)
print(f"cuBLAS 8192^3 {2*8192**3/t/1e9:.0f} TF/s")
