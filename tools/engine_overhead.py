"""Per-launch floor of the tcgen05 engine (tiny GEMMs back to back in one graph)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402

for (m, n, k) in ((128, 64, 64), (128, 64, 512), (2048, 64, 64), (2048, 64, 4096)):
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(k, n, device="cuda").bfloat16()
    o = torch.empty(m, n, device="cuda")
    t = timed([lambda: qb.gemm_bf16(a, b, out=o)] * 20, n=5) * 1e3 / 20
    print(f"gemm_bf16 {m}x{n}x{k}: {t:6.2f} us/launch")
x = torch.randn(1 << 20, device="cuda")
t = timed([lambda: x.add_(1.0)] * 20, n=5) * 1e3 / 20
print(f"torch add_ 4 MB: {t:6.2f} us/launch")
