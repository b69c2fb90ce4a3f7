"""Locate wrong tiles of the fused NF4 GEMM against a torch fp32 reference."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402


def check(m, k, n, r, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn(k, n, device="cuda", generator=g) * 0.02
    q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
    wd = qb.dequantize(q, torch.bfloat16).float()
    x = torch.randn(m, k, device="cuda", generator=g).bfloat16()
    lin = qb.QLinear(q, [])
    y, _ = lin.forward(x)
    ref = x.float() @ wd
    d = (y.float() - ref).abs()
    rel = d / ref.abs().max()
    bad = rel > 1e-2
    print(f"m={m} k={k} n={n}: max-rel {rel.max().item():.3e} bad {int(bad.sum())}")
    if bad.any():
        idx = bad.nonzero()
        toks = idx[:, 0]
        cols = idx[:, 1]
        print("  token tiles", torch.unique(toks // 256).tolist(), "col tiles", torch.unique(cols // 128).tolist())
        print("  cols mod 128 sample", torch.unique(cols % 128)[:20].tolist())
        print("  tokens sample", torch.unique(toks)[:20].tolist())


for shp in [(512, 1024, 2048, 0), (256, 1024, 2048, 0), (512, 512, 2048, 0), (512, 1024, 512, 0), (2048, 4096, 11008, 0)]:
    check(*shp)
