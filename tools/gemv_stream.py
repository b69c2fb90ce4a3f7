"""Batch-1 GEMV GB/s: one launch after an L2 flush ("single") and distinct
weights back to back, > 2x L2 ("stream", the decode regime), r = 0 and 64.
usage: python tools/gemv_stream.py [KxN ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402

HBM = 6550.0
cb = qb.get_codebook("nf4")
for shp in sys.argv[1:] or ["8192x8192", "8192x22016", "22016x8192"]:
    k, n = (int(v) for v in shp.split("x"))
    g = torch.Generator(device="cuda").manual_seed(k + n)
    gb = k * n // 2 + k * n // 64 + 4 * (k * n // 64 // 256) + 2 * k + 2 * n
    reps = max(2, -(-(256 << 20) // gb))
    qs = [qb.quantize(torch.randn(k, n, device="cuda", generator=g) * 0.02, cb, 64, double_quant=True)
          for _ in range(reps)]
    x = torch.randn(1, k, device="cuda", generator=g).bfloat16()
    ad = qb.LoraAdapter(64, 16.0, torch.randn(k, 64, device="cuda", generator=g) / 8,
                        torch.randn(64, n, device="cuda", generator=g) * 0.01)
    out = []
    for tag, ads in (("r0", []), ("r64", [ad])):
        lins = [qb.QLinear(q, ads) for q in qs]
        t1 = timed([lambda: lins[0].forward(x)], n=20)
        ts = timed([(lambda li: (lambda: li.forward(x)))(li) for li in lins], n=10) / reps
        out.append(f"{tag}: single {t1 * 1e3:6.1f} us {gb / t1 / 1e6:6.0f} GB/s | stream {ts * 1e3:6.1f} us "
                   f"{gb / ts / 1e6:6.0f} GB/s ({gb / ts / 1e6 / HBM:.3f})")
    print(f"{shp} x{reps}: " + " || ".join(out), flush=True)
    del qs
    torch.cuda.empty_cache()
