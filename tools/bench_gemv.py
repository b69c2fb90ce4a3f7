"""Batch-1 GEMV (M = 1) at the LLaMA shapes: tensor-core GEMV (QLRT_GEMV_MMA=1)
vs the FHFMA GEMV (=0), no adapter and with LoRA r = 64.  GB/s over the
algorithmic bytes n/2 + nb + 4 n2 + 2K + 2N; graph
replay between L2 flushes, CUDA events."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402

shapes = [(8192, 8192), (8192, 22016), (22016, 8192), (4096, 11008), (4096, 4096)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[1:]]
cb = qb.get_codebook("nf4")
res = {}
for k, n in shapes:
    g = torch.Generator(device="cuda").manual_seed(k + n)
    q = qb.quantize(torch.randn(k, n, device="cuda", generator=g) * 0.02, cb, 64, double_quant=True)
    x = torch.randn(1, k, device="cuda", generator=g).bfloat16()
    nb = k * n // 64
    byt = k * n // 2 + nb + 4 * ((nb + 255) // 256) + 2 * k + 2 * n
    lin0 = qb.QLinear(q, [])
    lin1 = qb.QLinear(q, [qb.LoraAdapter(64, 16.0, torch.randn(k, 64, device="cuda", generator=g) / 8,
                                         torch.randn(64, n, device="cuda", generator=g) * 0.01)])
    row = {"bytes": byt}
    for mma in (1, 0):
        qb.set_policy("QLRT_GEMV_MMA", mma)
        for tag, lin in (("r0", lin0), ("r64", lin1)):
            t = timed([lambda lin=lin: lin.forward(x)], n=20)
            row[f"mma{mma}_{tag}_us"] = round(t * 1e3, 2)
            row[f"mma{mma}_{tag}_gbs"] = round(byt / (t / 1e3) / 1e9, 1)
        y = lin0.forward(x)[0]
        row[f"mma{mma}_y"] = y.float()
    qb.set_policy("QLRT_GEMV_MMA", None)
    d = (row.pop("mma1_y") - row.pop("mma0_y")).abs()
    row["new_vs_old_max_abs"] = d.max().item()
    res[f"{k}x{n}"] = row
    print(f"{k}x{n}", json.dumps(row), flush=True)
