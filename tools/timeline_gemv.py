"""Kernel timeline (torch profiler) of back-to-back batch-1 GEMV calls."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402

k, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8192x22016").split("x"))
q = qb.quantize(torch.randn(k, n, device="cuda") * 0.02, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(1, k, device="cuda").bfloat16()
lin = qb.QLinear(q, [])
for _ in range(3):
    lin.forward(x)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3):
        lin.forward(x)
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:8.1f} {e['ts'] + e['dur'] - t0:8.1f} {e['dur']:7.1f}  {e['name'][:70]}")
