"""Kernel timeline of one QLinear fwd + bwd with a LoRA adapter (torch profiler, CUDA events)."""
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402

k, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "4096x11008").split("x"))
m, r = 2048, 64
w = torch.randn(k, n, device="cuda") * 0.02
q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
lin = qb.QLinear(q, [qb.LoraAdapter(r, 16.0, torch.randn(k, r, device="cuda") / 8,
                                    torch.randn(r, n, device="cuda") * .01)])
for _ in range(3):
    y, c = lin.forward(x)
    lin.backward(dy, c)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2):
        y, c = lin.forward(x)
        lin.backward(dy, c)
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
half = len(ev) // 2
ev = ev[half:]  # second iteration
t0 = ev[0]["ts"]
for e in ev:
    print(f"{e['ts'] - t0:8.1f} {e['ts'] + e['dur'] - t0:8.1f} {e['dur']:7.1f}  s{e['args'].get('stream', '?'):<3} "
          f"g{str(e['args'].get('grid', '')):<14} {e['name'][:60]}")
