import json, os, sys, tempfile
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2305_14314_b200 as qb
from paper_2305_14314_b200.blockquant import quantize_async
x = torch.randn(4096, 4096, device="cuda")
cb = qb.get_codebook("nf4")
for _ in range(3): quantize_async(x, cb, 64, double_quant=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(2): quantize_async(x, cb, 64, double_quant=True)
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json"); prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"]); t0 = ev[0]["ts"]
for e in ev: print(f"{e['ts']-t0:8.1f} {e['dur']:7.1f} {e['name'][:70]}")
