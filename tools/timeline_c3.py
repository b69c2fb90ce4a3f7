"""Kernel timeline of one C3 step (LLaMA-7B shapes, few layers) replayed from
its CUDA graph: per-kernel start / end / stream, and the busy time per kernel
family.  usage: python tools/timeline_c3.py [layers] [grouped 0|1]"""
import collections
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
grouped = bool(int(sys.argv[2])) if len(sys.argv) > 2 else True
cfg = LlamaConfig.llama7b(n_layers=layers)
m = LlamaQLoRA(cfg, seed=0, grouped=grouped)
g = torch.Generator(device="cuda").manual_seed(0)
tok = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
tgt = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        m.set_step_constants()
        m.train_step(tok, tgt)
torch.cuda.current_stream().wait_stream(s)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    m.train_step(tok, tgt)
for _ in range(3):
    gr.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    gr.replay()
    torch.cuda.synchronize()
fn = os.path.join(tempfile.mkdtemp(), "t.json")
prof.export_chrome_trace(fn)
ev = [e for e in json.load(open(fn))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
end = max(e["ts"] + e["dur"] for e in ev)
print(f"step {end - t0:.1f} us, {len(ev)} kernels")
fam = collections.Counter()
for e in ev:
    n = e["name"]
    key = ("fused NF4" if "true, true" in n else "skinny gemm" if "gemm_kernel" in n else
           "splitk reduce" if "splitk" in n else n.split("(")[0].split("<")[0][-40:])
    fam[key] += e["dur"]
for k, v in fam.most_common(20):
    print(f"{v:9.1f} us  {k}")
if os.environ.get("FULL"):
    for e in ev:
        print(f"{e['ts'] - t0:9.1f} {e['ts'] + e['dur'] - t0:9.1f} {e['dur']:7.1f} s{e['args'].get('stream', '?'):<3} "
              f"{e['name'][:70]}")
