"""Per-kernel GPU time of one C3 (LLaMA-7B shapes) QLoRA step (torch profiler, eager, 8 layers)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2305_14314_b200.llama import LlamaConfig, LlamaQLoRA  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 8
cfg = LlamaConfig.llama7b(n_layers=layers)
m = LlamaQLoRA(cfg, seed=0)
g = torch.Generator(device="cuda").manual_seed(0)
tok = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
tgt = torch.randint(0, cfg.vocab, (4, cfg.seq), device="cuda", generator=g)
for _ in range(3):
    m.set_step_constants()
    m.train_step(tok, tgt)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.train_step(tok, tgt)
    torch.cuda.synchronize()
tot = 0
rows = []
for e in prof.key_averages():
    if e.device_type.name == "CUDA" or getattr(e, "self_device_time_total", 0) > 0:
        t = getattr(e, "self_device_time_total", None) or getattr(e, "self_cuda_time_total", 0)
        if t > 0:
            rows.append((t, e.count, e.key))
            tot += t
rows.sort(reverse=True)
print(f"total GPU kernel time {tot / 1e3:.2f} ms for {layers} layers")
for t, c, k in rows[:25]:
    print(f"{t / 1e3:8.3f} ms {100 * t / tot:5.1f}% n={c:4d}  {k[:90]}")
