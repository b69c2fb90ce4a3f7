"""Achievable single-launch floor at C1 sizes: torch fill / copy of the same bytes, timed like bench_mem."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from tools.bench_mem import timed  # noqa: E402

res = {}
for mb in (34, 42, 128, 453):
    n = (mb << 20) // 2
    a = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    b = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    t = timed([lambda: a.fill_(1.0)])
    res[f"fill_{mb}MiB"] = {"us": t * 1e3, "gbs": 2 * n / t / 1e6}
    h = n // 2
    t = timed([lambda: a[:h].copy_(b[:h])])
    res[f"copy_{mb}MiB_total"] = {"us": t * 1e3, "gbs": 2 * n / t / 1e6}
t = timed([lambda: None])
res["empty_graph"] = {"us": t * 1e3}
print(json.dumps(res, indent=1))
