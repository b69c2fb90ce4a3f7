"""In-process A/B of engine policies on the fused NF4 GEMMs (alternating runs, same box/clocks).
usage: python tools/ab.py "QLRT_STREAMK=0" "QLRT_STREAMK=1" [--shape KxN] [--m M] [--rounds R]"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2305_14314_b200 as qb  # noqa: E402
from tools.bench_mem import timed  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("variants", nargs="+")
ap.add_argument("--shape", default="4096x11008")
ap.add_argument("--m", type=int, default=2048)
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--lora", action="store_true")
a = ap.parse_args()
k, n = (int(v) for v in a.shape.split("x"))
m, r = a.m, 64
w = torch.randn(k, n, device="cuda") * 0.02
q = qb.quantize(w, qb.get_codebook("nf4"), 64, double_quant=True)
x = torch.randn(m, k, device="cuda").bfloat16()
dy = torch.randn(m, n, device="cuda").bfloat16()
ads = [qb.LoraAdapter(r, 16.0, torch.randn(k, r, device="cuda") / 8, torch.randn(r, n, device="cuda") * .01)] \
    if a.lora else []
lin = qb.QLinear(q, ads)
fl = 2 * m * k * n
res = {v: {"fwd": [], "bwd": []} for v in a.variants}


ALL_KEYS = {kv.split("=")[0] for v in a.variants for kv in v.split(",")}


def setenv(v):
    """Exactly this variant's policies (qlrt_set_policy): keys set by other
    variants go back to their defaults."""
    from paper_2305_14314_b200._native import set_policy
    for kk in ALL_KEYS:
        set_policy(kk, None)
    for kv in v.split(","):
        kk, vv = kv.split("=")
        set_policy(kk, int(vv))


for _ in range(a.rounds):
    for v in a.variants:
        setenv(v)
        res[v]["fwd"].append(fl / timed([lambda: lin.forward(x)], n=10) / 1e9)
        _, c = lin.forward(x)
        res[v]["bwd"].append(fl / timed([lambda: lin.backward(dy, c)], n=10) / 1e9)
for v in a.variants:
    print(f"{v:40s} fwd {statistics.median(res[v]['fwd']):7.0f}  bwd {statistics.median(res[v]['bwd']):7.0f} TF/s"
          f"  ({a.shape}, M={m}{', lora' if a.lora else ''})")
