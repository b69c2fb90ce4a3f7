"""Per-SASS-line execution counts and stall samples of one kernel in an .ncu-rep.
usage: python tools/ncu_src.py rep [kernel-substring] [--top N]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
sections, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r[1], None, []]
        sections.append(cur)
    elif cur is not None and cur[1] is None:
        cur[1] = r
    elif cur is not None:
        cur[2].append(r)
for name, h, body in sections:
    if want not in name:
        continue
    ia, iss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    tot = sum(int(x[ia] or 0) for x in body)
    st = sum(int(x[iss] or 0) for x in body)
    print(f"== {name[:90]}: {tot} warp-instr, {st} samples")
    buckets = Counter()
    for x in body:
        e = int(x[ia] or 0)
        buckets[e] += 1
    for e, n in sorted(buckets.items(), key=lambda t: -t[0] * t[1])[:6]:
        print(f"   {n:5d} instrs executed {e} times each -> {n * e}")
    ops = Counter()
    hot = max(buckets, key=lambda e: e * buckets[e])
    for x in body:
        if int(x[ia] or 0) == hot:
            t = x[1].split()
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += 1
    print("   hottest block mix:", ops.most_common(16))
    cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not" not in c]
    tt = Counter()
    for x in body:
        for i in cols:
            tt[h[i]] += int(x[i] or 0)
    print("   stalls:", tt.most_common(8))
    for x in body:
        if int(x[iss] or 0) > st * 0.02:
            print("   ", x[0][-5:], x[ia], x[iss], x[1][:80])
