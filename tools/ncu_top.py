"""Top SASS lines of a kernel in an .ncu-rep by stall samples (with their top 2 reasons).
usage: python tools/ncu_top.py rep [N]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, body = None, []
for r in rows:
    if r and r[0] == "Kernel Name":
        h, body = None, []
        continue
    if h is None:
        h = r
        continue
    body.append(r)
iss, ia = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
order = sorted(range(len(body)), key=lambda j: -int(body[j][iss] or 0))
for j in order[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    x = body[j]
    st = sorted(((int(x[i] or 0), h[i][6:]) for i in cols), reverse=True)[:2]
    print(f"{j:5d} {x[0][-5:]} {x[ia]:>8} {x[iss]:>5} {x[1][:64]:64s} {st}")
