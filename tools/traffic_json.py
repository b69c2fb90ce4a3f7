"""profiles/roofline_traffic.json from the ncu --set full captures of tools/profile_all.sh:
per-launch DRAM bytes (read + write), duration and tensor-pipe activity of each roofline kernel."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
reps = {"fused_fwd_gu": ("prof_fused_gu", 0), "fused_fwd_c2": ("prof_fused_c2", 0), "fused_bwd_c2": ("prof_fused_c2", 1),
        "dequant_c1": ("prof_dequant_c1", 0), "gemv_8192x22016": ("prof_gemv_c4", 0)}


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], v)) for v in r[2:]]


def num(d, k):
    return float(d.get(k, "0").replace(",", "") or 0)


res = {}
for key, (rep, idx) in reps.items():
    path = os.path.join(ROOT, "gpurun_out", rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    d = rows(path)[idx]
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0}
    r = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    units = dict(zip(*list(csv.reader(r.splitlines()))[:2]))
    byt = sum(num(d, k) * scale.get(units.get(k, "byte"), 1.0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = num(d, "gpu__time_duration.sum") * (1e-3 if units.get("gpu__time_duration.sum") == "nsecond" else 1.0)
    res[key] = {"kernel": d["Kernel Name"][:80], "dram_bytes": byt, "duration_us": t,
                "tensor_active_pct": num(d, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                "source": f"ncu capture ({tag})/{rep}.ncu-rep"}
with open(os.path.join(ROOT, "profiles", "roofline_traffic.json"), "w") as fh:
    json.dump(res, fh, indent=1)
print(json.dumps(res, indent=1))
