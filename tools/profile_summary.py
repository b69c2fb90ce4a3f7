"""Write a markdown summary of ncu reports + a launch list into profiles/."""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg.per_second"]


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[1], [dict(zip(r[0], v)) for v in r[2:]]


def summarize_rep(path, title):
    units, rows = raw(path)
    hdr = list(rows[0].keys()) if rows else []
    unit = dict(zip(hdr, units))
    lines = [f"### {title}", "", f"source: `{path}` (ncu --set full --clock-control none)", ""]
    for d in rows:
        lines.append(f"kernel: `{d['Kernel Name'][:110]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for k in KEYS:
            lines.append(f"| {k} | {d.get(k)} | {unit.get(k, '')} |")
        st = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
                     if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")), key=lambda x: -x[1])
        lines.append("")
        lines.append("top stall reasons (pc samples): " + ", ".join(f"{k} {int(v)}" for k, v in st[:6]))
        lines.append("")
    return "\n".join(lines)


def summarize_launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    idx = {h: j for j, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[start:]:
        if len(r) != len(hdr):
            continue
        agg.setdefault(r[idx["Kernel Name"]][:90], []).append(float(r[idx["Metric Value"]].replace(",", "")))
    lines = ["### launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench.py --steps 2)", "",
             "cold-cache, serialised per launch: compare shares, not absolutes", "",
             "| launches | mean ns | kernel |", "|---|---|---|"]
    for k, v in agg.items():
        lines.append(f"| {len(v)} | {sum(v) / len(v):.0f} | `{k}` |")
    return "\n".join(lines)


if __name__ == "__main__":
    out, parts = sys.argv[1], []
    for arg in sys.argv[2:]:
        if arg.endswith(".csv"):
            parts.append(summarize_launches(arg))
        else:
            path, title = arg.split("=", 1) if "=" in arg else (arg, arg)
            parts.append(summarize_rep(path, title))
    with open(out, "w") as fh:
        fh.write("\n\n".join(parts) + "\n")
