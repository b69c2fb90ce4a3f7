"""Summarise an .ncu-rep: duration, DRAM bytes, tensor %, IPC, top stalls, top SASS lines."""
import csv
import subprocess
import sys


def raw(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], v)) for v in r[2:]]


def main(path, top=0):
    for d in raw(path):
        keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
                "l1tex__throughput.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "launch__registers_per_thread", "launch__grid_size"]
        print(d["Kernel Name"][:70])
        for k in keys:
            print(f"  {k} = {d.get(k)}")
        st = sorted(((k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
                     if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")), key=lambda x: -x[1])
        print("  stalls:", st[:7])
    if top:
        out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
        r = list(csv.reader(out.splitlines()))
        hdr = r[1]
        idx = {h: i for i, h in enumerate(hdr)}
        rows = r[2:]
        order = sorted(range(len(rows)), key=lambda i: -int(rows[i][idx["Warp Stall Sampling (All Samples)"]] or 0))
        for i in sorted(order[:top]):
            x = rows[i]
            print(i, x[idx["Warp Stall Sampling (All Samples)"]], x[idx["Instructions Executed"]], x[idx["Source"]][:90])


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
