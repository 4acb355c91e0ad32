"""Summarise an ncu --set full report (raw page) for the judged metrics.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json] [--stalls]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "lts__t_sector_hit_rate.pct",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    path = sys.argv[1]
    hdr, units, data = load(path)
    idx = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in data:
        d = {"kernel": r[idx["Kernel Name"]]}
        for k in KEYS:
            if k in idx:
                d[k] = r[idx[k]] + (" " + units[idx[k]] if units[idx[k]] else "")
        if "--stalls" in sys.argv:
            for h, i in idx.items():
                if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                    try:
                        v = float(r[i])
                    except ValueError:
                        continue
                    if v >= 0.05:
                        d[h.replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", "")] = v
        res.append(d)
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump(res, f, indent=1)
    for d in res:
        print("---", d["kernel"][:90])
        for k, v in d.items():
            if k != "kernel":
                print(f"   {k} = {v}")


if __name__ == "__main__":
    main()
