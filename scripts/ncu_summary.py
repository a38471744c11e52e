"""Summarise an `ncu --set full` report into the JSON kept under profiles/.

  python scripts/ncu_summary.py REPORT.ncu-rep OUT.json "capture command"

Reads the raw page (`ncu -i REPORT --page raw --csv`), keeps the metrics
DESIGN.md §6 cites for the first captured launch, and the top warp-stall
reasons from PC sampling."""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "smsp__warps_eligible.avg.per_cycle_active",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__grid_size",
    "launch__block_size",
]


def main():
    rep, out, capture = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(head)}
    res = {"kernel": vals[col["Kernel Name"]]}
    for k in KEEP:
        if k in col:
            res[k] = {"value": vals[col[k]], "unit": units[col[k]]}
    stalls = []
    pre = "smsp__pcsamp_warps_issue_stalled_"
    for h, i in col.items():
        if h.startswith(pre) and not h.endswith("_not_issued") and vals[i]:
            try:
                stalls.append((h[len(pre):], float(vals[i].replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in stalls) or 1.0
    stalls.sort(key=lambda x: -x[1])
    res["pc_sampling_stalls_top"] = [{"reason": r, "share": round(v / tot, 4)} for r, v in stalls[:8]]
    res["capture"] = capture
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
