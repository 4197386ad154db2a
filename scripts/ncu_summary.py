"""Markdown summary of one kernel's ncu capture (any kernel), for profiles/.

  python scripts/ncu_summary.py REPORT.ncu-rep --title "..." --source "..." [--bytes B] > profiles/x.md

--bytes: the kernel's algorithmic bytes per launch (adds achieved GB/s and the fraction of
MEASURED_PEAKS.json hbm_gbs).  Under ncu the clocks are ncu's, so the time is indicative only.
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sector_op_read_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--title", required=True)
    ap.add_argument("--source", default="")
    ap.add_argument("--bytes", type=float, default=0.0)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    get = {h: (v, u) for h, v, u in zip(hdr, val, units)}
    print(f"# {a.title}\n")
    if a.source:
        print(f"Source: {a.source}\n")
    print("| metric | value |\n|---|---|")
    for k in KEYS:
        if k in get:
            print(f"| `{k}` | {get[k][0]} {get[k][1]} |")
    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(v or 0) for h, v in zip(hdr, val)
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1.0
    print("\nWarp stall reasons (share of samples):\n")
    for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]:
        print(f"- {k}: {100 * v / tot:.1f}%")
    if a.bytes and "gpu__time_duration.sum" in get:
        t, unit = get["gpu__time_duration.sum"]
        t = float(t) * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit.strip(), 1e-6)
        try:
            peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except (OSError, ValueError, KeyError):
            peak = 6650.0
        gbs = a.bytes / t / 1e9
        print(f"\nAlgorithmic bytes per launch {a.bytes / 1e9:.3f} GB -> {gbs:.0f} GB/s under ncu "
              f"({100 * gbs / peak:.0f} % of the measured {peak:.0f} GB/s; ncu's clocks, indicative only).")


if __name__ == "__main__":
    main()
