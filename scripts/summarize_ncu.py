"""Summarise ncu outputs (brought back by gpurun into gpurun_out/) into profiles/.

  python scripts/summarize_ncu.py --launches gpurun_out/launches_r1a.csv \
      --full gpurun_out/prof_bench_verify.ncu-rep --tag r1

Writes profiles/launches_<tag>.md (per-kernel share of device time, cold-cache serialised
launch list), profiles/verify_ncu_<tag>.md (key metrics of one full capture of the verify
kernel) and profiles/verify_traffic.json (dram bytes per launch, read by bench.py).
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        v = float(r[vi].replace(",", ""))
        unit = hdr[vi]
        tot[name] += v
        cnt[name] += 1
    allt = sum(tot.values())
    out = [f"# Launch list summary ({tag})", "",
           f"Source: `{os.path.basename(path)}` — `ncu --metrics gpu__time_duration.sum "
           "--clock-control none` over `bench.py --steps 1 --warmup 0` (first launches of one RL "
           "step: synth bank, pool put, index build, decoding). Serialised, cold-cache: compare "
           "SHARES, not absolute times.", "",
           "| kernel | launches | total (ns) | mean (ns) | share |", "|---|---:|---:|---:|---:|"]
    for name, t in tot.most_common():
        out.append(f"| `{name}` | {cnt[name]} | {t:.0f} | {t / cnt[name]:.0f} | {100 * t / allt:.1f}% |")
    p = os.path.join(PROF, f"launches_{tag}.md")
    open(p, "w").write("\n".join(out) + "\n")
    print(p)


def full(path, tag):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

    def g(name):
        v, u = d.get(name, ("", ""))
        return v, u

    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "launch__shared_mem_per_block_dynamic"]
    stalls = []
    for h in hdr:
        if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                stalls.append((float(d[h][0].replace(",", "")), h.split("stalled_")[-1]))
            except ValueError:
                pass
    st = sum(x for x, _ in stalls) or 1
    out = [f"# verify kernel — one full ncu capture ({tag})", "",
           f"Source: `{os.path.basename(path)}` (`ncu --set full --clock-control none "
           "--import-source on -k regex:verify_cluster -s 200 -c 1` inside `bench.py --steps 1`: a full-batch launch early in the RL step).", "",
           "| metric | value |", "|---|---|"]
    for k in keys:
        v, u = g(k)
        out.append(f"| `{k}` | {v} {u} |")
    out += ["", "Warp stall reasons (share of samples):", ""]
    for x, n in sorted(stalls, reverse=True)[:8]:
        out.append(f"- {n}: {100 * x / st:.1f}%")
    p = os.path.join(PROF, f"verify_ncu_{tag}.md")
    open(p, "w").write("\n".join(out) + "\n")
    print(p)

    def num(k):
        v, u = g(k)
        x = float(v.replace(",", "")) if v else 0.0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return x * scale

    traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
    json.dump({"bytes_per_launch": traffic, "source": os.path.basename(path), "tag": tag},
              open(os.path.join(PROF, "verify_traffic.json"), "w"), indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", default="r1")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        launches(a.launches, a.tag)
    if a.full:
        full(a.full, a.tag)


if __name__ == "__main__":
    sys.exit(main())
