#!/bin/bash
# Round-2 (late) profile artifacts: launch list of one bench RL step and one full ncu capture of a
# full-batch verify launch with its per-line stall samples.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/r2k/prof; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches_r2k.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --no-sweep > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:verify_cluster -s 200 -c 1 -o $O/prof_verify_r2k python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra --no-sweep > $O/ncu_full.log 2>&1
ncu -i $O/prof_verify_r2k.ncu-rep --page raw --csv > $O/verify_raw.csv 2>&1
ncu -i $O/prof_verify_r2k.ncu-rep --page source --csv --print-source sass > $O/verify_src.csv 2>&1
ncu -i $O/prof_verify_r2k.ncu-rep --page details --csv > $O/verify_details.csv 2>&1
