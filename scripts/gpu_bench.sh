#!/bin/bash
# Bench + launch list + one full ncu capture of the verify kernel (outputs under gpurun_out/).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-r1c}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_cluster -s 200 -c 1 -o gpurun_out/prof_bench_verify_$TAG python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1
cat MEASURED_PEAKS.json > gpurun_out/peaks.json 2>/dev/null
