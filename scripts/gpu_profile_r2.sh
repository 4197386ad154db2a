#!/bin/bash
# Round-2 profile artifacts: launch list of one bench RL step, one full ncu capture of a
# full-batch verify launch, and compute-sanitizer over the round-2 kernels' tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/prof.build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2/launches_r2.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra > gpurun_out/r2/ncu_launch_r2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:verify_cluster -s 200 -c 1 -o gpurun_out/r2/prof_bench_verify_r2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-extra > gpurun_out/r2/ncu_full_r2.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 \
    python -m pytest tests/test_gpu_attention.py tests/test_gpu_lmhead.py tests/test_gpu_pregen.py tests/test_gpu_parity.py \
    -m gpu -q -p no:cacheprovider -k "not 151936 and (attention or lm_head or lmhead or fused_stats or pregen or bubble or ngram or top_k)" \
    > gpurun_out/r2/sanitize_new_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2/sanitize_new_$tool.log
done
