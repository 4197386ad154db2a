#!/bin/bash
# A/B of library variants on the filtered (top-p) verify: per-call latency and the LC bench line.
#   VARIANTS="base tpu4" OUT=gpurun_out/ab_topp bash scripts/ab_topp.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=${OUT:-gpurun_out/ab_topp}; mkdir -p $O
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then unset BS_LIB_VARIANT; else export BS_LIB_VARIANT=$v; fi
  timeout 300 python scripts/topp_latency.py --ns 1,8,64 > $O/toppl_$v.txt 2>&1
  timeout 600 python bench.py --config lc --steps ${STEPS:-2} --warmup 3 --no-extra --no-sweep --no-cpu-baseline > $O/bench_$v.json 2> $O/bench_$v.err
done
unset BS_LIB_VARIANT
