#!/bin/bash
# A/B of library variants (BS_LIB_VARIANT): verify latency vs batch size and the Q7 bench line.
#   VARIANTS="base d8 epi" OUT=gpurun_out/r2k bash scripts/ab_variants.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=${OUT:-gpurun_out/ab}; mkdir -p $O
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then unset BS_LIB_VARIANT; else export BS_LIB_VARIANT=$v; fi
  timeout 300 python scripts/verify_latency.py --ns ${NS:-1,8,64,128,256} > $O/lat_$v.txt 2>&1
  [ -n "$TAIL" ] && timeout 300 python scripts/tail_profile.py --no-events > $O/tail_$v.txt 2>&1
  timeout 600 python bench.py --steps ${STEPS:-3} --warmup 3 --no-extra --no-sweep --no-cpu-baseline > $O/bench_$v.json 2> $O/bench_$v.err
done
unset BS_LIB_VARIANT
