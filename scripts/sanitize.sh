#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the TINY-sized GPU tests:
# every verify kernel (cluster / split / rows / top-p), fused commit + lookup, graph replay,
# index build and lookup, the 1-rank NCCL exchange.  Output: gpurun_out/r2/sanitize_<tool>.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2/sanitize_build.log 2>&1
SEL=${SEL:-"tiny_rollouts_token_for_token or fused_lookup_matches_separate_lookup_tiny or verify_step_parity or verify_top_p_parity or eos_and_edge or lookup_parity_random_pools or lookup_stale or exchange_one_rank or graph_replay_staleness"}
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout ${TMO:-900} compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_rollout.py tests/test_gpu_parity.py tests/test_gpu_exchange.py \
    -m gpu -q -x -p no:cacheprovider -k "$SEL and not 151936 and not qwen" \
    > gpurun_out/r2/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2/sanitize_$tool.log
  tail -3 gpurun_out/r2/sanitize_$tool.log
done
