#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=${OUT:-gpurun_out/r2k/tr}; mkdir -p $O
python -m paper_2605_08862_b200.build --trace > $O/build_trace.log 2>&1
TRACE_SAVE=$O/ev_bench10.npy TRACE_PHASES=1 TRACE_FLIGHT=1 TRACE_BUSY=1 TRACE_GAPS=1 timeout 300 python scripts/trace_verify.py --bench 10 --iters 3 > $O/trace_bench10.txt 2>&1
TRACE_SAVE=$O/ev_n256.npy TRACE_PHASES=1 TRACE_GAPS=1 timeout 300 python scripts/trace_verify.py --n 256 --iters 4 > $O/trace_n256.txt 2>&1
TRACE_SAVE=$O/ev_live1.npy TRACE_PHASES=1 timeout 300 python scripts/trace_verify.py --n 256 --live 1 --iters 4 > $O/trace_live1.txt 2>&1
if [ -n "$TRACE_DEFS" ]; then
  python -m paper_2605_08862_b200.build --variant trace BS_TRACE $TRACE_DEFS > $O/build_trace2.log 2>&1
  TRACE_SAVE=$O/ev_n256_v.npy TRACE_PHASES=1 TRACE_GAPS=1 timeout 300 python scripts/trace_verify.py --n 256 --iters 4 > $O/trace_n256_v.txt 2>&1
  TRACE_SAVE=$O/ev_live1_v.npy TRACE_PHASES=1 timeout 300 python scripts/trace_verify.py --n 256 --live 1 --iters 4 > $O/trace_live1_v.txt 2>&1
fi
