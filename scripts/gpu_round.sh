#!/bin/bash
# One GPU session: build, gpu tests, raw verify throughput, bench.  Outputs gpurun_out/r2/$TAG.*
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-x}
O=gpurun_out/r2/$TAG
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build()" > $O.build.log 2>&1
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > $O.pytest.log 2>&1; echo "pytest rc=$?" >> $O.pytest.log
fi
if [ -z "$NOTPUT" ]; then
  BS_FORCE_EAGER=1 timeout 120 python scripts/verify_tput.py --ns 256 > $O.tput.txt 2>&1
  timeout 120 python scripts/verify_tput.py --ns 1,8,64,256 --beta 13.5 >> $O.tput.txt 2>&1
fi
if [ -z "$NOBENCH" ]; then
  timeout 600 python bench.py ${BENCH_ARGS:-} > $O.bench.json 2> $O.bench.err; echo "bench rc=$?" >> $O.bench.err
fi
