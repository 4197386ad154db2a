#!/bin/bash
# Quick GPU check: build, a pytest selection (-k $SEL, default all gpu tests), smoke.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2
TAG=${TAG:-q}
O=gpurun_out/r2/$TAG
python -c "import __graft_entry__ as g; g.build()" > $O.build.log 2>&1
timeout ${TMO:-900} python -m pytest tests -m gpu -x -q ${SEL:+-k "$SEL"} > $O.pytest.log 2>&1; echo "pytest rc=$?" >> $O.pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1; echo "smoke rc=$?" >> $O.smoke.log
