#!/bin/bash
# Round-2 GPU session: build, all GPU tests, smoke, bench (with the sweep), f2 attention bench
# (two head shapes) + ncu, f1 bubble measurement.  Outputs gpurun_out/r2/$TAG.*
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/r2
TAG=${TAG:-x}
O=gpurun_out/r2/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O.gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O.build.log 2>&1
if [ -z "$NOTEST" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O.pytest.log 2>&1; echo "pytest rc=$?" >> $O.pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O.smoke.log 2>&1; echo "smoke rc=$?" >> $O.smoke.log
fi
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > $O.bench.json 2> $O.bench.err; echo "bench rc=$?" >> $O.bench.err
fi
if [ -z "$NOATTN" ]; then
  timeout 300 python scripts/attn_bench.py > $O.attn.json 2>&1
  timeout 300 python scripts/attn_bench.py --heads 32,8 >> $O.attn.json 2>&1
  timeout 300 ncu --set full --import-source on -k regex:unified_attn -c 1 -o $O.attn python scripts/attn_bench.py --iters 1 --warmup 0 > $O.attn_ncu.log 2>&1
fi
if [ -z "$NOBUBBLE" ]; then
  timeout 600 python scripts/bubble_pregen.py --steps 3 > $O.bubble.txt 2>&1
fi
