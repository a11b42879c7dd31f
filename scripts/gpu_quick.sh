#!/bin/bash
# Quick GPU session: smoke, GPU parity tests, bench (tag = output dir).
# Usage (repo root, under gpurun): bash scripts/gpu_quick.sh tag [pytest -k expr]
TAG=${1:-q}; K=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export PSN_WAIT_LIMIT_MS=20000
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
if [ -n "$K" ]; then
  timeout 1200 python -m pytest tests -q -m gpu -x -k "$K" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
else
  timeout 1200 python -m pytest tests -q -m gpu -x --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
fi
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
tail -25 $OUT/pytest_gpu.log
tail -c 3000 $OUT/bench.json; tail -5 $OUT/bench.err
