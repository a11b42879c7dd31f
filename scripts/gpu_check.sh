#!/bin/bash
# Bounded GPU session: hangcheck, smoke, GPU parity tests, bench (fused and generic).
# Usage (repo root, under gpurun): bash scripts/gpu_check.sh [tag]
TAG=${1:-check}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/nvsmi.txt 2>&1
timeout 180 python scripts/hangcheck.py > $OUT/hangcheck.log 2>&1; echo "hangcheck rc=$?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
PSN_FORCE_GENERIC=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > $OUT/bench_generic.json 2> $OUT/bench_generic.err; echo "bench generic rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
tail -3 $OUT/hangcheck.log $OUT/smoke.log $OUT/pytest_gpu.log
cat $OUT/bench.json $OUT/bench_generic.json
