#!/bin/bash
# One GPU session: smoke, GPU parity tests, bench, ncu launch list + full capture.
# Usage (from repo root, under gpurun): bash scripts/gpu_round.sh [tag]
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.draw --format=csv > $OUT/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 900 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 20 -c 16 --csv \
   --log-file $OUT/launches.csv python bench.py --steps 4 --warmup 5 --no-cpu-baseline --no-e2e --no-suite > $OUT/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fused|fwd_stats|fwd_spike|bwd_reduce|bwd_dx" -s 6 -c 2 \
   -o $OUT/prof python bench.py --steps 2 --warmup 4 --no-cpu-baseline --no-e2e --no-suite > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
tail -3 $OUT/pytest_gpu.log
cat $OUT/bench.json
