#!/bin/bash
# Bounded profiling session: pipe microbenchmark, ncu launch list, ncu --set full captures.
# Usage (repo root, under gpurun): bash scripts/gpu_profile.sh [tag] [bench args...]
TAG=${1:-prof}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
BARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-suite $*"
if [ -n "$MICROBENCH" ]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb scripts/microbench_pipes.cu && timeout 60 /tmp/mb > $OUT/microbench.txt 2>&1
fi
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file $OUT/launches.csv python bench.py $BARGS > $OUT/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"psn_stream_kernel" -s 6 -c 2 \
   -o $OUT/prof_stream python bench.py $BARGS > $OUT/ncu_full.log 2>&1
echo "ncu full fused rc=$?" >> $OUT/status.txt
[ -n "$PROFILE_GENERIC" ] && PSN_FORCE_GENERIC=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fwd_stats|fwd_spike|bwd_reduce|bwd_dx" -s 12 -c 4 \
   -o $OUT/prof_generic python bench.py $BARGS > $OUT/ncu_full_generic.log 2>&1
echo "ncu full generic rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
