#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the streamed
# kernels at BASELINE config 1 and at T < halo; summary lines to gpurun_out/$TAG.
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export PSN_WAIT_LIMIT_MS=0   # no watchdog: the tools slow the kernels down by orders of magnitude
for tool in memcheck racecheck synccheck initcheck; do
  for shape in "250 32 128 4 3" "9 16 64 8 3" "300 20 96 4 2"; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_step.py $shape \
      > $OUT/${tool}_$(echo $shape | tr ' ' '_').log 2>&1
    echo "$tool [$shape] rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/${tool}_$(echo $shape | tr ' ' '_').log | tail -1)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
