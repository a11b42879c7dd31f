#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) on the streamed
# kernels and on the generic kernels (cp.async rings: 16-B pieces at C = 128 /
# 96 / 64, scalar copies at C = 45, k = 16) at BASELINE config 1, T < halo and
# ragged shapes; summary lines to gpurun_out/$TAG.
TAG=${1:-san}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export PSN_WAIT_LIMIT_MS=0   # no watchdog: the tools slow the kernels down by orders of magnitude
for tool in memcheck racecheck synccheck initcheck; do
  for shape in "250 32 128 4 3 stream" "9 16 64 8 3 stream" "300 20 96 4 2 stream" \
               "250 32 128 4 3 generic" "70 6 45 16 2 generic" "9 16 64 8 3 generic"; do
    log=$OUT/${tool}_$(echo $shape | tr ' ' '_').log
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/san_step.py $shape > $log 2>&1
    echo "$tool [$shape] rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> $OUT/summary.txt
  done
done
cat $OUT/summary.txt
