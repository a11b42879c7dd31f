# Launch lists (and optionally one --set full capture) of the generic k=16 path.
OUT=gpurun_out/k16; mkdir -p $OUT
B="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-suite"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l_k16d3.csv python bench.py $B --k 16 --d 3 > $OUT/a.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/l_cifar.csv python bench.py $B --T 32 --B 128 --C 4096 --k 16 --d 1 > $OUT/b.log 2>&1
[ -n "$FULL" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fwd_stats|fwd_spike|bwd_reduce|bwd_dx" -s 12 -c 4 -o $OUT/gen python bench.py $B --k 16 --d 3 > $OUT/c.log 2>&1
echo done
