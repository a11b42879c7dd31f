#!/bin/bash
# Sweep plan knobs (env) on the bench; one JSON summary line per setting.
# Usage: bash scripts/sweep_env.sh <tag> "<ENV1=.. ENV2=..>" ["..."] ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-suite $BENCH_ARGS > $OUT/tmp.json 2>$OUT/tmp.err
  python - "$cfg" $OUT/tmp.json <<'PY' >> $OUT/sweep.txt
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    s=d["step_roofline"]
    print(f'{sys.argv[1]:40s} value={d["value"]:.1f} fwd_ms={s["fwd_ms"]:.4f} bwd_ms={s["bwd_ms"]:.4f} frac={s["frac"]:.3f}')
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
done
cat $OUT/sweep.txt
