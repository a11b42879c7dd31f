#!/bin/bash
# A/B experiment builds (python -m paper_2501_14490_b200._build --variant NAME -D...)
# against the default library on one box, interleaved, two rounds.
# Usage (repo root, under gpurun): bash scripts/variant_bench.sh <tag> name1 name2 ...
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT; : > $OUT/variants.txt
for rep in 1 2; do
  for v in base "$@"; do
    lib=""; [ $v != base ] && lib=$PWD/paper_2501_14490_b200/_lib_$v/libpsn_b200.so
    PSN_B200_LIB=$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-suite > $OUT/tmp.json 2>$OUT/tmp.err
    python - $v $OUT/tmp.json >> $OUT/variants.txt <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); s=d["step_roofline"]
    print(f'{sys.argv[1]:10s} value={d["value"]:.1f} fwd_ms={s["fwd_ms"]:.4f} bwd_ms={s["bwd_ms"]:.4f}')
except Exception as e:
    print(sys.argv[1], "FAILED", e)
PY
  done
done
cat $OUT/variants.txt
