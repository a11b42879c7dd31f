#!/bin/bash
# A/B the bench on one box: current tree vs the ab_old worktree, interleaved.
OUT=gpurun_out/ab; mkdir -p $OUT; : > $OUT/ab.txt
for rep in 1 2; do
  for side in new old; do
    dir=.; [ $side = old ] && dir=ab_old
    (cd $dir && timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-suite > /tmp/ab.json 2>/tmp/ab.err)
    python - $side /tmp/ab.json >> $OUT/ab.txt <<'PY'
import json,sys
d=json.loads(open(sys.argv[2]).read().strip().splitlines()[-1]); s=d["step_roofline"]
print(f'{sys.argv[1]:4s} value={d["value"]:.1f} fwd_ms={s["fwd_ms"]:.4f} bwd_ms={s["bwd_ms"]:.4f}')
PY
  done
done
cat $OUT/ab.txt
