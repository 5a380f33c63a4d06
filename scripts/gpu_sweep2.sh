#!/bin/bash
# option sweep on the product build: per-layer µs for each --opt setting
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${CFGS:-few_shot reasoning}; do
  for o in ${SWEEP}; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --headline-only --opt $o > gpurun_out/sw.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/sw.log').read().strip().splitlines()[-1]); print('$c $o', round(d['us_per_layer'],2))" 2>/dev/null || tail -2 gpurun_out/sw.log
  done
done
