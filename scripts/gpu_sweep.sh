#!/bin/bash
# Option sweep on one config: SWEEP="opt=v,opt=v opt=v ..." CFG=few_shot
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for o in ${SWEEP}; do
  OPTS=$(echo $o | tr ',' '\n' | sed 's/^/--opt /' | tr '\n' ' ')
  timeout 300 python bench.py --config ${CFG:-few_shot} --steps 50 --warmup 3 --no-cpu-baseline --no-e2e $OPTS > gpurun_out/sweep.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/sweep.log').read().strip().splitlines()[-1]); print('$o', round(d['value'],1), 'us/step', round(d['us_per_layer'],2), 'us/layer frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -3 gpurun_out/sweep.log
done
