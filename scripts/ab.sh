#!/bin/bash
# A/B on one box: LIBS="a.so b.so" CFGS="few_shot reasoning" OPTS_b="--opt x=1"
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for rep in 1 2; do
for c in ${CFGS:-few_shot}; do
  for l in ${LIBS}; do
    for o in "${AB_OPTS:-}" ; do
      TREEATTN_B200_LIB=$PWD/paper_2404_00242_b200/$l timeout 300 python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --no-e2e $o > gpurun_out/ab.log 2>&1
      python -c "import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$rep $c $l $o', round(d['us_per_layer'],2), 'us/layer')" 2>/dev/null || tail -2 gpurun_out/ab.log
    done
  done
done
done
