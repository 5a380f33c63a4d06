#!/bin/bash
# A/B of library variants: VARIANTS="base pub1 ..." (base = the in-tree build), CFGS, MARKS=1 for phase marks
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in ${VARIANTS:-base}; do
  if [ "$v" = base ]; then unset TREEATTN_B200_LIB; else export TREEATTN_B200_LIB=$PWD/build/variants/$v.so; fi
  for c in ${CFGS:-few_shot}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e --headline-only ${BENCH_ARGS} > gpurun_out/ab_${v}_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_$c.log').read().strip().splitlines()[-1]); print('$v $c', round(d['value']/d['config']['n_layers'],2), 'us/layer')" 2>/dev/null || tail -3 gpurun_out/ab_${v}_$c.log
    if [ -n "$MARKS" ]; then timeout 300 python scripts/trace_marks.py $c > gpurun_out/marks_${v}_$c.txt 2>&1; sed -n '/critical/,$p' gpurun_out/marks_${v}_$c.txt; fi
  done
done
