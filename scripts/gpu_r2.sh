#!/bin/bash
# Round-2 iteration on the GPU box: GPU tests, then an A/B of bench configs.
#   TESTS="tests/test_gpu_configs.py"  CFGS="few_shot reasoning"  AB="fused_merge=0"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ "${TESTS:-all}" != "none" ]; then
  T=${TESTS:-tests}
  timeout ${TEST_TIMEOUT:-1500} python -m pytest $T -m gpu -q -x -p no:cacheprovider --durations=8 > gpurun_out/pytest_gpu.log 2>&1
  tail -15 gpurun_out/pytest_gpu.log
fi
for c in ${CFGS:-few_shot}; do
  for o in "" ${AB}; do
    arg=""; [ -n "$o" ] && arg="--opt $o"
    timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e $arg ${BENCH_ARGS} > gpurun_out/bench_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c [$o]', round(d['value'],1), 'us/step', round(d['us_per_layer'],2), 'us/layer frac', round(d['roofline']['frac'],3), d['roofline']['bound'], 'launches', d['gpu_launches'], d['schedule'])" 2>/dev/null || tail -5 gpurun_out/bench_$c.log
  done
done
for c in ${PHASES}; do
  timeout 300 python scripts/trace_marks.py $c $OPTS > gpurun_out/marks_$c.txt 2>&1; cat gpurun_out/marks_$c.txt
done
