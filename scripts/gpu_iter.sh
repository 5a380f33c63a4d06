#!/bin/bash
# One iteration on the GPU box: parity tests (one process each), pipeline
# trace, bench.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash scripts/gpu_isolate.sh > /dev/null 2>&1
grep -c PASS gpurun_out/isolate.log; grep -A3 FAIL gpurun_out/isolate.log | head -20
timeout 300 python scripts/trace_mma.py ${TRACE_CFG:-few_shot} ${TRACE_OPTS} > gpurun_out/trace.log 2>&1
head -${TRACE_LINES:-40} gpurun_out/trace.log
for c in ${BENCH_CFGS:-few_shot}; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$c.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_$c.log').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), 'us/step', round(d['us_per_layer'],2), 'us/layer frac', round(d['roofline']['frac'],3), 'e2e', d['e2e'] and round(d['e2e']['value'],1), d['schedule'])" 2>/dev/null || tail -3 gpurun_out/bench_$c.log
done
if [ -n "$LAUNCHES" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_|merge" -s 64 -c 8 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-graph ${BENCH_ARGS} > /dev/null 2>&1
  python - <<'PY'
import csv
rows = [r for r in csv.DictReader(open('gpurun_out/launches.csv')) if r.get('Metric Name') == 'gpu__time_duration.sum']
for r in rows: print(r['Kernel Name'][:40], r['Metric Value'], r['Metric Unit'])
PY
fi
