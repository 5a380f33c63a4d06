#!/bin/bash
# Perf round trip: parity (fast), option sweep, ncu launch list of attention kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 200 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
for o in ${SWEEP:-"fma_max_rows=8" "fma_max_rows=1" "fma_max_rows=4"}; do
  OPTS=$(echo $o | tr ',' '\n' | sed 's/^/--opt /' | tr '\n' ' ')
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} $OPTS > gpurun_out/bench_$o.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$o.log').read().strip().splitlines()[-1]); print('$o', round(d['value'],1), 'us/step', round(d['us_per_layer'],2), 'us/layer frac', round(d['roofline']['frac'],3), d['schedule'])" 2>/dev/null || tail -3 gpurun_out/bench_$o.log
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn|merge" -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS} > gpurun_out/ncu_bench.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader(open('gpurun_out/launches.csv')))
agg = collections.defaultdict(list)
for r in rows:
    if r.get('Metric Name') == 'gpu__time_duration.sum':
        agg[r['Kernel Name'][:60]].append(float(r['Metric Value'].replace(',', '')))
for k, v in agg.items():
    print(f"{k:60s} n={len(v)} mean={sum(v)/len(v):.1f} {rows[0].get('Metric Unit','')}")
PY
