# Repeated default bench runs (hang / failure check): each run bounded by timeout
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in $(seq 1 ${N:-4}); do
  s=$(date +%s)
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-replay > gpurun_out/stress$i.json 2> gpurun_out/stress$i.err
  rc=$?
  python -c "import json; d=json.loads(open('gpurun_out/stress$i.json').read().strip().splitlines()[-1]); dl=d['decode_loop']; print('run $i rc=$rc', $(date +%s)-$s, 's device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'decode', dl.get('us_per_step', dl), [k for k,v in d['configs'].items() if 'error' in v])" 2>/dev/null || { echo "run $i rc=$rc FAILED"; tail -5 gpurun_out/stress$i.err; }
done
