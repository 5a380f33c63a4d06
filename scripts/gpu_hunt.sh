cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for i in $(seq 1 ${N:-8}); do
  s=$(date +%s)
  WATCHDOG=150 timeout 200 python scripts/bench_watchdog.py --steps 20 --warmup 5 --no-cpu-baseline --no-replay > gpurun_out/hunt$i.json 2> gpurun_out/hunt$i.err
  rc=$?
  python -c "import json; d=json.loads(open('gpurun_out/hunt$i.json').read().strip().splitlines()[-1]); dl=d['decode_loop']; print('run $i rc=$rc', $(date +%s)-$s, 's device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'decode', dl.get('us_per_step', dl), [k for k,v in d['configs'].items() if 'error' in v])" 2>/dev/null || { echo "run $i rc=$rc FAILED after $(( $(date +%s)-s )) s"; grep -v "^\s*$" gpurun_out/hunt$i.err | tail -25; }
done
