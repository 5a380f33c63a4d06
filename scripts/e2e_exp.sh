cd $GRAFT_REPO_ROOT
for e in 0 1 2 3; do
  TA_E2E_EXP=$e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/e2e_exp$e.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/e2e_exp$e.json').read().strip().splitlines()[-1]); print('exp $e device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
