cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/qflag_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/qflag_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --headline-only > gpurun_out/qflag$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/qflag$i.json').read().strip().splitlines()[-1]); print('device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
timeout 200 python scripts/e2e_host.py | tail -2
