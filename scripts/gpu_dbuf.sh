cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/dbuf_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/dbuf_pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-replay > gpurun_out/dbuf$i.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/dbuf$i.json').read().strip().splitlines()[-1]); print('device', round(d['value'],1), 'per layer', round(d['us_per_layer'],2), 'e2e', round(d['e2e']['value'],1), 'decode', round(d['decode_loop']['us_per_step'],1), {k: round(v['value'],1) for k,v in d['configs'].items()})"
done
