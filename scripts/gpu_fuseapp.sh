cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fuseapp_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/fuseapp_pytest.log
timeout 400 python scripts/decode_kv_append_cost.py 2>&1 | tail -1
for o in 1 0; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --opt fuse_append=$o --no-replay > gpurun_out/fuseapp$o.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/fuseapp$o.json').read().strip().splitlines()[-1]); print('fuse_append=$o headline', round(d['value'],1), 'decode', round(d['decode_loop']['us_per_step'],1), d['decode_loop']['host_prepare_us'])"
done
