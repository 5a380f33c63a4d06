cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in spec_t64 few_shot spec_t256; do for o in 1 0 1 0; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --headline-only --opt host_q_poll=$o > gpurun_out/qp_$c$o.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/qp_$c$o.json').read().strip().splitlines()[-1]); print('$c poll=$o device', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done; done
