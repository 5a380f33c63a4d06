cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
i=0
while IFS= read -r OPTS; do
  for c in ${CFGS:-spec_t256 reasoning spec_t64}; do
    timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --headline-only $OPTS > gpurun_out/swi_${i}_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/swi_${i}_$c.log').read().strip().splitlines()[-1]); print('[$OPTS] $c', round(d['value']/d['config']['n_layers'],2))" 2>/dev/null || tail -2 gpurun_out/swi_${i}_$c.log
  done
  i=$((i+1))
done <<< "${GRID:-
--opt item_cost_many=800
--opt item_cost_many=1200
--opt item_cost_many=800 --opt many_items=2
--opt item_cost_many=1200 --opt many_items=3
--opt item_cost=500 --opt item_cost_many=1200}"
