# Fit the schedule cost model on the light-trace build, then A/B the fitted
# constants (and a grid) on the product build with the bench.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TREEATTN_B200_LIB=$PWD/build/variants/light.so timeout 600 python scripts/calibrate2.py ${CALCFGS:-few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard} 2>&1 | tee gpurun_out/calibrate2.txt | tail -9
FIT=$(cat gpurun_out/calibrate2_opts.txt 2>/dev/null)
i=0
while IFS= read -r OPTS; do
  [ "$OPTS" = FIT ] && OPTS="$FIT"
  for c in ${CFGS:-few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard}; do
    timeout 300 python bench.py --config $c --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e --headline-only $OPTS > gpurun_out/cal_${i}_$c.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/cal_${i}_$c.log').read().strip().splitlines()[-1]); print('[$OPTS] $c', round(d['value']/d['config']['n_layers'],2), 'us/layer')" 2>/dev/null || tail -3 gpurun_out/cal_${i}_$c.log
  done
  i=$((i+1))
done <<< "${GRID:-
FIT
--opt tile_cost=100 --opt item_cost=500
--opt tile_cost=100 --opt box_cost=20 --opt item_cost=500}"
