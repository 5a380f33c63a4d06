#!/bin/bash
# ncu --set full capture of the attention kernels (one launch each) + launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
for k in ${KERNELS:-attn_mma attn_fma merge}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 4 -c 1 -f -o gpurun_out/prof_$k $B > gpurun_out/ncu_$k.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn|merge" -c 60 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
for o in ${SWEEP:-"fma_max_rows=8" "fma_max_rows=1"}; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e ${BENCH_ARGS} --opt $o > gpurun_out/bench_$o.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$o.log').read().strip().splitlines()[-1]); print('$o', round(d['value'],1), 'us/step', round(d['us_per_layer'],2), 'us/layer frac', round(d['roofline']['frac'],3), d['schedule'])" 2>/dev/null || tail -3 gpurun_out/bench_$o.log
done
ls -la gpurun_out/
