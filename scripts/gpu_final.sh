#!/bin/bash
# Round-end evidence: GPU tests, the default bench line (CPU baseline + e2e),
# the reference arm, every config's bench line, ncu captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; tail -2 gpurun_out/final/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; tail -c 600 gpurun_out/final/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; tail -c 400 gpurun_out/final/bench_reference.json
for c in ${CFGS:-demo reasoning spec_t64 spec_t256 few_shot_70b}; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/final/bench_$c.json 2> gpurun_out/final/bench_$c.err
  python -c "import json; d=json.loads(open('gpurun_out/final/bench_$c.json').read().strip().splitlines()[-1]); print('$c', round(d['value'],1), round(d['us_per_layer'],2), round(d['roofline']['frac'],3), d['e2e'] and round(d['e2e']['value'],1))" || tail -3 gpurun_out/final/bench_$c.err
done
for c in few_shot reasoning spec_t64 demo; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_|merge" -s 40 -c 2 -f -o gpurun_out/final/prof_$c $B > gpurun_out/final/ncu_$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_|merge" -s 40 -c 16 --csv --log-file gpurun_out/final/launches_$c.csv $B > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_mma|attn_fma|merge_kernel" -c 256 --csv --log-file gpurun_out/final/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls gpurun_out/final
