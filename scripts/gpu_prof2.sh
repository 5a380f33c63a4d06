#!/bin/bash
# ncu evidence for the round: full capture of one attention launch + one merge
# launch per config, and the launch list of a bench step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CFGS:-few_shot}; do
  B="python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --headline-only"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_|merge" -s 40 -c 2 -f -o gpurun_out/prof_$c $B > gpurun_out/ncu_$c.log 2>&1
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_|merge" -s 40 -c 16 --csv --log-file gpurun_out/launches_$c.csv $B > /dev/null 2>&1
  tail -2 gpurun_out/ncu_$c.log
done
ls gpurun_out/
