#!/bin/bash
# ncu --set full of one attention launch (after warm-up) + launch-time list; bench first.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e ${BENCH_ARGS}"
K=${KERNEL:-attn_}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-40} -c 1 -f -o gpurun_out/prof $B > gpurun_out/ncu_full.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:$K -s 32 -c 64 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_list.log 2>&1
tail -3 gpurun_out/ncu_full.log
