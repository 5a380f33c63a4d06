#!/bin/bash
# Round-end evidence (session 2): GPU tests, smoke, the default bench line,
# the reference arm, the launch list of a default step, one full ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final2/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/final2/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/final2/bench_default.json 2> gpurun_out/final2/bench_default.err; echo "bench rc=$?"; tail -c 400 gpurun_out/final2/bench_default.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final2/bench_reference.json 2> gpurun_out/final2/bench_reference.err; echo "ref rc=$?"; tail -c 300 gpurun_out/final2/bench_reference.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"attn_mma|attn_fma|merge_kernel|kv_" -c 256 --csv --log-file gpurun_out/final2/launches_default.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --headline-only > /dev/null 2>&1; echo "ncu list rc=$?"
B="python bench.py --config few_shot --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph --headline-only"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_mma" -s 40 -c 1 -f -o gpurun_out/final2/prof_few_shot $B > gpurun_out/final2/ncu_few_shot.log 2>&1; echo "ncu full rc=$?"
ls gpurun_out/final2
