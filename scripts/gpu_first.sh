#!/bin/bash
# First GPU call of a session: GPU tests, smoke, then the default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout ${TEST_TIMEOUT:-1200} python -m pytest ${TESTS:-tests} -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -30 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
if [ "${BENCH:-1}" = 1 ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench.log; tail -5 gpurun_out/bench.err
fi
