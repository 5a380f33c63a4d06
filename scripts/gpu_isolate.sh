#!/bin/bash
# Run every GPU test in its own process (a sticky CUDA error cannot cascade),
# then the first failing one under compute-sanitizer.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -m gpu --collect-only -q -p no:cacheprovider 2>/dev/null | grep '::' > gpurun_out/gpu_ids.txt
: > gpurun_out/isolate.log
first=""
while read id; do
  if timeout 120 python -m pytest "$id" -q -x -p no:cacheprovider > gpurun_out/one.log 2>&1; then
    echo "PASS $id" >> gpurun_out/isolate.log
  else
    echo "FAIL $id" >> gpurun_out/isolate.log
    grep -E "^E " gpurun_out/one.log | head -5 >> gpurun_out/isolate.log
    [ -z "$first" ] && first="$id"
  fi
done < gpurun_out/gpu_ids.txt
if [ -n "$first" ] && [ -n "$SANITIZE" ]; then
  timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest "$first" -q -x -p no:cacheprovider > gpurun_out/sanitizer.log 2>&1
  grep -E "Invalid|misaligned|at 0x|by thread|Address" gpurun_out/sanitizer.log | head -40
fi
cat gpurun_out/isolate.log
if [ -n "$BENCH_ANYWAY" ]; then
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
  tail -c 1500 gpurun_out/bench.log
fi
