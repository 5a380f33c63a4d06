#!/bin/bash
# compute-sanitizer on a small decode (the smoke case: FMA fp32 MHA + tcgen05 bf16 GQA): memcheck, synccheck, racecheck
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
# larger trees through the fused merge: config B at full size and random trees (memcheck only; slow)
if [ -n "$BIG" ]; then
  timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 7 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "few_shot_full_size or random_trees or fused" > gpurun_out/sanitizer_memcheck_big.log 2>&1
  echo "memcheck big rc=$?"; tail -4 gpurun_out/sanitizer_memcheck_big.log
fi
