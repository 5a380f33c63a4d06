#!/bin/bash
# compute-sanitizer on a small decode (the smoke case: FMA fp32 MHA + tcgen05 bf16 GQA): memcheck, synccheck, racecheck
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 7 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitizer_$tool.log
done
