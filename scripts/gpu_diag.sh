#!/bin/bash
# Diagnostic traces of the attention launch (debug instantiation) per config.
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for c in ${CFGS:-few_shot reasoning}; do
  timeout 300 python scripts/trace_phases.py $c $OPTS > gpurun_out/phases_$c.txt 2>&1; cat gpurun_out/phases_$c.txt | tail -8
  timeout 300 python scripts/trace_mma.py $c $OPTS > gpurun_out/trace_$c.txt 2>&1; head -3 gpurun_out/trace_$c.txt
  timeout 300 python scripts/timeline.py $c $OPTS > gpurun_out/timeline_$c.txt 2>&1; cat gpurun_out/timeline_$c.txt
done
