#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for v in ${VARIANTS:-light}; do
  export TREEATTN_B200_LIB=$PWD/build/variants/$v.so
  for c in ${CFGS:-few_shot}; do
    timeout 120 python scripts/light_spans.py $c $OPTS > gpurun_out/spans_${v}_$c.txt 2>&1; echo "== $v"; cat gpurun_out/spans_${v}_$c.txt | tail -9
  done
done
