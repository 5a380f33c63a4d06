cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
export TREEATTN_B200_LIB=$PWD/build/variants/light.so
for c in ${CFGS:-few_shot reasoning}; do timeout 300 python scripts/cta_variance.py $c > gpurun_out/var_$c.txt 2>&1; cat gpurun_out/var_$c.txt | tail -14; done
