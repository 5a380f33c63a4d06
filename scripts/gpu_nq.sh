cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TREEATTN_B200_LIB=$PWD/build/variants/nq4.so timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/nq4_pytest.log 2>&1; echo "pytest nq4 rc=$?"; tail -3 gpurun_out/nq4_pytest.log
VARIANTS="nq2 nq4" CFGS="few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard" bash scripts/gpu_ab.sh
