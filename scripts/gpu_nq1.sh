cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TREEATTN_B200_LIB=$PWD/build/variants/nq1.so timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/nq1_pytest.log 2>&1; echo "pytest nq1 rc=$?"; tail -3 gpurun_out/nq1_pytest.log
VARIANTS="base nq1" CFGS="few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard" bash scripts/gpu_ab.sh
