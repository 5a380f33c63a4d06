cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/defer_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/defer_pytest.log
VARIANTS="base nodefer" CFGS="few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard" bash scripts/gpu_ab.sh
