cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TREEATTN_B200_LIB=$PWD/build/variants/direct.so timeout 900 python -m pytest tests -m gpu -x -q -k "parity or decode" > gpurun_out/direct_pytest.log 2>&1; echo "pytest direct rc=$?"; tail -2 gpurun_out/direct_pytest.log
VARIANTS="base direct" CFGS="few_shot reasoning spec_t64 spec_t256 few_shot_70b_shard" bash scripts/gpu_ab.sh
TREEATTN_B200_LIB=$PWD/build/variants/direct.so timeout 200 python scripts/trace_items.py spec_t256 2>&1 | grep -A1 "first switch\|phases"
