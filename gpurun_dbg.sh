cd $GRAFT_REPO_ROOT
for d in 0 4 1; do
python scripts/trace_mma.py few_shot debug=$d > gpurun_out/trace_d$d.log 2>&1
echo "debug=$d"; head -1 gpurun_out/trace_d$d.log; grep "item epilogue" gpurun_out/trace_d$d.log | head -4
done
