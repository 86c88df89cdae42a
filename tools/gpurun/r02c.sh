# full GPU suite + BASELINE-scale parity, parity table
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02c.jsonl
rm -f $KWB_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_r02c.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02c.log
echo done
