# split tests (fixed) + lane balance over a C2 run
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py -q -m gpu --timeout 600 > gpurun_out/pytest_r02n.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02n.log
timeout 600 python tools/imbalance.py --config c2 --steps 60 --every 5 > gpurun_out/imbalance_c2.txt 2>&1
echo done
