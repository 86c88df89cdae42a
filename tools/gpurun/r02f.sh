# 1. full GPU suite (floor-free gather, copysign quotients: particles must stay bitwise)
# 2. the same suite on the bounds-checked debug library (compute-sanitizer stand-in)
# 3. negative control: PCS warp boxes without __syncwarp must fail the dense test
# 4. A/B of experiment builds on C2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02f.jsonl
rm -f $KWB_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_r02f.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02f.log
unset KWB_PARITY_LOG
KWB_LIB_PATH=$PWD/exp/libkwb200_checks.so timeout 3000 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/checks_r02f.log 2>&1
echo "checks pytest exit $?" >> gpurun_out/checks_r02f.log
KWB_LIB_PATH=$PWD/exp/libkwb200_noboxsync.so timeout 600 python -m pytest tests/test_gpu_dense.py -q -m gpu -k pcs > gpurun_out/negctl_r02f.log 2>&1
echo "negative-control pytest exit $? (expected nonzero)" >> gpurun_out/negctl_r02f.log
timeout 1200 python tools/ab.py --rounds 2 --steps 20 paper_1606_02862_b200/libkwb200.so exp/libkwb200_earlys0.so exp/libkwb200_oldgather.so > gpurun_out/ab_r02f.txt 2>&1
echo done
