# parity subset (all failures listed) + A/B of the register-window variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02b.jsonl
rm -f $KWB_PARITY_LOG
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_dense.py tests/test_gpu_edges.py -q -m gpu --timeout 600 > gpurun_out/pytest_r02b.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02b.log
timeout 900 python tools/ab.py --rounds 2 --steps 20 paper_1606_02862_b200/libkwb200.so exp/libkwb200_winsmem.so exp/libkwb200_minb1.so > gpurun_out/ab_r02b.txt 2>&1
echo done
