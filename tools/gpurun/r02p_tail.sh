# tail in round-robin order: quick parity subset, A/B of tail cost (steady state), ncu of the tail build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_parity.py -q -m gpu -x --timeout 600 > gpurun_out/pytest_r02p.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02p.log
L=paper_1606_02862_b200/libkwb200.so
timeout 1500 python tools/ab.py --config c2 --rounds 1 --steps 20 --warmup 40 exp/libkwb200_tail0.so exp/libkwb200_tail2.so $L exp/libkwb200_tail4.so exp/libkwb200_tail6.so > gpurun_out/ab_r02p_steady.txt 2>&1
KWB_LIB_PATH=$PWD/exp/libkwb200_tail4.so timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 60 -c 1 -o gpurun_out/r02p_tail4 python bench.py --config c2 --steps 2 --warmup 40 --no-cpu > gpurun_out/ncu_r02p.log 2>&1
echo done
