# lane-balance tail: parity subset on the default build, then A/B of the tail cost (early and steady state)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_edges.py tests/test_gpu_scale.py tests/test_gpu_split.py -q -m gpu --timeout 900 > gpurun_out/pytest_r02o.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02o.log
L=paper_1606_02862_b200/libkwb200.so
timeout 1200 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 3 exp/libkwb200_tail0.so exp/libkwb200_tail2.so $L exp/libkwb200_tail4.so > gpurun_out/ab_r02o_early.txt 2>&1
timeout 1200 python tools/ab.py --config c2 --rounds 1 --steps 20 --warmup 40 exp/libkwb200_tail0.so exp/libkwb200_tail2.so $L exp/libkwb200_tail4.so > gpurun_out/ab_r02o_steady.txt 2>&1
timeout 600 python tools/imbalance.py --config c2 --steps 60 --every 10 > gpurun_out/imbalance_c2_tail.txt 2>&1
echo done
