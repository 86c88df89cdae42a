# lane balance by ranking x-rows: parity subset + A/B vs identity (early + steady)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_edges.py tests/test_gpu_scale.py -q -m gpu --timeout 900 > gpurun_out/pytest_r02w.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02w.log
L=paper_1606_02862_b200/libkwb200.so
timeout 1500 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 5 exp/libkwb200_norow.so $L > gpurun_out/ab_r02w_early.txt 2>&1
timeout 1500 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 40 exp/libkwb200_norow.so $L > gpurun_out/ab_r02w_steady.txt 2>&1
timeout 900 python tools/ab.py --config c4_tsc --rounds 1 --steps 20 --warmup 40 exp/libkwb200_norow.so $L > gpurun_out/ab_r02w_c4.txt 2>&1
echo done
