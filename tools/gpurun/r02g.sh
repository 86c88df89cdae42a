# TMA E/B staging + J reduce-add: parity suite, then A/B against KWB_NO_TMA=1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_random.py tests/test_gpu_dense.py tests/test_gpu_edges.py tests/test_gpu_decomp.py -q -m gpu --timeout 900 > gpurun_out/pytest_r02g.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02g.log
timeout 1200 python tools/ab.py --rounds 3 --steps 20 paper_1606_02862_b200/libkwb200.so "paper_1606_02862_b200/libkwb200.so@KWB_NO_TMA=1" > gpurun_out/ab_r02g.txt 2>&1
echo done
