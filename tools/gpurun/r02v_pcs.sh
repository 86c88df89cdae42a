# PCS box: innermost edge loops unrolled (no register rotations): PCS/dense parity subset + A/B on C4 PCS
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_scale.py -q -m gpu -k "pcs or dense or random" --timeout 900 > gpurun_out/pytest_r02v.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02v.log
L=paper_1606_02862_b200/libkwb200.so
timeout 1500 python tools/ab.py --config c4_pcs --rounds 2 --steps 10 --warmup 5 exp/libkwb200_base.so $L > gpurun_out/ab_r02v_pcs.txt 2>&1
echo done
