# cells sorted by column length (lane balance): parity subset, A/B vs identity (early + steady), imbalance
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_edges.py tests/test_gpu_scale.py tests/test_gpu_split.py -q -m gpu --timeout 900 > gpurun_out/pytest_r02q.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02q.log
L=paper_1606_02862_b200/libkwb200.so
timeout 1200 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 3 exp/libkwb200_nosort.so $L > gpurun_out/ab_r02q_early.txt 2>&1
timeout 1200 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 40 exp/libkwb200_nosort.so $L $L@KWB_SPLIT=1 > gpurun_out/ab_r02q_steady.txt 2>&1
timeout 900 python tools/ab.py --config c4_cic --rounds 1 --steps 20 --warmup 40 exp/libkwb200_nosort.so $L > gpurun_out/ab_r02q_c4cic.txt 2>&1
timeout 600 python tools/imbalance.py --config c2 --steps 60 --every 10 > gpurun_out/imbalance_c2_sort.txt 2>&1
echo done
