# PCS back at 2 CTAs/SM (32-record ring) + FFMA box: parity subset, PCS bench, C2 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dense.py tests/test_gpu_random.py tests/test_gpu_scale.py tests/test_gpu_edges.py -q -m gpu --timeout 900 > gpurun_out/pytest_r02l.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02l.log
timeout 600 python bench.py --config c4_pcs --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r02l_pcs.json 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_r02l_c2.json 2>&1
timeout 300 python tools/step_breakdown.py --config c2 --steps 20 > gpurun_out/breakdown_r02l.txt 2>&1
echo done
