cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02a.jsonl
rm -f $KWB_PARITY_LOG
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_dense.py tests/test_gpu_edges.py -q -m gpu -x --timeout 600 > gpurun_out/pytest_r02a.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02a.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err
echo done
