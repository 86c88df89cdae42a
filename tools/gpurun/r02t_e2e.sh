# e2e path: batched species uploads, pinned fields; GPU suite subset that loads state; e2e breakdown; bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/pytest_r02t.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02t.log
timeout 800 python tools/e2e_breakdown.py --config c2 > gpurun_out/e2e_breakdown2.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02t.json 2> gpurun_out/bench_r02t.err
echo done
