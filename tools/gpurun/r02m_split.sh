# split advance (push_kernel + deposit kernel): tests, then A/B vs fused on C2/C2_f64/C1
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py -x -q -m gpu --timeout 600 > gpurun_out/pytest_r02m.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02m.log
timeout 900 python tools/ab.py --config c2 --rounds 2 --steps 30 paper_1606_02862_b200/libkwb200.so paper_1606_02862_b200/libkwb200.so@KWB_SPLIT=1 > gpurun_out/ab_r02m_c2.txt 2>&1
timeout 600 python tools/ab.py --config c2_f64 --rounds 1 --steps 20 paper_1606_02862_b200/libkwb200.so paper_1606_02862_b200/libkwb200.so@KWB_SPLIT=1 > gpurun_out/ab_r02m_c2f64.txt 2>&1
KWB_SPLIT=1 timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_r02m_split.json 2>gpurun_out/bench_r02m_split.err
KWB_SPLIT=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"push_kernel|advance_kernel" -c 12 --csv --log-file gpurun_out/launches_r02m.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
echo done
