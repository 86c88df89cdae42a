# full GPU suite + compute-sanitizer (racecheck, synccheck, memcheck) on small cases + C2 bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02e.jsonl
rm -f $KWB_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_r02e.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02e.log
for tool in racecheck synccheck memcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_r02e.json 2> gpurun_out/bench_r02e.err
echo done
