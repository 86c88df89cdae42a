# Round-2 evidence on the final build:
#  1 full GPU suite with the parity log      2 the same on the bounds-checked library
#  3 C2 bench (contract line)                 4 reference arm
#  5 ncu launch list of the bench command     6 ncu --set full of the C2 advance
#  7 every config                             8 C2 step breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_final.jsonl
rm -f $KWB_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_final.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_final.log
unset KWB_PARITY_LOG
KWB_LIB_PATH=$PWD/exp/libkwb200_checks.so timeout 3000 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/checks_final.log 2>&1
echo "checks pytest exit $?" >> gpurun_out/checks_final.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final_c2.json 2> gpurun_out/bench_final_c2.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_final_ref.json 2> gpurun_out/bench_final_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launches_final.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance -s 8 -c 1 -o gpurun_out/final_c2_adv -f python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_final_c2.log 2>&1
bash tools/config_sweep.sh
timeout 300 python tools/step_breakdown.py --config c2 --steps 20 > gpurun_out/breakdown_final.txt 2>&1
echo done
