# why the C2 step time drifts up over thousands of steps: leavers per step, and ncu of the advance at step ~3000
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/long_run.py --config c2 --steps 3000 --every 500 > gpurun_out/long_run_c2_leavers.txt 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 6000 -c 1 -o gpurun_out/r02_drift_step3000 -f python tools/long_run.py --config c2 --steps 3001 --every 3001 > gpurun_out/ncu_drift.log 2>&1
echo done
