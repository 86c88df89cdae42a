# every BASELINE config on the current build + the C2 step breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/config_sweep.sh
timeout 300 python tools/step_breakdown.py --config c2 --steps 20 > gpurun_out/breakdown_c2.txt 2>&1
echo done
