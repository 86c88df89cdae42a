# final build: long-run stability (C2 2000 steps, C4 PCS 300 steps) and validate=True at full size on every config
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python tools/long_run.py --config c2 --steps 2000 --every 200 > gpurun_out/long_run_c2.txt 2>&1
timeout 900 python tools/long_run.py --config c4_pcs --steps 300 --every 50 > gpurun_out/long_run_c4pcs.txt 2>&1
timeout 1800 python tools/validate_sweep.py > gpurun_out/validate_sweep_r02.txt 2>&1
echo done
