# C2 long run with nvidia-smi sampling (clock / power / temperature drift under sustained load)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 1000 > gpurun_out/smi_longrun.csv 2>&1 &
SMI=$!
timeout 900 python tools/long_run.py --config c2 --steps 3000 --every 250 > gpurun_out/long_run_c2_clk.txt 2>&1
kill $SMI
echo done
