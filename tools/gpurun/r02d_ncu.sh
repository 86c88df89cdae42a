# C2 bench (no CPU leg) then one full ncu capture of a steady-state advance launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r02d.json 2> gpurun_out/bench_r02d.err || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:advance -s 10 -c 1 \
    -o gpurun_out/r02d_adv -f python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_r02d.log 2>&1
echo done
