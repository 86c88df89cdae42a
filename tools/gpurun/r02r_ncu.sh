# ncu --set full of the C2 advance at the steady state (launch 61 = step ~30, species 0) on the current build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 60 -c 1 -o gpurun_out/r02r_c2_steady python bench.py --config c2 --steps 2 --warmup 40 --no-cpu > gpurun_out/ncu_r02r.log 2>&1
echo done
