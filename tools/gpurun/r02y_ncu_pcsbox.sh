# ncu of the experimental conflict-free PCS box build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 20 -c 1 -o gpurun_out/r02y_pcsbox -f python bench.py --config c4_pcs --steps 2 --warmup 20 --no-cpu > gpurun_out/ncu_r02y.log 2>&1
echo done
