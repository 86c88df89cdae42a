# ncu --set full of the C4 PCS advance after 20 steps (current build)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 20 -c 1 -o gpurun_out/r02s_pcs python bench.py --config c4_pcs --steps 2 --warmup 20 --no-cpu > gpurun_out/ncu_r02s.log 2>&1
echo done
