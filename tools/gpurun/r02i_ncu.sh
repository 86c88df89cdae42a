# ncu: fused (NS=2) vs per-species (NS=1) advance on C2, key sections only
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --section LaunchStats --section Occupancy --section WarpStateStats --section SpeedOfLight \
   --section InstructionStats --clock-control none -k regex:advance -s 4 -c 1 \
   python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_r02i_fused.txt 2>&1
KWB_PER_SPECIES=1 timeout 600 ncu --section LaunchStats --section Occupancy --section WarpStateStats --section SpeedOfLight \
   --section InstructionStats --clock-control none -k regex:advance -s 8 -c 1 \
   python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_r02i_single.txt 2>&1
echo done
