# the CPU reference arm (oracle port, all host cores) on every config, for a GPU-vs-CPU table
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in c1 c1_tsc c2 c2_f64 c3 c4_cic c4_tsc c4_pcs c5; do
  timeout 600 python bench.py --impl reference --config $c --steps 5 --warmup 1 > gpurun_out/refsweep_$c.json 2> gpurun_out/refsweep_$c.err
done
nproc > gpurun_out/refsweep_nproc.txt; lscpu | head -20 > gpurun_out/refsweep_lscpu.txt
echo done
