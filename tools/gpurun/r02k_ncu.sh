# ncu --set full of the PCS advance (C4) and of the C3-physics advance (128^3 proxy) + C2 breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/step_breakdown.py --config c2 --steps 20 > gpurun_out/breakdown_c2.txt 2>&1
timeout 300 python bench.py --config c4_pcs --steps 3 --warmup 3 --no-cpu > gpurun_out/pcs_plain.json 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance -s 4 -c 1 \
   -o gpurun_out/r02k_pcs -f python bench.py --config c4_pcs --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_r02k_pcs.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:advance -s 8 -c 1 \
   -o gpurun_out/r02k_c3 -f python bench.py --config c3_128 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_r02k_c3.log 2>&1
echo done
