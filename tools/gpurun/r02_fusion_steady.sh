# species fusion (two species per launch) vs per-species launches in the steady state
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
L=paper_1606_02862_b200/libkwb200.so
timeout 1500 python tools/ab.py --config c2 --rounds 2 --steps 20 --warmup 40 $L $L@KWB_SPECIES_FUSION=1 > gpurun_out/ab_fusion_steady.txt 2>&1
timeout 1500 python tools/ab.py --config c2 --rounds 1 --steps 20 --warmup 5 $L $L@KWB_SPECIES_FUSION=1 > gpurun_out/ab_fusion_early.txt 2>&1
echo done
