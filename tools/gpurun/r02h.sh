# species fusion: GPU suite, then A/B fused vs per-species launches, both with TMA
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
export KWB_PARITY_LOG=$PWD/gpurun_out/parity_r02h.jsonl
rm -f $KWB_PARITY_LOG
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -x > gpurun_out/pytest_r02h.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_r02h.log
unset KWB_PARITY_LOG
timeout 1500 python tools/ab.py --rounds 3 --steps 20 paper_1606_02862_b200/libkwb200.so "paper_1606_02862_b200/libkwb200.so@KWB_PER_SPECIES=1" "paper_1606_02862_b200/libkwb200.so@KWB_NO_TMA=1" > gpurun_out/ab_r02h.txt 2>&1
echo done
