# closing check on the final tree: full GPU suite on the normal and on the bounds-checked library, smoke()
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/pytest_final2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_final2.log
KWB_LIB_PATH=$PWD/exp/libkwb200_checks.so timeout 3000 python -m pytest tests -q -m gpu --timeout 1200 -p no:cacheprovider > gpurun_out/checks_final2.log 2>&1
echo "checks pytest exit $?" >> gpurun_out/checks_final2.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final2.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_final2.log
echo done
