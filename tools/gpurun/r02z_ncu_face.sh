# launch list + ncu of the face-kernel PCS variant
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"advance_kernel|face_deposit" -c 12 --csv --log-file gpurun_out/launches_r02z.csv python bench.py --config c4_pcs --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:advance_kernel --launch-skip 6 -c 1 -o gpurun_out/r02z_face -f python bench.py --config c4_pcs --steps 2 --warmup 6 --no-cpu > gpurun_out/ncu_r02z.log 2>&1
echo done
