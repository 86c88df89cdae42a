#!/bin/bash
# Every BASELINE config on one GPU (device-timed bench lines) -> gpurun_out/sweep_<cfg>.json
cd "$(dirname "$0")/.."
for c in c1 c1_tsc c2 c2_f64 c3 c4_cic c4_tsc c4_pcs c5; do
  steps=20; [ "$c" = c2 ] && steps=40; [ "${c:0:2}" = c1 ] && steps=100
  timeout 600 python bench.py --config $c --steps $steps --warmup 3 --no-cpu > gpurun_out/sweep_$c.json 2> gpurun_out/sweep_$c.err
done
timeout 600 python bench.py --config c2 --steps 40 --warmup 3 --no-cpu --zslab > gpurun_out/sweep_c2_zslab.json 2> gpurun_out/sweep_c2_zslab.err
