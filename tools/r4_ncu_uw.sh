#!/bin/bash
# ncu captures of unweighted 2 / 4 / 1 on the first 4000 sets of configs[2], summarised on the box
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -f"
for a in ${ALGOS:-unweighted2 unweighted4 unweighted1}; do
  python tools/ncu_driver_cfg.py config3 $a 4096 4000 > /dev/null 2>&1
  timeout 600 $N -k regex:sketch_sets -c 1 -o gpurun_out/uw_$a python tools/ncu_driver_cfg.py config3 $a 4096 4000 > gpurun_out/uw_$a.log 2>&1
done
bash tools/r3_ncu_sum.sh
