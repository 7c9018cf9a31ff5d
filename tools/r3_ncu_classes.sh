#!/bin/bash
# ncu captures of the ProbMinHash kernels on size classes of configs[1]
mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -f"
python tools/ncu_driver.py probminhash3 1 1 1024 3 >/dev/null 2>&1 && \
  timeout 300 $N -k regex:sketch_flat -c 1 -o gpurun_out/c_flat_tiny python tools/ncu_driver.py probminhash3 1 1 1024 3 > gpurun_out/c1.log 2>&1
timeout 300 $N -k regex:sketch_flat -c 1 -o gpurun_out/c_flat_mid python tools/ncu_driver.py probminhash3 256 1 1024 1023 > gpurun_out/c2.log 2>&1
timeout 300 $N -k regex:sketch_ -c 2 -o gpurun_out/c_pmh1_tiny python tools/ncu_driver.py probminhash1 1 1 1024 7 > gpurun_out/c3.log 2>&1
timeout 300 $N -k regex:sketch_sets -c 1 -o gpurun_out/c_pmh1_mid python tools/ncu_driver.py probminhash1 16 1 1024 63 > gpurun_out/c4.log 2>&1
timeout 300 $N -k regex:sketch_sets -c 1 -o gpurun_out/c_pmh2_mid python tools/ncu_driver.py probminhash2 256 1 1024 1023 > gpurun_out/c5.log 2>&1
ls -la gpurun_out/*.ncu-rep
