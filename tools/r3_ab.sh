#!/bin/bash
# A/B: class timings of the default lib vs tools/libpmh_cta.so
mkdir -p gpurun_out
timeout 600 python tools/profile_classes.py ${VARS:-probminhash1} > gpurun_out/ab_a.log 2>&1
PMH_LIB_PATH=$PWD/tools/libpmh_cta.so timeout 600 python tools/profile_classes.py ${VARS:-probminhash1} > gpurun_out/ab_b.log 2>&1
echo "== A (default)"; grep -E "sum over|ms=" gpurun_out/ab_a.log | cut -c1-75
echo "== B (cta)"; grep -E "sum over|ms=" gpurun_out/ab_b.log | cut -c1-75
