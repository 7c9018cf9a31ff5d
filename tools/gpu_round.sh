#!/bin/bash
# one GPU round: parity tests, class profile, bench (development helper)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
grep -E "Error|assert|FAILED" gpurun_out/pytest_gpu.log | head -10
if [ "$1" != "notiming" ]; then
timeout 600 python tools/profile_classes.py ${VARS:-pminhash,probminhash1,probminhash2,probminhash3,probminhash4} > gpurun_out/classes.log 2>&1
grep -E "sum over" gpurun_out/classes.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2>gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], {k: round(v,2) for k,v in d['per_variant_ms'].items()}, d['clocks'])" || tail -5 gpurun_out/bench.err
fi
