#!/bin/bash
# iteration helper: parity tests + per-class timings + bench (no cpu baseline)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_caps.py -q -m gpu -x -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1
echo "pytest: $(tail -n 1 gpurun_out/it_pytest.log)"
grep -E "Error|assert|FAILED" gpurun_out/it_pytest.log | head -10
timeout 600 python tools/profile_classes.py ${VARS:-probminhash1,probminhash3} > gpurun_out/it_classes.log 2>&1
grep -E "sum over|ms=" gpurun_out/it_classes.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/it_bench.json 2>gpurun_out/it_bench.err
python -c "import json; d=json.load(open('gpurun_out/it_bench.json')); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -5 gpurun_out/it_bench.err
