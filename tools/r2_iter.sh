# quick GPU iteration: parity subset + class profile + short bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q -p no:cacheprovider > gpurun_out/it_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/it_pytest.log
tail -3 gpurun_out/it_pytest.log
grep -E "Error|assert|FAILED" gpurun_out/it_pytest.log | head -10
timeout 600 python tools/profile_classes.py ${VARS:-probminhash1,probminhash2,probminhash3,probminhash4} > gpurun_out/it_classes.log 2>&1
grep -E "sum over" gpurun_out/it_classes.log
timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/it_bench.json 2>gpurun_out/it_bench.err
python -c "import json; d=json.load(open('gpurun_out/it_bench.json')); print(round(d['value']/1e9,3), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -5 gpurun_out/it_bench.err
