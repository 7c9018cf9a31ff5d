# A/B of library builds on the class profile + short bench: LIBS="a b" (paper_1911_00675_b200/libpmh_<x>.so)
mkdir -p gpurun_out
for L in $LIBS; do
  export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so
  if [ -n "$PARITY" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py -m gpu -x -q -p no:cacheprovider > gpurun_out/ab_pytest_$L.log 2>&1; echo "$L pytest: $(tail -1 gpurun_out/ab_pytest_$L.log)"; fi
  if [ -n "$CLASSES" ]; then timeout 600 python tools/profile_classes.py ${VARS:-probminhash1,probminhash2,probminhash3,probminhash4} > gpurun_out/ab_classes_$L.log 2>&1; echo "$L $(grep -E 'sum over' gpurun_out/ab_classes_$L.log | tr '\n' ' ')"; fi
  timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_bench_$L.json 2>gpurun_out/ab_bench_$L.err
  python -c "import json; d=json.load(open('gpurun_out/ab_bench_$L.json')); print('$L', round(d['value']/1e9,3), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -5 gpurun_out/ab_bench_$L.err
done
