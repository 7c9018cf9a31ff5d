for L in A D; do
  export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_stats.py -m gpu -x -q -p no:cacheprovider > gpurun_out/d_pytest_$L.log 2>&1; echo "$L pytest: $(tail -1 gpurun_out/d_pytest_$L.log)"
  timeout 600 python tools/bench_configs.py --configs 3,4 > gpurun_out/d_cfg_$L.jsonl 2> gpurun_out/d_cfg_$L.err; echo "$L"; cat gpurun_out/d_cfg_$L.jsonl | cut -c1-300
done
