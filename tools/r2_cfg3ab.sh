for L in $LIBS; do
  export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so
  if [ -n "$PARITY" ]; then timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_api.py tests/test_gpu_stats.py -m gpu -x -q -p no:cacheprovider > gpurun_out/e_pytest_$L.log 2>&1; echo "$L pytest: $(tail -n 1 gpurun_out/e_pytest_$L.log)"; fi
  timeout 600 python tools/bench_configs.py --configs ${CFGS:-4} > gpurun_out/e_cfg_$L.jsonl 2> gpurun_out/e_cfg_$L.err; python3 -c "
import json
for l in open('gpurun_out/e_cfg_$L.jsonl'): d=json.loads(l); print('$L', d.get('config','')[:12], d.get('algo'), round(d.get('ms_min',0),2))
" || tail -3 gpurun_out/e_cfg_$L.err
done
