export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_L.so
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/fl_pytest.log 2>&1; echo "pytest: $(tail -n 1 gpurun_out/fl_pytest.log)"
grep -E "^FAILED|Error" gpurun_out/fl_pytest.log | head -5
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fl_bench.json 2> gpurun_out/fl_bench.err
python -c "import json; d=json.load(open('gpurun_out/fl_bench.json')); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -3 gpurun_out/fl_bench.err
timeout 900 python tools/bench_configs.py --configs 1,2 > gpurun_out/fl_cfg.jsonl 2> gpurun_out/fl_cfg.err
python3 -c "
import json
for l in open('gpurun_out/fl_cfg.jsonl'): d=json.loads(l); print(d.get('config','')[:12], d.get('algo'), round(d.get('ms_min',0),2))
" || tail -3 gpurun_out/fl_cfg.err
