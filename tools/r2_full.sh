# full GPU pass: all gpu tests, bench, configs table
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1; echo "pytest: $(tail -n 1 gpurun_out/f_pytest.log)"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/f_bench.json')); print(round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), {k: round(v,2) for k,v in d['per_variant_ms'].items()})"
timeout 900 python tools/bench_configs.py > gpurun_out/f_configs.jsonl 2> gpurun_out/f_configs.err; echo "configs rc=$?"
python3 -c "
import json
for l in open('gpurun_out/f_configs.jsonl'): d=json.loads(l); print(d.get('config','')[:14], d.get('algo'), round(d.get('ms_min',0),2))
"
