mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/sw_pytest.log 2>&1; echo "pytest: $(tail -n 1 gpurun_out/sw_pytest.log)"
for f in "" "--no-shared-w"; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 $f > gpurun_out/sw_bench.json 2> gpurun_out/sw_bench.err
python -c "import json; d=json.load(open('gpurun_out/sw_bench.json')); print('$f', round(d['value']/1e9,3), round(d['e2e']['value']/1e9,3), round(d['ms_per_step'],2), round(d['set_weights_ms'],3), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -3 gpurun_out/sw_bench.err
done
timeout 600 python tools/bench_configs.py --configs 4 > gpurun_out/sw_cfg.jsonl 2> gpurun_out/sw_cfg.err
python3 -c "
import json
for l in open('gpurun_out/sw_cfg.jsonl'): d=json.loads(l); print(d.get('config','')[:12], d.get('algo'), round(d.get('ms_min',0),2))
" || tail -3 gpurun_out/sw_cfg.err
