mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c2_pytest.log 2>&1; echo "pytest: $(tail -n 1 gpurun_out/c2_pytest.log)"
timeout 900 python tools/bench_configs.py --configs ${CFGS:-1,3} > gpurun_out/c2_cfg.jsonl 2> gpurun_out/c2_cfg.err
python3 -c "
import json
for l in open('gpurun_out/c2_cfg.jsonl'): d=json.loads(l); print(d.get('config','')[:12], d.get('algo'), round(d.get('ms_min',0),2))
" || tail -3 gpurun_out/c2_cfg.err
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err
python -c "import json; d=json.load(open('gpurun_out/c2_bench.json')); print(round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['per_variant_ms'].items()})" || tail -3 gpurun_out/c2_bench.err
