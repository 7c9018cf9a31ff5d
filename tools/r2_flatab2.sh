for L in $LIBS; do
export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/fab2_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/fab2_$L.json')); print('$L', round(d['value']/1e9,3), round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['per_variant_ms'].items()})"
timeout 600 python tools/bench_configs.py --configs 1,3 2>/dev/null > gpurun_out/fab2_cfg_$L.jsonl
python3 -c "
import json
for l in open('gpurun_out/fab2_cfg_$L.jsonl'): d=json.loads(l); print('$L', d.get('config','')[:10], d.get('algo'), round(d.get('ms_min',0),2))
"
done
