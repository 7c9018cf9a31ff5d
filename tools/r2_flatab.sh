for L in $LIBS; do
export PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so
timeout 600 python tools/profile_classes.py probminhash3 > gpurun_out/fab_cls_$L.log 2>&1
echo "$L $(grep -E 'sum over' gpurun_out/fab_cls_$L.log)"; awk '{print $5, $6}' gpurun_out/fab_cls_$L.log | head -8 | tr '\n' ' '; echo
timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --variants probminhash3,probminhash3a,pminhash > gpurun_out/fab_b_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/fab_b_$L.json')); print('$L', {k: round(v,2) for k,v in d['per_variant_ms'].items()})"
timeout 600 python tools/bench_configs.py --configs 1,2 2>/dev/null | python3 -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print('$L', d.get('config','')[:10], d.get('algo'), round(d.get('ms_min',0),2))
" | grep -E "probminhash3$|unweighted3$"
done
