for V in pminhash,probminhash1 pminhash,probminhash3 pminhash,probminhash4 probminhash3,pminhash; do
for L in J K1; do
PMH_LIB_PATH=paper_1911_00675_b200/libpmh_$L.so timeout 300 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --variants $V > gpurun_out/pmab_$L.json 2>/dev/null
python -c "import json; d=json.load(open('gpurun_out/pmab_$L.json')); print('$V $L', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['per_variant_ms'].items()})"
done; done
