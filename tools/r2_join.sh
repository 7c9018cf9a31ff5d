timeout 900 python -m pytest tests/test_gpu_join.py tests/test_gpu_pairs_e2e.py tests/test_gpu_stats.py -m gpu -x -q -p no:cacheprovider > gpurun_out/jn_pytest.log 2>&1; echo "pytest: $(tail -n 1 gpurun_out/jn_pytest.log)"
grep -E "^FAILED|Error" gpurun_out/jn_pytest.log | head -5
timeout 600 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/jn_cfg5.json 2> gpurun_out/jn_cfg5.err
python -c "
import json
d=[json.loads(l) for l in open('gpurun_out/jn_cfg5.json') if l.startswith('{')][0]
print(d['value'], d['stage_ms'], d['statistics']['ok'], d['statistics']['max_abs_z_mean'])" || tail -5 gpurun_out/jn_cfg5.err
