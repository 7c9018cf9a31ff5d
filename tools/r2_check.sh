# round-2 GPU check: full gpu suite, bench (config2 + config5), --gpus 2 refusal
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
tail -3 gpurun_out/r2_pytest.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/r2_cfg5.json 2> gpurun_out/r2_cfg5.err; echo "cfg5 rc=$?"
timeout 120 python bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/r2_g2.out 2> gpurun_out/r2_g2.err; echo "gpus2 rc=$?"
