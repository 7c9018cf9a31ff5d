#!/bin/bash
# Full measurement pass for profiles/ (run under gpurun; each ncu pass only
# after the same command exited 0 without ncu):
#   bench (default flags, with cpu_baseline), the reference arm, the per-config
#   table, the serialised launch list of one bench step, and one full ncu
#   capture of the dominant kernel.  Post-process here with
#   tools/launch_table.py and tools/ncu_summary.py.
set -u
mkdir -p gpurun_out
TAG=${TAG:-final}
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
echo "ref rc=$?"; cat gpurun_out/bench_ref_$TAG.json
timeout 900 python tools/bench_configs.py --configs 1,2,3,4,5 > gpurun_out/bench_configs_$TAG.jsonl 2> gpurun_out/bench_configs_$TAG.err
echo "configs rc=$?"
python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 0 --e2e-steps 0 \
    --no-cpu-baseline > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
python tools/ncu_driver.py pminhash > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:pminhash64 -c 1 \
    -f -o gpurun_out/pm64_$TAG python tools/ncu_driver.py pminhash > gpurun_out/ncu_pm64_$TAG.log 2>&1
echo "ncu full rc=$?"
