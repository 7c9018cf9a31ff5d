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
# configs[4] end to end (NCCL path) and the ProbMinHash kernels of one step
timeout 600 python bench.py --workload config5 --steps 3 --warmup 1 > gpurun_out/bench_cfg5_$TAG.json 2> gpurun_out/bench_cfg5_$TAG.err
echo "config5 rc=$?"
python tools/ncu_driver_cfg.py config4 probminhash4 64 200000 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sketch_wps -c 1 \
    -f -o gpurun_out/wps_$TAG python tools/ncu_driver_cfg.py config4 probminhash4 64 200000 > gpurun_out/ncu_wps_$TAG.log 2>&1
echo "ncu wps rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"sketch_sets|sketch_small" \
    -f -o gpurun_out/pmh_$TAG python tools/ncu_driver.py probminhash4 > gpurun_out/ncu_pmh_$TAG.log 2>&1
echo "ncu pmh4 rc=$?"
