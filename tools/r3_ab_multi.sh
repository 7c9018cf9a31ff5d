#!/bin/bash
# bench step per library (LIBS="a.so b.so ..."), 2 alternating rounds
mkdir -p gpurun_out
for i in 1 2; do
for L in $LIBS; do
  PMH_LIB_PATH=$PWD/$L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 ${BARGS:-} > gpurun_out/ab.json 2>gpurun_out/ab.err
  python - "$L" <<'PY'
import json, sys
d = json.load(open("gpurun_out/ab.json"))
print(sys.argv[1].split("/")[-1], round(d["ms_per_step"], 2), {k: round(v, 2) for k, v in d["per_variant_ms"].items()}, d["clocks"].get("sm_mhz"))
PY
done; done
