"""Host-core scaling of the CPU reference arm (bench.py --impl reference):
the oracle's equal-cost work items (oracle.sketch_csr_balanced) on a
stratified configs[1] sample, 1 thread vs all host threads.  Test
infrastructure (uses the oracle); prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_1911_00675_b200 import datagen  # noqa: E402
import bench  # noqa: E402

target = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
full = datagen.config2()
sub = full.subset(bench._reference_sample(full, target))
cores = bench._cores()
orc.lib()
res = {"sample_sets": sub.nsets, "sample_elements": sub.nelems, "cores": cores}
for th in (1, cores):
    t0 = time.perf_counter()
    bench._oracle_step(orc, sub, th)
    res[f"s_{th}"] = time.perf_counter() - t0
res["speedup"] = res["s_1"] / res[f"s_{cores}"]
print(json.dumps(res))
