"""points_min of SURVEY.md §8d for a config batch (development tool; uses the
CPU oracle, so it is test infrastructure, never the measured path).

points_min(set, variant) = the reference loop's point count when every
stop-limit read is pinned to nextafter(H, +inf), H = the set's final stop
limit: the schedule-free lower bound on the points any exact schedule must
generate.  Written to profiles/points_min_<config>_m<m>.json and read by
bench.py for the per-variant issue-slot roofline.

    python tools/points_min.py [config2] [threads]
"""
import json
import math
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402
from paper_1911_00675_b200 import datagen  # noqa: E402

VARIANTS = ["probminhash1", "probminhash2", "probminhash3", "probminhash4"]


def points_min_batch(algo, m, batch, threads):
    off = batch.offsets
    ns = batch.nsets

    def one(s):
        ids, w = batch.set(s)
        _, _, h = orc.sketch(algo, ids, w, m, want_h=True)
        _, st = orc.sketch(algo, ids, w, m, pin=math.nextafter(h, math.inf))
        return int(st[0])

    with ThreadPoolExecutor(threads) as ex:
        pts = np.array(list(ex.map(one, range(ns))), np.int64)
    return pts


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "config2"
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else (os.cpu_count() or 8)
    if cfg == "config2":
        batch, m = datagen.config2(), 1024
    else:
        raise SystemExit(f"unknown config {cfg}")
    out = {"config": cfg, "m": m, "nsets": batch.nsets, "nelems": batch.nelems,
           "definition": "sum over sets of the oracle's points_generated with every stop-limit "
                         "read pinned to nextafter(H, +inf), H = the set's final stop limit "
                         "(SURVEY.md §8d)", "points_min": {}}
    for v in VARIANTS:
        t = time.time()
        pts = points_min_batch(v, m, batch, threads)
        out["points_min"][v] = int(pts.sum())
        print(v, int(pts.sum()), round(pts.sum() / batch.nelems, 4), "pts/elt",
              round(time.time() - t, 1), "s", flush=True)
    out["points_min"]["probminhash1a"] = out["points_min"]["probminhash1"]
    out["points_min"]["probminhash3a"] = out["points_min"]["probminhash3"]
    out["points_min"]["pminhash"] = int(batch.nelems) * m
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                        f"points_min_{cfg}_m{m}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)


if __name__ == "__main__":
    main()
