"""Device-side RandomnessFailureError (reference loop caps K:279-281 coupon
cap, K:37/K:109/K:150 rejection cap).  The caps are never hit with
splitmix64 at the reference values, so the test lowers them through the
library's test hook (PMH_TEST_COUPON_CAP / PMH_TEST_REJECT_CAP, read once per
process) in a subprocess and checks that the device flag surfaces as
RandomnessFailureError naming the lowest failing set."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))

SCRIPT = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
from paper_1911_00675_b200 import datagen, sketch_batch, RandomnessFailureError
from paper_1911_00675_b200.batch import to_device_f64, to_device_i64, to_device_u64
algo, m = sys.argv[1], int(sys.argv[2])
sizes = [int(v) for v in sys.argv[3].split(",")]
b = datagen.random_sets(17, sizes, "uniform")
out = {}
for path in ("device", "host"):
    try:
        if path == "device":
            sketch_batch(algo, to_device_u64(b.ids), to_device_f64(b.weights),
                         to_device_i64(b.offsets), m)
        else:
            sketch_batch(algo, b.ids, b.weights, b.offsets, m)
        out[path] = "ok"
    except RandomnessFailureError as e:
        out[path] = "randomness: " + str(e)
print(json.dumps(out))
""" % ROOT


def _run(env_extra, algo, m, sizes):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT, algo, str(m), ",".join(map(str, sizes))],
                       capture_output=True, text=True, env=env, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("algo", ["probminhash1", "probminhash1a", "probminhash3", "probminhash3a"])
def test_coupon_cap_raises_with_lowest_failing_set(algo):
    # large sets: every element stays far below 40 points; the singletons at
    # indices 2 and 4 need ~m ln m points in one element and hit the cap
    sizes = [3000, 3000, 1, 3000, 1]
    out = _run({"PMH_TEST_COUPON_CAP": "40"}, algo, 64, sizes)
    for path in ("device", "host"):
        assert out[path].startswith("randomness:"), out
        assert "in set 2" in out[path], out


def test_reject_cap_raises_for_fisher_yates_labels():
    # non-power-of-two m: label draws reject (K:97-110); cap 0 fails at the
    # first rejection of a lane-per-element label
    out = _run({"PMH_TEST_REJECT_CAP": "0"}, "probminhash2", 1000, [3000, 2000, 5000])
    assert out["device"].startswith("randomness:"), out


def test_reference_caps_do_not_fail():
    out = _run({}, "probminhash1", 64, [3000, 3000, 1, 3000, 1])
    assert out == {"device": "ok", "host": "ok"}
