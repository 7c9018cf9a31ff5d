"""Loaders for the committed golden fixtures (tests/golden/*.npz)."""
import os

import numpy as np

from paper_1911_00675_b200.datagen import CSRBatch

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
WEIGHTED_NAMES = ["pminhash", "probminhash1", "probminhash1a", "probminhash2",
                  "probminhash3", "probminhash3a", "probminhash4"]
UNWEIGHTED_NAMES = ["unweighted1", "unweighted1a", "unweighted2", "unweighted3",
                    "unweighted3a", "unweighted4", "minhash", "superminhash", "oph"]


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def weighted_cases():
    """Yields (case_key, m, batch, algo, sig, stats); sets whose stats[0] == -1
    were not run by the reference (too expensive) and must be skipped."""
    z = load("weighted")
    ci = 0
    while f"c{ci}_ids" in z:
        batch = CSRBatch(z[f"c{ci}_ids"], z[f"c{ci}_w"], z[f"c{ci}_off"], f"c{ci}")
        m = int(z[f"c{ci}_m"])
        for algo in WEIGHTED_NAMES:
            k = f"c{ci}_{algo}_sig"
            if k in z:
                yield f"c{ci}", m, batch, algo, z[k], z[f"c{ci}_{algo}_stats"]
        ci += 1


def unweighted_cases():
    z = load("unweighted")
    ci = 0
    while f"u{ci}_ids" in z:
        batch = CSRBatch(z[f"u{ci}_ids"], None, z[f"u{ci}_off"], f"u{ci}")
        m = int(z[f"u{ci}_m"])
        for algo in UNWEIGHTED_NAMES:
            k = f"u{ci}_{algo}_sig"
            if k in z:
                yield f"u{ci}", m, batch, algo, z[k], z[f"u{ci}_{algo}_stats"]
        ci += 1


def config_cases():
    z = load("configs")
    yield ("c1", 256, CSRBatch(z["c1_ids"], z["c1_w"], z["c1_off"]),
           "probminhash3", z["c1_sig"], z["c1_stats"])
    c2 = CSRBatch(z["c2_ids"], z["c2_w"], z["c2_off"])
    for algo in WEIGHTED_NAMES:
        sig = z[f"c2_{algo}_sig"]
        b = c2 if sig.shape[0] == c2.nsets else c2.subset(np.arange(sig.shape[0]))
        yield "c2", 1024, b, algo, sig, z[f"c2_{algo}_stats"]
    c4 = CSRBatch(z["c4_ids"], z["c4_w"], z["c4_off"])
    for algo in ("probminhash2", "probminhash4"):
        yield "c4", 64, c4, algo, z[f"c4_{algo}_sig"], z[f"c4_{algo}_stats"]
