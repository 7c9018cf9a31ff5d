"""Build libpmh.so in-tree with nvcc for sm_100a.

    python -m paper_1911_00675_b200.build [--force] [--debug]

--debug builds libpmh_debug.so with -DPMH_DEBUG_BOUNDS (device-side index
checks that trap); run the tests against it with PMH_LIB_PATH pointing there.

-fmad=false keeps every device floating-point operation a single IEEE
rounding (the reference has no FMA contraction);
explicit fma() calls in pmh_math.cuh reproduce the host glibc's own FMAs.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpmh.so")
OUT_DEBUG = os.path.join(HERE, "libpmh_debug.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-shared", "-diag-suppress", "177",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.inc"))
                  + [os.path.join(HERE, "..", "include", "pmh.h")])


def needs_build(out: str = OUT) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    out = OUT_DEBUG if debug else OUT
    if not force and not needs_build(out):
        return out
    extra = ["-DPMH_DEBUG_BOUNDS"] if debug else []
    cmd = [NVCC, *NVCC_FLAGS, *extra, "-o", out + ".tmp", os.path.join(CSRC, "pmh_capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, debug="--debug" in sys.argv))
