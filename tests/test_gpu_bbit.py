"""Packed b-bit signatures on the GPU: fused reduction +
packing against the reference's b-bit vectors (tests/golden/bbit.npz, from
K._k_bbit via estimate.bbit_reduce), and the SWAR all-pairs count against a
brute-force count, for powers of two and odd b."""
import numpy as np
import pytest

from golden_io import load
from paper_1911_00675_b200.batch import (allpairs_bbit_hist_device, bbit_device, bbit_estimate,
                                         bbit_pack_device, bbit_unpack, to_device_u64)

pytestmark = pytest.mark.gpu


def test_pack_matches_reference_bbit():
    z = load("bbit")
    sig = z["sig"]
    for rows in (1, 4):
        t = to_device_u64(sig).view(rows, -1)
        m = t.shape[1]
        for b in (1, 2, 4, 8, 16):
            got = bbit_unpack(bbit_pack_device(t, b).cpu().numpy(), m, b).reshape(-1)
            ref = z[f"bbit_{b}"]
            if rows == 1:
                assert np.array_equal(got, ref), b
            else:  # component index restarts per row
                assert np.array_equal(got, bbit_device(t, b).cpu().numpy().reshape(-1)), b


@pytest.mark.parametrize("b", [1, 3, 5, 8, 13, 16])
def test_pack_equals_unpacked_reduction(b):
    rng = np.random.default_rng(b)
    t = to_device_u64(rng.integers(0, 2**63, size=(37, 129)).astype(np.uint64))
    packed = bbit_pack_device(t, b).cpu().numpy()
    assert np.array_equal(bbit_unpack(packed, 129, b), bbit_device(t, b).cpu().numpy())
    # unused fields / bits stay zero
    fpw = 64 // b
    pv = packed.view(np.uint64)
    if fpw * b < 64:
        assert not (pv >> np.uint64(fpw * b)).any()


@pytest.mark.parametrize("b", [1, 2, 3, 7, 8, 16])
def test_allpairs_bbit_matches_brute_force(b):
    rng = np.random.default_rng(100 + b)
    n, m = 333, 200
    base = rng.integers(0, 2**63, size=(40, m)).astype(np.uint64)
    sig = base[rng.integers(0, 40, size=n)].copy()
    flip = rng.random((n, m)) < 0.3          # correlated rows: many partial matches
    sig[flip] = rng.integers(0, 2**63, size=int(flip.sum())).astype(np.uint64)
    t = to_device_u64(sig)
    comp = bbit_device(t, b).cpu().numpy()
    full = (comp[:, None, :] == comp[None, :, :]).sum(axis=2)
    iu = np.triu_indices(n, 1)
    thr = int(np.percentile(full[iu], 99))
    hist, pairs, k = allpairs_bbit_hist_device(bbit_pack_device(t, b), m, b, threshold=thr)
    np.testing.assert_array_equal(hist.cpu().numpy(), np.bincount(full[iu], minlength=m + 1))
    exp = {(int(i), int(j), int(full[i, j])) for i, j in zip(*iu) if full[i, j] >= thr}
    assert {tuple(map(int, r)) for r in pairs} == exp and k == len(exp)
    # split block rows give the same histogram
    h2 = None
    for r0 in range(0, n, 64):
        h2, _, _ = allpairs_bbit_hist_device(bbit_pack_device(t, b), m, b, r0, min(n, r0 + 64),
                                             r0, n, threshold=m + 1, hist=h2)
    np.testing.assert_array_equal(h2.cpu().numpy(), hist.cpu().numpy())
    est = bbit_estimate(full[iu][:5], m, b)
    assert ((est >= 0) & (est <= 1)).all()
