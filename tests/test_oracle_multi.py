"""Pins of the oracle's multi-label output (oracle_classify_multi; SURVEY.md Sec. 8(f) row f4's optional
half: the original DWM assignment to every bundle within threshold).  Bit b of a fiber's mask
is set iff D_b <= thr_b (D_b: the bundle's minimum Eq. 2 distance), so the closest-bundle label is the
argmin of D_b over the set bits; bits within the 1e-3 mm band of their threshold are flagged ambiguous."""
import numpy as np
import pytest

import oracle
from seg_testutil import fiber_A
from synth import atlas_for_config, fibers_for_config


def test_multi_constructed():
    a = fiber_A()[None]
    cents = np.stack([fiber_A() + np.float32([3, 0, 0]),       # bundle 0 at 3 (thr 4): set
                      fiber_A() + np.float32([0, 5, 0]),       # bundle 1 at 5 (thr 6): set
                      fiber_A() + np.float32([0, 0, 7]),       # bundle 2 at 7 (thr 6): not set
                      fiber_A() + np.float32([2, 0, 0]),       # bundle 3 at exactly its thr 2: set
                      fiber_A() + np.float32([0, 2 + 2 ** -11, 0])])   # bundle 4 just above thr 2: unset, ambiguous
    bid = np.arange(5, dtype=np.int32)
    thr = np.array([4, 6, 6, 2, 2], np.float32)
    r = oracle.classify_multi(a, cents, bid, thr)
    assert r["mask"].shape == (1, 1)
    assert r["mask"][0, 0] == 0b01011
    assert r["amb"][0, 0] == 0b11000        # bundle 3 (d = thr) and bundle 4 (thr + 2^-11) lie in the band


def test_multi_brute_force_and_single_label():
    """Against a numpy brute force on 300 cfg-0 fibers, and consistent with the closest-bundle label."""
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 300)
    r = oracle.classify_multi(fib, at.centroids, at.bundle_id, at.thresh)
    s = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, want_d2b=True)
    d = np.sqrt(s["d2b"])                                            # [n, B]
    want = d <= at.thresh[None, :].astype(np.float64)
    bits = (r["mask"][:, 0][:, None] >> np.arange(at.B)[None, :]) & 1
    assert np.array_equal(bits.astype(bool), want)
    lab = s["label"]
    for i in range(fib.shape[0]):
        if lab[i] >= 0:
            assert bits[i, lab[i]] == 1
            assert lab[i] == np.nonzero(bits[i])[0][np.argmin(d[i][bits[i] == 1])]
        elif s["decidable"][i]:
            assert bits[i].sum() == 0


def test_multi_wide_masks_and_non_finite():
    """100 bundles (cfg 1): four 32-bit words; a non-finite fiber is unassigned (all zero)."""
    at = atlas_for_config(1)
    fib = fibers_for_config(1, 0, 60)
    fib[5, 3, 1] = np.nan
    r = oracle.classify_multi(fib, at.centroids, at.bundle_id, at.thresh)
    assert r["mask"].shape == (60, 4)
    assert np.all(r["mask"][5] == 0)
    s = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    for i in np.nonzero(s["label"] >= 0)[0]:
        b = s["label"][i]
        assert (r["mask"][i, b >> 5] >> (b & 31)) & 1
    with pytest.raises(ValueError):
        oracle.classify_multi(fib, at.centroids, at.bundle_id, at.thresh, words=3)   # 100 bundles need 4 words
