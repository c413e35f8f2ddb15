"""The parity rule's valid-answer check for undecidable fibers (tests/parity_util.py), on constructed
per-bundle intervals and on the oracle's own answers (which must always be valid)."""
import numpy as np

import oracle
from parity_util import valid_answers
from seg_testutil import fiber_A
from synth import atlas_for_config, fibers_for_config

INF = np.inf


def test_valid_answers_constructed():
    thr = np.array([4.0, 8.0], np.float32)
    # bundle 0 at 3.9995 (inside the band below thr 4), bundle 1 at 6 (certainly accepted)
    lo = np.array([[3.9995, 6.0]])
    hi = lo.copy()
    assert valid_answers([0], [3.9995], lo, hi, thr).all()             # the oracle's answer
    assert valid_answers([1], [6.0], lo, hi, thr).all()                # 0 may be read as beyond its threshold
    lo1 = np.array([[3.5, 6.0]])
    assert not valid_answers([1], [6.0], lo1, lo1, thr).all()          # 0 at 3.5 is certain and closer
    # bundle 0 just above its threshold (inside thr + delta): -1 ... only if nothing is certain; here 1 is
    lo2 = np.array([[4.0005, 6.0]])
    assert valid_answers([1], [6.0], lo2, lo2, thr).all()
    assert valid_answers([0], [4.0005], lo2, lo2, thr).all()          # accepting 0 within the band is valid too
    assert not valid_answers([-1], [INF], lo2, lo2, thr).all()         # 1 is certainly accepted
    lo3 = np.array([[4.0005, 8.0005]])
    assert valid_answers([-1], [INF], lo3, lo3, thr).all()
    assert not valid_answers([-1], [7.0], lo3, lo3, thr).all()         # -1 must carry +inf
    # runner-up within delta: both labels valid, each with its own distance only
    lo4 = np.array([[3.0, 3.0005]])
    assert valid_answers([0, 1], [3.0, 3.0005], np.repeat(lo4, 2, 0), np.repeat(lo4, 2, 0), thr).all()
    assert not valid_answers([1], [3.0], lo4, lo4, thr).all()          # wrong distance for bundle 1
    # an orientation-ambiguous bundle (paper mode): any value in [lo, hi] is a correct distance
    lo5, hi5 = np.array([[1.0, INF]]), np.array([[12.0, INF]])
    assert valid_answers([0], [1.0], lo5, hi5, np.array([20.0, 8.0], np.float32)).all()
    assert valid_answers([0], [12.0], lo5, hi5, np.array([20.0, 8.0], np.float32)).all()
    assert not valid_answers([0], [13.0], lo5, hi5, np.array([20.0, 8.0], np.float32)).all()


def test_oracle_answers_are_valid_in_the_band():
    """With thresholds moved onto fibers' own distances, every oracle answer (decidable or not) is
    valid under its own intervals."""
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 300)
    for mode in ("exact", "paper"):
        r0 = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode=mode)
        thr = at.thresh.copy()
        lab = r0["label"]
        for b in np.unique(lab[lab >= 0])[:5]:
            thr[b] = np.float32(r0["dist"][np.nonzero(lab == b)[0][0]] + 2e-4)
        r = oracle.classify(fib, at.centroids, at.bundle_id, thr, mode=mode, want_bands=True)
        assert (~r["decidable"]).sum() > 0
        assert valid_answers(r["label"], r["dist"], r["lo"], r["hi"], thr).all()


def test_exact_bands_are_the_bundle_distances():
    a = fiber_A()[None]
    c = np.stack([fiber_A() + np.float32([3, 0, 0]), fiber_A() + np.float32([0, 5, 0])])
    r = oracle.classify(a, c, np.array([0, 1], np.int32), np.array([4.0, 8.0], np.float32), want_bands=True)
    assert np.array_equal(r["lo"], np.array([[3.0, 5.0]])) and np.array_equal(r["hi"], r["lo"])
