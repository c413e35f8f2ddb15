"""Pins of the oracle's sound-discard variants (oracle_classify_sound / _paper_sound) to the plain
definition (oracle/oracle.c header).

The sound variants run Alg. 1's cascade (discardCenter, discardExtremes,
discardFourPoints, discarded21points with the early exit of PAPER.md:159) cut at (thr + 2 delta)^2.
They exist only to make the full-size oracle affordable, so they must return bitwise the plain
definition's label, dist and decidable flag, which these tests require on whole and sampled seeded
workloads, on constructed cases at the threshold and inside the tie band (where a cut at thr instead
of thr + 2 delta would drop the values the band reads), and on non-finite fibers.
"""
import numpy as np
import pytest

import oracle
from seg_testutil import fiber_A
from synth import atlas_for_config, fibers_for_config, sample_indices


def same(p, s):
    return (np.array_equal(p["label"], s["label"]) and np.array_equal(p["decidable"], s["decidable"])
            and np.array_equal(p["dist"].view(np.int64), s["dist"].view(np.int64)))


def both(fib, cen, bid, thr, mode, threads=None):
    p = oracle.classify(fib, cen, bid, thr, mode=mode, threads=threads)
    s = oracle.classify(fib, cen, bid, thr, mode=mode, threads=threads, sound=True)
    return p, s


@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_sound_equals_plain_cfg0_full(mode):
    at = atlas_for_config(0)
    fib = fibers_for_config(0)
    p, s = both(fib, at.centroids, at.bundle_id, at.thresh, mode)
    assert same(p, s)
    assert (p["label"] >= 0).sum() > 1000


@pytest.mark.parametrize("cfg,k", [(1, 300), (3, 120), (4, 120)])
@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_sound_equals_plain_sampled(cfg, k, mode):
    at = atlas_for_config(cfg)
    fib = fibers_for_config(cfg, 0, 65536)
    sub = fib[sample_indices(fib.shape[0], k, seed=31 + cfg)]
    p, s = both(sub, at.centroids, at.bundle_id, at.thresh, mode)
    assert same(p, s)


@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_sound_equals_plain_in_the_tie_band(mode):
    """Thresholds set to each fiber's own best distance -/+ a fraction of delta, so the deciding value
    sits at, inside or just beyond the band: the sound variant must still read it exactly."""
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 400)
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode=mode)
    lab = ref["label"]
    rng = np.random.default_rng(3)
    n_undec = 0
    for off in (-1.5e-3, -5e-4, 0.0, 5e-4, 1.5e-3, 1.9e-3):
        thr = at.thresh.copy()
        for b in np.unique(lab[lab >= 0])[:6]:
            i = rng.choice(np.nonzero(lab == b)[0])
            thr[b] = np.float32(ref["dist"][i] + off)
        p, s = both(fib, at.centroids, at.bundle_id, thr, mode)
        assert same(p, s), f"offset {off}"
        n_undec += int((~p["decidable"]).sum())
    assert n_undec > 0   # the constructed cases really exercise the band


def test_cut_at_thr_would_fail_the_band_case():
    """A fiber whose best is inside (thr, thr + delta]: plain and sound agree that it is undecidable
    (a cut at thr would have discarded that bundle and called the fiber decidable)."""
    a = fiber_A()[None]
    c = (fiber_A() + np.float32([4.0 + 2 ** -11, 0, 0]))[None]
    for mode in ("exact", "paper"):
        p, s = both(a, c, np.array([0], np.int32), np.array([4.0], np.float32), mode)
        assert same(p, s)
        assert p["label"][0] == -1 and not p["decidable"][0]


@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_sound_threshold_equality_and_non_finite(mode):
    at = atlas_for_config(0)
    f = at.centroids[:6].copy()
    f[1, 5, 2] = np.nan
    f[2, 0, 0] = np.inf
    f[3] = f[3] + np.float32([0, 0, 0.5])
    thr = at.thresh.copy()
    thr[at.bundle_id[3]] = np.float32(0.5)        # d = thr exactly (dyadic translation): accepted
    p, s = both(f, at.centroids, at.bundle_id, thr, mode)
    assert same(p, s)
    assert p["label"][1] == -1 and np.isnan(p["dist"][1]) and p["label"][2] == -1


@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_sound_empty_bundle_and_threads(mode):
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 300)
    thr = np.concatenate([at.thresh, np.float32([7.0])])   # bundle 10 has no centroid
    s1 = oracle.classify(fib, at.centroids, at.bundle_id, thr, mode=mode, sound=True, threads=1)
    s8 = oracle.classify(fib, at.centroids, at.bundle_id, thr, mode=mode, sound=True, threads=8)
    p = oracle.classify(fib, at.centroids, at.bundle_id, thr, mode=mode)
    assert same(p, s1) and same(p, s8)
