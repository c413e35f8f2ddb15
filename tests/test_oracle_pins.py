"""Pins for the CPU oracle (oracle/oracle.c) against what the paper and mathematics fix.

The paper prints no worked numeric example (PAPER.md has no per-fiber result), so
the pins are: SPEC.md's hand-worked examples (tests/golden/spec_examples.jsonl,
each with its citation), closed forms of Eq. 2, a special case that
reduces to a library routine (numpy norm), metric invariants, constructed
labelling cases for Alg. 1 / PAPER.md:163, and pure-Python brute force on tiny inputs.
Each pin is written as a check over an implementation so that the same checks are
also run against deliberately broken variants (mutants) -- every plausible mistake
(dropped orientation, wrong inverse index, max/min swap, dropped coordinate, wrong
tie rule, strict threshold) must fail at least one pin.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from seg_testutil import fiber_A, parse_fiber

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.jsonl")


# ----------------------------------------------------------------------------------
# implementations under test: the oracle, and mutants of it
# ----------------------------------------------------------------------------------
class OracleImpl:
    name = "oracle"

    def d_me(self, a, b):
        return oracle.d_me(a, b)

    def max_pw(self, a, b, inverse):
        return oracle.max_pointwise(a, b, inverse)

    def classify(self, fibers, cents, bid, thr):
        r = oracle.classify(fibers, cents, bid, thr, threads=1)
        return r["label"], r["dist"]


def _pw(a, b, idx_fn, ncoord=3):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return max(math.sqrt(sum((a[i, k] - b[idx_fn(i), k]) ** 2 for k in range(ncoord))) for i in range(21))


class Mutant:
    """Pure-Python variants; each overrides one step with a plausible mistake."""

    def __init__(self, name, inv_idx=lambda i: 20 - i, combine=min, ncoord=3, sq=False,
                 tie_high=False, strict=False, first=False):
        self.name, self.inv_idx, self.combine, self.ncoord = name, inv_idx, combine, ncoord
        self.sq, self.tie_high, self.strict, self.first = sq, tie_high, strict, first

    def max_pw(self, a, b, inverse):
        v = _pw(a, b, self.inv_idx if inverse else (lambda i: i), self.ncoord)
        return v * v if self.sq else v

    def d_me(self, a, b):
        return self.combine(self.max_pw(a, b, False), self.max_pw(a, b, True))

    def classify(self, fibers, cents, bid, thr):
        labels, dists = [], []
        B = len(thr)
        for f in fibers:
            Db = [math.inf] * B
            for c, b in zip(cents, bid):
                Db[b] = min(Db[b], self.d_me(f, c))
            best = -1
            for b in range(B):
                ok = Db[b] < thr[b] if self.strict else Db[b] <= thr[b]
                if not ok:
                    continue
                if best < 0:
                    best = b
                elif self.first:
                    continue
                elif Db[b] < Db[best] or (self.tie_high and Db[b] == Db[best]):
                    best = b
            labels.append(best)
            dists.append(Db[best] if best >= 0 else math.inf)
        return np.array(labels), np.array(dists)


MUTANTS = [
    Mutant("inverse index b_{21-i} (mod 21)", inv_idx=lambda i: (21 - i) % 21),
    Mutant("inverse index b_{19-i} (clamped)", inv_idx=lambda i: max(19 - i, 0)),
    Mutant("max over orientations instead of min", combine=max),
    Mutant("direct orientation only", combine=lambda d, i: d),
    Mutant("inverse orientation only", combine=lambda d, i: i),
    Mutant("dropped z coordinate", ncoord=2),
    Mutant("squared distance returned", sq=True),
    Mutant("ties to the highest bundle id", tie_high=True),
    Mutant("strict threshold (d < thr)", strict=True),
    Mutant("first accepted bundle, not the closest", first=True),
]


# ----------------------------------------------------------------------------------
# pins (each returns None or raises AssertionError)
# ----------------------------------------------------------------------------------
def pin_golden(impl):
    """SPEC.md hand-worked examples (tests/golden/spec_examples.jsonl)."""
    with open(GOLDEN) as fh:
        rows = [json.loads(l) for l in fh if l.strip()]
    for r in rows:
        if r["op"] == "point_distance":
            if isinstance(impl, OracleImpl):
                got = math.sqrt(oracle.point_d2(r["p"], r["q"]))
            else:
                p, q = np.array(r["p"], float), np.array(r["q"], float)
                got = math.sqrt(sum((p[k] - q[k]) ** 2 for k in range(impl.ncoord)))
                got = got * got if impl.sq else got
            assert got == pytest.approx(r["expect"], abs=1e-12), r["cite"]
        elif r["op"] == "max_pointwise":
            got = impl.max_pw(parse_fiber(r["a"]), parse_fiber(r["b"]), r["inverse"])
            assert got == pytest.approx(r["expect"], abs=1e-12), r["cite"]
        elif r["op"] == "d_me":
            got = impl.d_me(parse_fiber(r["a"]), parse_fiber(r["b"]))
            assert got == pytest.approx(r["expect"], abs=1e-12), r["cite"]
        elif r["op"] == "closest":
            a = parse_fiber(r["a"])[None]
            cents = np.stack([parse_fiber(c) for c in r["centroids"]])
            lab, dist = impl.classify(a, cents, np.array(r["bundle_id"], np.int32),
                                      np.array(r["thresh"], np.float32))
            assert lab[0] == r["expect_label"], r["cite"]
            exp = math.inf if r["expect_dist"] == "inf" else r["expect_dist"]
            assert dist[0] == pytest.approx(exp, abs=1e-12), r["cite"]


def _dyadic_fibers(rng, n):
    """Random curved fibers with coordinates on a 1/8 grid (exact in FP32 and double)."""
    steps = rng.integers(-24, 25, size=(n, 21, 3)).astype(np.float64) / 8.0
    start = rng.integers(-400, 400, size=(n, 1, 3)).astype(np.float64) / 8.0
    return (start + np.cumsum(steps, axis=1)).astype(np.float32)


def pin_translation(impl):
    """Closed form (Eq. 2): d_ME(a + t, a) = |t| for ANY 21-point a -- every direct pair
    is |t| and the inverse max is >= |t| because index 10 pairs with itself."""
    rng = np.random.default_rng(1)
    for a in _dyadic_fibers(rng, 6):
        for t in ([3, 4, 0], [2, 3, 6], [1, 2, 2], [0.5, 0, 0], [-1.5, 2, -6]):
            t = np.array(t, np.float32)
            exp = float(np.sqrt(np.sum(t.astype(np.float64) ** 2)))
            assert impl.d_me(a + t, a) == pytest.approx(exp, rel=1e-14, abs=1e-14)


def pin_identity_reverse(impl):
    """d_ME(a, a) = 0 and d_ME(reverse(a), a) = 0 (Eq. 2 inverse term)."""
    rng = np.random.default_rng(2)
    for a in _dyadic_fibers(rng, 6):
        assert impl.d_me(a, a) == 0.0
        assert impl.d_me(np.ascontiguousarray(a[::-1]), a) == 0.0
        assert impl.d_me(a, np.ascontiguousarray(a[::-1])) == 0.0


def pin_collinear(impl):
    """Closed form: a_i = i s u, b_i = i s' u (s, s' > 0) -> d_ME = 20 |s - s'|
    (direct max at i = 20; the inverse max is 20 max(s, s') >= 20 |s - s'|)."""
    u = np.array([1.0, 2.0, 2.0]) / 3.0   # unit vector
    i = np.arange(21, dtype=np.float64)[:, None]
    for s, s2 in [(1.0, 1.25), (2.0, 0.5), (0.75, 3.0)]:
        a = (i * s * u).astype(np.float32)
        b = (i * s2 * u).astype(np.float32)
        exp = float(np.linalg.norm(a[20].astype(np.float64) - b[20].astype(np.float64)))
        assert impl.d_me(a, b) == pytest.approx(exp, rel=1e-12)
        assert exp == pytest.approx(20 * abs(s - s2), rel=1e-6)


def pin_library_special_case(impl):
    """Single-orientation max equals numpy's row-norm maximum (special case -> library)."""
    rng = np.random.default_rng(3)
    for _ in range(20):
        a = rng.normal(0, 30, (21, 3)).astype(np.float32)
        b = rng.normal(0, 30, (21, 3)).astype(np.float32)
        a64, b64 = a.astype(np.float64), b.astype(np.float64)
        exp_d = np.linalg.norm(a64 - b64, axis=1).max()
        exp_i = np.linalg.norm(a64 - b64[::-1], axis=1).max()
        assert impl.max_pw(a, b, False) == pytest.approx(exp_d, rel=1e-13)
        assert impl.max_pw(a, b, True) == pytest.approx(exp_i, rel=1e-13)
        assert impl.d_me(a, b) == pytest.approx(min(exp_d, exp_i), rel=1e-13)


def pin_invariants(impl):
    """Symmetry, flip invariance and the triangle inequality
    (d_ME is a metric on fibers modulo reversal)."""
    rng = np.random.default_rng(4)
    f = rng.normal(0, 10, (12, 21, 3)).astype(np.float32)
    for k in range(0, 12, 3):
        a, b, c = f[k], f[k + 1], f[k + 2]
        ra, rb = np.ascontiguousarray(a[::-1]), np.ascontiguousarray(b[::-1])
        dab = impl.d_me(a, b)
        assert impl.d_me(b, a) == dab
        assert impl.d_me(ra, b) == dab and impl.d_me(a, rb) == dab and impl.d_me(ra, rb) == dab
        assert impl.d_me(a, c) <= dab + impl.d_me(b, c) + 1e-9


def pin_threshold_equality(impl):
    """A distance exactly equal to the threshold is accepted; just above is not
    (PAPER.md:93 'above the threshold' -> discarded; reading R4)."""
    a = fiber_A()[None]
    thr = np.array([4.0], np.float32)
    lab, dist = impl.classify(a, (fiber_A() + np.float32([4, 0, 0]))[None], np.array([0], np.int32), thr)
    assert lab[0] == 0 and dist[0] == 4.0
    lab, _ = impl.classify(a, (fiber_A() + np.float32([4 + 2 ** -10, 0, 0]))[None],
                           np.array([0], np.int32), thr)
    assert lab[0] == -1


def pin_tie_lowest_bundle(impl):
    """Equal distances in two bundles -> the lower bundle id (Alg. 1 strict '<' with j
    ascending; reading R5)."""
    a = fiber_A()[None]
    c = np.stack([fiber_A() + np.float32([0, 0, 3]), fiber_A() + np.float32([0, 3, 0]),
                  fiber_A() + np.float32([3, 0, 0])])
    lab, dist = impl.classify(a, c, np.array([2, 1, 3], np.int32), np.full(4, 5, np.float32))
    assert lab[0] == 1 and dist[0] == 3.0


def pin_closest_not_first(impl):
    """Only the closest bundle under threshold labels the fiber."""
    a = fiber_A()[None]
    c = np.stack([fiber_A() + np.float32([0, 0, 4]), fiber_A() + np.float32([2, 0, 0])])
    lab, dist = impl.classify(a, c, np.array([0, 1], np.int32), np.full(2, 5, np.float32))
    assert lab[0] == 1 and dist[0] == 2.0


PINS = [pin_golden, pin_translation, pin_identity_reverse, pin_collinear, pin_library_special_case,
        pin_invariants, pin_threshold_equality, pin_tie_lowest_bundle, pin_closest_not_first]


@pytest.mark.parametrize("pin", PINS, ids=[p.__name__ for p in PINS])
def test_oracle_passes_pin(pin):
    pin(OracleImpl())


@pytest.mark.parametrize("mutant", MUTANTS, ids=[m.name for m in MUTANTS])
def test_every_mutant_fails_some_pin(mutant):
    failed = []
    for pin in PINS:
        try:
            pin(mutant)
        except AssertionError:
            failed.append(pin.__name__)
    assert failed, f"mutant '{mutant.name}' passes every pin"


# ----------------------------------------------------------------------------------
# classification-level pins on the oracle
# ----------------------------------------------------------------------------------
def _brute_classify(fibers, cents, bid, thr):
    """Pure-Python brute force: enumerate all 42 point distances of every pair."""
    B = len(thr)
    out = []
    for f in np.asarray(fibers, np.float64):
        Db = [math.inf] * B
        for c, b in zip(np.asarray(cents, np.float64), bid):
            dd = max(math.dist(f[i], c[i]) for i in range(21))
            di = max(math.dist(f[i], c[20 - i]) for i in range(21))
            Db[b] = min(Db[b], min(dd, di))
        acc = [b for b in range(B) if Db[b] <= float(thr[b])]
        best = min(acc, key=lambda b: (Db[b], b)) if acc else -1
        out.append((best, Db[best] if best >= 0 else math.inf))
    return out


def test_oracle_matches_brute_force_tiny():
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0)
    sel = np.arange(0, at.M, 10)                     # 50 centroids over all 10 bundles
    fib = fibers_for_config(0, 0, 40)
    thr = at.thresh * 1.5                            # wider thresholds -> more accepted pairs
    exp = _brute_classify(fib, at.centroids[sel], at.bundle_id[sel], thr)
    r = oracle.classify(fib, at.centroids[sel], at.bundle_id[sel], thr)
    for k, (lab, d) in enumerate(exp):
        assert r["label"][k] == lab
        if lab >= 0:
            assert r["dist"][k] == pytest.approx(d, rel=1e-12)
        else:
            assert r["dist"][k] == math.inf
    assert (r["label"] >= 0).sum() >= 5               # the case exercises assignment


def test_self_segmentation():
    """Atlas centroids as subject -> own bundle at distance 0."""
    from synth import atlas_for_config
    at = atlas_for_config(0)
    r = oracle.classify(at.centroids[::7], at.centroids, at.bundle_id, at.thresh)
    assert np.array_equal(r["label"], at.bundle_id[::7])
    assert np.all(r["dist"] == 0.0)


def test_threshold_monotonicity():
    """Raising thresholds never unassigns a fiber nor increases its distance."""
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 200)
    r1 = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    r2 = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh * 1.3)
    was = r1["label"] >= 0
    assert np.all(r2["label"][was] >= 0)
    assert np.all(r2["dist"][was] <= r1["dist"][was])
    assert np.all(r1["dist"][was] <= at.thresh[r1["label"][was]])


def test_non_finite_fiber():
    """A fiber with a NaN/Inf coordinate -> label -1, dist NaN (reading R12)."""
    from synth import atlas_for_config
    at = atlas_for_config(0)
    f = at.centroids[:3].copy()
    f[1, 5, 2] = np.nan
    f[2, 0, 0] = np.inf
    r = oracle.classify(f, at.centroids, at.bundle_id, at.thresh)
    assert r["label"][0] == at.bundle_id[0]
    assert r["label"][1] == -1 and np.isnan(r["dist"][1])
    assert r["label"][2] == -1 and np.isnan(r["dist"][2])


def test_tie_band_flag():
    """decidable = False within 1e-3 mm of a threshold or of the runner-up bundle."""
    a = fiber_A()[None]
    bid = np.array([0, 1], np.int32)
    thr = np.array([4.0, 8.0], np.float32)

    def run(t0, t1):
        c = np.stack([fiber_A() + np.float32([t0, 0, 0]), fiber_A() + np.float32([0, t1, 0])])
        return oracle.classify(a, c, bid, thr)

    assert run(2.0, 6.0)["decidable"][0]                      # clear winner
    r = run(4.0 - 2 ** -11, 6.0)                              # within 1e-3 of thr_0
    assert r["label"][0] == 0 and not r["decidable"][0]
    r = run(4.0 + 2 ** -11, 6.0)                              # just above thr_0, within band
    assert r["label"][0] == 1 and not r["decidable"][0]
    r = run(3.0, 3.0 + 2 ** -11)                              # runner-up within 1e-3
    assert r["label"][0] == 0 and not r["decidable"][0]
    assert run(3.0, 3.0 + 2 ** -8)["decidable"][0]            # runner-up 3.9e-3 away
    assert run(9.0, 9.0)["decidable"][0]                      # nothing within thr + delta


def test_oracle_threads_do_not_change_results():
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 300)
    r1 = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, threads=1)
    r4 = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, threads=4)
    for k in ("label", "dist", "decidable"):
        assert np.array_equal(r1[k], r4[k])


def test_generator_ground_truth_sanity():
    """Generator sanity (not a pin of the oracle's arithmetic): most matched fibers
    land in their source bundle and no background fiber is mostly assigned."""
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0)
    fib, truth = fibers_for_config(0, 0, 400, with_truth=True)
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    m = truth >= 0
    assert (r["label"][m] == truth[m]).mean() > 0.9
    assert (r["label"][~m] >= 0).mean() < 0.2
