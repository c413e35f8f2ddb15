"""Pins for the oracle's paper-semantics mode (oracle/oracle.c).

The paper's final classifier scores a pair by d_ME in the orientation the end points infer
 plus the length term TN of Eq. 3 ("the complete distance metric
(d_ME + TN)").  The paper prints no worked example, so the pins are SPEC.md's
hand-evaluated examples of Eq. 3 and of the complete metric (tests/golden/spec_examples.jsonl),
closed forms (straight and staircase polylines, a uniformly scaled copy, a pair whose end points
and interior disagree about the orientation), invariants (TN symmetric and scale-free, score >=
exact d_ME), constructed labelling cases and a pure-Python brute force on tiny inputs.  Every pin
is a check over an implementation, run against the oracle and against deliberately broken
variants (mutants): each plausible mistake must fail at least one pin.
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
# implementations under test
# ----------------------------------------------------------------------------------
class OracleImpl:
    name = "oracle"

    def tn(self, ls, lc):
        return oracle.tn(ls, lc)

    def length(self, a):
        return oracle.polyline_length(a)

    def orientation(self, a, c):
        return oracle.endpoint_orientation(a, c)

    def score(self, a, c):
        return oracle.paper_score(a, c)

    def classify(self, fibers, cents, bid, thr):
        r = oracle.classify(fibers, cents, bid, thr, threads=1, mode="paper")
        return r["label"], r["dist"]


def _d(p, q):
    return float(np.sqrt(((np.asarray(p, np.float64) - np.asarray(q, np.float64)) ** 2).sum()))


class Mutant:
    """A numpy re-implementation of paper mode with one deliberate mistake."""

    def __init__(self, name, tn=None, length=None, orient=None, score=None, strict=False):
        self.name = name
        self._tn, self._length, self._orient, self._score, self.strict = tn, length, orient, score, strict

    def tn(self, ls, lc):
        if self._tn:
            return self._tn(ls, lc)
        return (abs(ls - lc) / max(ls, lc) + 1.0) ** 2 - 1.0

    def length(self, a):
        a = np.asarray(a, np.float64).reshape(21, 3)
        if self._length:
            return self._length(a)
        return float(np.sqrt(((a[1:] - a[:-1]) ** 2).sum(1)).sum())

    def orientation(self, a, c):
        a, c = np.asarray(a, np.float64).reshape(21, 3), np.asarray(c, np.float64).reshape(21, 3)
        mdir = max(_d(a[0], c[0]), _d(a[20], c[20]))
        minv = max(_d(a[0], c[20]), _d(a[20], c[0]))
        if self._orient:
            return self._orient(mdir, minv)
        return 1 if minv < mdir else 0

    def _max(self, a, c, o):
        a, c = np.asarray(a, np.float64).reshape(21, 3), np.asarray(c, np.float64).reshape(21, 3)
        cc = c[::-1] if o else c
        return float(np.sqrt(((a - cc) ** 2).sum(1)).max())

    def score(self, a, c):
        if self._score:
            return self._score(self, a, c)
        return self._max(a, c, self.orientation(a, c)) + self.tn(self.length(a), self.length(c))

    def classify(self, fibers, cents, bid, thr):
        fibers = np.asarray(fibers, np.float32).reshape(-1, 21, 3)
        labels, dists = [], []
        for a in fibers:
            sb = {}
            for c, b in zip(np.asarray(cents, np.float32).reshape(-1, 21, 3), bid):
                s = self.score(a, c)
                sb[int(b)] = min(sb.get(int(b), math.inf), s)
            best, bs = -1, math.inf
            for b in sorted(sb):
                ok = sb[b] < thr[b] if self.strict else sb[b] <= thr[b]
                if ok and sb[b] < bs:
                    best, bs = b, sb[b]
            labels.append(best)
            dists.append(bs)
        return np.array(labels), np.array(dists)


MUTANTS = [
    Mutant("tn without the square", tn=lambda ls, lc: abs(ls - lc) / max(ls, lc)),
    Mutant("tn over min length", tn=lambda ls, lc: (abs(ls - lc) / min(ls, lc) + 1.0) ** 2 - 1.0
           if min(ls, lc) > 0 else math.inf),
    Mutant("tn without -1", tn=lambda ls, lc: (abs(ls - lc) / max(ls, lc) + 1.0) ** 2),
    Mutant("length = chord of the end points", length=lambda a: float(np.sqrt(((a[20] - a[0]) ** 2).sum()))),
    Mutant("orientation = argmax", orient=lambda mdir, minv: 1 if minv > mdir else 0),
    Mutant("orientation ties -> inverse", orient=lambda mdir, minv: 1 if minv <= mdir else 0),
    Mutant("exact min orientation instead of inferred",
           score=lambda m, a, c: min(m._max(a, c, 0), m._max(a, c, 1)) + m.tn(m.length(a), m.length(c))),
    Mutant("no TN", score=lambda m, a, c: m._max(a, c, m.orientation(a, c))),
    Mutant("strict threshold", strict=True),
]


# ----------------------------------------------------------------------------------
# pins
# ----------------------------------------------------------------------------------
def _golden(op):
    with open(GOLDEN) as fh:
        return [r for r in map(json.loads, fh) if r["op"] == op]


def pin_golden(impl):
    for r in _golden("tn"):
        assert impl.tn(*r["args"]) == pytest.approx(r["expect"], abs=1e-12), r["cite"]
    for r in _golden("paper_score"):
        assert impl.score(parse_fiber(r["a"]), parse_fiber(r["b"])) == pytest.approx(r["expect"], abs=1e-9), r["cite"]


def pin_tn_closed_forms(impl):
    for l in (0.5, 3.0, 17.25, 100.0):
        assert impl.tn(l, l) == 0.0
        assert impl.tn(l, 2 * l) == pytest.approx(1.25, abs=1e-12)       # (1/2 + 1)^2 - 1
        assert impl.tn(3 * l, l) == pytest.approx(16.0 / 9.0, abs=1e-12)  # (2/3 + 1)^2 - 1 = 25/9 - 1
        assert impl.tn(l, 5 * l) == pytest.approx(impl.tn(5 * l, l), abs=1e-12)


def pin_length_closed_forms(impl):
    s = np.float32(0.75)
    straight = np.zeros((21, 3), np.float32)
    straight[:, 0] = np.arange(21, dtype=np.float32) * s
    assert impl.length(straight) == pytest.approx(20 * 0.75, abs=1e-12)
    stair = np.zeros((21, 3), np.float32)   # alternating unit steps in x and y: 20 unit segments
    for i in range(1, 21):
        stair[i] = stair[i - 1] + (np.float32([1, 0, 0]) if i % 2 else np.float32([0, 1, 0]))
    assert impl.length(stair) == pytest.approx(20.0, abs=1e-12)


def pin_orientation(impl):
    a = fiber_A()
    assert impl.orientation(a, a[::-1].copy()) == 1
    assert impl.score(a, a[::-1].copy()) == pytest.approx(0.0, abs=1e-9)
    assert impl.orientation(a, a + np.float32([0, 2, 0])) == 0
    # a palindromic fiber: both orientations tie exactly -> direct (reading R17)
    p = np.zeros((21, 3), np.float32)
    p[:, 0] = np.abs(np.arange(21, dtype=np.float32) - 10)
    p[:, 1] = np.arange(21, dtype=np.float32) * 0
    q = p + np.float32([0, 0, 1])
    assert impl.orientation(p, q) == 0


def pin_inferred_not_exact(impl):
    """End points match directly (m_dir = 0 < m_inv = 20) but point 2 is displaced, so the direct
    maximum (23) exceeds the inverse one (20): the inferred orientation is direct, score 23 + TN."""
    a = np.zeros((21, 3), np.float32)
    a[:, 0] = np.arange(21, dtype=np.float32)
    c = a.copy()
    c[2] = (25, 0, 0)
    lc = 20 - 2 + 24 + 22          # segments a1->c2 (24) and c2->a3 (22) replace two unit segments
    tn = (abs(20 - lc) / lc + 1) ** 2 - 1
    assert impl.orientation(a, c) == 0
    assert impl.score(a, c) == pytest.approx(23 + tn, abs=1e-9)
    assert oracle.d_me(a, c) == pytest.approx(20.0, abs=1e-12)   # the exact Eq. 2 distance differs


def pin_scaled_copy(impl):
    """c = a scaled by k about a_10 (direct orientation): d = |1 - k| max_i |a_i - a_10|, l_C = k l_S."""
    a = np.zeros((21, 3), np.float32)
    a[:, 0] = np.arange(21, dtype=np.float32) - 10
    k = np.float32(1.5)
    c = a * k
    assert impl.orientation(a, c) == 0
    expect = 0.5 * 10 + ((abs(20 - 30) / 30.0 + 1) ** 2 - 1)
    assert impl.score(a, c) == pytest.approx(expect, abs=1e-9)


def pin_threshold_and_tn_cut(impl):
    a = fiber_A()
    c = a + np.float32([3, 0, 0])                    # score exactly 3 (TN = 0)
    lab, dist = impl.classify(a[None], c[None], np.array([0], np.int32), np.array([3.0], np.float32))
    assert lab[0] == 0 and dist[0] == pytest.approx(3.0, abs=1e-9)
    # d_ME <= thr but d_ME + TN > thr: scaled copy, d = 5, TN = 1/9 -> 5.111 > 5.05
    s = np.zeros((21, 3), np.float32)
    s[:, 0] = np.arange(21, dtype=np.float32) - 10
    lab, _ = impl.classify(s[None], (s * np.float32(1.5))[None], np.array([0], np.int32), np.array([5.05], np.float32))
    assert lab[0] == -1


def pin_score_at_least_exact(impl):
    rng = np.random.default_rng(11)
    for _ in range(40):
        a = np.cumsum(rng.normal(0, 2, (21, 3)), 0).astype(np.float32)
        c = (a + rng.normal(0, 1.5, (21, 3))).astype(np.float32)
        if rng.random() < 0.5:
            c = c[::-1].copy()
        assert impl.score(a, c) >= oracle.d_me(a, c) - 1e-9


PINS = [pin_golden, pin_tn_closed_forms, pin_length_closed_forms, pin_orientation, pin_inferred_not_exact,
        pin_scaled_copy, pin_threshold_and_tn_cut, pin_score_at_least_exact]


@pytest.mark.parametrize("pin", PINS, ids=[p.__name__ for p in PINS])
def test_oracle_passes_pin(pin):
    pin(OracleImpl())


@pytest.mark.parametrize("mutant", MUTANTS, ids=[m.name for m in MUTANTS])
def test_every_mutant_fails_some_pin(mutant):
    failed = []
    for pin in PINS:
        try:
            pin(mutant)
        except (AssertionError, ZeroDivisionError, ValueError):
            failed.append(pin.__name__)
    assert failed, f"mutant '{mutant.name}' passes every paper-mode pin"


# ----------------------------------------------------------------------------------
# brute force and invariants on small seeded inputs
# ----------------------------------------------------------------------------------
def _small_problem(seed, n=60, bundles=4, per=5):
    rng = np.random.default_rng(seed)
    base = [np.cumsum(rng.normal(0, 3, (21, 3)), 0) for _ in range(bundles)]
    cents, bid = [], []
    for b in range(bundles):
        for _ in range(per):
            cents.append(base[b] + rng.normal(0, 1.0, (21, 3)))
            bid.append(b)
    fibers = []
    for _ in range(n):
        b = rng.integers(bundles)
        f = base[b] + rng.normal(0, 1.2, (21, 3))
        fibers.append(f[::-1] if rng.random() < 0.5 else f)
    thr = rng.uniform(3, 6, bundles)
    return (np.array(fibers, np.float32), np.array(cents, np.float32), np.array(bid, np.int32),
            thr.astype(np.float32))


def test_paper_mode_matches_brute_force_tiny():
    fib, cen, bid, thr = _small_problem(5)
    r = oracle.classify(fib, cen, bid, thr, threads=1, mode="paper")
    ref = Mutant("reference")   # the mistake-free numpy re-implementation (orientation in double)
    for i, a in enumerate(fib):
        # skip fibers whose end-point orientation decision is within FP32 reach of a tie
        gaps = []
        for c in cen:
            mdir = max(_d(a[0], c[0]), _d(a[20], c[20]))
            minv = max(_d(a[0], c[20]), _d(a[20], c[0]))
            gaps.append(abs(mdir - minv))
        if min(gaps) < 1e-4:
            continue
        lab, dist = ref.classify(a[None], cen, bid, thr)
        assert r["label"][i] == lab[0]
        if lab[0] >= 0:
            assert r["dist"][i] == pytest.approx(dist[0], rel=1e-12)


def test_paper_mode_accepts_a_subset_of_exact():
    fib, cen, bid, thr = _small_problem(7, n=200)
    p = oracle.classify(fib, cen, bid, thr, threads=2, mode="paper")
    e = oracle.classify(fib, cen, bid, thr, threads=2, mode="exact")
    for i in range(len(fib)):
        if p["label"][i] >= 0:
            assert e["label"][i] >= 0 and e["dist"][i] <= p["dist"][i] + 1e-12


def test_paper_self_segmentation_and_monotonicity():
    fib, cen, bid, thr = _small_problem(9)
    r = oracle.classify(cen, cen, bid, thr, threads=1, mode="paper")
    assert np.array_equal(r["label"], bid) and np.all(r["dist"] == 0.0)
    lo = oracle.classify(fib, cen, bid, thr, threads=1, mode="paper")
    hi = oracle.classify(fib, cen, bid, thr * np.float32(1.5), threads=1, mode="paper")
    assert np.all((lo["label"] < 0) | (hi["label"] >= 0))
    assert np.all(hi["dist"][lo["label"] >= 0] <= lo["dist"][lo["label"] >= 0] + 1e-12)


# ----------------------------------------------------------------------------------
# the paper-mode tie band (decidable flag; oracle/oracle.c label_paper, readings R17 + R20)
# ----------------------------------------------------------------------------------
def test_paper_tie_band_flag():
    """decidable = False within 1e-3 mm of a threshold or of the runner-up bundle (scores with TN = 0:
    translated copies have the fiber's own length), mirroring tests/test_oracle_pins.py's exact case."""
    a = fiber_A()[None]
    bid = np.array([0, 1], np.int32)
    thr = np.array([4.0, 8.0], np.float32)

    def run(t0, t1):
        c = np.stack([fiber_A() + np.float32([t0, 0, 0]), fiber_A() + np.float32([0, t1, 0])])
        return oracle.classify(a, c, bid, thr, mode="paper")

    r = run(2.0, 6.0)
    assert r["label"][0] == 0 and r["dist"][0] == 2.0 and r["decidable"][0]      # clear winner
    r = run(4.0 - 2 ** -11, 6.0)                              # within 1e-3 of thr_0
    assert r["label"][0] == 0 and not r["decidable"][0]
    r = run(4.0 + 2 ** -11, 6.0)                              # just above thr_0, within band
    assert r["label"][0] == 1 and not r["decidable"][0]
    r = run(3.0, 3.0 + 2 ** -11)                              # runner-up within 1e-3
    assert r["label"][0] == 0 and not r["decidable"][0]
    assert run(3.0, 3.0 + 2 ** -8)["decidable"][0]            # runner-up 3.9e-3 away
    r = run(9.0, 9.0)
    assert r["label"][0] == -1 and r["decidable"][0]          # nothing within thr + delta


def _loop_fiber():
    """A closed, non-palindromic loop: a_0 = a_20 (so every centroid's end-point maxima tie exactly)."""
    t = np.arange(21, dtype=np.float64) * (2 * np.pi / 20)
    f = np.stack([8 * np.cos(t) - 8, 6 * np.sin(t), 2 * np.sin(2 * t)], 1)
    return (np.round(f * 64) / 64).astype(np.float32)   # dyadic: translations stay exact in FP32


def test_paper_orientation_band_makes_a_loop_undecidable():
    """Reading R20: a_0 = a_20 ties the orientation decision exactly; the direct score (1, a translated
    copy) and the inverse one differ, so either is a correct answer and the fiber is undecidable."""
    a = _loop_fiber()
    a[20] = a[0]
    c = a + np.float32([0, 0, 1])
    assert oracle.orientation_ambiguous(a, c) and oracle.endpoint_orientation(a, c) == 0
    inv = oracle.max_pointwise(a, c, inverse=True)
    assert inv > 5.0
    r = oracle.classify(a[None], c[None], np.array([0], np.int32), np.array([4.0], np.float32), mode="paper",
                        want_bands=True)
    assert r["label"][0] == 0 and r["dist"][0] == pytest.approx(1.0, abs=1e-12)   # ties -> direct
    assert not r["decidable"][0]
    assert r["lo"][0, 0] == pytest.approx(1.0, abs=1e-12) and r["hi"][0, 0] == pytest.approx(inv, abs=1e-9)
    # with a threshold no inverse score can reach, the label is still -1 or 0 depending on the choice:
    # undecidable; with a palindromic fiber both orientations score alike and the fiber is decidable
    p = np.zeros((21, 3), np.float32)
    p[:, 0] = np.abs(np.arange(21, dtype=np.float32) - 10)
    q = p + np.float32([0, 0, 1])
    assert oracle.orientation_ambiguous(p, q)
    r = oracle.classify(p[None], q[None], np.array([0], np.int32), np.array([4.0], np.float32), mode="paper")
    assert r["label"][0] == 0 and r["dist"][0] == 1.0 and r["decidable"][0]


def test_paper_orientation_band_edges():
    """Just outside the band the orientation is a plain decision (decidable); just inside it is not."""
    a = _loop_fiber()
    a[20] = a[0] + np.float32([0.5, 0, 0])
    c = a + np.float32([0, 0, 1])
    # m_dir^2 = 1 (a translated copy); m_inv^2 = max(|a0 - c20|, |a20 - c0|)^2 = 0.25 + 1 = 1.25: direct
    assert not oracle.orientation_ambiguous(a, c) and oracle.endpoint_orientation(a, c) == 0
    r = oracle.classify(a[None], c[None], np.array([0], np.int32), np.array([40.0], np.float32), mode="paper")
    assert r["label"][0] == 0 and r["decidable"][0] and r["dist"][0] == 1.0
    # the band is 2^-18 relative on the squared maxima: an end-point offset e gives m_dir^2 = 1 and
    # m_inv^2 = 1 + e^2, i.e. a relative gap e^2 -- inside for e = 2^-12 (2^-24), outside for 2^-8 (2^-16)
    for e, inside in ((2.0 ** -12, True), (2.0 ** -8, False)):
        a2 = _loop_fiber()
        a2[20] = a2[0] + np.float32([e, 0, 0])
        c2 = a2 + np.float32([0, 0, 1])
        assert oracle.orientation_ambiguous(a2, c2) == inside and oracle.endpoint_orientation(a2, c2) == 0
        r = oracle.classify(a2[None], c2[None], np.array([0], np.int32), np.array([40.0], np.float32),
                            mode="paper")
        assert r["label"][0] == 0 and r["dist"][0] == 1.0
        assert r["decidable"][0] == (not inside)
