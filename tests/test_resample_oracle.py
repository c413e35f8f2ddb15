"""Pins for the row-f2 oracle (oracle/resample.py): 21 points equidistant in chord length.

Against SPEC.md's examples for resample (a straight segment, idempotence on an
equidistant fiber, end points preserved), closed forms (an L-shaped polyline), and an independent
arc-position check: every output point must lie on the input polyline at arc length k L / 20,
measured by walking the segments.  Mutants (arc positions over 21 instead of 20, index instead of
chord-length parameterisation, end points not copied exactly) must each fail a pin.
"""
import math

import numpy as np
import pytest

import oracle.resample as R


def _mut_over21(P):
    P = np.asarray(P, np.float64)
    s = np.concatenate([[0.0], np.cumsum(np.sqrt(((P[1:] - P[:-1]) ** 2).sum(1)))])
    t = np.arange(21) * s[-1] / 21.0
    return np.stack([np.interp(t, s, P[:, c]) for c in range(3)], 1).astype(np.float32)


def _mut_index(P):
    P = np.asarray(P, np.float64)
    x = np.arange(P.shape[0], dtype=np.float64)
    t = np.linspace(0, P.shape[0] - 1, 21)
    return np.stack([np.interp(t, x, P[:, c]) for c in range(3)], 1).astype(np.float32)


def _mut_ends(P):
    out = R.resample_one(P).astype(np.float64)
    out[0] += 1e-3
    out[20] -= 1e-3
    return out.astype(np.float32)


IMPLS = [("oracle", R.resample_one), ("over21", _mut_over21), ("index", _mut_index), ("ends", _mut_ends)]


def pin_straight(f):
    out = f(np.array([[0, 0, 0], [20, 0, 0]], np.float32))
    assert np.array_equal(out[:, 0], np.arange(21, dtype=np.float32)) and not out[:, 1:].any()


def pin_idempotent(f):
    i = np.arange(21, dtype=np.float32)
    P = np.stack([2 * i - 20, 0.5 * i, 0 * i], 1).astype(np.float32)   # equidistant, straight
    assert np.abs(f(P) - P).max() <= 1e-5


def pin_L_shape(f):
    out = f(np.array([[0, 0, 0], [3, 0, 0], [3, 4, 0]], np.float32)).astype(np.float64)
    for k in range(21):
        a = 7.0 * k / 20
        want = (a, 0.0, 0.0) if a <= 3 else (3.0, a - 3.0, 0.0)
        assert np.allclose(out[k], want, atol=2e-6), (k, out[k], want)


def pin_arc_positions_random(f):
    rng = np.random.default_rng(4)
    P = np.cumsum(rng.normal(0, 1.5, (50, 3)), 0).astype(np.float32)
    out = f(P).astype(np.float64)
    Pd = P.astype(np.float64)
    seg = np.sqrt(((Pd[1:] - Pd[:-1]) ** 2).sum(1))
    s = np.concatenate([[0.0], np.cumsum(seg)])
    L = s[-1]
    assert np.array_equal(out[0], Pd[0]) and np.array_equal(out[20], Pd[-1])
    for k in range(1, 20):
        # arc position of out[k]: the segment it lies on (distance to the segment ~ 0)
        best = None
        for j in range(49):
            d = Pd[j + 1] - Pd[j]
            u = np.clip(np.dot(out[k] - Pd[j], d) / np.dot(d, d), 0, 1)
            dist = np.linalg.norm(Pd[j] + u * d - out[k])
            if best is None or dist < best[0]:
                best = (dist, s[j] + u * seg[j])
        assert best[0] < 1e-4 and abs(best[1] - k * L / 20) < 1e-4 * L, (k, best, k * L / 20)


PINS = [pin_straight, pin_idempotent, pin_L_shape, pin_arc_positions_random]


@pytest.mark.parametrize("pin", PINS, ids=[p.__name__ for p in PINS])
def test_oracle_passes(pin):
    pin(R.resample_one)


@pytest.mark.parametrize("name,f", IMPLS[1:], ids=[n for n, _ in IMPLS[1:]])
def test_mutant_fails_a_pin(name, f):
    failed = 0
    for pin in PINS:
        try:
            pin(f)
        except AssertionError:
            failed += 1
    assert failed, f"mutant {name} passes every pin"


def test_invalid_inputs_are_nan():
    assert np.isnan(R.resample_one(np.zeros((1, 3), np.float32))).all()
    assert np.isnan(R.resample_one(np.ones((5, 3), np.float32))).all()          # zero length
    bad = np.zeros((4, 3), np.float32)
    bad[2, 1] = np.nan
    assert np.isnan(R.resample_one(bad)).all()
