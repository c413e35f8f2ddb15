"""Seeded raw (not resampled) streamlines for row f2 -- an input generator only.

Real tractography streamlines have hundreds of points at a fixed integration step; the paper
resamples them to 21 points before classification.  The stand-in here: a Catmull-Rom
spline through each 21-point synthetic fiber, sampled at m uniformly spaced *spline parameters*
(m ~ U[mmin, mmax] per fiber), plus isotropic Gaussian jitter.  Spline parameters are not arc
length, so the chord spacing of the raw points is uneven, as resampling must handle.  Returns CSR
arrays: points float32 [P, 3], offsets int64 [N + 1].
"""
from __future__ import annotations

import numpy as np


def raw_streamlines(fibers: np.ndarray, seed: int, mmin: int = 30, mmax: int = 200, jitter: float = 0.05):
    fibers = np.asarray(fibers, np.float64)
    n = fibers.shape[0]
    rng = np.random.default_rng([1912, 11494, 77, seed])
    m = rng.integers(mmin, mmax + 1, n)
    offsets = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    points = np.empty((int(offsets[-1]), 3), np.float32)
    for mv in np.unique(m):
        idx = np.nonzero(m == mv)[0]
        u = np.linspace(0.0, 20.0, int(mv))
        i = np.minimum(np.floor(u).astype(np.int64), 19)
        t = (u - i)[None, :, None]
        f = fibers[idx]
        p0, p1 = f[:, np.maximum(i - 1, 0)], f[:, i]
        p2, p3 = f[:, i + 1], f[:, np.minimum(i + 2, 20)]
        c = 0.5 * (2 * p1 + (p2 - p0) * t + (2 * p0 - 5 * p1 + 4 * p2 - p3) * t ** 2
                   + (3 * p1 - p0 - 3 * p2 + p3) * t ** 3)
        c += rng.normal(0.0, jitter, c.shape)
        pos = offsets[idx][:, None] + np.arange(int(mv))[None, :]
        points[pos] = c.astype(np.float32)
    return points, offsets
