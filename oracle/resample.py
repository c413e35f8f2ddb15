"""Oracle of row f2 (resampling) -- TEST INFRASTRUCTURE ONLY; shares nothing with the CUDA path.

The plain definition ("resampled using 21 equidistant points"; reading R19 after
SPEC.md:63-71): s_j = cumulative chord length at input point j (double), L = s_last; output point
k = the point at arc position k L / 20 on the polyline, found by walking the segments and linearly
interpolating inside the segment that holds it; points 0 and 20 are the input end points exactly.
Fewer than 2 points, zero length or non-finite input -> 63 NaNs.  Each coordinate rounded to FP32
once.  Pure Python / numpy loops: for test-sized inputs.
"""
from __future__ import annotations

import math

import numpy as np


def resample_one(P) -> np.ndarray:
    P = np.asarray(P, np.float64).reshape(-1, 3)
    out = np.full((21, 3), np.nan, np.float32)
    m = P.shape[0]
    if m < 2 or not np.all(np.isfinite(P)):
        return out
    seg = [math.sqrt(float(((P[j + 1] - P[j]) ** 2).sum())) for j in range(m - 1)]
    s = [0.0]
    for L in seg:
        s.append(s[-1] + L)
    L = s[-1]
    if not L > 0.0:
        return out
    out[0] = P[0].astype(np.float32)
    out[20] = P[-1].astype(np.float32)
    j = 0
    for k in range(1, 20):
        t = k * L / 20.0
        while j < m - 2 and s[j + 1] < t:     # the first segment whose end reaches t
            j += 1
        u = min(max((t - s[j]) / seg[j], 0.0), 1.0) if seg[j] > 0 else 0.0
        out[k] = (P[j] + u * (P[j + 1] - P[j])).astype(np.float32)
    return out


def resample(points, offsets) -> np.ndarray:
    points = np.asarray(points, np.float32)
    offsets = np.asarray(offsets, np.int64)
    n = offsets.shape[0] - 1
    out = np.empty((n, 21, 3), np.float32)
    for f in range(n):
        out[f] = resample_one(points[offsets[f]:offsets[f + 1]])
    return out
