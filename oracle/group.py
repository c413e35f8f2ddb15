"""Oracle of row f3 (the segmented bundles) -- TEST INFRASTRUCTURE ONLY.

The plain definition with library primitives, no reordering beyond what the definition states:
bins = label for 0 <= label < B, else B (unassigned last); order = a STABLE argsort of the bins
(numpy's mergesort); offsets = the exclusive prefix of the bin counts; per bundle the min / max / sum
of dist over its fibers (sum in double), +inf / 0 / 0 for an empty bundle.
"""
from __future__ import annotations

import numpy as np


def group_by_bundle(label, dist, B: int):
    label = np.asarray(label, np.int64)
    bins = np.where((label >= 0) & (label < B), label, B)
    order = np.argsort(bins, kind="stable").astype(np.int32)
    counts = np.bincount(bins, minlength=B + 1)
    offsets = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    out = dict(order=order, offsets=offsets, counts=counts)
    if dist is not None:
        dist = np.asarray(dist, np.float32)
        dmin = np.full(B, np.inf, np.float32)
        dmax = np.zeros(B, np.float32)
        dsum = np.zeros(B, np.float64)
        for b in range(B):
            d = dist[order[offsets[b]:offsets[b + 1]]]
            if d.size:
                dmin[b], dmax[b], dsum[b] = d.min(), d.max(), d.astype(np.float64).sum()
        out.update(dmin=dmin, dmax=dmax, dsum=dsum)
    return out
