"""Offline: how many (fiber, tile) pairs the live tile bound passes with boxes of more centroid points.

The kernel bounds a tile by the boxes of points 0/10/20 (canonical orientation).  Adding boxes of
points 5/15 (or more) can only reject more pairs; this counts by how much, at the final cutoff
tau = min(thr^2, d_final^2) (every fiber seeded with its final best: the live cutoff's limit) and at
1.3x that distance.  CPU only.   python scripts/box_eval.py [cfg] [n_fibers]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from scripts.tile_eval import canon_flips, current_plan, feats
from synth import atlas_for_config, fibers_for_config, sample_indices

EPS = 1e-3


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
    at = atlas_for_config(cfg)
    full = fibers_for_config(cfg, 0, 200000)
    fib = full[sample_indices(len(full), n, seed=5)]
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    dfin = np.where(r["label"] >= 0, r["dist"], np.inf)
    fl = canon_flips(at)
    Cc, _ = feats(at, fl)
    tb, mem, _ = current_plan(at)
    T = len(tb)
    thr2 = (at.thresh.astype(np.float64) ** 2)[tb]
    F = fib.astype(np.float64)
    sets = {"0/10/20": (0, 10, 20), "+5/15": (0, 5, 10, 15, 20), "+3/7/13/17": (0, 3, 5, 7, 10, 13, 15, 17, 20)}
    lo = {p: Cc[mem, p].min(1) for p in range(21)}    # [T, 3]
    hi = {p: Cc[mem, p].max(1) for p in range(21)}

    def boxd(P, p):   # [n, T] distance from fiber point P [n, 3] to box p of every tile
        d = np.maximum(np.maximum(lo[p][None] - P[:, None], P[:, None] - hi[p][None]), 0.0)
        return np.sqrt((d ** 2).sum(-1))

    for scale in (1.0, 1.3):
        s = np.sqrt(np.minimum(thr2[None], (scale * dfin[:, None]) ** 2)) + EPS
        out = []
        for name, pts in sets.items():
            ok_d = np.ones((n, T), bool)
            ok_i = np.ones((n, T), bool)
            for p in pts:
                ok_d &= boxd(F[:, p], p) <= s
                ok_i &= boxd(F[:, 20 - p], p) <= s
            out.append(f"{name}: {np.count_nonzero(ok_d | ok_i) / n:7.3f}")
        print(f"cutoff {scale} x final  passes per fiber  " + "  ".join(out), flush=True)


if __name__ == "__main__":
    main()
