"""Offline estimate (CPU only) of a window-level tile pre-test for k_cull.

k_cull tests every fiber of a 256-fiber window (one k_classify CTA, Morton-ordered by point 10) against
every tile of every bundle some fiber of the window may need.  A window-level test -- the window's
bounding boxes of points 0 / 10 / 20 against a tile's spheres grown by the threshold -- could drop tiles
no fiber of the window can pass before the per-fiber loop.  This counts, over a sample of windows:
  per_fiber_now   tiles of the bundles passing the window (what the per-fiber loop walks today)
  window_pass     of those, tiles passing the window-box test (what it would walk)
  listed          tiles some fiber passes (the list k_classify streams)

python scripts/sim_cull.py [cfg] [n_windows]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1912_11494_b200 import binding
from synth import atlas_for_config, fibers_for_config

TILE, EPS, FPC = 32, 1e-3, 256


def spread3(v):
    v = v.astype(np.uint64)
    out = np.zeros_like(v)
    for b in range(10):
        out |= ((v >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b)
    return out


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    nwin = int(sys.argv[2]) if len(sys.argv) > 2 else 400
    at = atlas_for_config(cfg)
    T = binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, 0)
    tb = np.zeros(T, np.int32)
    mem = np.zeros(T * TILE, np.int32)
    sph = np.zeros(T * 12, np.float32)
    binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, T, tb, mem, sph)
    sph = sph.reshape(T, 3, 4).astype(np.float64)          # points 0 / 10 / 20: centre, radius
    thr = at.thresh.astype(np.float64)[tb]
    R = sph[:, :, 3] + thr[:, None] + EPS                     # grown radii [T, 3]
    # bundle point-10 spheres (the CTA-level bundle test): the sphere over the tiles' point-10 spheres
    bc, br = np.zeros((at.B, 3)), np.zeros(at.B)
    for b in range(at.B):
        s = sph[tb == b, 1]
        lo, hi = (s[:, :3] - s[:, 3:]).min(0), (s[:, :3] + s[:, 3:]).max(0)
        bc[b] = (lo + hi) / 2
        br[b] = np.sqrt(((s[:, :3] - bc[b]) ** 2).sum(1)).max() + s[:, 3].max()
    bR = br + at.thresh + EPS
    F = fibers_for_config(cfg)
    P0, P10, P20 = F[:, 0].astype(np.float64), F[:, 10].astype(np.float64), F[:, 20].astype(np.float64)
    del F
    C10 = at.centroids[:, 10].astype(np.float64)
    lo, hi = C10.min(0), C10.max(0)
    q = np.clip((P10 - lo) / (hi - lo) * 127, 0, 127).astype(np.int64)
    key = spread3(q[:, 0]) | (spread3(q[:, 1]) << np.uint64(1)) | (spread3(q[:, 2]) << np.uint64(2))
    order = np.argsort(key, kind="stable")
    nw = len(order) // FPC
    rng = np.random.default_rng(5)
    wins = rng.choice(nw, size=min(nwin, nw), replace=False)

    def box_sphere_d2(blo, bhi, c):
        d = np.maximum(np.maximum(blo[None] - c, c - bhi[None]), 0)
        return (d ** 2).sum(-1)

    tot = dict(per_fiber_now=0, window_pass=0, window_pass_10only=0, listed=0, bundles=0)
    for w in wins:
        idx = order[w * FPC:(w + 1) * FPC]
        a0, a10, a20 = P0[idx], P10[idx], P20[idx]
        # bundles: any fiber's point 10 inside the grown bundle sphere
        bpass = (((a10[:, None] - bc[None]) ** 2).sum(-1) <= bR[None] ** 2).any(0)
        tiles = np.nonzero(bpass[tb])[0]
        tot["bundles"] += int(bpass.sum())
        tot["per_fiber_now"] += len(tiles)
        if len(tiles) == 0:
            continue
        c0, c10, c20 = sph[tiles, 0, :3], sph[tiles, 1, :3], sph[tiles, 2, :3]
        r0, r10, r20 = R[tiles, 0] ** 2, R[tiles, 1] ** 2, R[tiles, 2] ** 2
        w10 = box_sphere_d2(a10.min(0), a10.max(0), c10) <= r10
        b0lo, b0hi, b2lo, b2hi = a0.min(0), a0.max(0), a20.min(0), a20.max(0)
        wd = (box_sphere_d2(b0lo, b0hi, c0) <= r0) & (box_sphere_d2(b2lo, b2hi, c20) <= r20)
        wi = (box_sphere_d2(b0lo, b0hi, c20) <= r20) & (box_sphere_d2(b2lo, b2hi, c0) <= r0)
        tot["window_pass_10only"] += int(w10.sum())
        tot["window_pass"] += int((w10 & (wd | wi)).sum())
        # per fiber: the exact three-sphere test (the list)
        d10 = ((a10[:, None] - c10[None]) ** 2).sum(-1) <= r10[None]
        dd = (((a0[:, None] - c0[None]) ** 2).sum(-1) <= r0[None]) & (((a20[:, None] - c20[None]) ** 2).sum(-1) <= r20[None])
        di = (((a0[:, None] - c20[None]) ** 2).sum(-1) <= r20[None]) & (((a20[:, None] - c0[None]) ** 2).sum(-1) <= r0[None])
        tot["listed"] += int((d10 & (dd | di)).any(0).sum())
    n = len(wins)
    print(f"cfg{cfg}: {n} windows of {FPC} fibers (Morton 7-bit on point 10), T={T}")
    for k, v in tot.items():
        print(f"  {k:22s} {v / n:8.1f} per window")


if __name__ == "__main__":
    main()
