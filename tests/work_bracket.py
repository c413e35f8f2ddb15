"""An independent CPU check of the roofline numerator W (bench.py's lane_point_dists).

The stats kernel counts the point distances its cascade rules needed (one unit =
Eq. 1 squared = 6 FP32 lane-instructions), in four terms:
  T1 = 5 per (fiber, listed tile)          live tile bound (boxes of points 0/10/20)
  T2 = 32 per (fiber, tile passing it)     test1 for every lane of the tile
  T3 = 4 per (fiber, centroid) whose test1 passes in such a tile (test2, both end points)
  T4 = the test3/test4 points the candidate rounds computed
Each term depends on the order the kernel meets tiles and candidates (its running best), so it is not
a fixed number; but every execution of those rules lies between two bounds computed here on the host
from the fibers, the tile plan (seg_plan_tiles, host-only) and the oracle's final distances:
  lower: the work that remains when every fiber starts with its final best as the cutoff, over the
         tiles it is guaranteed to be listed for;
  upper: the work with the threshold as the cutoff, over every tile that could pass (a box test on
         orientation-symmetric boxes, which contain the kernel's boxes).
Margins (1e-5 relative, the screen's 2^-15 (|a|^2 + |c|^2)) cover the FP32 roundings in the
conservative direction.  Arithmetic in double with numpy; no code shared with the kernel.
"""
import numpy as np

CULL_EPS = 1e-3
REL = 1e-5


def _d2(a, b):
    return ((a.astype(np.float64) - b.astype(np.float64)) ** 2).sum(-1)


def bounds(fibers, centroids, bundle_id, thresh, tile_bundle, tile_members, final_d2, chunk=128):
    """Per-term (lower, upper) bounds, summed over the fibers.  final_d2[n]: the oracle's squared
    distance of each fiber's label (+inf when unlabelled)."""
    fib = np.asarray(fibers, np.float32)
    cen = np.asarray(centroids, np.float32)
    thr = np.asarray(thresh, np.float32).astype(np.float64)
    T = tile_bundle.shape[0]
    tb = np.asarray(tile_bundle)
    mem = np.asarray(tile_members).reshape(T, 32)
    thr2_t = (thr ** 2)[tb]                                                  # [T]
    # orientation-symmetric boxes per tile: point 10, and points 0 and 20 together
    c10m, c0m, c20m = cen[mem, 10], cen[mem, 0], cen[mem, 20]                # [T, 32, 3]
    b10lo, b10hi = c10m.min(1).astype(np.float64), c10m.max(1).astype(np.float64)
    ends = np.concatenate([c0m, c20m], 1)
    belo, behi = ends.min(1).astype(np.float64), ends.max(1).astype(np.float64)
    s_up = (np.sqrt(thr2_t) * (1 + REL) + CULL_EPS) ** 2 * (1 + REL)        # [T]

    def box_d2(p, lo, hi):                                                    # p [n,3], lo/hi [T,3] -> [n,T]
        d = np.maximum(np.maximum(lo[None] - p[:, None], p[:, None] - hi[None]), 0.0)
        return (d ** 2).sum(-1)

    lo_t = np.zeros(4)
    hi_t = np.zeros(4)
    hi_t[0] = 5.0 * T * fib.shape[0]
    for s in range(0, fib.shape[0], chunk):
        f = fib[s:s + chunk]
        n = f.shape[0]
        d10 = _d2(f[:, None, 10], cen[None, :, 10])                          # [n, M]
        d00, d2020 = _d2(f[:, None, 0], cen[None, :, 0]), _d2(f[:, None, 20], cen[None, :, 20])
        d020, d200 = _d2(f[:, None, 0], cen[None, :, 20]), _d2(f[:, None, 20], cen[None, :, 0])
        r_dir = np.maximum(d10, np.maximum(d00, d2020))                     # 3-point maxima per orientation
        r_inv = np.maximum(d10, np.maximum(d020, d200))
        r_min = np.minimum(r_dir, r_inv)
        # per (fiber, tile, lane)
        R = r_min[:, mem]                                                     # [n, T, 32]
        D10 = d10[:, mem]
        RD, RI = r_dir[:, mem], r_inv[:, mem]
        tau_min = np.minimum(thr2_t[None], np.asarray(final_d2[s:s + n], np.float64)[:, None])   # [n, T]
        listed = (R <= (thr2_t[None, :, None] * (1 - REL))).any(-1)         # guaranteed listed
        fin = (R <= (tau_min[:, :, None] * (1 - REL))).any(-1)              # guaranteed to pass at any cutoff
        must = listed & fin
        lo_t[0] += 5.0 * listed.sum()
        lo_t[1] += 32.0 * must.sum()
        lo_t[2] += 4.0 * ((D10 <= tau_min[:, :, None] * (1 - REL)) & must[:, :, None]).sum()
        lo_t[3] += 18.0 * np.isfinite(final_d2[s:s + n]).sum()
        # upper bounds
        may = (box_d2(f[:, 10].astype(np.float64), b10lo, b10hi) <= s_up[None]) & \
              (box_d2(f[:, 0].astype(np.float64), belo, behi) <= s_up[None]) & \
              (box_d2(f[:, 20].astype(np.float64), belo, behi) <= s_up[None])  # [n, T]
        hi_t[1] += 32.0 * may.sum()
        norm = (f[:, None, 10].astype(np.float64) ** 2).sum(-1)[:, :, None] + (c10m.astype(np.float64) ** 2).sum(-1)[None]
        scr = D10 <= thr2_t[None, :, None] * (1 + REL) + 2.0 ** -15 * norm
        hi_t[2] += 4.0 * (scr & may[:, :, None]).sum()
        cut = thr2_t[None, :, None] * (1 + REL)
        hi_t[3] += 18.0 * (((RD <= cut).astype(np.int64) + (RI <= cut)) * may[:, :, None]).sum()
    return lo_t, hi_t


def kernel_terms(stats):
    """The stats kernel's four terms (T1..T4) from seg_classify_stats counters."""
    t1 = 5.0 * stats["lane_bound_tests"]
    t2 = float(stats["lane_test1"])
    t3 = 4.0 * stats["lane_test2"]
    t4 = float(stats["lane_point_dists"]) - t1 - t2 - t3
    return np.array([t1, t2, t3, t4])
