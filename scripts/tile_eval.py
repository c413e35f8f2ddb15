"""Offline evaluation of tile plans (row a0) on a fiber sample, CPU only.

For a plan (tiles of 32 same-bundle centroids, each bounded by spheres of points 0/10/20) count, over
a sample of fibers, the (fiber, tile) pairs the exact tile bound passes and, among them, the centroid
pairs surviving test1 / test2.  Two cutoffs bracket the kernel's live one: tau = thr^2 (no best yet)
and tau = min(thr^2, d_final^2) (every fiber seeded with its final best; d_final from the oracle).
Dense work in k_classify is ~32 lanes x passing pairs, so fewer passes at equal survivors is better.

python scripts/tile_eval.py [cfg] [n_fibers]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_1912_11494_b200 import binding
from synth import atlas_for_config, fibers_for_config, sample_indices

TILE = 32
EPS = 1e-3


def current_plan(at):
    T = binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, 0)
    tb = np.zeros(T, np.int32)
    mem = np.zeros(T * TILE, np.int32)
    sph = np.zeros(T * 12, np.float32)
    binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, T, tb, mem, sph)
    return tb, mem.reshape(T, TILE), sph.reshape(T, 3, 4)


def canon_flips(at):
    """The same canonicalisation as seg_create: reverse a centroid if that brings its end points
    closer to its bundle's first member."""
    C = at.centroids.astype(np.float64)
    fl = np.zeros(at.M, bool)
    for b in range(at.B):
        ids = np.nonzero(at.bundle_id == b)[0]
        if len(ids) == 0:
            continue
        r = C[ids[0]]
        same = ((C[ids, 0] - r[0]) ** 2).sum(1) + ((C[ids, 20] - r[20]) ** 2).sum(1)
        rev = ((C[ids, 20] - r[0]) ** 2).sum(1) + ((C[ids, 0] - r[20]) ** 2).sum(1)
        fl[ids] = rev < same
    return fl


def feats(at, fl):
    C = at.centroids.astype(np.float64)
    Cc = np.where(fl[:, None, None], C[:, ::-1], C)
    return Cc, np.concatenate([Cc[:, 0], Cc[:, 10], Cc[:, 20]], 1)   # [M, 9]


def split_pca(F, ids, out):
    n = len(ids)
    if n <= TILE:
        out.append(ids)
        return
    left = ((n + TILE - 1) // TILE // 2) * TILE
    X = F[ids] - F[ids].mean(0)
    w, v = np.linalg.eigh(X.T @ X)
    proj = X @ v[:, -1]
    o = np.argsort(proj, kind="stable")
    split_pca(F, ids[o[:left]], out)
    split_pca(F, ids[o[left:]], out)


def plan_pca(at, fl):
    _, F = feats(at, fl)
    tiles, tb = [], []
    for b in range(at.B):
        ids = np.nonzero(at.bundle_id == b)[0]
        if len(ids) == 0:
            continue
        out = []
        split_pca(F, ids, out)
        for t in out:
            tiles.append(np.sort(t))
            tb.append(b)
    return np.array(tb, np.int32), tiles


def refine_kmeans(at, fl, tb, tiles, iters=10):
    """Balanced k-means within each bundle: every tile keeps its size, members swap between tiles of
    the same bundle toward the nearest tile mean (9-D), by a greedy sorted assignment."""
    _, F = feats(at, fl)
    tiles = [np.array(t) for t in tiles]
    for b in range(at.B):
        ks = [k for k in range(len(tiles)) if tb[k] == b]
        if len(ks) < 2:
            continue
        ids = np.concatenate([tiles[k] for k in ks])
        cap = np.array([len(tiles[k]) for k in ks])
        for _ in range(iters):
            mu = np.stack([F[tiles[k]].mean(0) for k in ks])
            D = ((F[ids][:, None, :] - mu[None]) ** 2).sum(-1)   # [n, K]
            # greedy: pairs in increasing distance, respecting the capacities
            order = np.argsort(D, axis=None, kind="stable")
            assigned = -np.ones(len(ids), int)
            fill = np.zeros(len(ks), int)
            left = len(ids)
            for flat in order:
                i, k = divmod(int(flat), len(ks))
                if assigned[i] >= 0 or fill[k] >= cap[k]:
                    continue
                assigned[i] = k
                fill[k] += 1
                left -= 1
                if left == 0:
                    break
            new = [np.sort(ids[assigned == j]) for j in range(len(ks))]
            same = all(np.array_equal(new[j], tiles[ks[j]]) for j in range(len(ks)))
            for j, k in enumerate(ks):
                tiles[k] = new[j]
            if same:
                break
    return tiles


def spheres_bbox(Cc, t):
    out = np.zeros((3, 4))
    for q, pt in enumerate((0, 10, 20)):
        P = Cc[t, pt]
        c = 0.5 * (P.min(0) + P.max(0))
        c = c.astype(np.float32).astype(np.float64)
        out[q, :3] = c
        out[q, 3] = np.sqrt(((P - c) ** 2).sum(1).max())
    return out


def spheres_meb(Cc, t, iters=400):
    """Approximate minimum enclosing ball (Badoiu-Clarkson), then the exact radius about that centre."""
    out = np.zeros((3, 4))
    for q, pt in enumerate((0, 10, 20)):
        P = Cc[t, pt]
        c = 0.5 * (P.min(0) + P.max(0))
        for i in range(1, iters + 1):
            far = P[np.argmax(((P - c) ** 2).sum(1))]
            c = c + (far - c) / (i + 1)
        c = c.astype(np.float32).astype(np.float64)
        r_bb = spheres_bbox(Cc, t)[q, 3]
        r = np.sqrt(((P - c) ** 2).sum(1).max())
        if r > r_bb:   # keep the better of the two centres
            out[q] = spheres_bbox(Cc, t)[q]
        else:
            out[q, :3] = c
            out[q, 3] = r
    return out


def evaluate(name, at, Cc, tb, tiles, S, fib, dfin):
    """S [T, 3, 4] spheres.  Returns pass counts and test1/test2 survivors for both cutoffs."""
    T = len(tiles)
    TM = np.stack([np.concatenate([t, np.full(TILE - len(t), t[0])]) for t in tiles])     # [T, 32]
    TV = np.stack([np.arange(TILE) < len(t) for t in tiles])                              # [T, 32]
    thr2 = (at.thresh.astype(np.float64) ** 2)[tb]                     # [T]
    f0, f10, f20 = (fib[:, p].astype(np.float64) for p in (0, 10, 20))
    res = {}
    for tname, seeded in (("static", False), ("seeded", True)):
        npass = nt1 = nt2 = 0
        for a in range(0, len(fib), 500):
            sl = slice(a, a + 500)
            tau = np.broadcast_to(thr2[None], (len(f0[sl]), T)).copy()
            if seeded:
                tau = np.minimum(tau, (dfin[sl, None].astype(np.float64) ** 2))
            s = np.sqrt(tau) + EPS

            def inside(P, q):
                d = np.sqrt(((P[:, None, :] - S[None, :, q, :3]) ** 2).sum(-1))
                return d <= S[None, :, q, 3] + s
            p10 = inside(f10[sl], 1)
            pd = inside(f0[sl], 0) & inside(f20[sl], 2)
            pi = inside(f20[sl], 0) & inside(f0[sl], 2)
            ps = p10 & (pd | pi)
            fi, ti = np.nonzero(ps)
            npass += len(fi)
            if len(fi):
                M, V = TM[ti], TV[ti]                                    # [P, 32]
                tt = tau[fi, ti][:, None]
                m10 = ((f10[sl][fi][:, None] - Cc[M, 10]) ** 2).sum(-1)
                t1 = (m10 <= tt) & V
                nt1 += int(t1.sum())
                e00 = ((f0[sl][fi][:, None] - Cc[M, 0]) ** 2).sum(-1)
                e22 = ((f20[sl][fi][:, None] - Cc[M, 20]) ** 2).sum(-1)
                e02 = ((f0[sl][fi][:, None] - Cc[M, 20]) ** 2).sum(-1)
                e20 = ((f20[sl][fi][:, None] - Cc[M, 0]) ** 2).sum(-1)
                t2 = t1 & ((np.maximum(e00, e22) <= tt) | (np.maximum(e02, e20) <= tt))
                nt2 += int(t2.sum())
        res[tname] = (npass, nt1, nt2)
    n = len(fib)
    print(f"{name:28s} T={T:5d} | static: pass/fiber {res['static'][0] / n:7.2f} t1 {res['static'][1] / n:7.2f} "
          f"t2 {res['static'][2] / n:6.2f} | seeded: pass/fiber {res['seeded'][0] / n:6.2f} "
          f"t1 {res['seeded'][1] / n:6.2f} t2 {res['seeded'][2] / n:5.2f}", flush=True)
    return res


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 4000
    at = atlas_for_config(cfg)
    full = fibers_for_config(cfg, 0, 200000)
    idx = sample_indices(len(full), n, seed=5)
    fib = full[idx]
    t0 = time.time()
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    lab, dist = r["label"], r["dist"]
    dfin = np.where(lab >= 0, dist, np.inf)
    print(f"oracle {time.time() - t0:.1f}s; labelled {np.mean(lab >= 0):.3f}", flush=True)
    fl = canon_flips(at)
    Cc, _ = feats(at, fl)

    tb, mem, sph = current_plan(at)
    tiles_cur = [np.unique(m) for m in mem]
    evaluate("current (C plan)", at, Cc, tb, tiles_cur, sph.astype(np.float64), fib, dfin)
    evaluate("current + MEB spheres", at, Cc, tb, tiles_cur, np.stack([spheres_meb(Cc, t) for t in tiles_cur]),
             fib, dfin)
    tbp, tiles_p = plan_pca(at, fl)
    evaluate("pca split", at, Cc, tbp, tiles_p, np.stack([spheres_bbox(Cc, t) for t in tiles_p]), fib, dfin)
    evaluate("pca split + MEB", at, Cc, tbp, tiles_p, np.stack([spheres_meb(Cc, t) for t in tiles_p]), fib, dfin)
    tiles_k = refine_kmeans(at, fl, tbp, tiles_p)
    evaluate("pca + kmeans + MEB", at, Cc, tbp, tiles_k, np.stack([spheres_meb(Cc, t) for t in tiles_k]), fib, dfin)


if __name__ == "__main__":
    main()


def seed_eval(cfg=3, n=2000, reps=1):
    """Quality of a cheap seed: the fiber's nearest tile by sphere centres (max of the point-10 and the
    better-orientation end-point centre distances), then the exact d_ME against that tile's
    representative member (the member nearest its sphere centres)."""
    at = atlas_for_config(cfg)
    full = fibers_for_config(cfg, 0, 200000)
    fib = full[sample_indices(len(full), n, seed=5)].astype(np.float64)
    r = oracle.classify(fib.astype(np.float32), at.centroids, at.bundle_id, at.thresh)
    lab, dfin = r["label"], np.where(r["label"] >= 0, r["dist"], np.inf)
    tb, mem, sph = current_plan(at)
    S = sph.astype(np.float64)
    C = at.centroids.astype(np.float64)
    fl = canon_flips(at)
    Cc, _ = feats(at, fl)
    # representative of each tile: member minimising the max distance to the three sphere centres
    rep = np.zeros(len(tb), int)
    for t in range(len(tb)):
        m = np.unique(mem[t])
        d = np.max([np.sqrt(((Cc[m, p] - S[t, q, :3]) ** 2).sum(1)) for q, p in enumerate((0, 10, 20))], axis=0)
        rep[t] = m[np.argmin(d)]
    f0, f10, f20 = fib[:, 0], fib[:, 10], fib[:, 20]
    dc = lambda P, q: np.sqrt(((P[:, None] - S[None, :, q, :3]) ** 2).sum(-1))
    prox = np.maximum(dc(f10, 1), np.minimum(np.maximum(dc(f0, 0), dc(f20, 2)), np.maximum(dc(f20, 0), dc(f0, 2))))
    order = np.argsort(prox, axis=1)[:, :reps]
    thr = at.thresh.astype(np.float64)
    dseed = np.full(n, np.inf)
    for k in range(reps):
        t = order[:, k]
        c = C[rep[t]]
        dd = np.minimum(np.sqrt(((fib - c) ** 2).sum(-1)).max(1), np.sqrt(((fib - c[:, ::-1]) ** 2).sum(-1)).max(1))
        ok = dd <= thr[tb[t]]
        dseed = np.where(ok, np.minimum(dseed, dd), dseed)
    lbl = np.isfinite(dfin)
    print(f"reps={reps}: labelled {lbl.mean():.3f}; seeded {np.isfinite(dseed).mean():.3f} "
          f"(of labelled {np.isfinite(dseed[lbl]).mean():.3f}); seed == final {np.mean(dseed[lbl] <= dfin[lbl] * (1 + 1e-6)):.3f}; "
          f"median d_seed/d_final {np.median(dseed[lbl & np.isfinite(dseed)] / dfin[lbl & np.isfinite(dseed)]):.3f}")
    return dseed, dfin
