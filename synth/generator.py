"""Seeded synthetic stand-ins for the paper's workloads (BASELINE.json configs 0-4).

The paper measures on real ARCHI tractography segmented with the LNAO-SWM79 atlas
(100 bundles / 7,753 centroids, Sec. 2.2) and a whole-brain atlas
(62 bundles / 44,345 centroids).  Neither dataset is available, so
these generators reproduce their *shapes*: fiber counts, bundle and centroid
counts, 21 points per fiber, per-bundle thresholds.  The
recipe is the one DESIGN.md Sec. "Input recipe" states; it is frozen here.

Everything is float64 internally and returned as float32 [*, 21, 3] (mm).
Randomness comes from numpy PCG64 streams keyed by SeedSequence entropy lists,
so any contiguous fiber range can be regenerated independently (chunks of
CHUNK fibers), which is what the multi-rank bench and the sampled parity tests use.
"""
from __future__ import annotations

import dataclasses
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np

N_POINTS = 21            # every fiber / centroid has 21 points
CHUNK = 1 << 16          # fibers per independently seeded chunk
_N_CURVE = 201           # samples of the analytic curve before resampling
BOX_LO = np.array([-70.0, -90.0, -60.0])   # BASELINE.json configs[0]
BOX_HI = np.array([70.0, 90.0, 80.0])

# cfg -> workload description (BASELINE.json configs[0..4])
CONFIGS = {
    0: dict(name="cfg0-tiny", n_fibers=2_000, atlas_key=0, n_bundles=10, n_centroids=500,
            split="even", lengths=(20.0, 80.0), thresh=(4.0, 8.0), p_match=0.7, sigma_fiber=1.5),
    1: dict(name="cfg1-swm79-100k", n_fibers=100_000, atlas_key=1, n_bundles=100, n_centroids=7_753,
            split="dirichlet", lengths=(20.0, 80.0), thresh=(4.0, 8.0), p_match=0.7, sigma_fiber=1.5),
    2: dict(name="cfg2-swm79-955k", n_fibers=955_000, atlas_key=1, n_bundles=100, n_centroids=7_753,
            split="dirichlet", lengths=(20.0, 80.0), thresh=(4.0, 8.0), p_match=0.7, sigma_fiber=1.5),
    3: dict(name="cfg3-wholebrain-4.145M", n_fibers=4_145_000, atlas_key=3, n_bundles=62,
            n_centroids=44_345, split="dirichlet", lengths=(30.0, 150.0), thresh=(5.0, 10.0),
            p_match=0.7, sigma_fiber=1.5),
    4: dict(name="cfg4-adversarial-8M", n_fibers=8_000_000, atlas_key=3, n_bundles=62,
            n_centroids=44_345, split="dirichlet", lengths=(30.0, 150.0), thresh=(5.0, 10.0),
            p_match=1.0, sigma_fiber=3.0),
}
SIGMA_CENTROID = 2.0     # BASELINE.json configs[0]: centroid = base curve + smooth N(0, 2 mm)
P_REVERSE = 0.5          # BASELINE.json configs[0]: matched fibers reversed with p = 0.5


def _rng(*entropy: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([1912, 11494, *entropy])))


# --------------------------------------------------------------------------------------
# geometry helpers (input construction only)
# --------------------------------------------------------------------------------------
def resample_equidistant(pts: np.ndarray, n: int = N_POINTS) -> np.ndarray:
    """Resample polylines [m, K, 3] to n points equidistant in arc length.

    Chord-length parameterisation with linear interpolation;
    endpoints are kept exactly.
    """
    pts = np.asarray(pts, dtype=np.float64)
    m, k, _ = pts.shape
    seg = np.linalg.norm(np.diff(pts, axis=1), axis=2)             # [m, K-1]
    cum = np.concatenate([np.zeros((m, 1)), np.cumsum(seg, axis=1)], axis=1)
    total = cum[:, -1:]
    targets = total * (np.arange(n, dtype=np.float64) / (n - 1))[None, :]
    big = float(np.max(total)) * 2.0 + 1.0
    off = (np.arange(m, dtype=np.float64) * big)[:, None]
    idx = np.searchsorted((cum + off).ravel(), (targets + off).ravel(), side="right")
    idx = idx.reshape(m, n) - 1 - (np.arange(m) * k)[:, None]
    idx = np.clip(idx, 0, k - 2)
    rows = np.arange(m)[:, None]
    c0 = cum[rows, idx]
    sl = seg[rows, idx]
    w = np.where(sl > 0, (targets - c0) / np.where(sl > 0, sl, 1.0), 0.0)
    w = np.clip(w, 0.0, 1.0)[..., None]
    p0 = pts[rows, idx]
    p1 = pts[rows, idx + 1]
    out = p0 + w * (p1 - p0)
    out[:, 0] = pts[:, 0]
    out[:, -1] = pts[:, -1]
    return out


def reverse_fibers(f: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(f[:, ::-1, :])


def _unit(v: np.ndarray) -> np.ndarray:
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


_T = np.linspace(0.0, 1.0, _N_CURVE)
# canonical curve: cubic Bezier P0=(0,0), P1=(1/3,h), P2=(2/3,h), P3=(1,0) in the
# (chord, normal) plane; it evaluates to x(t)=t, y(t)=3 h t (1-t).
_H_GRID = np.linspace(0.0, 4.0, 4097)


def _canon_len(h: np.ndarray) -> np.ndarray:
    y = 3.0 * h[:, None] * (_T * (1.0 - _T))[None, :]
    dx = np.diff(_T)[None, :]
    dy = np.diff(y, axis=1)
    return np.sqrt(dx * dx + dy * dy).sum(axis=1)


_L_GRID = _canon_len(_H_GRID)        # monotone increasing in h


def _base_curves(rng: np.random.Generator, n: int, lmin: float, lmax: float) -> np.ndarray:
    """n random curved fibers of length ~U(lmin,lmax), resampled to 21 points.

    P0 ~ U(box); chord = u L, u ~ U(0.7, 0.95); chord direction uniform on S^2;
    P3 = P0 + chord * dir must fall inside the box (rejection); the bend h is
    chosen so that the canonical arc length equals 1/u (table inversion).
    """
    out = np.empty((n, N_POINTS, 3))
    got = 0
    while got < n:
        k = max(2 * (n - got), 64)
        length = rng.uniform(lmin, lmax, size=k)
        u = rng.uniform(0.7, 0.95, size=k)
        p0 = rng.uniform(BOX_LO, BOX_HI, size=(k, 3))
        d = _unit(rng.standard_normal((k, 3)))
        g = rng.standard_normal((k, 3))
        nrm = _unit(g - (g * d).sum(axis=1, keepdims=True) * d)
        chord = u * length
        p3 = p0 + chord[:, None] * d
        ok = np.all((p3 >= BOX_LO) & (p3 <= BOX_HI), axis=1)
        idx = np.nonzero(ok)[0][: n - got]
        if idx.size == 0:
            continue
        h = np.interp(1.0 / u[idx], _L_GRID, _H_GRID)
        y = 3.0 * h[:, None] * (_T * (1.0 - _T))[None, :]
        curve = (p0[idx, None, :]
                 + chord[idx, None, None] * (_T[None, :, None] * d[idx, None, :]
                                              + y[:, :, None] * nrm[idx, None, :]))
        out[got:got + idx.size] = resample_equidistant(curve)
        got += idx.size
    return out


_TK = np.arange(N_POINTS) / (N_POINTS - 1.0)
_BERN = np.stack([(1 - _TK) ** 3, 3 * (1 - _TK) ** 2 * _TK, 3 * (1 - _TK) * _TK ** 2, _TK ** 3], axis=1)
_BERN_N = _BERN / np.sqrt((_BERN ** 2).sum(axis=1, keepdims=True))   # [21, 4], rows unit norm


def _smooth_displace(rng: np.random.Generator, f: np.ndarray, sigma: float) -> np.ndarray:
    """f + smooth Gaussian displacement with marginal SD sigma per coordinate, re-resampled."""
    eps = rng.standard_normal((f.shape[0], 4, 3)) * sigma
    disp = np.einsum("kj,njc->nkc", _BERN_N, eps)
    return resample_equidistant(f + disp)


# --------------------------------------------------------------------------------------
# atlas
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class Atlas:
    centroids: np.ndarray    # float32 [M, 21, 3]
    bundle_id: np.ndarray    # int32 [M]
    thresh: np.ndarray       # float32 [B]

    @property
    def M(self) -> int:
        return int(self.centroids.shape[0])

    @property
    def B(self) -> int:
        return int(self.thresh.shape[0])


def _split_counts(rng: np.random.Generator, m: int, b: int, split: str) -> np.ndarray:
    if split == "even":
        assert m % b == 0
        return np.full(b, m // b, dtype=np.int64)
    w = rng.dirichlet(np.ones(b))
    raw = w * (m - b)
    counts = 1 + np.floor(raw).astype(np.int64)
    rem = m - counts.sum()
    order = np.argsort(-(raw - np.floor(raw)), kind="stable")
    counts[order[:rem]] += 1
    return counts


_ATLAS_CACHE: dict[int, Atlas] = {}


def atlas_for_config(cfg: int) -> Atlas:
    """Atlas of config cfg (configs 1-2 share atlas key 1, configs 3-4 share key 3)."""
    spec = CONFIGS[cfg]
    key = spec["atlas_key"]
    if key in _ATLAS_CACHE:
        return _ATLAS_CACHE[key]
    rng = _rng(key, 0)
    b, m = spec["n_bundles"], spec["n_centroids"]
    counts = _split_counts(rng, m, b, spec["split"])
    lmin, lmax = spec["lengths"]
    base = _base_curves(rng, b, lmin, lmax)
    bundle_id = np.repeat(np.arange(b, dtype=np.int32), counts)
    cents = _smooth_displace(rng, base[bundle_id], SIGMA_CENTROID)
    thresh = rng.uniform(*spec["thresh"], size=b).astype(np.float32)
    # centroids are stored shuffled: the library must not rely on grouping by bundle
    perm = rng.permutation(m)
    at = Atlas(np.ascontiguousarray(cents[perm], dtype=np.float32),
               np.ascontiguousarray(bundle_id[perm], dtype=np.int32), thresh)
    _ATLAS_CACHE[key] = at
    return at


# --------------------------------------------------------------------------------------
# subject fibers
# --------------------------------------------------------------------------------------
def _chunk(cfg: int, c: int, subject: int) -> tuple[np.ndarray, np.ndarray]:
    spec = CONFIGS[cfg]
    at = atlas_for_config(cfg)
    n_total = spec["n_fibers"]
    start = c * CHUNK
    n = min(CHUNK, n_total - start)
    rng = _rng(cfg, 1, c) if subject == 0 else _rng(cfg, 1, c, subject)
    matched = rng.random(n) < spec["p_match"]
    nm = int(matched.sum())
    src = rng.integers(0, at.M, size=nm)
    f = np.empty((n, N_POINTS, 3))
    mf = _smooth_displace(rng, at.centroids[src].astype(np.float64), spec["sigma_fiber"])
    rev = rng.random(nm) < P_REVERSE
    mf[rev] = mf[rev, ::-1, :]
    f[matched] = mf
    lmin, lmax = spec["lengths"]
    if n - nm:
        f[~matched] = _base_curves(rng, n - nm, lmin, lmax)
    truth = np.full(n, -1, dtype=np.int32)
    truth[matched] = at.bundle_id[src]
    return f.astype(np.float32), truth


def _chunk_star(args):
    return _chunk(*args)


def fibers_for_config(cfg: int, start: int = 0, stop: int | None = None, subject: int = 0,
                      workers: int | None = None, with_truth: bool = False):
    """Subject fibers [start, stop) of config cfg as float32 [n, 21, 3].

    subject > 0 selects an independent subject of the same shape (weak-scaling
    ranks); subject 0 is the config's canonical subject.
    """
    n_total = CONFIGS[cfg]["n_fibers"]
    stop = n_total if stop is None else min(stop, n_total)
    if stop <= start:
        e = np.empty((0, N_POINTS, 3), np.float32)
        return (e, np.empty(0, np.int32)) if with_truth else e
    c0, c1 = start // CHUNK, (stop - 1) // CHUNK + 1
    jobs = [(cfg, c, subject) for c in range(c0, c1)]
    atlas_for_config(cfg)  # build once before forking
    if workers is None:
        workers = min(len(jobs), os.cpu_count() or 1, 32)
    if workers > 1 and len(jobs) > 1:
        import multiprocessing as mp
        with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork")) as ex:
            parts = list(ex.map(_chunk_star, jobs))
    else:
        parts = [_chunk(*j) for j in jobs]
    f = np.concatenate([p[0] for p in parts])
    t = np.concatenate([p[1] for p in parts])
    lo = start - c0 * CHUNK
    f = np.ascontiguousarray(f[lo:lo + (stop - start)])
    t = t[lo:lo + (stop - start)]
    return (f, t) if with_truth else f


def sample_indices(n: int, k: int, seed: int = 0) -> np.ndarray:
    """k distinct sorted fiber indices in [0, n), always including the first and last."""
    rng = _rng(999, seed)
    if k >= n:
        return np.arange(n)
    idx = rng.choice(n, size=k, replace=False)
    idx[0], idx[-1] = 0, n - 1
    return np.unique(idx)
