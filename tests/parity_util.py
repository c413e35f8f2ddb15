"""Parity rule of the hot path (BASELINE.json north_star; DESIGN.md Sec. 2 'Parity rule').

Labels must equal the oracle's for every decidable fiber (deciding distance more than
1e-3 mm from its threshold and from the runner-up bundle; paper mode also outside the
orientation band of reading R20); winning distances within 1e-5 relative (0 <-> 0 exactly);
unlabelled fibers carry +inf; non-finite fibers NaN.

Undecidable fibers have several correct answers.  check_valid() holds the GPU's answer for them
to being one of those, from the oracle's per-bundle intervals [lo_b, hi_b] of correct values
(exact mode lo = hi = d_b; paper mode [L_b, H_b]):
  label g >= 0 : lo_g (1 - 1e-5) <= dist <= hi_g (1 + 1e-5), dist <= thr_g + delta, and no other
                 bundle b is certainly accepted (hi_b < thr_b - delta) and certainly closer
                 (hi_b < dist - delta);
  label -1     : dist = +inf and no bundle is certainly accepted.
"""
import numpy as np

DIST_RTOL = 1e-5
DELTA_MM = 1e-3


def check_parity(label, dist, ref, what=""):
    label = np.asarray(label)
    dist = np.asarray(dist, np.float64)
    rl, rd, dec = ref["label"], ref["dist"], ref["decidable"]
    bad = np.nonzero(dec & (label != rl))[0]
    assert bad.size == 0, (f"{what}: {bad.size} decidable label mismatches, first {bad[:10]} "
                           f"gpu={label[bad[:10]]} oracle={rl[bad[:10]]} "
                           f"gpu_d={dist[bad[:10]]} oracle_d={rd[bad[:10]]}")
    same = (label == rl) & (rl >= 0) & dec
    err = np.abs(dist[same] - rd[same])
    lim = DIST_RTOL * rd[same]
    worst = np.nonzero(err > lim)[0]
    assert worst.size == 0, f"{what}: {worst.size} distances outside 1e-5 rel, e.g. {dist[same][worst[:5]]} vs {rd[same][worst[:5]]}"
    un = (rl < 0) & dec & ~np.isnan(rd)
    assert np.all(np.isinf(dist[un]) & (dist[un] > 0)), f"{what}: unlabelled fibers must carry +inf"
    nan = np.isnan(rd)
    assert np.all(np.isnan(dist[nan]) & (label[nan] == -1)), f"{what}: non-finite fibers must be -1/NaN"
    return dict(n=int(label.size), tie_band=int((~dec).sum()), labelled=int((rl >= 0).sum()))


def valid_answers(label, dist, lo, hi, thresh, delta=DELTA_MM):
    """Boolean per fiber: is (label, dist) one of the correct answers given the per-bundle intervals
    lo, hi [n, B] (mm) of the oracle?  (See the module docstring.)"""
    label = np.asarray(label)
    dist = np.asarray(dist, np.float64)
    thr = np.asarray(thresh, np.float64)[None, :]
    certain = hi < thr - delta                                   # [n, B] certainly accepted
    ok = np.zeros(label.size, bool)
    for i in range(label.size):
        g, d = int(label[i]), float(dist[i])
        if g < 0:
            ok[i] = np.isinf(d) and d > 0 and not certain[i].any()
            continue
        if g >= lo.shape[1] or not np.isfinite(d):
            continue
        in_band = lo[i, g] * (1 - DIST_RTOL) <= d <= hi[i, g] * (1 + DIST_RTOL) and d <= thr[0, g] + delta
        others = certain[i].copy()
        others[g] = False
        beaten = np.any(others & (hi[i] < d - delta))
        ok[i] = bool(in_band and not beaten)
    return ok


def check_valid(label, dist, idx, lo, hi, thresh, what=""):
    """Assert that the answers at fiber indices idx (the undecidable ones) are valid."""
    if len(idx) == 0:
        return 0
    label = np.asarray(label)[idx]
    dist = np.asarray(dist, np.float64)[idx]
    ok = valid_answers(label, dist, lo, hi, thresh)
    bad = np.nonzero(~ok)[0]
    assert bad.size == 0, (f"{what}: {bad.size} of {len(idx)} tie-band answers are not valid, e.g. fiber "
                           f"{np.asarray(idx)[bad[:5]]} gpu=({label[bad[:5]]}, {dist[bad[:5]]})")
    return int(len(idx))


def check_parity_full(label, dist, fibers, ref, centroids, bundle_id, thresh, mode="exact", what=""):
    """check_parity plus the valid-answer check of every undecidable fiber (bands from the plain oracle)."""
    import oracle
    r = check_parity(label, dist, ref, what)
    und = np.nonzero(~np.asarray(ref["decidable"]))[0]
    if und.size:
        b = oracle.classify(np.asarray(fibers)[und], centroids, bundle_id, thresh, mode=mode, want_bands=True)
        r["tie_band_valid"] = check_valid(label, dist, und, b["lo"], b["hi"], thresh, what)
    return r
