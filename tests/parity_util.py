"""Parity rule of the hot path (BASELINE.json north_star; DESIGN.md Sec. 3 'Parity').

Labels must equal the oracle's for every decidable fiber (deciding distance more than
1e-3 mm from its threshold and from the runner-up bundle); winning distances within
1e-5 relative (0 <-> 0 exactly); unlabelled fibers carry +inf; non-finite fibers NaN.
"""
import numpy as np

DIST_RTOL = 1e-5


def check_parity(label, dist, ref, what=""):
    label = np.asarray(label)
    dist = np.asarray(dist, np.float64)
    rl, rd, dec = ref["label"], ref["dist"], ref["decidable"]
    bad = np.nonzero(dec & (label != rl))[0]
    assert bad.size == 0, (f"{what}: {bad.size} decidable label mismatches, first {bad[:10]} "
                           f"gpu={label[bad[:10]]} oracle={rl[bad[:10]]} "
                           f"gpu_d={dist[bad[:10]]} oracle_d={rd[bad[:10]]}")
    same = (label == rl) & (rl >= 0)
    err = np.abs(dist[same] - rd[same])
    lim = DIST_RTOL * rd[same]
    worst = np.nonzero(err > lim)[0]
    assert worst.size == 0, f"{what}: {worst.size} distances outside 1e-5 rel, e.g. {dist[same][worst[:5]]} vs {rd[same][worst[:5]]}"
    un = (rl < 0) & dec & ~np.isnan(rd)
    assert np.all(np.isinf(dist[un]) & (dist[un] > 0)), f"{what}: unlabelled fibers must carry +inf"
    nan = np.isnan(rd)
    assert np.all(np.isnan(dist[nan]) & (label[nan] == -1)), f"{what}: non-finite fibers must be -1/NaN"
    return dict(n=int(label.size), tie_band=int((~dec).sum()), labelled=int((rl >= 0).sum()))
