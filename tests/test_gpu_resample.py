"""GPU parity of row f2 (seg_resample) against oracle/resample.py.

Both sides compute arc lengths and the interpolation in double (summation orders differ) and round
each coordinate to FP32 once, so the outputs agree to within one FP32 ulp; end
points are copied exactly.  Invalid fibers come out as NaN on both sides.
"""
import numpy as np
import pytest
import torch

import oracle
import oracle.resample as R
from parity_util import check_parity
from synth import atlas_for_config, fibers_for_config, sample_indices
from synth.raw import raw_streamlines

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas, SegError, resample


def _gpu(points, offsets):
    out = resample(torch.from_numpy(points).cuda(), torch.from_numpy(offsets).cuda())
    torch.cuda.synchronize()
    return out.cpu().numpy()


def _ulp_ok(got, want):
    fin = np.isfinite(want)
    assert np.array_equal(np.isnan(got), np.isnan(want))
    diff = np.abs(got[fin].astype(np.float64) - want[fin].astype(np.float64))
    ulp = np.spacing(np.abs(want[fin])).astype(np.float64)
    assert np.all(diff <= ulp), f"max {np.max(diff / ulp):.2f} ulp"


@pytest.mark.parametrize("n,seed", [(1, 0), (31, 1), (2000, 2), (20_000, 3)])
def test_resample_parity(n, seed):
    fib = fibers_for_config(0, 0, min(n, 2000))
    if n > fib.shape[0]:
        fib = np.concatenate([fib] * (-(-n // fib.shape[0])))[:n]
    pts, off = raw_streamlines(fib, seed)
    got = _gpu(pts, off)
    k = min(n, 3000)
    _ulp_ok(got[:k], R.resample(pts, off[:k + 1]))
    assert np.array_equal(got[:, 0], pts[off[:-1]]) and np.array_equal(got[:, 20], pts[off[1:] - 1])


def test_resample_long_and_degenerate():
    rng = np.random.default_rng(5)
    polys = [np.cumsum(rng.normal(0, 1, (m, 3)), 0) for m in (2, 3, 33, 64, 65, 1000, 4097)]
    polys += [np.ones((7, 3)), np.zeros((1, 3)), np.array([[0, 0, 0], [0, 0, 0], [1, 0, 0]])]
    bad = np.cumsum(rng.normal(0, 1, (10, 3)), 0)
    bad[4, 2] = np.inf
    polys.append(bad)
    off = np.concatenate([[0], np.cumsum([p.shape[0] for p in polys])]).astype(np.int64)
    pts = np.concatenate(polys).astype(np.float32)
    _ulp_ok(_gpu(pts, off), R.resample(pts, off))


def test_resample_equidistant_is_identity():
    """a fiber that already has 21 equidistant points comes back unchanged (1e-5 per
    coordinate).  Helices sampled at equal parameter steps have exactly equal chords."""
    rng = np.random.default_rng(6)
    fibs = []
    for _ in range(500):
        r, th, c = rng.uniform(5, 30), rng.uniform(0.05, 0.4), rng.uniform(-3, 3)
        k = np.arange(21)
        fibs.append(np.stack([r * np.cos(k * th), r * np.sin(k * th), c * k], 1) + rng.uniform(-50, 50, 3))
    fib = np.array(fibs, np.float32)
    off = np.arange(0, 21 * 501, 21, dtype=np.int64)
    got = _gpu(np.ascontiguousarray(fib.reshape(-1, 3)), off)
    assert np.abs(got - fib).max() <= 1e-5


def test_resample_then_classify_matches_oracle_chain():
    """The whole front end: raw streamlines -> seg_resample -> seg_classify, against the oracle's
    resampling followed by the oracle's classification (cfg 0)."""
    at = atlas_for_config(0)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    pts, off = raw_streamlines(fibers_for_config(0), 7)
    f = resample(torch.from_numpy(pts).cuda(), torch.from_numpy(off).cuda())
    lab, d = A.classify(f)
    torch.cuda.synchronize()
    ref_fib = R.resample(pts, off)
    ref = oracle.classify(ref_fib, at.centroids, at.bundle_id, at.thresh)
    check_parity(lab.cpu().numpy(), d.cpu().numpy(), ref, "raw -> resample -> classify")


def test_resample_errors():
    p = torch.zeros((4, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(SegError):
        from paper_1912_11494_b200 import binding
        binding.seg_resample(p, torch.zeros(2, dtype=torch.int64), 1, p, None)   # host offsets
    assert resample(p, torch.zeros(1, dtype=torch.int64, device="cuda")).shape == (0, 21, 3)
