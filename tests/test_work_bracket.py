"""The roofline numerator's independent CPU bracket (tests/work_bracket.py): host-side sanity (no GPU)
and, on the GPU, the stats kernel's counters inside the bracket term by term (W must be
reproducible from outside the kernel)."""
import numpy as np
import pytest

import oracle
from synth import atlas_for_config, fibers_for_config, sample_indices
from work_bracket import bounds, kernel_terms


def _plan(at):
    from paper_1912_11494_b200 import binding
    T = binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, 0)
    tb = np.empty(T, np.int32)
    tm = np.empty((T, 32), np.int32)
    binding.seg_plan_tiles(at.centroids, at.bundle_id, at.M, at.B, T, tb, tm, None)
    return tb, tm


def _sample(cfg, k, seed):
    at = atlas_for_config(cfg)
    fib = fibers_for_config(cfg, 0, 65536)
    sub = np.ascontiguousarray(fib[sample_indices(fib.shape[0], k, seed=seed)])
    r = oracle.classify(sub, at.centroids, at.bundle_id, at.thresh)
    final = np.where(r["label"] >= 0, r["dist"] ** 2, np.inf)
    return at, sub, final


def test_bracket_is_ordered_cpu():
    at, sub, final = _sample(0, 400, 5)
    tb, tm = _plan(at)
    lo, hi = bounds(sub, at.centroids, at.bundle_id, at.thresh, tb, tm, final)
    assert np.all(lo <= hi) and lo.sum() > 0
    # the winner's full evaluation alone: 18 points per labelled fiber
    assert lo[3] == 18.0 * np.isfinite(final).sum()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,k", [(1, 2000), (3, 600)])
def test_kernel_work_inside_the_bracket(cfg, k):
    import torch
    from paper_1912_11494_b200 import Atlas
    at, sub, final = _sample(cfg, k, 11)
    tb, tm = _plan(at)
    lo, hi = bounds(sub, at.centroids, at.bundle_id, at.thresh, tb, tm, final)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    _, _, st = A.classify_stats(torch.from_numpy(sub).cuda())
    torch.cuda.synchronize()
    w = kernel_terms(st)
    names = ("T1 bound tests", "T2 test1 lanes", "T3 test2", "T4 candidate points")
    for i in range(4):
        assert lo[i] <= w[i] <= hi[i], f"{names[i]}: {lo[i]:.4g} <= {w[i]:.4g} <= {hi[i]:.4g} violated"
    assert lo.sum() <= st["lane_point_dists"] <= hi.sum()
