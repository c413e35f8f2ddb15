"""GPU parity of the paper-semantics mode (SEG_MODE_PAPER) against the
oracle's paper mode: score = d_ME in the end-point-inferred orientation + TN (Eq. 3).

Same rule as the exact mode (tests/parity_util.py): labels exact for decidable fibers (the winning
score more than 1e-3 mm from its threshold and from the runner-up bundle), scores within 1e-5
relative.  The FP32 TN term (lengths summed in FP32) differs from the oracle's double by ~1e-7
relative, far inside the tolerance.
"""
import numpy as np
import pytest
import torch

import oracle
from parity_util import check_parity, check_parity_full
from seg_testutil import fiber_A
from synth import atlas_for_config, fibers_for_config, sample_indices

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas


def _atlas(at, mode="paper"):
    return Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
                 torch.from_numpy(at.thresh).cuda(), mode=mode)


def _gpu(atlas, fib):
    f = torch.from_numpy(np.ascontiguousarray(fib)).cuda()
    lab, d = atlas.classify(f)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), d.cpu().numpy()


@pytest.fixture(scope="module")
def cfg0p():
    at = atlas_for_config(0)
    return at, _atlas(at)


def test_paper_mode_info(cfg0p):
    _, A = cfg0p
    assert A.info["mode"] == 1 and A.mode == "paper"


def test_paper_cfg0_full_parity(cfg0p):
    at, A = cfg0p
    fib = fibers_for_config(0)
    lab, d = _gpu(A, fib)
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode="paper")
    info = check_parity_full(lab, d, fib, ref, at.centroids, at.bundle_id, at.thresh, "paper", "cfg0 paper")
    assert info["labelled"] > 500


@pytest.mark.parametrize("n", [1, 129, 4095, 5001])
def test_paper_ragged_sizes(cfg0p, n):
    at, A = cfg0p
    fib = fibers_for_config(0, 0, min(n, 2000))
    if n > fib.shape[0]:
        fib = np.ascontiguousarray(np.concatenate([fib] * (-(-n // fib.shape[0])))[:n])
    lab, d = _gpu(A, fib)
    k = min(n, 2000)
    ref = oracle.classify(fib[:k], at.centroids, at.bundle_id, at.thresh, mode="paper")
    check_parity(lab[:k], d[:k], ref, f"paper n={n}")


def test_paper_cfg1_subset_parity():
    at = atlas_for_config(1)
    A = _atlas(at)
    fib = fibers_for_config(1, 0, 4000)
    lab, d = _gpu(A, fib)
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode="paper")
    check_parity_full(lab, d, fib, ref, at.centroids, at.bundle_id, at.thresh, "paper", "cfg1[:4000] paper")


@pytest.mark.parametrize("cfg,k", [(3, 2000), (4, 2000)])
def test_paper_full_size_sampled(cfg, k):
    """Full-size subject (launched as bench.py launches it), compared on a seeded sample."""
    at = atlas_for_config(cfg)
    A = _atlas(at)
    fib = fibers_for_config(cfg)
    lab, d = _gpu(A, fib)
    idx = sample_indices(fib.shape[0], k, seed=91)
    ref = oracle.classify(fib[idx], at.centroids, at.bundle_id, at.thresh, mode="paper")
    check_parity_full(lab[idx], d[idx], fib[idx], ref, at.centroids, at.bundle_id, at.thresh, "paper",
                      f"cfg{cfg} paper sample")


def test_paper_subset_of_exact_and_reversal(cfg0p):
    """Paper scores are >= the exact d_ME, so every paper-labelled fiber is exact-labelled with a
    distance no larger; a reversed fiber infers the mirrored orientation and gets the same score."""
    at, A = cfg0p
    E = _atlas(at, mode="exact")
    fib = fibers_for_config(0)
    lp, dp = _gpu(A, fib)
    le, de = _gpu(E, fib)
    m = lp >= 0
    assert np.all(le[m] >= 0) and np.all(de[m] <= dp[m] * (1 + 1e-6))
    lr, dr = _gpu(A, np.ascontiguousarray(fib[:, ::-1]))
    ref = oracle.classify(np.ascontiguousarray(fib[:, ::-1]), at.centroids, at.bundle_id, at.thresh, mode="paper")
    check_parity(lr, dr, ref, "cfg0 paper reversed")


def test_paper_constructed_cases():
    """a vs a + (3,0,0) scores exactly 3 (TN = 0); a TN push past the threshold
    (scaled copy: d = 5, TN = 1/9) leaves the fiber unlabelled; ties -> lowest bundle."""
    a = fiber_A()
    s = np.zeros((21, 3), np.float32)
    s[:, 0] = np.arange(21, dtype=np.float32) - 10
    cents = np.stack([a + np.float32([3, 0, 0]), a + np.float32([0, 3, 0]), s * np.float32(1.5)]).astype(np.float32)
    bid = np.array([1, 0, 2], np.int32)
    thr = np.array([3.0, 3.0, 5.05], np.float32)
    A = Atlas(torch.from_numpy(cents).cuda(), torch.from_numpy(bid).cuda(), torch.from_numpy(thr).cuda(),
              mode="paper")
    lab, d = _gpu(A, np.stack([a, s]).astype(np.float32))
    assert lab[0] == 0 and d[0] == 3.0          # both bundles score 3.0 exactly: lowest id wins
    assert lab[1] == -1 and np.isinf(d[1])


def test_paper_host_buffers_equal_device(cfg0p):
    """The host-buffer pipeline (chunked H2D / classify / D2H) computes the same bits in paper mode."""
    _, A = cfg0p
    fib = fibers_for_config(0)
    lab, d = _gpu(A, fib)
    hl, hd = A.classify(np.ascontiguousarray(fib))
    assert np.array_equal(hl, lab) and np.array_equal(hd.view(np.int32), d.view(np.int32))


def _loop_fiber():
    """A closed, non-palindromic loop with dyadic coordinates: a_0 = a_20, so every centroid's end-point
    maxima tie exactly (tests/test_oracle_paper_pins.py)."""
    t = np.arange(21, dtype=np.float64) * (2 * np.pi / 20)
    f = np.stack([8 * np.cos(t) - 8, 6 * np.sin(t), 2 * np.sin(2 * t)], 1)
    f = (np.round(f * 64) / 64).astype(np.float32)
    f[20] = f[0]
    return f


def test_paper_tie_picks_the_callers_direct_orientation():
    """seg_create stores some centroids reversed (canonical orientation within a bundle: the
    orientation closer to the bundle's first member).  A loop fiber (a_0 = a_20) ties the end-point maxima
    exactly against every centroid; the tie must pick the caller's direct orientation whatever the stored
    one, as the oracle's 'ties -> direct' does, so the result cannot depend on the centroid order.  Order
    [r, c] stores c reversed, order [c, r] stores it forward: both must give the same bits.  The oracle
    marks the fiber undecidable (both orientations are correct answers, reading R20); the GPU's answer is
    also required to be the tie-direct one."""
    a = _loop_fiber()
    c = a + np.float32([0, 0, 1])
    c[20] += np.float32([0.25, 0, 0])                      # an open centroid: c_0 != c_20
    r = c[::-1].copy() + np.float32([0, 0, 40])            # far away, opposite orientation
    cents = np.stack([r, c]).astype(np.float32)
    bid = np.array([0, 0], np.int32)
    thr = np.array([4.0], np.float32)
    assert oracle.orientation_ambiguous(a, c) and oracle.endpoint_orientation(a, c) == 0
    direct = oracle.max_pointwise(a, c) + oracle.tn(oracle.polyline_length(a), oracle.polyline_length(c))
    assert oracle.max_pointwise(a, c, inverse=True) > 5.0
    bits = []
    for order in ([0, 1], [1, 0]):
        A = Atlas(torch.from_numpy(cents[order]).cuda(), torch.from_numpy(bid).cuda(), torch.from_numpy(thr).cuda(),
                  mode="paper")
        lab, d = _gpu(A, a[None])
        ref = oracle.classify(a[None], cents[order], bid, thr, mode="paper")
        assert ref["label"][0] == 0 and ref["dist"][0] == pytest.approx(direct, rel=1e-12) and not ref["decidable"][0]
        assert lab[0] == 0 and abs(d[0] - direct) <= 1e-5 * direct, (order, lab, d, direct)
        check_parity_full(lab, d, a[None], ref, cents[order], bid, thr, "paper", f"loop order {order}")
        bits.append((int(lab[0]), int(d.view(np.int32)[0])))
    assert bits[0] == bits[1]
