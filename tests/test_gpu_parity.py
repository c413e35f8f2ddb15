"""GPU parity of the CUDA hot path (through the C ABI) against the CPU oracle.

Element-by-element on the same seeded inputs: labels exact for decidable fibers,
distances within 1e-5 relative (tests/parity_util.py).  Small sizes are compared in
full; the BASELINE.json full-size configs are launched exactly as bench.py launches
them and compared on seeded samples the oracle computes one by one.
"""
import numpy as np
import pytest
import torch

import oracle
from parity_util import check_parity, check_parity_full
from synth import CONFIGS, atlas_for_config, fibers_for_config, sample_indices

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas, binding


def _atlas(at):
    return Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
                 torch.from_numpy(at.thresh).cuda())


def _gpu(atlas, fib):
    f = torch.from_numpy(np.ascontiguousarray(fib)).cuda()
    lab, d = atlas.classify(f)
    torch.cuda.synchronize()
    return lab.cpu().numpy(), d.cpu().numpy()


@pytest.fixture(scope="module")
def cfg0():
    at = atlas_for_config(0)
    return at, _atlas(at)


def test_cfg0_full_parity(cfg0):
    at, A = cfg0
    fib = fibers_for_config(0)
    lab, d = _gpu(A, fib)
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    info = check_parity(lab, d, ref, "cfg0")
    assert info["labelled"] > 1000


@pytest.mark.parametrize("n", [1, 31, 129, 1000, 4095, 4096, 5001, 12345])
def test_ragged_sizes(cfg0, n):
    """Sizes spanning the no-prepass path (< 4096), the prepass path, partial warps and CTAs."""
    at, A = cfg0
    fib = fibers_for_config(0, 0, min(n, 2000))
    if n > fib.shape[0]:
        reps = -(-n // fib.shape[0])
        fib = np.ascontiguousarray(np.concatenate([fib] * reps)[:n])
    lab, d = _gpu(A, fib)
    k = min(n, 2000)
    ref = oracle.classify(fib[:k], at.centroids, at.bundle_id, at.thresh)
    check_parity(lab[:k], d[:k], ref, f"n={n}")
    if n > k:   # repeated fibers must repeat their results bit for bit
        assert np.array_equal(lab[k:], lab[np.arange(k, n) % 2000])
        assert np.array_equal(d[k:].view(np.int32), d[np.arange(k, n) % 2000].view(np.int32))


def test_empty_input(cfg0):
    _, A = cfg0
    f = torch.empty((0, 21, 3), dtype=torch.float32, device="cuda")
    lab, d = A.classify(f)
    assert lab.numel() == 0 and d.numel() == 0


def test_cfg1_subset_full_parity():
    at = atlas_for_config(1)
    A = _atlas(at)
    fib = fibers_for_config(1, 0, 6000)
    lab, d = _gpu(A, fib)
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    check_parity_full(lab, d, fib, ref, at.centroids, at.bundle_id, at.thresh, "exact", "cfg1[:6000]")


@pytest.mark.parametrize("cfg,k", [(1, 5000), (2, 3000), (3, 3000), (4, 3000)])
def test_full_size_sampled_parity(cfg, k):
    """BASELINE.json configs at full size, launched like bench.py; sampled oracle check."""
    at = atlas_for_config(cfg)
    A = _atlas(at)
    fib = fibers_for_config(cfg)
    assert fib.shape[0] == CONFIGS[cfg]["n_fibers"]
    lab, d = _gpu(A, fib)
    idx = sample_indices(fib.shape[0], k, seed=cfg)
    ref = oracle.classify(fib[idx], at.centroids, at.bundle_id, at.thresh)
    info = check_parity_full(lab[idx], d[idx], fib[idx], ref, at.centroids, at.bundle_id, at.thresh, "exact",
                             f"cfg{cfg} sampled")
    # properties that hold at any size: labelled -> dist <= thr; unlabelled -> +inf
    m = lab >= 0
    assert np.all(d[m] <= at.thresh[lab[m]])
    assert np.all(np.isinf(d[~m]))
    assert 0.5 < m.mean() < 1.0
    assert info["labelled"] > 0


# ----------------------------------------------------------------------------------
# constructed edge cases
# ----------------------------------------------------------------------------------
def _fiber_A():
    i = np.arange(21, dtype=np.float64)
    return np.stack([2 * i - 20, i * i / 8.0, (i % 3) / 2.0], axis=1).astype(np.float32)


def test_threshold_equality_and_ties():
    """d == thr accepted, d just above rejected, equal distances -> lowest bundle id."""
    a = _fiber_A()
    cents = np.stack([a + np.float32([4, 0, 0]),        # bundle 2 at exactly its thr 4
                      a + np.float32([0, 0, 3]),        # bundle 3 at 3
                      a + np.float32([0, 3, 0]),        # bundle 1 at 3 (tie with 3 -> 1 wins)
                      a + np.float32([6, 0, 0])])       # bundle 0 at 6 > thr 5
    bid = np.array([2, 3, 1, 0], np.int32)
    thr = np.array([5, 5, 4, 5], np.float32)
    A = Atlas(cents, bid, thr)
    probes = np.stack([a, a + np.float32([0, 0, 0]), a[::-1].copy()])
    lab, d = _gpu(A, probes)
    assert np.all(lab == 1) and np.all(d == 3.0)
    # only bundle 2 at exactly thr
    A2 = Atlas(cents[:1].copy(), np.array([0], np.int32), np.array([4], np.float32))
    lab, d = _gpu(A2, np.stack([a, a - np.float32([2 ** -10, 0, 0])]))
    assert lab[0] == 0 and d[0] == 4.0
    assert lab[1] == -1 and np.isinf(d[1])


def test_self_segmentation_and_nonfinite(cfg0):
    at, A = cfg0
    f = at.centroids.copy()
    f[7, 3, 1] = np.nan
    f[9, 20, 2] = np.inf
    lab, d = _gpu(A, f)
    ok = np.ones(at.M, bool)
    ok[[7, 9]] = False
    assert np.array_equal(lab[ok], at.bundle_id[ok])
    assert np.all(d[ok] == 0.0)
    assert lab[7] == -1 and np.isnan(d[7]) and lab[9] == -1 and np.isnan(d[9])


def test_far_fibers_unlabelled(cfg0):
    at, A = cfg0
    f = fibers_for_config(0, 0, 500) + np.float32([500, 0, 0])
    lab, d = _gpu(A, np.ascontiguousarray(f))
    assert np.all(lab == -1) and np.all(np.isinf(d))


# ----------------------------------------------------------------------------------
# invariants (bitwise)
# ----------------------------------------------------------------------------------
def test_flip_permutation_and_determinism():
    at = atlas_for_config(1)
    A = _atlas(at)
    fib = fibers_for_config(1, 0, 20000)
    lab, d = _gpu(A, fib)
    lab2, d2 = _gpu(A, fib)
    assert np.array_equal(lab, lab2) and np.array_equal(d.view(np.int32), d2.view(np.int32))
    rev = np.ascontiguousarray(fib[:, ::-1, :])
    lab3, d3 = _gpu(A, rev)
    assert np.array_equal(lab, lab3) and np.array_equal(d.view(np.int32), d3.view(np.int32))
    perm = np.random.default_rng(0).permutation(fib.shape[0])
    lab4, d4 = _gpu(A, np.ascontiguousarray(fib[perm]))
    assert np.array_equal(lab[perm], lab4) and np.array_equal(d[perm].view(np.int32), d4.view(np.int32))


def test_centroid_order_and_orientation_do_not_matter():
    at = atlas_for_config(1)
    fib = fibers_for_config(1, 0, 20000)
    lab, d = _gpu(_atlas(at), fib)
    rng = np.random.default_rng(5)
    perm = rng.permutation(at.M)
    c = at.centroids[perm].copy()
    flip = rng.random(at.M) < 0.5
    c[flip] = c[flip, ::-1, :]
    A2 = Atlas(np.ascontiguousarray(c), np.ascontiguousarray(at.bundle_id[perm]), at.thresh)
    lab2, d2 = _gpu(A2, fib)
    assert np.array_equal(lab, lab2) and np.array_equal(d.view(np.int32), d2.view(np.int32))


def test_host_buffer_path_matches_device_path():
    at = atlas_for_config(1)
    A = _atlas(at)
    fib = fibers_for_config(1, 0, 100_000)
    lab, d = _gpu(A, fib)
    pin = torch.from_numpy(fib).pin_memory()
    hl = torch.empty(fib.shape[0], dtype=torch.int32).pin_memory()
    hd = torch.empty(fib.shape[0], dtype=torch.float32).pin_memory()
    A.classify(pin, hl, hd)
    assert np.array_equal(lab, hl.numpy()) and np.array_equal(d.view(np.int32), hd.numpy().view(np.int32))
    nl, nd = A.classify(fib)                       # pageable numpy
    assert np.array_equal(lab, nl) and np.array_equal(d.view(np.int32), nd.view(np.int32))


def test_stats_kernel_matches_and_counts():
    at = atlas_for_config(1)
    A = _atlas(at)
    fib = torch.from_numpy(fibers_for_config(1, 0, 50_000)).cuda()
    lab, d = A.classify(fib)
    lab2, d2, st = A.classify_stats(fib)
    torch.cuda.synchronize()
    assert torch.equal(lab, lab2) and torch.equal(d.view(torch.int32), d2.view(torch.int32))
    assert st["fibers"] == 50_000
    assert st["lane_test1"] >= st["lane_test2"] >= st["lane_test34"] >= st["lane_full21"]
    assert st["best_updates"] >= int((lab >= 0).sum())
    assert st["ctas"] == -(-50_000 // 256)


def test_argument_errors_on_gpu(cfg0):
    _, A = cfg0
    f = torch.zeros((8, 21, 3), dtype=torch.float32, device="cuda")
    lab = torch.zeros(8, dtype=torch.int32, device="cuda")
    d = torch.zeros(8, dtype=torch.float32, device="cuda")
    hl = np.zeros(8, np.int32)
    with pytest.raises(binding.SegError) as ei:          # mixed host/device
        binding.seg_classify(A.handle, f, 8, hl, d)
    assert ei.value.code == binding.SEG_EINVAL
    with pytest.raises(binding.SegError) as ei:          # misaligned
        binding.seg_classify(A.handle, f.data_ptr() + 2, 7, lab, d)
    assert ei.value.code == binding.SEG_EINVAL
    with pytest.raises(binding.SegError) as ei:          # null with N > 0
        binding.seg_classify(A.handle, None, 8, lab, d)
    assert ei.value.code == binding.SEG_EINVAL
    bad = np.array([0, 1, 10], np.int32)
    with pytest.raises(binding.SegError) as ei:          # bundle id out of range
        binding.seg_create(np.zeros((3, 21, 3), np.float32), bad, 3, np.ones(10, np.float32), 10)
    assert ei.value.code == binding.SEG_EINVAL
    with pytest.raises(binding.SegError):                # threshold <= 0
        binding.seg_create(np.zeros((1, 21, 3), np.float32), np.zeros(1, np.int32), 1,
                           np.zeros(1, np.float32), 1)
    c = np.zeros((1, 21, 3), np.float32)
    c[0, 4, 1] = np.nan
    with pytest.raises(binding.SegError):                # non-finite centroid
        binding.seg_create(c, np.zeros(1, np.int32), 1, np.ones(1, np.float32), 1)


def test_empty_bundle_and_unaligned_fiber_pointer():
    """A bundle with no centroid never wins; a 4-byte (not 16-byte) aligned fiber pointer works."""
    at = atlas_for_config(0)
    bid = at.bundle_id.copy()
    bid[bid == 3] = 4                                      # bundle 3 now empty
    A = Atlas(at.centroids, bid, at.thresh)
    fib = fibers_for_config(0, 0, 999)
    buf = torch.from_numpy(np.concatenate([np.zeros(63, np.float32), fib.ravel()])).cuda()
    f_off = buf[63:].view(999, 21, 3)                      # 252 B offset: 4-byte aligned only
    lab = torch.empty(999, dtype=torch.int32, device="cuda")
    d = torch.empty(999, dtype=torch.float32, device="cuda")
    binding.seg_classify(A.handle, f_off.data_ptr(), 999, lab, d)
    torch.cuda.synchronize()
    ref = oracle.classify(fib, at.centroids, bid, at.thresh)
    check_parity(lab.cpu().numpy(), d.cpu().numpy(), ref, "empty bundle")
    assert not np.any(lab.cpu().numpy() == 3)
