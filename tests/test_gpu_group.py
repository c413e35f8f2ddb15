"""GPU parity of row f3 (seg_group_by_bundle) against oracle/group.py: order, offsets, min and max
bit-exact (integer / selection work), sums within 1e-12 relative (double atomics, order-dependent
rounding only)."""
import numpy as np
import pytest
import torch

from oracle.group import group_by_bundle as ref_group
from synth import atlas_for_config, fibers_for_config

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas, SegError, group_by_bundle


def _check(label, dist, B):
    lt = torch.from_numpy(label).cuda()
    dt = torch.from_numpy(dist).cuda() if dist is not None else None
    order, off, dmin, dmax, dsum = group_by_bundle(lt, dt, B)
    torch.cuda.synchronize()
    r = ref_group(label, dist, B)
    assert np.array_equal(order.cpu().numpy(), r["order"])
    assert np.array_equal(off.cpu().numpy(), r["offsets"])
    if dist is not None:
        assert np.array_equal(dmin.cpu().numpy().view(np.int32), r["dmin"].view(np.int32))
        assert np.array_equal(dmax.cpu().numpy().view(np.int32), r["dmax"].view(np.int32))
        np.testing.assert_allclose(dsum.cpu().numpy(), r["dsum"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("n,B", [(0, 5), (1, 1), (2047, 7), (2048, 7), (2049, 62), (100_000, 100), (70_001, 4095)])
def test_group_random(n, B):
    rng = np.random.default_rng(n + B)
    label = rng.integers(-1, B + 3, n).astype(np.int32)
    dist = np.where(label >= 0, rng.uniform(0, 10, n), np.inf).astype(np.float32)
    _check(label, dist, B)
    _check(label, None, B)


def test_group_skewed_and_empty_bundles():
    rng = np.random.default_rng(1)
    label = np.where(rng.random(50_000) < 0.9, 3, rng.integers(0, 10, 50_000)).astype(np.int32)
    label[::7] = -1
    _check(label, rng.uniform(0, 5, 50_000).astype(np.float32), 12)   # bundles 10, 11 empty


def test_group_of_a_classification():
    at = atlas_for_config(1)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    fib = torch.from_numpy(fibers_for_config(1, 0, 60_000)).cuda()
    lab, d = A.classify(fib)
    torch.cuda.synchronize()
    _check(lab.cpu().numpy(), d.cpu().numpy(), at.B)


def test_group_argument_errors():
    lab = torch.zeros(4, dtype=torch.int32, device="cuda")
    with pytest.raises(SegError):
        group_by_bundle(lab, None, 0)
    with pytest.raises(SegError):
        group_by_bundle(lab, None, 4096)
