"""GPU parity of the multi-label output (seg_classify_multi; row f4's optional half, the original DWM
assignment of PAPER.md:163) against oracle_classify_multi: every mask bit equal except the bits the
oracle flags as lying within 1e-3 mm of their threshold (either value is correct there); the closest
bundle of seg_classify is one of the set bits."""
import numpy as np
import pytest
import torch

import oracle
from seg_testutil import fiber_A
from synth import atlas_for_config, fibers_for_config, sample_indices

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas, SegError


def _atlas(at, mode="exact"):
    return Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
                 torch.from_numpy(at.thresh).cuda(), mode=mode)


def _check(gpu, ref, what):
    gpu = np.asarray(gpu).view(np.uint32)
    diff = (gpu ^ ref["mask"]) & ~ref["amb"]
    bad = np.nonzero(diff.any(1))[0]
    assert bad.size == 0, f"{what}: {bad.size} fibers with mask mismatches outside the band, e.g. {bad[:5]}"


@pytest.mark.parametrize("cfg,n", [(0, None), (1, 6000)])
def test_multi_parity_prefix(cfg, n):
    at = atlas_for_config(cfg)
    A = _atlas(at)
    fib = fibers_for_config(cfg, 0, n)
    fib[7, 4, 2] = np.nan
    m = A.classify_multi(torch.from_numpy(fib).cuda())
    lab, _ = A.classify(torch.from_numpy(fib).cuda())
    torch.cuda.synchronize()
    m, lab = m.cpu().numpy(), lab.cpu().numpy()
    ref = oracle.classify_multi(fib, at.centroids, at.bundle_id, at.thresh)
    _check(m, ref, f"cfg{cfg}")
    assert np.all(m[7] == 0)
    mu = m.view(np.uint32)
    for i in np.nonzero(lab >= 0)[0]:
        assert (mu[i, lab[i] >> 5] >> (lab[i] & 31)) & 1


@pytest.mark.parametrize("cfg,k", [(2, 2000), (3, 1000)])
def test_multi_full_size_sampled(cfg, k):
    """Launched on the full-size subject, compared on a seeded sample (cfg 3: 62 bundles, 2 words)."""
    at = atlas_for_config(cfg)
    A = _atlas(at)
    fib = fibers_for_config(cfg)
    m = A.classify_multi(torch.from_numpy(fib).cuda())
    torch.cuda.synchronize()
    idx = sample_indices(fib.shape[0], k, seed=5)
    ref = oracle.classify_multi(fib[idx], at.centroids, at.bundle_id, at.thresh)
    _check(m.cpu().numpy()[idx], ref, f"cfg{cfg} sample")


def test_multi_constructed_and_errors():
    a = fiber_A()
    cents = np.stack([a + np.float32([3, 0, 0]), a + np.float32([0, 5, 0]), a + np.float32([0, 0, 7]),
                      a + np.float32([2, 0, 0])]).astype(np.float32)
    bid = np.arange(4, dtype=np.int32)
    thr = np.array([4, 6, 6, 2], np.float32)
    A = Atlas(torch.from_numpy(cents).cuda(), torch.from_numpy(bid).cuda(), torch.from_numpy(thr).cuda())
    m = A.classify_multi(torch.from_numpy(np.stack([a, a[::-1].copy()])).cuda())
    torch.cuda.synchronize()
    assert m.cpu().numpy().view(np.uint32)[:, 0].tolist() == [0b1011, 0b1011]   # d = thr accepted; reversal-invariant
    P = _atlas(atlas_for_config(0), mode="paper")
    with pytest.raises(SegError):
        P.classify_multi(torch.zeros((4, 21, 3), device="cuda"))
    with pytest.raises(SegError):                                               # too few words for 4 bundles? 1 is enough;
        A.classify_multi(torch.zeros((4, 21, 3), device="cuda"),                # 0 words is not
                         masks=torch.zeros((4, 0), dtype=torch.int32, device="cuda"))
