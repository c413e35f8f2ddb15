"""A large atlas: config 3's atlas replicated 14 times with small seeded displacements and distinct bundle
ids (620,830 centroids, 868 bundles, ~19,400 tiles of 32).  This exercises the paths small atlases do not
reach: k_cull's bundle spheres read from global memory (B > 512 staged in shared memory), its ~150 KB of
dynamic shared memory, and the u16 per-CTA tile lists far above config 3's 1,417 tiles.  Parity against the
oracle on a sample of config-3 fibers (they match several replicas: the near ties exercise the lexicographic
(distance, bundle) rule)."""
import numpy as np
import pytest
import torch

import oracle
from parity_util import check_parity
from synth import atlas_for_config, fibers_for_config, sample_indices

pytestmark = pytest.mark.gpu

REPS = 14


@pytest.fixture(scope="module")
def big():
    at = atlas_for_config(3)
    rng = np.random.default_rng(20261020)
    cents, bids, thr = [], [], []
    for r in range(REPS):
        shift = rng.normal(0.0, 0.6, size=(1, 1, 3)).astype(np.float32) * (r > 0)
        cents.append((at.centroids + shift).astype(np.float32))
        bids.append(at.bundle_id + r * at.B)
        thr.append(at.thresh)
    return (np.ascontiguousarray(np.concatenate(cents)), np.ascontiguousarray(np.concatenate(bids).astype(np.int32)),
            np.ascontiguousarray(np.concatenate(thr).astype(np.float32)))


def test_large_atlas_parity(big):
    from paper_1912_11494_b200 import Atlas
    cents, bid, thr = big
    A = Atlas(*(torch.from_numpy(x).cuda() for x in (cents, bid, thr)))
    assert A.info["n_bundles"] == 62 * REPS and A.info["n_tiles"] > 15000
    full = fibers_for_config(3, 0, 200000)
    fib = np.ascontiguousarray(full[sample_indices(len(full), 6000, seed=44)])
    lab, d = A.classify(torch.from_numpy(fib).cuda())
    torch.cuda.synchronize()
    k = 400
    ref = oracle.classify(fib[:k], cents, bid, thr)
    info = check_parity(lab.cpu().numpy()[:k], d.cpu().numpy()[:k], ref, "large atlas")
    assert info["labelled"] > 150
    # the same answer through the host-buffer pipeline
    hl, hd = A.classify(fib)
    assert np.array_equal(hl, lab.cpu().numpy()) and np.array_equal(hd.view(np.int32), d.cpu().numpy().view(np.int32))


def _one_centroid_bundles(nb, seed):
    """nb bundles of one centroid each (one tile each): centroids drawn from config 3's atlas, jittered."""
    at = atlas_for_config(3)
    rng = np.random.default_rng(seed)
    pick = rng.integers(0, at.M, size=nb)
    cents = (at.centroids[pick] + rng.normal(0, 1.0, size=(nb, 1, 3))).astype(np.float32)
    return (np.ascontiguousarray(cents), np.arange(nb, dtype=np.int32),
            np.ascontiguousarray(rng.uniform(5, 10, nb).astype(np.float32)))


def test_max_tiles_atlas_parity_and_limit():
    """Exactly the build's tile limit (30,000 tiles) works and matches the oracle; one more is refused."""
    from paper_1912_11494_b200 import Atlas, binding
    cents, bid, thr = _one_centroid_bundles(30000, 7)
    A = Atlas(*(torch.from_numpy(x).cuda() for x in (cents, bid, thr)))
    assert A.info["n_tiles"] == 30000
    full = fibers_for_config(3, 0, 100000)
    fib = np.ascontiguousarray(full[sample_indices(len(full), 5000, seed=45)])
    lab, d = A.classify(torch.from_numpy(fib).cuda())
    torch.cuda.synchronize()
    ref = oracle.classify(fib[:500], cents, bid, thr)
    info = check_parity(lab.cpu().numpy()[:500], d.cpu().numpy()[:500], ref, "30000-tile atlas")
    assert info["labelled"] > 50
    A.close()
    c2, b2, t2 = _one_centroid_bundles(30001, 8)
    with pytest.raises(binding.SegError) as ei:
        Atlas(*(torch.from_numpy(x).cuda() for x in (c2, b2, t2)))
    assert ei.value.code == binding.SEG_EINVAL and "30001 tiles" in str(ei.value)
