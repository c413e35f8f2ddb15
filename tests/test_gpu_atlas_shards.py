"""Row f4 on one GPU: atlas shards emulated on a single device.  The element-wise MIN of the shards'
keys, decoded, must equal the unsharded seg_classify bit for bit (both modes): a (fiber, centroid)
pair's FP32 distance does not depend on which shard holds the centroid.  Each shard's own keys, and
the reduced keys, are also held to the oracle directly: a shard's keys decode to the oracle's
classification against that shard's centroids (global bundle ids and thresholds), and the MIN over
the shards to the oracle's classification against the whole atlas (Alg. 1's closest bundle,
PAPER.md:129-133, :163)."""
import numpy as np
import pytest
import torch

import oracle
from parity_util import check_parity_full
from synth import atlas_for_config, fibers_for_config

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas, keys_to_labels
    from paper_1912_11494_b200.dist import shard_atlas


@pytest.mark.parametrize("cfg,n,world,mode", [(0, 2000, 2, "exact"), (0, 2000, 3, "paper"), (1, 30_000, 4, "exact"),
                                              (3, 20_000, 2, "exact"), (3, 20_000, 3, "paper")])
def test_sharded_min_equals_unsharded(cfg, n, world, mode):
    at = atlas_for_config(cfg)
    c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
    fib = fibers_for_config(cfg, 0, n)
    fib[3, 5, 0] = np.inf
    f = torch.from_numpy(fib).cuda()
    full = Atlas(c, b, t, mode=mode)
    lab, d = full.classify(f)
    keys = None
    for r in range(world):
        k = shard_atlas(c, b, t, world, r, mode=mode).classify_keys(f)
        keys = k if keys is None else torch.minimum(keys, k)
    lab2, d2 = keys_to_labels(keys, mode)
    torch.cuda.synchronize()
    assert torch.equal(lab, lab2)
    assert torch.equal(d.view(torch.int32), d2.view(torch.int32))
    assert lab2[3].item() == -1 and torch.isnan(d2[3])


@pytest.mark.parametrize("cfg,n,world,mode", [(0, 2000, 2, "exact"), (0, 2000, 3, "paper"), (1, 3000, 4, "exact"),
                                              (3, 1500, 2, "exact"), (3, 1500, 3, "paper")])
def test_shard_keys_match_the_oracle(cfg, n, world, mode):
    from paper_1912_11494_b200.dist import shard_bundles
    at = atlas_for_config(cfg)
    c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
    fib = fibers_for_config(cfg, 0, n)
    fib[3, 5, 0] = np.inf
    f = torch.from_numpy(fib).cuda()
    keys = None
    for r in range(world):
        k = shard_atlas(c, b, t, world, r, mode=mode).classify_keys(f)
        lab, d = keys_to_labels(k, mode)
        torch.cuda.synchronize()
        mine = shard_bundles(np.bincount(at.bundle_id, minlength=at.B), world)[r]
        sel = np.nonzero(np.isin(at.bundle_id, mine))[0]
        ref = oracle.classify(fib, at.centroids[sel], at.bundle_id[sel], at.thresh, mode=mode)
        check_parity_full(lab.cpu().numpy(), d.cpu().numpy(), fib, ref, at.centroids[sel], at.bundle_id[sel],
                          at.thresh, mode, f"cfg{cfg} {mode} shard {r}/{world}")
        keys = k if keys is None else torch.minimum(keys, k)
    lab, d = keys_to_labels(keys, mode)
    torch.cuda.synchronize()
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode=mode)
    check_parity_full(lab.cpu().numpy(), d.cpu().numpy(), fib, ref, at.centroids, at.bundle_id, at.thresh, mode,
                      f"cfg{cfg} {mode} MIN over {world} shards")


def test_keys_argument_errors():
    from paper_1912_11494_b200 import SegError, binding
    at = atlas_for_config(0)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    f = torch.zeros((8, 21, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(SegError):                                   # host keys
        binding.seg_classify_keys(A.handle, f, 8, np.zeros(8, np.int64), None)
    with pytest.raises(TypeError):
        A.classify_keys(f.cpu())
    k = A.classify_keys(f)                                          # a zero fiber: finite, unassigned
    lab, d = keys_to_labels(k)
    torch.cuda.synchronize()
    assert torch.all(lab == -1) and torch.all(torch.isinf(d))
