"""Row f4 on one GPU: atlas shards emulated on a single device.  The element-wise MIN of the shards'
keys, decoded, must equal the unsharded seg_classify bit for bit (both modes): a (fiber, centroid)
pair's FP32 distance does not depend on which shard holds the centroid."""
import numpy as np
import pytest
import torch

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
