"""The library keeps its per-call scratch in a memory pool of its own (one per atlas, seg_api.cu): creating
and using an atlas must not change the device's default pool, which belongs to the caller's process."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _default_pool_threshold(rt):
    err, pool = rt.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
    assert err == rt.cudaError_t.cudaSuccess
    err, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReleaseThreshold)
    assert err == rt.cudaError_t.cudaSuccess
    return int(v)


def test_default_pool_untouched():
    rt = pytest.importorskip("cuda.bindings.runtime")
    from paper_1912_11494_b200 import Atlas
    from synth import atlas_for_config, fibers_for_config
    torch.cuda.init()
    before = _default_pool_threshold(rt)
    at = atlas_for_config(0)
    A = Atlas(*(torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh)))
    f = torch.from_numpy(fibers_for_config(0)).cuda()
    lab, d = A.classify(f)
    hl, hd = A.classify(np.ascontiguousarray(fibers_for_config(0)))
    torch.cuda.synchronize()
    assert np.array_equal(lab.cpu().numpy(), hl)
    assert _default_pool_threshold(rt) == before
    A.close()
