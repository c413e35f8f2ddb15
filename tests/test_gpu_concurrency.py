"""include/seg.h: an atlas may be used from several host threads at once (only the profiling hook is
not thread-safe).  Two threads classify different fiber sets through one atlas concurrently, each on
its own CUDA stream (ctypes releases the GIL during the calls), device and host-buffer paths; the
results equal the sequential ones bit for bit."""
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_two_threads_one_atlas():
    from paper_1912_11494_b200 import Atlas
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(1)
    A = Atlas(*(torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh)))
    sets = [fibers_for_config(1, 0, 60000), fibers_for_config(1, 40000, 100000)]
    seq = []
    for f in sets:
        lab, d = A.classify(torch.from_numpy(f).cuda())
        torch.cuda.synchronize()
        seq.append((lab.cpu().numpy(), d.cpu().numpy()))
    out = [None, None]
    err = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            f = torch.from_numpy(sets[i]).cuda()
            res = []
            for rep in range(4):
                with torch.cuda.stream(s):
                    lab, d = A.classify(f, stream=s)
                s.synchronize()
                res.append((lab.cpu().numpy(), d.cpu().numpy()))
                hl, hd = A.classify(np.ascontiguousarray(sets[i]))      # host-buffer pipeline
                res.append((hl, hd))
            out[i] = res
        except Exception as e:   # surfaced below
            err.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not err, err
    for i in range(2):
        for lab, d in out[i]:
            assert np.array_equal(lab, seq[i][0])
            assert np.array_equal(d.view(np.int32), seq[i][1].view(np.int32))
