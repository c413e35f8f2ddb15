"""Experiment: how much faster is the kernel when every fiber starts with its final best
(a perfect best-first order)?  Prints normal vs seeded kernel time on a config."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_11494_b200 import Atlas, binding
from synth import atlas_for_config, fibers_for_config

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
at = atlas_for_config(cfg)
A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(), torch.from_numpy(at.thresh).cuda())
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
lab = torch.empty(N, dtype=torch.int32, device="cuda")
d = torch.empty(N, dtype=torch.float32, device="cuda")


def timeit(fn, n=10):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


t0 = timeit(lambda: A.classify(fib, lab, d))
_, _, st = A.classify_stats(fib)
lab0, d0 = lab.clone(), d.clone()
d2 = (d0.double() ** 2 * (1 + 1e-6)).float()
key = (d2.view(torch.int32).to(torch.int64) << 32) | lab0.to(torch.int64).bitwise_and(0xffffffff)
key = torch.where(lab0 >= 0, key, torch.full_like(key, -1))
lab2 = torch.empty_like(lab)
d2o = torch.empty_like(d)
t1 = timeit(lambda: binding.seg_debug_classify_seeded(A.handle, fib, N, key, lab2, d2o, None,
                                                      torch.cuda.current_stream().cuda_stream))
st2 = np.zeros(binding.SEG_NSTATS, np.uint64)
binding.seg_debug_classify_seeded(A.handle, fib, N, key, lab2, d2o, st2, torch.cuda.current_stream().cuda_stream)
same = bool(torch.equal(lab0, lab2)) and bool(torch.equal(d0.view(torch.int32), d2o.view(torch.int32)))
print(f"cfg{cfg}: normal {t0:.3f} ms, seeded {t1:.3f} ms, identical={same}")
print("stats normal", st)
print("stats seeded", dict(zip(binding.STAT_NAMES, (int(v) for v in st2))))
