"""Measure the widened rows on B200, cfg 3 inputs, CUDA events on the launching
stream after warm-up.  Prints one JSON line per row.  (The headline bench line is bench.py's.)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1912_11494_b200 import Atlas, group_by_bundle
from synth import atlas_for_config, fibers_for_config

PEAKS = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
at = atlas_for_config(cfg)
A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(), torch.from_numpy(at.thresh).cuda())
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
N = fib.shape[0]
lab, d = A.classify(fib)
torch.cuda.synchronize()
ms = timeit(lambda: group_by_bundle(lab, d, at.B))
# algorithmic bytes: label + dist read by the count pass, label read by the scatter pass, order written
alg = N * (4 + 4 + 4 + 4)
print(json.dumps(dict(row="f3 seg_group_by_bundle", config=f"cfg{cfg} labels of {N:,} fibers, B={at.B}",
                      ms=ms, fibers_per_s=N / (ms * 1e-3), algorithmic_bytes=alg,
                      achieved_gbs=alg / (ms * 1e-3) / 1e9, hbm_peak_gbs=PEAKS["hbm_gbs"],
                      frac=alg / (ms * 1e-3) / 1e9 / PEAKS["hbm_gbs"])))
