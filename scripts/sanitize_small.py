"""Small invocations of every kernel for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1912_11494_b200 import Atlas, group_by_bundle, keys_to_labels, resample
from synth import atlas_for_config, fibers_for_config
from synth.raw import raw_streamlines

at = atlas_for_config(0)
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
fib = fibers_for_config(0, 0, 5000 if len(sys.argv) < 2 else int(sys.argv[1]))
fib[3, 4, 1] = np.nan
f = torch.from_numpy(fib).cuda()
for mode in ("exact", "paper"):
    A = Atlas(c, b, t, mode=mode)
    lab, d = A.classify(f)
    lab2, d2, st = A.classify_stats(f)
    k = A.classify_keys(f)
    l3, d3 = keys_to_labels(k, mode)
    hl, hd = A.classify(np.ascontiguousarray(fib[:777]))
torch.cuda.synchronize()
order, off, dmin, dmax, dsum = group_by_bundle(lab, d, at.B)
pts, offs = raw_streamlines(fib[:300], 1)
r = resample(torch.from_numpy(pts).cuda(), torch.from_numpy(offs).cuda())
torch.cuda.synchronize()
print("sanitize run ok", int((lab >= 0).sum()))
