"""Print the stats-kernel counters for one config (GPU)."""
import sys, json, torch
sys.path.insert(0, ".")
from paper_1912_11494_b200 import Atlas
from synth import atlas_for_config, fibers_for_config
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
at = atlas_for_config(cfg)
A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(), torch.from_numpy(at.thresh).cuda())
fib = torch.from_numpy(fibers_for_config(cfg)).cuda()
_, _, st = A.classify_stats(fib)
print(json.dumps(st))
