"""Measure the widened rows on B200, cfg 3 inputs, CUDA events on the launching
stream after warm-up.  Prints one JSON line per row.  (The headline bench line is bench.py's.)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1912_11494_b200 import Atlas, group_by_bundle, keys_to_labels, resample
from paper_1912_11494_b200.dist import shard_atlas
from synth.raw import raw_streamlines
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

# row f2: raw streamlines (Catmull-Rom stand-ins, 30-200 points each) of the first 1,000,000 fibers
NR = min(N, 1_000_000)
pts, off = raw_streamlines(fibers_for_config(cfg, 0, NR), seed=11)
P = int(off[-1])
pts_d, off_d = torch.from_numpy(pts).cuda(), torch.from_numpy(off).cuda()
ms = timeit(lambda: resample(pts_d, off_d))
alg = 12 * P + 8 * (NR + 1) + 4 * 63 * NR
print(json.dumps(dict(row="f2 seg_resample", config=f"cfg{cfg} first {NR:,} fibers as raw streamlines, {P:,} points "
                      f"(30-200 per fiber, synth/raw.py)", ms=ms, fibers_per_s=NR / (ms * 1e-3),
                      points_per_s=P / (ms * 1e-3), algorithmic_bytes=alg, achieved_gbs=alg / (ms * 1e-3) / 1e9,
                      hbm_peak_gbs=PEAKS["hbm_gbs"], frac=alg / (ms * 1e-3) / 1e9 / PEAKS["hbm_gbs"])))

# row f4: atlas shards (emulated one after another on this GPU): the per-shard keys kernel time is what
# one rank of a world-N atlas-sharded run spends; the MIN over the shards + decode is checked bitwise
c_d, b_d, t_d = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
full_ms = timeit(lambda: A.classify(fib, lab, d), reps=10)
for world in (2, 4, 8):
    shards = [shard_atlas(c_d, b_d, t_d, world, r) for r in range(world)]
    per = []
    keys = None
    for sh in shards:
        kk = torch.empty(N, dtype=torch.int64, device="cuda")
        per.append(timeit(lambda: sh.classify_keys(fib, kk), reps=5))
        keys = kk.clone() if keys is None else torch.minimum(keys, kk)
    l2, d2 = keys_to_labels(keys)
    torch.cuda.synchronize()
    same = bool(torch.equal(l2, lab)) and bool(torch.equal(d2.view(torch.int32), d.view(torch.int32)))
    print(json.dumps(dict(row="f4 atlas shards", config=f"cfg{cfg}, {N:,} fibers, world={world}",
                          unsharded_ms=full_ms, shard_ms=per, max_shard_ms=max(per), sum_shard_ms=sum(per),
                          strong_scaling_speedup=full_ms / max(per), min_decode_equals_unsharded=same)))


# row f4's optional half: the multi-label (DWM) masks, every bundle within threshold (seg_classify_multi)
masks = torch.empty((N, (at.B + 31) // 32), dtype=torch.int32, device="cuda")
ms = timeit(lambda: A.classify_multi(fib, masks), reps=10)
m64 = masks.to(torch.int64)
nmulti = int((sum((m64 >> k) & 1 for k in range(32)).sum(-1) > 1).sum())
print(json.dumps(dict(row="f4 multi-label seg_classify_multi", config=f"cfg{cfg}, {N:,} fibers x {at.M:,} centroids",
                      ms=ms, comparisons_per_s=N * at.M / (ms * 1e-3), fibers_per_s=N / (ms * 1e-3),
                      single_label_ms=full_ms, fibers_with_several_bundles=nmulti)))
