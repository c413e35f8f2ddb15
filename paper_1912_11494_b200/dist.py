"""Multi-GPU driver: one process per GPU, torch.distributed over NCCL.

Fibers are independent units (Alg. 1's outer loop "has no collision problems",
PAPER.md:152), so the data path needs no collective: each rank classifies its own
contiguous shard.  The only exchanges are
  * the atlas, replicated once at setup by a broadcast from rank 0 (C1), and
  * optionally the labels, gathered after the classification (C2).
Shard boundaries are multiples of 4 fibers so every shard starts 16-byte aligned.  The gather is
either NCCL's all_gather (classify_sharded) or fused into the classify kernel's epilogue, which stores
each fiber's result straight into rank 0's memory over NVLink (PeerResults, classify_sharded_p2p).

Row f4: the atlas can be sharded instead (atlases beyond one GPU, or more GPUs
than subjects): every rank holds a subset of the bundles (shard_bundles / shard_atlas) and writes
each fiber's best key over its shard (Atlas.classify_keys); one all_reduce(MIN) over the int64 keys
gives the key of the whole atlas, exactly (include/seg.h row f4), and keys_to_labels decodes it.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank `rank`; chunk = 4 * ceil(n / (4 world))."""
    chunk = 4 * (-(-n // (4 * world))) if n else 0
    lo = min(n, rank * chunk)
    return lo, min(n, lo + chunk)


def broadcast_atlas(at, M: int, B: int, device, world: int):
    """Replicate (centroids f32[M,21,3], bundle_id i32[M], thresh f32[B]) from rank 0 (C1).

    `at` (a synth.Atlas or any object with .centroids/.bundle_id/.thresh numpy arrays) is
    only needed on rank 0.  Returns tensors on `device`.
    """
    if at is not None:
        c = torch.from_numpy(at.centroids).to(device)
        b = torch.from_numpy(at.bundle_id).to(device)
        t = torch.from_numpy(at.thresh).to(device)
    else:
        c = torch.empty((M, 21, 3), dtype=torch.float32, device=device)
        b = torch.empty(M, dtype=torch.int32, device=device)
        t = torch.empty(B, dtype=torch.float32, device=device)
    if world > 1:
        for x in (c, b, t):
            dist.broadcast(x, src=0)
    return c, b, t


def classify_sharded(classify, fibers: torch.Tensor, n_total: int, world: int, rank: int,
                     gather: bool = True):
    """Strong-scaling path for one subject: this rank labels its shard `fibers`
    (= fibers[shard_range(n_total, world, rank)]) with `classify(fibers) -> (label, dist)`,
    then (gather=True) the padded shards are all-gathered (C2).  Returns the full
    (label, dist) on every rank, or this rank's shard when gather=False."""
    lab, dst = classify(fibers)
    if not gather or world == 1:
        return lab, dst
    lo, hi = shard_range(n_total, world, rank)
    chunk = shard_range(n_total, world, 0)[1]
    packed = torch.full((chunk, 2), -1, dtype=torch.int32, device=lab.device)
    packed[: hi - lo, 0] = lab
    packed[: hi - lo, 1] = dst.view(torch.int32)
    out = torch.empty((world * chunk, 2), dtype=torch.int32, device=lab.device)
    dist.all_gather_into_tensor(out, packed)
    rows = []
    for r in range(world):
        a, b = shard_range(n_total, world, r)
        rows.append(out[r * chunk: r * chunk + (b - a)])
    full = torch.cat(rows)
    return full[:, 0].contiguous(), full[:, 1].contiguous().view(torch.float32)


class PeerResults:
    """The fused gather (the NVLink-native option for C2): rank 0 owns the whole
    subject's label int32[n] / dist float32[n]; every other rank maps them through CUDA IPC, so each rank's
    seg_classify epilogue stores its shard's results straight into rank 0's memory over NVLink (include/seg.h:
    label / dist may be peer memory).  One slot per fiber, so no two ranks ever write the same word
    (PAPER.md:152).  The IPC handles travel once, at setup, as pickled torch IPC descriptors."""

    def __init__(self, n_total: int, world: int, rank: int, device):
        from torch.multiprocessing.reductions import reduce_tensor
        self.n, self.world, self.rank = n_total, world, rank
        if rank == 0:
            self.label = torch.empty(n_total, dtype=torch.int32, device=device)
            self.dist = torch.empty(n_total, dtype=torch.float32, device=device)
            desc = [reduce_tensor(self.label), reduce_tensor(self.dist)]
        else:
            desc = [None, None]
        if world > 1:
            dist.broadcast_object_list(desc, src=0)
        if rank != 0:
            with torch.cuda.device(device):
                self.label = desc[0][0](*desc[0][1])
                self.dist = desc[1][0](*desc[1][1])
        lo, hi = shard_range(n_total, world, rank)
        self.my_label, self.my_dist = self.label[lo:hi], self.dist[lo:hi]
        self.flag = torch.zeros(1, dtype=torch.int32, device=device)


def classify_sharded_p2p(classify_into, fibers: torch.Tensor, peer: PeerResults):
    """This rank's shard classified with its results stored straight into rank 0's buffers (fused gather),
    then a stream-ordered one-element all_reduce that completes only after every rank's kernel did, so rank
    0's later work on the same stream sees every shard.  classify_into(fibers, label, dist) is
    Atlas.classify.  Returns rank 0's full (label, dist) on rank 0, this rank's views elsewhere."""
    classify_into(fibers, peer.my_label, peer.my_dist)
    if peer.world > 1:
        dist.all_reduce(peer.flag)
    return (peer.label, peer.dist) if peer.rank == 0 else (peer.my_label, peer.my_dist)


def shard_bundles(counts, world: int) -> list:
    """Deterministic bundle -> rank assignment balancing the centroid counts: bundles by decreasing
    count (ties: lower id first), each to the rank with the least load so far (ties: lower rank).
    Returns one sorted list of bundle ids per rank.  Empty bundles are not assigned."""
    import numpy as np
    counts = np.asarray(counts, np.int64)
    order = sorted((b for b in range(counts.size) if counts[b] > 0), key=lambda b: (-int(counts[b]), b))
    if len(order) < world:
        raise ValueError(f"cannot shard {len(order)} non-empty bundles over {world} ranks")
    load = [0] * world
    out = [[] for _ in range(world)]
    for b in order:
        r = min(range(world), key=lambda i: (load[i], i))
        out[r].append(b)
        load[r] += int(counts[b])
    return [sorted(x) for x in out]


def shard_atlas(centroids, bundle_id, thresh, world: int, rank: int, mode: str = "exact", device: int = -1):
    """This rank's atlas shard: the centroids of its bundles, with the global bundle count and
    thresholds (so labels stay global).  Inputs: numpy arrays or tensors (host or device)."""
    import numpy as np
    from . import Atlas
    bid = bundle_id.cpu().numpy() if hasattr(bundle_id, "cpu") else np.asarray(bundle_id)
    B = int(thresh.shape[0])
    mine = shard_bundles(np.bincount(bid, minlength=B), world)[rank]
    sel = np.nonzero(np.isin(bid, mine))[0]
    if hasattr(centroids, "index_select"):
        idx = torch.from_numpy(sel).to(centroids.device)
        c, b = centroids.index_select(0, idx).contiguous(), bundle_id.index_select(0, idx).contiguous()
    else:
        c, b = np.ascontiguousarray(centroids[sel]), np.ascontiguousarray(bid[sel])
    return Atlas(c, b, thresh, device=device, mode=mode)


def reduce_keys(keys: torch.Tensor, world: int) -> torch.Tensor:
    """all_reduce(MIN) of the shards' best keys (int64, every key < 2^63), in place."""
    if world > 1:
        dist.all_reduce(keys, op=dist.ReduceOp.MIN)
    return keys


def classify_atlas_sharded(atlas_shard, fibers: torch.Tensor, world: int):
    """Atlas-sharded classification of `fibers` (the same fibers on every rank): this rank's keys,
    the MIN over the ranks, decoded.  Returns (label, dist) on every rank."""
    from . import keys_to_labels
    keys = reduce_keys(atlas_shard.classify_keys(fibers), world)
    return keys_to_labels(keys, atlas_shard.mode)

