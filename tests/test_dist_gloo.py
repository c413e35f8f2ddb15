"""World-size-2 CPU (gloo) tests of the multi-GPU driver's host logic:
shard arithmetic, the atlas broadcast and the padded label gather.  The per-rank classify
is the oracle here (CPU); on the GPU box it is Atlas.classify."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1912_11494_b200.dist import broadcast_atlas, classify_sharded, shard_range


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 17, 1000, 4_145_000])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(n, world):
    ranges = [shard_range(n, world, r) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == n
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c
    for a, b in ranges:
        assert (a % 4 == 0 or a == b == n) and a <= b


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0) if rank == 0 else None
    c, b, t = broadcast_atlas(at, 500, 10, torch.device("cpu"), world)
    n = 301
    fib = fibers_for_config(0, 0, n)
    lo, hi = shard_range(n, world, rank)

    def classify(f):
        r = oracle.classify(f.numpy(), c.numpy(), b.numpy(), t.numpy(), threads=1)
        return torch.from_numpy(r["label"]), torch.from_numpy(r["dist"].astype(np.float32))

    lab, d = classify_sharded(classify, torch.from_numpy(fib[lo:hi]), n, world, rank)
    q.put((rank, lab.numpy(), d.numpy(), c.numpy().sum()))
    dist.destroy_process_group()


def test_two_rank_gloo_matches_single_process():
    import oracle
    from synth import atlas_for_config, fibers_for_config
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    at = atlas_for_config(0)
    ref = oracle.classify(fibers_for_config(0, 0, 301), at.centroids, at.bundle_id, at.thresh)
    for rank, lab, d, csum in out:
        assert csum == pytest.approx(float(at.centroids.sum()))     # broadcast delivered the atlas
        assert np.array_equal(lab, ref["label"])
        assert np.array_equal(d, ref["dist"].astype(np.float32))
