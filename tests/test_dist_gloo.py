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
    lo, hi = shard_range(n, world, rank)
    fib_shard = fibers_for_config(0, lo, hi)        # each rank generates only its shard, as bench.py does

    def classify(f):
        r = oracle.classify(f.numpy(), c.numpy(), b.numpy(), t.numpy(), threads=1)
        return torch.from_numpy(r["label"]), torch.from_numpy(r["dist"].astype(np.float32))

    lab, d = classify_sharded(classify, torch.from_numpy(fib_shard), n, world, rank)
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


# ----------------------------------------------------------------------------------
# row f4: atlas sharding -- the bundle assignment and the MIN reduction of the best keys
# ----------------------------------------------------------------------------------
from paper_1912_11494_b200.dist import reduce_keys, shard_bundles  # noqa: E402

KEY_NONE, KEY_NONFINITE = 0x7FFFFFFFFFFFFFFF, 0x7FFFFFFFFFFFFFFE


@pytest.mark.parametrize("world", [1, 2, 3, 7])
def test_shard_bundles_partition_and_balance(world):
    rng = np.random.default_rng(world)
    counts = rng.integers(0, 900, 62)
    counts[5] = 0
    shards = shard_bundles(counts, world)
    flat = sorted(b for s in shards for b in s)
    assert flat == [b for b in range(62) if counts[b] > 0]
    loads = [int(counts[s].sum()) for s in shards]
    assert max(loads) - min(loads) <= counts.max()
    assert shard_bundles(counts, world) == shards                     # deterministic
    with pytest.raises(ValueError):
        shard_bundles([1, 0, 0], 2)


def _oracle_keys(fib, at, bundles):
    """Best key of each fiber over `bundles` from the oracle's per-bundle minimum d_ME^2."""
    import oracle
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, threads=1, want_d2b=True)
    keys = np.full(fib.shape[0], KEY_NONE, np.int64)
    for i in range(fib.shape[0]):
        if np.isnan(r["dist"][i]):
            keys[i] = KEY_NONFINITE
            continue
        for b in bundles:
            d2 = r["d2b"][i, b]
            if d2 <= float(at.thresh[b]) ** 2:
                k = (int(np.float32(d2).view(np.uint32)) << 32) | b
                keys[i] = min(keys[i], k)
    return keys


def _shard_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 200)
    fib[7, 3, 1] = np.nan
    mine = shard_bundles(np.bincount(at.bundle_id, minlength=at.B), world)[rank]
    keys = torch.from_numpy(_oracle_keys(fib, at, mine))
    reduce_keys(keys, world)
    q.put((rank, keys.numpy()))
    dist.destroy_process_group()


def test_two_rank_gloo_atlas_sharding_matches_unsharded():
    import oracle
    from synth import atlas_for_config, fibers_for_config
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    at = atlas_for_config(0)
    fib = fibers_for_config(0, 0, 200)
    fib[7, 3, 1] = np.nan
    ref = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh)
    for rank, keys in out:
        lab = np.where(keys >= KEY_NONFINITE, -1, keys & 0xFFFFFFFF).astype(np.int32)
        dec = ref["decidable"]
        assert np.array_equal(lab[dec], ref["label"][dec])
        assert keys[7] == KEY_NONFINITE
        assert np.array_equal(keys, out[0][1])
