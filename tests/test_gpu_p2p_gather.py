"""The fused gather (dist.PeerResults / classify_sharded_p2p): every rank's classify epilogue stores its
shard's results straight into rank 0's buffers (CUDA IPC mapping; NVLink on a multi-GPU box).  Only one GPU
is available here, so two ranks share cuda:0 with a gloo process group -- the IPC mapping, the peer-output
path of the C ABI (include/seg.h) and the completion ordering run for real; the link is the same device.
No rank waits on another rank's kernel (the completion is a host-side gloo all_reduce)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1912_11494_b200 import Atlas
    from paper_1912_11494_b200.dist import PeerResults, classify_sharded_p2p, shard_range
    from synth import atlas_for_config, fibers_for_config
    at = atlas_for_config(1)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    peer = PeerResults(n, world, rank, torch.device("cuda", 0))
    lo, hi = shard_range(n, world, rank)
    fib = torch.from_numpy(fibers_for_config(1, lo, hi)).cuda()
    for _ in range(2):                                   # twice: the buffers are reused across steps
        lab, d = classify_sharded_p2p(A.classify, fib, peer)
    torch.cuda.synchronize()
    dist.barrier()
    if rank == 0:
        q.put((lab.cpu().numpy(), d.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_equals_single_process(world):
    import torch.multiprocessing as mp
    from paper_1912_11494_b200 import Atlas
    from synth import atlas_for_config, fibers_for_config
    n = 20_001
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    lab, d = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    at = atlas_for_config(1)
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda())
    rl, rd = A.classify(torch.from_numpy(fibers_for_config(1, 0, n)).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(lab, rl.cpu().numpy())
    assert np.array_equal(d.view(np.int32), rd.cpu().numpy().view(np.int32))
