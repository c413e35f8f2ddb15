"""bench.py's multi-rank paths end to end (one process per rank under torch.distributed.run): with one GPU
here, two ranks share cuda:0 over a gloo process group (SEG_BENCH_ONE_DEVICE, SEG_BENCH_BACKEND) -- a
functional check of the strong-scaling partition the driver's scaling run uses (one subject sharded, the
gather in every step, the per-rank e2e path and its equality check), not a timing."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("extra", [[], ["--gather", "p2p"], ["--scaling", "weak"]])
def test_bench_two_ranks(extra):
    env = dict(os.environ, SEG_BENCH_ONE_DEVICE="1", SEG_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "3", "--e2e-steps", "1", "--no-stats",
           *extra]
    r = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]          # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    weak = "--scaling" in extra
    assert d["scaling"] == ("weak" if weak else "strong")
    assert d["config"]["fibers"] == (200_000 if weak else 100_000)
    assert d["config"]["fibers_per_gpu"] == (100_000 if weak else 50_000)
