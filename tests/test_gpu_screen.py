"""The dot-product screen (seg_internal.cuh) never drops a candidate, in either mode.

The dense test1 / test2 of exact mode compare estimates h <= tau / 2 that are provably never above
d2 / 2, and the candidate rounds re-evaluate the three points with d2; so the results must be the same
BITS as the d2 form of the loop (-DSEG_NOSCREEN).  The test builds that library (about a minute of
nvcc), runs both in subprocesses (SEG_LIB) on inputs chosen against the screen's error argument --
large translations (norms up to 1e13 mm^2, where the 2^-18 lowering is widest), coordinates beyond the
2^50 safety limit (-inf half norms), coordinates small enough that squares are subnormal, and exact
ties between bundles -- and requires identical labels and distance bits.  Paper mode (round 2) screens
too and decides the end-point orientation in the candidate round; it must give the same bits as the
round-1 form that decided it in the dense loop on exact distances (-DSEG_PAPER_D2).
"""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1912_11494_b200 import Atlas
from synth import atlas_for_config, fibers_for_config
h = lambda t: hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).hexdigest()
out = {}
MODE = sys.argv[2] if len(sys.argv) > 2 else "exact"
def run(name, C, bid, thr, F):
    A = Atlas(torch.from_numpy(np.ascontiguousarray(C, np.float32)).cuda(), torch.from_numpy(bid).cuda(),
              torch.from_numpy(np.ascontiguousarray(thr, np.float32)).cuda(), mode=MODE)
    lab, d = A.classify(torch.from_numpy(np.ascontiguousarray(F, np.float32)).cuda())
    torch.cuda.synchronize()
    out[name] = [h(lab), h(d.view(torch.int32)), int((lab >= 0).sum())]
for cfg, n in ((0, None), (1, 20000)):
    at = atlas_for_config(cfg)
    F = fibers_for_config(cfg, 0, n)
    C, bid, thr = at.centroids, at.bundle_id, at.thresh
    run(f"{cfg}", C, bid, thr, F)
    for off in (1e4, -3e6):
        run(f"{cfg}off{off}", C + np.float32(off), bid, thr, F + np.float32(off))
    # a third of the fibers and one bundle far beyond the 2^50 limit (the -inf half-norm path)
    Fu, Cu = F.copy(), C.copy()
    Fu[::3] += np.float32(2.0 ** 52)
    Cu[bid == 0] += np.float32(2.0 ** 52)
    run(f"{cfg}unsafe", Cu, bid, thr, Fu)
    # tiny coordinates: squared distances and thresholds near and below the FP32 normal range
    for sc in (1e-17, 1e-19):
        run(f"{cfg}tiny{sc}", C * np.float32(sc), bid, thr * np.float32(sc), F * np.float32(sc))
    # exact ties: every centroid duplicated into a second bundle (smaller bundle id must win)
    B = len(thr)
    run(f"{cfg}ties", np.concatenate([C, C]), np.concatenate([bid, (bid + 1) % B]).astype(np.int32),
        np.concatenate([thr]), F)
print(json.dumps(out))
"""


def _run(env_extra, mode="exact"):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", PROBE, ROOT, mode], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def noscreen_lib():
    from paper_1912_11494_b200 import _build
    out = os.path.join(ROOT, "build", "noscreen", "libsegb200.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run([_build.nvcc(), *_build.NVCC_FLAGS, "-DSEG_NOSCREEN", "-o", out, *_build.SOURCES], check=True,
                   capture_output=True, timeout=900)
    return out


def test_screen_matches_d2_form_bit_for_bit(noscreen_lib):
    assert torch.cuda.is_available()
    prod = _run({"SEG_LIB": ""})
    ref = _run({"SEG_LIB": noscreen_lib})
    assert set(prod) == set(ref)
    bad = {k: (prod[k], ref[k]) for k in prod if prod[k] != ref[k]}
    assert not bad, bad
    assert prod["1"][2] > 10000 and prod["1off10000.0"][2] > 10000   # the cases label fibers


@pytest.fixture(scope="module")
def paper_d2_lib():
    from paper_1912_11494_b200 import _build
    out = os.path.join(ROOT, "build", "paperd2", "libsegb200.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run([_build.nvcc(), *_build.NVCC_FLAGS, "-DSEG_PAPER_D2", "-o", out, *_build.SOURCES], check=True,
                   capture_output=True, timeout=900)
    return out


def test_paper_screen_matches_d2_form_bit_for_bit(paper_d2_lib):
    prod = _run({"SEG_LIB": ""}, "paper")
    ref = _run({"SEG_LIB": paper_d2_lib}, "paper")
    assert set(prod) == set(ref)
    bad = {k: (prod[k], ref[k]) for k in prod if prod[k] != ref[k]}
    assert not bad, bad
    assert prod["1"][2] > 10000
