"""The checked build (-DSEG_DEBUG, scripts/checked_build.sh) on the GPU: every shared-memory queue index,
ring stage, tile index and scatter position is bounds-checked on the device and a violation traps.  The
GPU pool offers no compute-sanitizer, so this is its stand-in.

The test compiles the checked library (about a minute of nvcc), runs every entry point through it in a
subprocess (SEG_LIB), and requires the same bits as the production library: the checks only observe.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# runs under either library; prints a JSON digest of every output
PROBE = r"""
import hashlib, json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1912_11494_b200 import Atlas, group_by_bundle, keys_to_labels, resample
from synth import atlas_for_config, fibers_for_config
from synth.raw import raw_streamlines
h = lambda t: hashlib.sha256(np.ascontiguousarray(t.cpu().numpy() if torch.is_tensor(t) else t).tobytes()).hexdigest()
out = {}
for cfg, n in ((0, None), (1, 20000)):
    at = atlas_for_config(cfg)
    c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
    fib = fibers_for_config(cfg, 0, n)
    fib[5, 3, 2] = np.nan
    f = torch.from_numpy(fib).cuda()
    for mode in ("exact", "paper"):
        A = Atlas(c, b, t, mode=mode)
        lab, d = A.classify(f)
        k = A.classify_keys(f)
        l2, d2 = keys_to_labels(k, mode)
        hl, hd = A.classify(np.ascontiguousarray(fib[:3001]))
        torch.cuda.synchronize()
        out[f"{cfg}{mode}"] = [h(lab), h(d), h(k), h(l2), h(d2), h(hl), h(hd)]
        if mode == "exact":
            order, off, dmin, dmax, dsum = group_by_bundle(lab, d, at.B)
            torch.cuda.synchronize()
            out[f"{cfg}group"] = [h(order), h(off), h(dmin), h(dmax), h(dsum)]
pts, offs = raw_streamlines(fibers_for_config(0, 0, 500), 1)
r = resample(torch.from_numpy(pts).cuda(), torch.from_numpy(offs).cuda())
torch.cuda.synchronize()
out["resample"] = h(r)
print(json.dumps(out))
"""


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", PROBE, ROOT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


@pytest.fixture(scope="module")
def checked_lib():
    from paper_1912_11494_b200 import _build
    out = os.path.join(ROOT, "build", "checked", "libsegb200.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    subprocess.run([_build.nvcc(), *_build.NVCC_FLAGS, "-DSEG_DEBUG", "-o", out, *_build.SOURCES], check=True,
                   capture_output=True, timeout=900)
    return out


def test_checked_build_matches_production(checked_lib):
    assert torch.cuda.is_available()
    prod = _run({"SEG_LIB": ""})
    chk = _run({"SEG_LIB": checked_lib})
    assert chk == prod
