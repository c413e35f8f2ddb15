"""Device-resident calls are classified in slices of at most 2^23 fibers (seg_api.cu, classify_device_sliced)
to bound the scratch memory.  Fibers are independent, so the slicing must not change a single bit.  The
slice is forced small here (SEG_DEV_CHUNK, read once per process) with a ragged last slice."""
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
from paper_1912_11494_b200 import Atlas, binding
from synth import atlas_for_config, fibers_for_config
h = lambda t: hashlib.sha256(np.ascontiguousarray(t.cpu().numpy()).tobytes()).hexdigest()
at = atlas_for_config(1)
c, b, t = (torch.from_numpy(x).cuda() for x in (at.centroids, at.bundle_id, at.thresh))
f = torch.from_numpy(fibers_for_config(1)).cuda()
out = {}
for mode in ("exact", "paper"):
    A = Atlas(c, b, t, mode=mode)
    binding.seg_profile_enable(A._h, 16)              # one profile slot per slice
    lab, d = A.classify(f)
    z = np.zeros(16, np.float32)
    nslices = binding.seg_profile_read(A._h, z, z.copy(), z.copy(), 16)
    k = A.classify_keys(f)
    torch.cuda.synchronize()
    out[mode] = [h(lab), h(d), h(k), int((lab >= 0).sum())]
    out[mode + "_slices"] = nslices
print(json.dumps(out))
"""


def _run(chunk):
    env = dict(os.environ)
    env.pop("SEG_DEV_CHUNK", None)
    if chunk:
        env["SEG_DEV_CHUNK"] = str(chunk)
    r = subprocess.run([sys.executable, "-c", PROBE, ROOT], env=env, cwd=ROOT, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_slicing_is_bit_identical():
    assert torch.cuda.is_available()
    whole = _run(None)
    sliced = _run(30001)          # 100,000 fibers -> slices of 30,001 + a ragged 9,997
    assert whole["exact_slices"] == 1 and sliced["exact_slices"] == 4 and sliced["paper_slices"] == 4
    for m in ("exact", "paper"):
        assert sliced[m] == whole[m]
    assert whole["exact"][3] > 50000
