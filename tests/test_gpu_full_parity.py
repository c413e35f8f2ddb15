"""Full-size parity on every fiber (configs 1-4, both modes), against the oracle outputs cached by
scripts/oracle_full.py (the sound-discard oracle, pinned bitwise to the plain definition by
tests/test_oracle_sound.py; the cache is refused when the inputs or oracle/oracle.c changed).

The cache is hundreds of MB and does not travel with every GPU call; without it these tests skip and
scripts/full_parity.py (which computes the oracle on the host when needed) is the full-size run.  The
always-on full-size checks are tests/test_gpu_parity.py's sampled ones.
"""
import os
import sys

import numpy as np
import pytest
import torch

from parity_util import check_parity, check_valid
from synth import atlas_for_config, fibers_for_config

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "scripts"))

if torch.cuda.is_available():
    from paper_1912_11494_b200 import Atlas


@pytest.mark.parametrize("cfg", [1, 2, 3, 4])
@pytest.mark.parametrize("mode", ["exact", "paper"])
def test_every_fiber_matches_the_cached_oracle(cfg, mode):
    import oracle_full
    at = atlas_for_config(cfg)
    fib = fibers_for_config(cfg)
    ref = oracle_full.load(cfg, mode, fib, at)
    if ref is None:
        pytest.skip(f"no current oracle cache for cfg{cfg} {mode} (run scripts/oracle_full.py)")
    A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
              torch.from_numpy(at.thresh).cuda(), mode=mode)
    lab, d = A.classify(torch.from_numpy(fib).cuda())
    torch.cuda.synchronize()
    lab, d = lab.cpu().numpy(), d.cpu().numpy()
    info = check_parity(lab, d, ref, f"cfg{cfg} {mode} full")
    assert info["n"] == fib.shape[0]
    check_valid(lab, d, ref["undec_idx"], ref["undec_lo"], ref["undec_hi"], at.thresh, f"cfg{cfg} {mode} tie band")
    assert np.all(d[lab >= 0] <= at.thresh[lab[lab >= 0]] + 1e-3)
