#!/usr/bin/env python
"""Full-size oracle outputs for the parity run (scripts/full_parity.py, tests/test_gpu_full_parity.py).

    python scripts/oracle_full.py [--configs 0 1 2 3 4] [--modes exact paper] [--threads N]

Calls only oracle/ (the sound-discard variant, pinned bitwise to the plain definition by
tests/test_oracle_sound.py) and synth/ (the seeded inputs).  For every fiber of the config it stores
the oracle's label, dist and decidable flag in cache/oracle/cfg{K}_{mode}.npz, with the sha256 of
the fiber and atlas arrays and of oracle/oracle.c, so a stale cache (other inputs, other oracle
arithmetic) is detected and refused.  For the undecidable fibers it also stores the per-bundle
intervals [lo, hi] of correct values from the plain oracle (want_bands), which the valid-answer
check of tests/parity_util.py reads.  Nothing here comes from the CUDA path.

cache/ is git-ignored (hundreds of MB) and gpurun-ignored by default; the parity call ships it.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CACHE = os.path.join(ROOT, "cache", "oracle")


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).reshape(-1))
    return h.hexdigest()


def oracle_src_sha() -> str:
    with open(os.path.join(ROOT, "oracle", "oracle.c"), "rb") as fh:
        return hashlib.sha256(fh.read()).hexdigest()


def cache_path(cfg: int, mode: str) -> str:
    return os.path.join(CACHE, f"cfg{cfg}_{mode}.npz")


def load(cfg: int, mode: str, fibers: np.ndarray | None = None, atlas=None):
    """The cached outputs as a dict, or None when absent or stale (inputs or oracle changed)."""
    p = cache_path(cfg, mode)
    if not os.path.exists(p):
        return None
    z = np.load(p)
    meta = json.loads(str(z["meta"]))
    if meta["oracle_sha"] != oracle_src_sha():
        return None
    if fibers is not None and meta["fibers_sha"] != sha(fibers):
        return None
    if atlas is not None and meta["atlas_sha"] != sha(atlas.centroids, atlas.bundle_id, atlas.thresh):
        return None
    out = dict(label=z["label"].astype(np.int32), dist=z["dist"], decidable=z["decidable"],
               undec_idx=z["undec_idx"], undec_lo=z["undec_lo"], undec_hi=z["undec_hi"], meta=meta)
    return out


def compute(cfg: int, mode: str, threads: int, fibers=None, atlas=None, log=print):
    import oracle
    from synth import atlas_for_config, fibers_for_config
    at = atlas if atlas is not None else atlas_for_config(cfg)
    fib = fibers if fibers is not None else fibers_for_config(cfg)
    t0 = time.perf_counter()
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode=mode, sound=True, threads=threads)
    dt = time.perf_counter() - t0
    und = np.nonzero(~r["decidable"])[0]
    if und.size:
        b = oracle.classify(fib[und], at.centroids, at.bundle_id, at.thresh, mode=mode, threads=threads,
                            want_bands=True)
        lo, hi = b["lo"], b["hi"]
        assert np.array_equal(b["label"], r["label"][und]), "sound and plain oracles disagree"
    else:
        lo = hi = np.zeros((0, at.B))
    meta = dict(cfg=cfg, mode=mode, n=int(fib.shape[0]), M=at.M, B=at.B, seconds=dt, threads=threads,
                fibers_sha=sha(fib), atlas_sha=sha(at.centroids, at.bundle_id, at.thresh),
                oracle_sha=oracle_src_sha(), numpy=np.__version__, variant="oracle_classify_sound",
                labelled=int((r["label"] >= 0).sum()), undecidable=int(und.size))
    log(f"cfg{cfg} {mode}: {fib.shape[0]:,} fibers x {at.M:,} centroids in {dt:.1f} s on {threads} threads; "
        f"{meta['labelled']:,} labelled, {und.size} undecidable")
    return dict(label=r["label"], dist=r["dist"], decidable=r["decidable"], undec_idx=und, undec_lo=lo,
                undec_hi=hi, meta=meta)


def save(cfg: int, mode: str, res) -> str:
    os.makedirs(CACHE, exist_ok=True)
    p = cache_path(cfg, mode)
    tmp = p + ".tmp.npz"
    np.savez(tmp, label=res["label"].astype(np.int16), dist=res["dist"], decidable=res["decidable"],
             undec_idx=res["undec_idx"], undec_lo=res["undec_lo"], undec_hi=res["undec_hi"],
             meta=json.dumps(res["meta"]))
    os.replace(tmp, p)
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2, 3, 4])
    ap.add_argument("--modes", nargs="+", default=["exact", "paper"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    from synth import atlas_for_config, fibers_for_config
    for cfg in a.configs:
        at = atlas_for_config(cfg)
        fib = fibers_for_config(cfg)
        for mode in a.modes:
            if not a.force and load(cfg, mode, fib, at) is not None:
                print(f"cfg{cfg} {mode}: cached", flush=True)
                continue
            res = compute(cfg, mode, a.threads, fib, at, log=lambda s: print(s, flush=True))
            print("  ->", save(cfg, mode, res), flush=True)
        del fib


if __name__ == "__main__":
    main()
