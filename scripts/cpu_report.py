#!/usr/bin/env python
"""The CPU side of the SURVEY.md Sec. 8(d) report: the oracle timed on this machine's host cores.

    python scripts/cpu_report.py > cpu_report.jsonl

Per config and mode: the sound-discard oracle (oracle_classify_sound -- Alg. 1's cascade with the early
exit; bitwise the plain definition's labels, tests/test_oracle_sound.py) on all
host cores, at full size for configs 0-2 and "extrapolated x100 from a 1% seeded subsample" (stream-2
seeds) for configs 3-4 (fibers are i.i.d., so time is proportional to N); the same single-threaded on
configs 0-1; and the plain brute force (every pair, 42 distances) on config 0, all cores and one.
The paper's own multi-threaded C++ (i7-6700K, 4 cores / 8 threads) took about 6 min for the 4,145,000-
fiber subject against 44,345 centroids: 5.1e8 comparisons/s (derived in BASELINE.md).
"""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import CONFIGS, atlas_for_config, fibers_for_config, sample_indices  # noqa: E402


def lscpu_model():
    out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    return next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name:")), "unknown")


def timed(fib, at, mode, threads, sound):
    t0 = time.perf_counter()
    r = oracle.classify(fib, at.centroids, at.bundle_id, at.thresh, mode=mode, threads=threads, sound=sound)
    return time.perf_counter() - t0, r


def main():
    cores = os.cpu_count() or 1
    head = dict(cpu_model=lscpu_model(), nproc=cores)
    print(json.dumps(head), flush=True)
    for cfg in range(5):
        at = atlas_for_config(cfg)
        n = CONFIGS[cfg]["n_fibers"]
        fib = fibers_for_config(cfg)
        if cfg <= 2:
            sub, how = fib, "full size"
        else:
            idx = sample_indices(n, n // 100, seed=2)
            sub, how = fib[idx], f"extrapolated x100 from a 1% seeded subsample ({idx.size:,} fibers, seed 2)"
        for mode in ("exact", "paper"):
            runs = [("sound", cores)] + ([("sound", 1)] if cfg <= 1 else []) + \
                   ([("plain", cores), ("plain", 1)] if cfg == 0 else [])
            for variant, th in runs:
                dt, r = timed(sub, at, mode, th, variant == "sound")
                scale = n / sub.shape[0]
                rec = dict(cfg=cfg, mode=mode, oracle=("sound-discard (Alg. 1 cascade, fp64)" if variant == "sound"
                                                        else "plain brute force (every pair, fp64)"),
                           threads=th, fibers=n, centroids=at.M, sample=how, seconds_measured=round(dt, 3),
                           seconds_full=round(dt * scale, 2), comparisons_per_s=n * at.M / (dt * scale),
                           fibers_per_s=n / (dt * scale), labelled=int((r["label"] >= 0).sum()),
                           undecidable=int((~r["decidable"]).sum()))
                print(json.dumps(rec), flush=True)
        del fib


if __name__ == "__main__":
    main()
