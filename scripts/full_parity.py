#!/usr/bin/env python
"""Full-size parity: every fiber of configs 0-4, both modes, CUDA path vs the oracle (GPU).

    python scripts/full_parity.py [--configs 0 1 2 3 4] [--modes exact paper] [--out FILE.json]

Each config is classified through the C ABI exactly as bench.py launches it (one seg_classify of the
whole device-resident subject).  The oracle side is the sound-discard oracle's output for every fiber,
from cache/oracle/ (scripts/oracle_full.py, checked against the sha256 of these very inputs and of
oracle/oracle.c), or computed here on the host cores when the cache is absent or stale.  The rule is
tests/parity_util.py's: labels bit-identical on every decidable fiber, distances within 1e-5
relative, +inf / NaN conventions, and every undecidable (tie-band) fiber's answer checked to be one of
the correct answers from the plain oracle's per-bundle intervals.  Prints one JSON record per
(config, mode) and writes them all to --out.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "scripts"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2, 3, 4])
    ap.add_argument("--modes", nargs="+", default=["exact", "paper"])
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "full_parity.json"))
    a = ap.parse_args()
    import torch

    import oracle_full
    from paper_1912_11494_b200 import Atlas
    from parity_util import check_parity, valid_answers
    from synth import atlas_for_config, fibers_for_config

    recs = []
    for cfg in a.configs:
        at = atlas_for_config(cfg)
        fib = fibers_for_config(cfg)
        f = torch.from_numpy(fib).cuda()
        for mode in a.modes:
            t0 = time.perf_counter()
            ref = oracle_full.load(cfg, mode, fib, at)
            source = "cache/oracle (scripts/oracle_full.py)"
            if ref is None:
                ref = oracle_full.compute(cfg, mode, os.cpu_count() or 1, fib, at)
                source = f"computed here on {os.cpu_count()} host threads"
            t_or = time.perf_counter() - t0
            A = Atlas(torch.from_numpy(at.centroids).cuda(), torch.from_numpy(at.bundle_id).cuda(),
                      torch.from_numpy(at.thresh).cuda(), mode=mode)
            lab, d = A.classify(f)
            torch.cuda.synchronize()
            lab, d = lab.cpu().numpy(), d.cpu().numpy()
            rec = dict(cfg=cfg, mode=mode, n=int(fib.shape[0]), M=at.M, oracle=source, oracle_s=round(t_or, 1),
                       oracle_variant=ref["meta"]["variant"], oracle_sha=ref["meta"]["oracle_sha"][:16],
                       fibers_sha=ref["meta"]["fibers_sha"][:16])
            dec = ref["decidable"]
            rec["decidable"] = int(dec.sum())
            rec["undecidable"] = int((~dec).sum())
            rec["labelled_oracle"] = int((ref["label"] >= 0).sum())
            rec["label_mismatch_decidable"] = int((dec & (lab != ref["label"])).sum())
            same = dec & (lab == ref["label"]) & (ref["label"] >= 0)
            rel = np.abs(d[same].astype(np.float64) - ref["dist"][same]) / np.maximum(ref["dist"][same], 1e-300)
            rel[ref["dist"][same] == 0] = np.abs(d[same][ref["dist"][same] == 0])
            rec["dist_max_rel_err"] = float(rel.max()) if rel.size else 0.0
            rec["dist_outside_1e-5"] = int((rel > 1e-5).sum())
            try:
                check_parity(lab, d, ref, f"cfg{cfg} {mode}")
                rec["parity"] = "pass"
            except AssertionError as e:
                rec["parity"] = "FAIL: " + str(e)[:300]
            und = ref["undec_idx"]
            if und.size:
                ok = valid_answers(lab[und], d[und], ref["undec_lo"], ref["undec_hi"], at.thresh)
                rec["tie_band_valid"] = int(ok.sum())
                rec["tie_band_invalid"] = int((~ok).sum())
                rec["tie_band_label_equal"] = int((lab[und] == ref["label"][und]).sum())
            else:
                rec["tie_band_valid"] = rec["tie_band_invalid"] = rec["tie_band_label_equal"] = 0
            print(json.dumps(rec), flush=True)
            recs.append(rec)
            del A
        del f, fib
        torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as fh:
        json.dump(recs, fh, indent=1)
    bad = [r for r in recs if r["parity"] != "pass" or r["tie_band_invalid"]]
    print(f"{len(recs)} (config, mode) runs, {len(bad)} failing", flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
