#!/usr/bin/env python
"""The GPU side of the SURVEY.md Sec. 8(d) report: one bench.py line per config (0-4) and mode at N=1.

    python scripts/report.py [--modes exact paper] > report_rows.jsonl

Each line is bench.py's own JSON (device-resident step, kernel times from the library's events, FP32
roofline fraction, e2e through the host-buffer path, clocks); configs 0-2 are timed step by step after
an L2 flush (their inputs fit in L2).  The oracle's timing for the same configs is scripts/cpu_report.py.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STEPS = {0: 50, 1: 50, 2: 30, 3: 30, 4: 20}

ap = argparse.ArgumentParser()
ap.add_argument("--modes", nargs="+", default=["exact", "paper"])
ap.add_argument("--configs", type=int, nargs="+", default=[0, 1, 2, 3, 4])
a = ap.parse_args()
for cfg in a.configs:
    for mode in a.modes:
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", str(cfg), "--mode", mode,
               "--steps", str(STEPS[cfg]), "--warmup", "3", "--no-cpu-baseline"]
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.returncode == 0 and r.stdout.strip() else None
        if line is None:
            print(json.dumps(dict(cfg=cfg, mode=mode, error=r.stderr[-500:])), flush=True)
            continue
        d = json.loads(line)
        d["report_cfg"], d["report_mode"] = cfg, mode
        print(json.dumps(d), flush=True)
