#!/usr/bin/env python
"""Copy a scripts/gpu/round_evidence.sh run (gpurun_out/) into profiles/<round>/ and regenerate the tables.

    python scripts/collect_evidence.py r02

- bench.json / bench_ref.json      -> bench_cfg3.json / bench_reference_cfg3.json (the default bench lines)
- bench_rows.jsonl, report_rows.jsonl (per-config bench lines), full_parity.log (+ .json: its JSON lines)
- pytest_gpu.log                   -> pytest_gpu.log (the GPU suite of the same call)
then scripts/refresh_profiles.py (launch list, ncu summaries, traffic.json) and scripts/make_tables.py.
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", RND)
os.makedirs(P, exist_ok=True)


def last_json_line(path):
    lines = [l for l in open(path) if l.strip().startswith("{")]
    return lines[-1].strip()


for src, dst in (("bench.json", "bench_cfg3.json"), ("bench_ref.json", "bench_reference_cfg3.json")):
    open(os.path.join(P, dst), "w").write(last_json_line(os.path.join(G, src)) + "\n")
for name in ("bench_rows.jsonl", "report_rows.jsonl", "full_parity.log", "pytest_gpu.log"):
    shutil.copy(os.path.join(G, name), os.path.join(P, name))
par = [json.loads(l) for l in open(os.path.join(G, "full_parity.log")) if l.strip().startswith("{")]
json.dump(par, open(os.path.join(P, "full_parity.json"), "w"), indent=1)
print(f"full parity: {len(par)} runs, failing: {[ (r['cfg'], r['mode']) for r in par if r['parity'] != 'pass']}")
for script in ("refresh_profiles.py", "make_tables.py"):
    subprocess.run([sys.executable, os.path.join(ROOT, "scripts", script), RND] if script == "refresh_profiles.py"
                   else [sys.executable, os.path.join(ROOT, "scripts", script)], check=True)
