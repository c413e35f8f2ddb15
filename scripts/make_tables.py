#!/usr/bin/env python
"""Regenerate BASELINE.md's 'Measured' section from the committed round evidence (profiles/r02/):
report_rows.jsonl (bench.py per config and mode), cpu_report.jsonl (oracle on the B200 box's host cores),
full_parity.json (every fiber vs the oracle).  Rewrites the text between the MEASURED markers."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles", "r02")
rows = [json.loads(l) for l in open(os.path.join(P, "report_rows.jsonl")) if l.strip()]
cpu = [json.loads(l) for l in open(os.path.join(P, "cpu_report.jsonl")) if l.strip()]
par = {(r["cfg"], r["mode"]): r for r in json.load(open(os.path.join(P, "full_parity.json")))}
head = cpu[0]
cpu_by = {}
for c in cpu[1:]:
    cpu_by.setdefault((c["cfg"], c["mode"], c["oracle"].split()[0], c["threads"]), c)


def sci(x):
    m, e = f"{x:.2e}".split("e")
    return f"{m}×10^{int(e)}"


out = ["| cfg | mode | N | M | step ms (prepass + k_cull + k_classify) | comparisons/s | fibers/s | FP32 frac (k_classify) | "
       "e2e ms (host buffers) | oracle, all cores | vs oracle | parity: decidable mismatches / tie-band (valid) |",
       "|---|---|---|---|---|---|---|---|---|---|---|---|"]
for d in rows:
    if "error" in d:
        continue
    cfg, mode = d["report_cfg"], d["report_mode"]
    r = d["roofline"]
    c = cpu_by.get((cfg, mode, "sound-discard", head["nproc"]))
    pr = par.get((cfg, mode))
    ctxt = (f"{sci(c['comparisons_per_s'])}/s" + (" (extrapolated ×100, 1% sample)" if cfg >= 3 else " (full size)")) if c else "—"
    ratio = f"{d['value'] / c['comparisons_per_s']:,.0f}×" if c else "—"
    ptxt = f"{pr['label_mismatch_decidable']} / {pr['undecidable']:,} ({pr['tie_band_valid']:,})" if pr else "—"
    out.append(f"| {cfg} | {mode} | {d['config']['fibers']:,} | {d['config']['centroids']:,} | {d['ms_per_step']:.3f} "
               f"({r['prepass_ms']:.3f} + {r['cull_ms']:.3f} + {r['kernel_ms']:.3f}) | {sci(d['value'])} | {sci(d['fibers_per_s'])} | "
               f"{r['frac']:.3f} | {d['e2e']['ms_per_step']:.2f} | {ctxt} | {ratio} | {ptxt} |")
extra = ["", f"Oracle machine: {head['cpu_model']}, {head['nproc']} host threads (the B200 box's host). "
         "Single-thread and brute-force oracle timings:", "",
         "| cfg | mode | oracle | threads | comparisons/s | seconds (full size) |", "|---|---|---|---|---|---|"]
for c in cpu[1:]:
    if c["threads"] == 1 or c["oracle"].startswith("plain"):
        extra.append(f"| {c['cfg']} | {c['mode']} | {c['oracle']} | {c['threads']} | {sci(c['comparisons_per_s'])}/s | {c['seconds_full']} |")
text = "\n".join(out + extra)
b = os.path.join(ROOT, "BASELINE.md")
s = open(b).read()
s = re.sub(r"<!-- MEASURED -->.*<!-- /MEASURED -->", "<!-- MEASURED -->\n" + text + "\n<!-- /MEASURED -->", s, flags=re.S)
open(b, "w").write(s)
print(text)
