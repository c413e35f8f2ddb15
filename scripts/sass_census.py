#!/usr/bin/env python
"""SASS census of one kernel in an ncu report: issued warp instructions and stall samples per basic block.

    python scripts/sass_census.py REPORT.ncu-rep KERNEL_REGEX [TOP]

Reads `ncu -i REPORT --page source --csv --print-source=sass` and groups consecutive SASS instructions with the same
execution count into blocks (a straight-line run executes as often as its first instruction), then lists the blocks
by their share of the kernel's issued instructions and of its warp-stall samples, with the first instruction of each.
This is how round 2 found the dense step's FLO -> LEA -> LDS head, the per-tile end-marker load and k_cull's
per-passing-tile ballots.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
ai, si = h.index("Address"), h.index("Source")
ie, ns = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
seen, recs = set(), []
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[ai].startswith("0x") or r[ai] in seen:
        continue
    seen.add(r[ai])
    recs.append((int(r[ai], 16), r[si].strip(), int(r[ie] or 0), int(r[ns] or 0)))
recs.sort()
base = recs[0][0]
tot_i = sum(x[2] for x in recs) or 1
tot_s = sum(x[3] for x in recs) or 1
blocks, cur = [], None
for a, src, e, st in recs:
    if cur is not None and cur["exec"] == e:
        cur["end"], cur["n"], cur["samples"] = a, cur["n"] + 1, cur["samples"] + st
    else:
        cur = dict(start=a, end=a, exec=e, n=1, samples=st, first=src)
        blocks.append(cur)
print(f"{kern}: {tot_i:,} warp instructions issued, {tot_s:,} stall samples")
print(f"{'block':>15s} {'instr':>5s} {'executions':>12s} {'% instr':>8s} {'% stalls':>8s}  first instruction")
for b in sorted(blocks, key=lambda b: -b["exec"] * b["n"])[:top]:
    print(f"{b['start'] - base:6x}-{b['end'] - base:6x}  {b['n']:5d} {b['exec']:12,d} {100 * b['exec'] * b['n'] / tot_i:7.1f}% "
          f"{100 * b['samples'] / tot_s:7.1f}%  {b['first'][:60]}")
