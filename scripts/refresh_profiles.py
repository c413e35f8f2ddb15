"""Copy a scripts/gpu/ncu.sh run (gpurun_out/) into profiles/<round>/: the launch list and per-kernel shares,
ncu summaries of k_classify (exact and paper mode) and k_cull, and profiles/traffic.json (k_classify DRAM
bytes per launch from the full captures, keyed by config and mode).

    python scripts/refresh_profiles.py r02
"""
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RND = sys.argv[1] if len(sys.argv) > 1 else "r02"
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", RND)
os.makedirs(P, exist_ok=True)
shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, "launches_cfg3.csv"))

rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
d = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = v / 1000 if r[ui] in ("nsecond", "ns") else (v * 1000 if r[ui] in ("msecond", "ms") else v)
    d[re.sub(r"seg::", "", r[ki]).strip()].append(v)
prod = {k: v for k, v in d.items() if "<1," not in k and "k_" in k}
tot = sum(sum(v) / len(v) for v in prod.values())
out = [f"{k:40s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  share of the production launches={100 * sum(v) / len(v) / tot:5.1f}%"
       for k, v in sorted(prod.items(), key=lambda x: -sum(x[1]) / len(x[1]))]
out += [f"{k:40s} n={len(v):3d} mean={sum(v) / len(v):9.1f} us  (stats instantiation, run once by bench.py for the "
        f"counters; not part of a step)" for k, v in d.items() if "<1," in k]
out.append("(ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache serialised launches of: "
           "python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline)")
open(os.path.join(P, "launch_shares_cfg3.txt"), "w").write("\n".join(out) + "\n")
print("\n".join(out))

tf = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(tf)) if os.path.exists(tf) else {}
for rep, dst, key in (("prof_classify", "ncu_k_classify_summary.txt", "cfg3_exact"),
                      ("prof_classify_paper", "ncu_k_classify_paper_summary.txt", "cfg3_paper"),
                      ("prof_cull", "ncu_k_cull_summary.txt", None)):
    path = os.path.join(G, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    s = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), path, "30"],
                       capture_output=True, text=True).stdout
    open(os.path.join(P, dst), "w").write(s)
    if key is None:
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    b = {n: float(v.replace(",", "")) * scale[u] for n, u, v in zip(rr[0], rr[1], rr[2]) if n.startswith("dram__bytes")}
    t[key] = dict(bytes=int(round(sum(b.values()))), kernel="k_classify",
                  source=(f"profiles/{RND}/{dst} (dram__bytes_read.sum {b['dram__bytes_read.sum'] / 1e9:.6f} GB + "
                          f"dram__bytes_write.sum {b['dram__bytes_write.sum'] / 1e6:.6f} MB, one ncu --set full capture)"),
                  algorithmic_bytes=4_145_000 * (252 + 8))
json.dump(t, open(tf, "w"), indent=1)
print(json.dumps(t, indent=1))
