"""Copy a gpu_round.sh run (gpurun_out/) into profiles/r01/: bench lines, launch list + shares, ncu summaries,
and profiles/traffic.json (k_classify DRAM bytes from the full capture)."""
import csv, collections, io, json, os, re, shutil, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles", "r01")
for src, dst in (("bench.json", "bench_cfg3.json"), ("bench_ref.json", "bench_reference_cfg3.json"),
                 ("bench_paper.json", "bench_cfg3_paper_mode.json"), ("bench_rows.jsonl", "bench_rows_cfg3.jsonl"),
                 ("launches.csv", "launches_cfg3.csv")):
    shutil.copy(os.path.join(G, src), os.path.join(P, dst))

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

for rep, dst in (("prof_classify", "ncu_k_classify_summary.txt"), ("prof_cull", "ncu_k_cull_summary.txt")):
    s = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_summary.py"), os.path.join(G, rep + ".ncu-rep"), "30"],
                       capture_output=True, text=True).stdout
    open(os.path.join(P, dst), "w").write(s)

raw = subprocess.run(["ncu", "-i", os.path.join(G, "prof_classify.ncu-rep"), "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], rr[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
b = {}
for n, u, v in zip(hdr, units, vals):
    if n.startswith("dram__bytes"):
        b[n] = float(v.replace(",", "")) * scale[u]
tf = os.path.join(ROOT, "profiles", "traffic.json")
t = json.load(open(tf))
t["cfg3"]["bytes"] = int(round(sum(b.values())))
t["cfg3"]["source"] = (f"profiles/r01/ncu_k_classify_summary.txt (dram__bytes_read.sum {b['dram__bytes_read.sum'] / 1e9:.6f} GB + "
                       f"dram__bytes_write.sum {b['dram__bytes_write.sum'] / 1e6:.6f} MB, one ncu --set full capture at HEAD)")
json.dump(t, open(tf, "w"), indent=1)
print(t)
