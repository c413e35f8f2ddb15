"""Summarise an ncu report: key SOL/scheduler metrics, stall reasons and per-source-line hot spots.

    python scripts/ncu_summary.py REPORT.ncu-rep [TOP_LINES] [KERNEL_REGEX]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
kern = sys.argv[3] if len(sys.argv) > 3 else None   # a kernel-name regex, for reports holding several kernels


def ncu(*args):
    filt = ["-k", f"regex:{kern}"] if kern else []
    return subprocess.run(["ncu", "-i", rep, *filt, *args], capture_output=True, text=True).stdout


rows = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
h = rows[0]
si, mi, ui, vi = h.index("Section Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
keep = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Avg. Active Threads Per Warp",
        "Warp Cycles Per Issued Instruction", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Issued Instructions", "L1/TEX Hit Rate", "L2 Hit Rate", "Theoretical Occupancy", "Eligible Warps Per Scheduler",
        "Dynamic Shared Memory Per Block", "Compute (SM) Throughput", "Memory Throughput"]
for r in rows[1:]:
    if len(r) > vi and r[mi] in keep:
        print(f"  {r[mi]:40s} {r[vi]} {r[ui]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, u, v = raw[0], raw[1], raw[2]
st = []
for name, unit, val in zip(h, u, v):
    if name.startswith("smsp__pcsamp_warps_issue_stalled") and not name.endswith("not_issued"):
        try:
            st.append((float(val.replace(",", "")), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    if name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                "smsp__thread_inst_executed_per_inst_executed.ratio"):
        print(f"  {name:60s} {val} {unit}")
tot = sum(x for x, _ in st) or 1
print("  stalls: " + ", ".join(f"{n} {100 * x / tot:.1f}%" for x, n in sorted(st, reverse=True)[:8]))
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source=cuda,sass"))))
cur, agg = None, {}
for r in rows:
    if len(r) < 9:
        continue
    if r[0] and r[0].isdigit():
        cur = (int(r[0]), r[1].strip()[:90])
    elif r[0]:
        continue
    try:
        s, e, t = int(r[4] or 0), int(r[7] or 0), int(r[8] or 0)
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0, 0])
    a[0] += s; a[1] += e; a[2] += t
tot = sum(x[0] for x in agg.values()) or 1
print(f"  source lines by stall samples (total {tot}):")
for k, x in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"  {k[0]:4d} {100 * x[0] / tot:5.1f}%  inst={x[1]:11d} thr/inst={x[2] / max(x[1], 1):5.1f}  {k[1]}")
