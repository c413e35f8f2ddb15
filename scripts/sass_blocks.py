"""Per-basic-block instruction and stall breakdown of an ncu report (SASS source page)."""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, wi, ie, te = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed'), h.index('Thread Instructions Executed')
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
data = []
for r in rows[2:]:
    try:
        data.append((r[si], int(r[wi] or 0), int(r[ie] or 0), int(r[te] or 0), {c: int(r[h.index(c)] or 0) for c in cols}))
    except (ValueError, IndexError):
        pass
blocks = []; start = 0
for i in range(1, len(data) + 1):
    if i == len(data) or data[i][2] != data[start][2]:
        seg = data[start:i]
        st = {c: sum(d[4][c] for d in seg) for c in cols}
        blocks.append((start, i - start, data[start][2], sum(d[1] for d in seg), sum(d[3] for d in seg), st, data[start][0][:40]))
        start = i
tot = sum(d[2] for d in data); totw = sum(d[1] for d in data)
print(f"total inst {tot/1e9:.3f}G, samples {totw}")
for s, n, e, w, t, st, txt in sorted(blocks, key=lambda b: -b[3])[:top]:
    top3 = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{s:5d} len={n:3d} exec={e:10d} inst={n*e/1e9:5.2f}G ({100*n*e/tot:4.1f}%) thr={t/max(n*e,1):4.1f} stall={100*w/totw:4.1f}% "
          + " ".join(f"{k[6:]}={100*v/max(w,1):.0f}%" for k, v in top3) + f"  {txt}")
