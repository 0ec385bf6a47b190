"""dev: per-SASS-region instruction histogram of one kernel from an ncu source-page CSV
(ncu -i X.ncu-rep --page source --csv --print-source sass -k regex:K > f.csv)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
his = [i for i, r in enumerate(rows) if 'Address' in r]
hi = his[0]
end = his[1] - 1 if len(his) > 1 else len(rows)
hdr = rows[hi]
data = [r for r in rows[hi + 1:end] if len(r) == len(hdr)]
isrc, iex, wf = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("L1 Wavefronts Shared")
tot = sum(int(r[iex] or 0) for r in data)
print("total warp inst", tot)
groups = []
for k, r in enumerate(data):
    n, w, s = int(r[iex] or 0), int(r[wf] or 0), r[isrc].strip()
    if groups and groups[-1][2] == n:
        groups[-1][1] += 1
        groups[-1][3] += w
        groups[-1][4].append(s)
    else:
        groups.append([k, 1, n, w, [s]])
groups.sort(key=lambda g: -g[1] * g[2])
for g in groups[:int(sys.argv[2]) if len(sys.argv) > 2 else 22]:
    print(f"start {g[0]:5d} len {g[1]:4d} exec {g[2]:>10d} share {g[1]*g[2]/tot:.3f} wf {g[3]:>10d}  "
          f"{g[4][0][:40]} | {g[4][-1][:36]}")
