"""Aggregate an ncu SASS source page (csv) into basic-block-ish segments:
instructions executed, avg active threads, stall samples.
usage: ncu -i rep --page source --csv --print-source sass > f.csv; python tools/sass_hot.py f.csv"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex = hdr.index("Instructions Executed")
ith = hdr.index("Thread Instructions Executed")
ism = hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= iex:
        continue
    try:
        data.append((int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[ith] or 0), int(r[ism] or 0)))
    except ValueError:
        pass
base = data[0][0]
tot_ex = sum(d[2] for d in data)
tot_sm = sum(d[4] for d in data)
# segments: break where the execution count changes
segs = []
cur = [data[0]]
for d in data[1:]:
    if d[2] != cur[-1][2]:
        segs.append(cur)
        cur = [d]
    else:
        cur.append(d)
segs.append(cur)
print(f"total warp instr {tot_ex:.3e}, samples {tot_sm}")
for s in sorted(segs, key=lambda s: -sum(d[2] for d in s))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    ex = sum(d[2] for d in s)
    th = sum(d[3] for d in s) / max(ex, 1)
    sm = sum(d[4] for d in s)
    print(f"{s[0][0]-base:#07x}-{s[-1][0]-base:#07x} n={len(s):3d} execs/instr={s[0][2]:.3e} "
          f"instr={100*ex/tot_ex:5.1f}% thr={th:5.1f} stall={100*sm/max(tot_sm,1):5.1f}%  "
          f"{s[0][1][:40]} .. {s[-1][1][:30]}")
