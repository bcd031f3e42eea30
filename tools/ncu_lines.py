"""Per-source-line profile of one kernel from an ncu report (--set full,
--import-source on, -lineinfo build): warp-stall samples, executed warp
instructions and the top stall reasons per CUDA line, hottest first.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
lines, cur, fname, hdr = {}, None, "", None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0]:  # a CUDA line summary row
        cur = (fname, int(r[0]), r[1].strip()[:70])
        d = dict(zip(hdr[2:], r[2:]))
        def num(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        stalls = {k[6:]: num(k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k}
        lines[cur] = (num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"), stalls)
tot = sum(v[0] for v in lines.values()) or 1
tinst = sum(v[1] for v in lines.values()) or 1
print(f"total samples {tot:.0f}, warp instructions {tinst:.0f}")
for k, (s, ins, st) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
    tops = ", ".join(f"{a} {b / max(s, 1):.0%}" for a, b in sorted(st.items(), key=lambda x: -x[1])[:3] if b)
    print(f"{s / tot:6.1%} {ins / tinst:6.1%}  {k[0]}:{k[1]:<5} {k[2]:<70} | {tops}")
