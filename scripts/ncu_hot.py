"""Per-instruction view of an ncu report (run here): executed counts and stall
samples per SASS line, plus the top stall sites with their dominant reasons.

    python scripts/ncu_hot.py rep.ncu-rep [min_count] [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
minc = int(sys.argv[2]) if len(sys.argv) > 2 else 1000000
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia = hdr.index("Instructions Executed")
ss = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
tot_s = sum(int(r[ss]) for r in data) or 1
print("total warp inst", sum(int(r[ia]) for r in data), "stall samples", tot_s)
lst = []
for k, r in enumerate(data):
    reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:2]
    lst.append((int(r[ss]), k, r[0][-5:], int(r[ia]), r[1].strip(), reasons))
print("--- top stall sites")
for s, k, a, c, txt, rs in sorted(lst, reverse=True)[:top]:
    print(f"{a} {c:>10d} {100*s/tot_s:5.1f}%  {txt[:60]:60s} {rs}")
