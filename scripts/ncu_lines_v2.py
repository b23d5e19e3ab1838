"""Stall samples and executed instructions per CUDA source line (cuda,sass view).

    python scripts/ncu_lines_v2.py rep.ncu-rep [file-substring]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
sub = sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
cur_file, hdr = None, None
acc = defaultdict(lambda: [0, 0, ""])
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    num = lambda v: int(v) if v.strip().lstrip('-').isdigit() else 0  # noqa: E731
    ss = num(r[4])
    ie = num(r[7])
    key = (cur_file, int(r[0]))
    acc[key][0] += ss
    acc[key][1] += ie
    if r[1]:
        acc[key][2] = r[1]
tot = sum(v[0] for v in acc.values()) or 1
toti = sum(v[1] for v in acc.values()) or 1
print(f"total stall samples {tot}, warp instructions {toti}")
for (f, ln), (s, i, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:60]:
    if sub and sub not in f:
        continue
    print(f"{f.split('/')[-1]:28s}:{ln:<5d} stall {100*s/tot:5.1f}%  inst {100*i/toti:5.1f}%  {src.strip()[:80]}")
