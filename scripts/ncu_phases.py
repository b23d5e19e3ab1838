"""Stall samples and executed warp instructions aggregated over line ranges of a
kernel source (phases), from an ncu report with -lineinfo.

    python scripts/ncu_phases.py rep.ncu-rep file-substring name:a-b [name:a-b ...]
Lines in other files (inlined helpers) are reported per file.
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, sub = sys.argv[1], sys.argv[2]
ranges = []
for s in sys.argv[3:]:
    name, ab = s.split(":")
    a, b = ab.split("-")
    ranges.append((name, int(a), int(b)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur_file, hdr = None, None
acc = defaultdict(lambda: [0, 0])
num = lambda v: int(v) if v.strip().lstrip('-').isdigit() else 0  # noqa: E731
for r in csv.reader(io.StringIO(raw)):
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
    ln = int(r[0])
    name = None
    if sub in (cur_file or ""):
        for nm, a, b in ranges:
            if a <= ln <= b:
                name = nm
                break
        name = name or f"other:{ln}"
    else:
        name = "file:" + (cur_file or "?").split("/")[-1]
    acc[name][0] += num(r[4])
    acc[name][1] += num(r[7])
tot = sum(v[0] for v in acc.values()) or 1
toti = sum(v[1] for v in acc.values()) or 1
print(f"total stall samples {tot}, warp instructions {toti}")
for k, (s, i) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:40]:
    print(f"{k:24s} stall {100*s/tot:5.1f}%  inst {100*i/toti:5.1f}%")
