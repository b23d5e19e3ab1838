"""Attribute ncu per-SASS stall samples to source lines (run here, no GPU).

    python scripts/ncu_lines.py <report.ncu-rep> <cubin-basename-in-lib> <kernel-substring> [top] [inst]

The cubin is extracted from paper_1310_5182_b200/liblagp_b200.so (cuobjdump
-xelf) and disassembled with nvdisasm -g (line info); the profile's SASS rows
are matched by offset from the kernel's first instruction.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, cub, kname = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
by_inst = len(sys.argv) > 5 and sys.argv[5] == "inst"  # rank by warp instructions executed
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1310_5182_b200", "liblagp_b200.so")], cwd=tmp,
               capture_output=True)
dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
# offset -> (file, line) within the requested kernel
lines, cur, inside = {}, None, False
for ln in dis.splitlines():
    if ln.startswith(".text.") or ln.startswith("//----"):
        inside = kname in ln
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and inside:
        lines[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Address")
data = rows[rows.index(hdr) + 1:]
iA, iW = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
iX = hdr.index("L1 Wavefronts Shared Excessive")
iI = hdr.index("Instructions Executed")
base = int(data[0][iA], 16)
agg = collections.Counter()
exc = collections.Counter()
for r in data:
    try:
        off = int(r[iA], 16) - base
    except ValueError:
        continue
    key = lines.get(off, ("?", 0))
    agg[key] += int(r[iI] or 0) if by_inst else int(r[iW] or 0)
    exc[key] += int(r[iX] or 0)
tot = sum(agg.values()) or 1
src = {}
for (f, l), v in agg.most_common(top):
    p = os.path.join(ROOT, "paper_1310_5182_b200", "csrc", f)
    if f not in src and os.path.exists(p):
        src[f] = open(p).read().splitlines()
    text = src[f][l - 1].strip()[:90] if f in src and 0 < l <= len(src[f]) else ""
    print(f"{100 * v / tot:5.1f}%  {f}:{l:<4} exc_wf={exc[(f, l)]:>11}  {text}")
