"""Top SASS instructions by warp-stall samples with their main stall reasons.

    python scripts/ncu_sass_stalls.py rep.ncu-rep [N] [--window A-B (hex addresses)]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if r and r[0] == "Address")
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
recs = []
for r in rows:
    if not r or not r[0].startswith("0x") or len(r) < len(hdr):
        continue
    num = lambda h: float(r[ix[h]] or 0)  # noqa: E731
    st = {h: num(h) for h in reasons}
    recs.append((int(r[0], 16), r[1].strip(), num("Warp Stall Sampling (All Samples)"), num("Instructions Executed"), st))
base = recs[0][0] if recs else 0
tot = sum(x[2] for x in recs) or 1
print(f"total samples {tot:.0f}")
for addr, src, s, ie, st in sorted(recs, key=lambda x: -x[2])[:N]:
    top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{addr - base:6x} {100 * s / tot:5.2f}% {src[:52]:52s} " + " ".join(f"{k[6:]}:{100 * v / max(s, 1):.0f}" for k, v in top))
agg = {}
for _, _, s, _, st in recs:
    for k, v in st.items():
        agg[k] = agg.get(k, 0) + v
ta = sum(agg.values()) or 1
print("by reason: " + ", ".join(f"{k[6:]} {100 * v / ta:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:12]))
if "--reason" in sys.argv:
    rs = "stall_" + sys.argv[sys.argv.index("--reason") + 1]
    print(f"top by {rs}:")
    for addr, src, s, ie, st in sorted(recs, key=lambda x: -x[4].get(rs, 0))[:40]:
        print(f"{addr - base:6x} {100 * st.get(rs, 0) / tot:5.2f}% {src[:60]}")
