"""Write profiles/ncu_traffic.json — DRAM bytes (read + write) per launch of each
bench kernel at each workload — from the round's ncu --set full reports (each a
single-launch capture, -c 1), for bench.py's roofline.traffic:

    python scripts/traffic_json.py rNN WORKLOAD:KEY:report.ncu-rep [...]
    -> {WORKLOAD: {KEY: {"bytes": B, "launches": 1, "profile": ..., "kernel": ..., "ncu_duration_ms": t}}}
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1]
out = {}
for spec in sys.argv[2:]:
    workload, key, rep = spec.split(":", 2)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        print(f"skip {spec}: no data")
        continue
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, val))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
              "s": 1e3}
    b = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = float(d["gpu__time_duration.sum"].replace(",", "")) * tscale[u["gpu__time_duration.sum"]]
    out.setdefault(workload, {})[key] = {"bytes": b, "launches": 1, "kernel": d["Kernel Name"][:80],
                                         "ncu_duration_ms": t,
                                         "profile": f"{os.path.basename(rep)} (ncu --set full, round {rnd})"}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
