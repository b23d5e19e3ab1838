"""Write profiles/ncu_traffic.json (dram bytes per launch of each bench kernel)
from the round's ncu --set full reports (run here after gpurun):

    python scripts/traffic_json.py rNN gpurun_out/prof_alc_incremental_rNN.ncu-rep:incremental \
        gpurun_out/prof_alc_explicit_dmma_rNN.ncu-rep:explicit gpurun_out/prof_nn_pool_rNN.ncu-rep:nn
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
    rep, key = spec.rsplit(":", 1)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, val = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, val))
    u = dict(zip(hdr, units))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tscale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}
    b = sum(float(d[k].replace(",", "")) * scale[u[k]] for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    t = float(d["gpu__time_duration.sum"].replace(",", "")) * tscale[u["gpu__time_duration.sum"]]
    out[key] = {"dram_bytes_per_launch": b, "kernel": d["Kernel Name"][:80], "ncu_duration_ms": t,
                "source": f"{os.path.basename(rep)} (ncu --set full, M=10000, round {rnd})"}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
