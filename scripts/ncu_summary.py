"""Print the key metrics of an ncu report (run here, no GPU): python scripts/ncu_summary.py rep.ncu-rep"""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_fp64.sum", "smsp__inst_executed.sum", "launch__grid_size",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
        "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for val in rows[2:]:
    d = dict(zip(hdr, val)); u = dict(zip(hdr, units))
    for k in want:
        if k in d: print(f"{k:70s} {d[k]:>20s} {u.get(k,'')}")
    st = [(h[len('smsp__pcsamp_warps_issue_stalled_'):], float(v.replace(',', '') or 0)) for h, v in d.items()
          if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")]
    tot = sum(v for _, v in st) or 1
    print("stalls:", ", ".join(f"{h} {100*v/tot:.0f}%" for h, v in sorted(st, key=lambda x: -x[1])[:7]))
