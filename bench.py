#!/usr/bin/env python
"""Benchmark of the greedy ALC local-design hot path (arXiv 1310.5182) on B200.

Workload (BASELINE.json configs[1], the metric's single-GPU configuration):
C2 — 8-d borehole, N = 100,000 LHS design, M = 10,000 LHS predictive locations
per GPU, n0 = 6, n = 50, N' = 1000, d = q10 rule, g = 1e-4.
A "step" is one laGP_alc_batch call over the rank's M locations (NN pool, ALC
greedy loop, partitioned-inverse updates, prediction — every §8(a) row), and
with N > 1 GPUs the all-gather of every rank's results (NCCL).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

Weak scaling: every rank processes its own M = 10,000 rows of a global
predictive set of N·10,000 LHS rows; X and Z are replicated. Rank 0 prints one
JSON line. The oracle (oracle/, CPU) is executed only in the cpu_baseline leg
and by --impl reference.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "C2"
METRIC = "local-GP predictions/sec"
UNIT = "predictions/s"


# The paper's own timings with their hardware: context, not the target.
PAPER_CONTEXT = {
    "note": "PAPER.md timings (FP64, 2012 hardware); whole local-approximation runs, possibly incl. local MLE "
            "(P:845-849); context only",
    "lgbb_n50_Np1000": {"locations": 644436, "wall_s": 21 * 60, "locations_per_s": 511,
                        "hardware": "4 nodes x (16 Sandy Bridge cores + 2 Tesla M2090), GPUs take 80% of ALC",
                        "cite": "P:1006-1015"},
    "borehole_table1_1024000": {"N=M": 1024000, "n": 60, "Nprime": 5772,
                                "cpu": {"wall_s": 2789.81, "locations_per_s": 367,
                                        "hardware": "96 nodes x 16 Sandy Bridge cores (1536 cores)"},
                                "gpu": {"wall_s": 13694.48, "locations_per_s": 75,
                                        "hardware": "5 nodes x (2 Tesla M2090 + 16 cores)"},
                                "cite": "P:1062-1127 (Table 1)"},
    "fig6_speedup_vs_1_core": {"16_cores_plus_2_gpus": [33, 50, 100], "nNp": [[50, 1000], [50, 2000], [128, 2000]],
                               "cite": "P:933-936"},
}


def alc_evals_per_location(n0, n, Nprime):
    """ALC candidate evaluations per location: sum_{j=n0}^{n-1} (N' - j)."""
    return sum(Nprime - j for j in range(n0, n))


def alc_paper_flops_per_location(n0, n, Nprime):
    """Paper-count ALC work: (N'-j)(2j^2 + 4j) flop per step j."""
    return sum((Nprime - j) * (2 * j * j + 4 * j) for j in range(n0, n))


def fp64_peak_tflops():
    """ALU roofline denominator: 148 SMs x 64 FP64 FMA/clk x 2 flop
    x 1.965 GHz (clocks.max.sm) = 37.2 TFLOP/s; the measured DFMA ceiling of
    scripts/fp64_peak.cu is recorded beside it when profiles/ has it."""
    nominal = 148 * 64 * 2 * 1.965e9 / 1e12
    meas = None
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(p):
        try:
            meas = json.load(open(p)).get("dfma_tflops")
        except Exception:
            meas = None
    return nominal, meas


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows if len(r) >= 9 for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


WORKLOADS = {
    "C2": "C2: 8-d borehole, N=100000 LHS design, M=10000 LHS locations per GPU, n0=6 n=50 N'=1000",
    "C3": "C3: 3-d LGBB-shaped grid, N=37908, M=500000 dense grid over all GPUs, n0=6 n=50 N'=1000",
    "C4": "C4: 8-d borehole, N=M=1000000 LHS over all GPUs, n0=6 n=50 N'=1000 (the north_star target shape)",
}


def make_inputs(world, workload=WORKLOAD):
    from lagp_data import borehole, lhs, make_config

    cfg = make_config(workload)
    if workload == "C2" and world > 1:  # weak scaling: a global LHS of world x M rows
        cfg["XX"] = lhs(cfg["XX"].shape[0] * world, cfg["X"].shape[1], 202)
    cfg["borehole"] = borehole
    return cfg


def rank_rows(workload, M_total, rank, world):
    """C2: weak scaling, 10,000 locations per rank; C3/C4: strong scaling, the config's
    fixed predictive set split into contiguous shards."""
    if workload == "C2":
        return rank * 10_000, 10_000, 10_000 * world
    import paper_1310_5182_b200 as lagp

    lo, hi, _ = lagp.shard_bounds(M_total, rank, world)
    return lo, hi - lo, M_total


def cpu_model():
    """The host CPU model (SURVEY §8d asks for it beside the oracle timing)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(cfg, budget_s=15.0, lo=0):
    """The oracle as it stands, on all host cores, on a bounded sample of the
    workload's locations (consecutive rows of the rank-0 shard)."""
    import oracle

    cores = os.cpu_count() or 1
    args = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    t0 = time.perf_counter()
    oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][lo:lo + 1], *args, threads=1)
    t1 = time.perf_counter() - t0
    S = int(max(cores, min(cfg["XX"].shape[0] - lo, budget_s * cores / max(t1, 1e-4))))
    S = min(S, cfg["XX"].shape[0] - lo)
    t0 = time.perf_counter()
    o = oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][lo:lo + S], *args, threads=cores)
    el = time.perf_counter() - t0
    return o, S, el, o["threads"]


def run_reference(args):
    """--impl reference: the oracle (the reference arm of this tier) timed on
    the host cores on the same config, metric and unit; bounded samples."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = make_inputs(1, args.workload)
    import oracle

    cores = os.cpu_count() or 1
    a = (cfg["d"], cfg["g"], cfg["n0"], cfg["n"], cfg["Nprime"])
    t0 = time.perf_counter()
    oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][:1], *a, threads=1)
    t1 = time.perf_counter() - t0
    per_step_budget = max(min(2.0, args.ref_budget), args.ref_budget / max(1, args.steps + args.warmup))
    S = int(min(cfg["XX"].shape[0], max(cores, per_step_budget * cores / max(t1, 1e-4))))
    times = []
    for it in range(args.warmup + args.steps):
        lo = (it * S) % max(1, cfg["XX"].shape[0] - S + 1)
        t0 = time.perf_counter()
        o = oracle.alc_batch(cfg["X"], cfg["Z"], cfg["XX"][lo:lo + S], *a, threads=cores)
        el = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(el)
    ms = 1000.0 * sum(times) / len(times)
    value = S / (ms / 1000.0)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak" if args.workload == "C2" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload] + ", d=q10 g=1e-4", "sample_locations_per_step": S},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": o["threads"], "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"{S} consecutive {args.workload} locations per step (of "
                                   f"{cfg['XX'].shape[0]}), OpenMP over locations"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def traffic_for(workload, form, launches):
    """DRAM bytes (read + write) per local-design launch of this workload and
    form, from the ncu --set full capture of the same workload
    (profiles/ncu_traffic.json: {workload: {form: {"bytes": B, "launches": L,
    "profile": file}}}); None when no capture of this workload exists."""
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        tr = json.load(open(tp)).get(workload, {}).get(form)
    except Exception:
        return None
    if not tr:
        return None
    return {"bytes_per_launch": tr["bytes"] / max(1, tr.get("launches", 1)), "profile": tr.get("profile"),
            "algorithmic_bytes_note": tr.get("note")}


# FP32 (non-tensor) peak of one B200: 148 SM x 128 FP32 FMA/clk x 2 flop x 1.965 GHz
FP32_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12


def nn_roofline(head, m_rank, N, p):
    """NN stage as work actually done (lagp_timing counters of the step): prefilter and
    threshold-sample (row, query) pairs evaluated per second, each 2(p+1) FP32 flop (the
    dot-form prefilter: p FMA + the norm FMA; the sample's difference form is 3p), against
    the FP32 FMA peak; the pruned fraction of the M x N exhaustive pairs the cell lists
    skipped; exact FP64 keys computed (filter survivors)."""
    w = head.get("nn_work") or {}
    fp, sp, ek = w.get("nn_filter_pairs", 0), w.get("nn_sample_pairs", 0), w.get("nn_exact_keys", 0)
    t = head["nn_ms"] / 1000.0
    flops = fp * 2 * (p + 1) + sp * 3 * p
    return {"evaluated_pairs_per_sec": (fp + sp) / t, "filter_pairs": fp, "sample_pairs": sp, "exact_keys": ek,
            "exhaustive_pairs": m_rank * N, "pruned_fraction": 1.0 - fp / float(m_rank * N),
            "exact_keys_per_location": ek / float(m_rank), "achieved_tflops": flops / t / 1e12,
            "peak": FP32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": flops / t / 1e12 / FP32_PEAK_TFLOPS,
            "peak_basis": "148 SM x 128 FP32 FMA/clk x 2 x 1.965 GHz (FP32 FFMA2 pipe; no FP32 entry in MEASURED_PEAKS.json)",
            "note": "whole NN stage time (cell prep, sample, filter, exact keys, selection) over the FP32 flops of "
                    "the evaluated pairs; logical pairs the cells prune are not counted as work"}


def form_work(form, n0, n, Np, p):
    """Algorithmic FP64 work per location of a local-design kernel.

    explicit forms: the paper count (N'-j)(2j^2 + 4j) per step j;
    incremental form: per candidate update at design size j, 2j (w_*^T w_c) +
    3p (distance) + 8 (new entry, s and cov downdates, Delta) flop, over the
    N'-j-1 unchosen candidates, for j = 0..n-1 (the NN appends included); the
    exp per update is not counted (as in §8d)."""
    if form == "incremental":
        return float(sum((Np - j - 1) * (2 * j + 3 * p + 8) for j in range(0, n)))
    return float(alc_paper_flops_per_location(n0, n, Np))


def self_launch(args) -> int:
    """--gpus N > 1 outside torchrun: launch N ranks (one per GPU) the way the
    driver does (torch.distributed.run, 127.0.0.1) and pass their output through."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.stderr.write(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible\n")
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--form", default="auto", choices=["auto", "explicit", "incremental", "explicit_dfma"],
                    help="formulation of the headline number (auto = laGP_alc_batch's choice)")
    ap.add_argument("--no-north-star", action="store_true",
                    help="skip the north_star C4 line (N = M = 10^6 split over the ranks: strong scaling)")
    ap.add_argument("--compare", default="explicit",
                    help="comma list of other forms timed the same way and reported under 'forms' ('' = none)")
    ap.add_argument("--workload", default=WORKLOAD, choices=sorted(WORKLOADS),
                    help="C2 (default, BASELINE configs[1], weak scaling) or the full C3 / C4 shapes (strong)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-two-stage", action="store_true",
                    help="skip the Fig 1 two-stage (design, local MLE, design, MLE, predict) timing")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--ref-budget", type=float, default=90.0,
                    help="--impl reference: host seconds for the whole warmup + timed run (bounded samples)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        return self_launch(args)
    if world_env is not None and int(world_env) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}\n")
        return 2

    import torch
    import torch.distributed as dist

    import paper_1310_5182_b200 as lagp

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    if args.workload != "C2":  # the big shapes: headline form only
        args.compare, args.no_two_stage = "", True
    cfg = make_inputs(world, args.workload)
    X = torch.from_numpy(cfg["X"]).to(dev)
    Z = torch.from_numpy(cfg["Z"]).to(dev)
    lo, M_rank, M_all = rank_rows(args.workload, cfg["XX"].shape[0], rank, world)
    XXr_np = np.ascontiguousarray(cfg["XX"][lo:lo + M_rank])
    XX = torch.from_numpy(XXr_np).to(dev)
    n0, n, Np, d, g = cfg["n0"], cfg["n"], cfg["Nprime"], cfg["d"], cfg["g"]
    p = cfg["X"].shape[1]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)
    nominal, meas = fp64_peak_tflops()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def time_form(form, clocks=None, Xd=None, Zd=None, XXd=None, c=None, m_rank=None, m_all=None, steps=None,
                  workload=None):
        """Warm-up, then `steps` timed steps (L2 flushed before each, barrier + sync on
        both sides, CUDA events on the launching stream, max over ranks)."""
        Xd = X if Xd is None else Xd
        Zd = Z if Zd is None else Zd
        XXd = XX if XXd is None else XXd
        c = cfg if c is None else c
        m_rank = M_rank if m_rank is None else m_rank
        m_all = M_all if m_all is None else m_all
        steps = args.steps if steps is None else steps
        workload = args.workload if workload is None else workload
        a = (c["d"], c["g"], c["n0"], c["n"], c["Nprime"])
        for _ in range(args.warmup):
            lagp.alc_batch(Xd, Zd, XXd, *a, form=form)
        torch.cuda.synchronize()
        if clocks:
            clocks.start()
        total = alc = nn = 0.0
        launches = 0
        res = None
        for _ in range(steps):
            flush.fill_(1.0)  # L2 flush between timed steps (untimed)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = lagp.alc_batch(Xd, Zd, XXd, *a, form=form, timing=True)
            if world > 1:  # the one collective, results all-gathered in input order
                lagp.gather_shards(res, m_all)
            e1.record(stream)
            barrier()
            total += e0.elapsed_time(e1)
            alc += res["timing"]["alc_ms"]
            nn += res["timing"]["nn_ms"]
            launches += res["timing"]["launches"]
        clk = clocks.stop() if clocks else None
        t = torch.tensor([total, alc, nn], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t[0]) / steps
        alc_step_ms = float(t[1]) / steps
        ran = res["timing"]["alc_form"]  # the resolved formulation (auto -> incremental / explicit)
        pp, Npp, nn_, n0_ = c["X"].shape[1], c["Nprime"], c["n"], c["n0"]
        design_launches = -(-m_rank // 65536)  # one local-design launch per 65,536-location chunk
        achieved = m_rank * form_work(ran, n0_, nn_, Npp, pp) / (alc_step_ms / 1000.0) / 1e12
        kern = {"incremental": ("alc_incremental_v2_kernel" if Npp <= 1024 and pp in (1, 2, 3, 4, 8)
                                else "alc_incremental_kernel"),
                "explicit": "alc_explicit_dmma_kernel" if nn_ <= 64 else "alc_explicit_kernel",
                "explicit_dfma": "alc_explicit_kernel"}[ran]
        roof = {"bound": "alu", "kernel": kern, "alc_form": ran,
                "achieved": achieved, "peak": nominal, "unit": "TFLOP/s", "frac": achieved / nominal,
                "traffic": (traffic_for(workload, ran, design_launches) or {}).get("bytes_per_launch"),
                "traffic_unit": "bytes per launch (dram read + write, ncu --set full of the same workload)",
                "traffic_source": (traffic_for(workload, ran, design_launches) or {}).get("profile"),
                "work": ("incremental: (N'-j-1)(2j+3p+8) flop per location-step j=0..n-1, FP64, exp not counted"
                         if ran == "incremental" else
                         "paper count (N'-j)(2j^2+4j) flop per location-step (SURVEY §8d), FP64"),
                "peak_basis": "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (no FP64 entry in MEASURED_PEAKS.json)",
                "peak_measured_dfma": meas,
                "kernel_ms_per_step": alc_step_ms, "kernel_launches_per_step": design_launches,
                "kernel_ms_per_launch": alc_step_ms / design_launches}
        if ran == "incremental":
            # secondary view: the per-candidate state w_c streamed every step (sum over steps
            # of (N'-j-1) j entries x 8 B per location) against the shared-memory bandwidth
            # (128 B/clk/SM x 148 x 1.965 GHz); part of it is served by registers / TMEM
            sb = m_rank * sum((Npp - jj - 1) * jj * 8.0 for jj in range(nn_)) / (alc_step_ms / 1000.0) / 1e9
            smem_peak = 128 * 148 * 1.965
            roof["state_stream"] = {"achieved_GBps": sb, "smem_peak_GBps": smem_peak, "frac": sb / smem_peak,
                                    "bytes": "sum_j (N'-j-1) j 8 B per location (w_c entries read per step)"}
        tmg = res["timing"]  # NN work counters of the last step (identical every step)
        return dict(ms_step=ms_step, value=m_all / (ms_step / 1000.0), alc_ms=alc_step_ms,
                    nn_ms=float(t[2]) / steps, launches=launches, res=res, clk=clk, roofline=roof,
                    form=ran, nn_work={k: int(tmg[k]) for k in ("nn_filter_pairs", "nn_sample_pairs", "nn_exact_keys")})

    head = time_form(args.form, ClockSampler(local))
    others = {}
    for f in [f for f in args.compare.split(",") if f and f != args.form]:
        o = time_form(f)
        others[f] = {"ms_per_step": o["ms_step"], "value": o["value"], "unit": UNIT,
                     "phase_ms_per_step": {"nn": o["nn_ms"], "local_design": o["alc_ms"]},
                     "roofline": o["roofline"]}
    ms_step, value, res = head["ms_step"], head["value"], head["res"]
    evals = alc_evals_per_location(n0, n, Np)

    # ---- row f2: the paper's two-stage scheme (Fig 1 steps 1-5) on the same
    # locations: theta_x = d, {design, local MLE} twice, predict. Reported beside the
    # headline (which is Fig 1 steps 2 + 5 at fixed d, the north_star path).
    two = None
    if not args.no_two_stage:
        lo_t, hi_t = 1e-3, 10.0
        for _ in range(max(1, args.warmup // 2)):
            lagp.local_fit(X, Z, XX, d, lo_t, hi_t, g, n0, n, Np, stages=2)
        tt = {"total": 0.0, "nn": 0.0, "designs": 0.0, "mle_predict": 0.0}
        r2 = None
        for _ in range(max(1, min(args.steps, 3))):
            flush.fill_(1.0)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            r2 = lagp.local_fit(X, Z, XX, d, lo_t, hi_t, g, n0, n, Np, stages=2, timing=True)
            e1.record(stream)
            barrier()
            tt["total"] += e0.elapsed_time(e1)
            tt["nn"] += r2["timing"]["nn_ms"]
            tt["designs"] += r2["timing"]["alc_ms"]
            tt["mle_predict"] += r2["timing"]["predict_ms"]
        ns = max(1, min(args.steps, 3))
        t2 = torch.tensor([tt["total"] / ns], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        two = {"ms_per_step": float(t2[0]), "value": M_all / (float(t2[0]) / 1000.0), "unit": UNIT,
               "phase_ms_per_step": {k: v / ns for k, v in tt.items() if k != "total"},
               "config": {"stages": 2, "theta0": d, "theta_bounds": [lo_t, hi_t]}, "res": r2}

    # ---- e2e: the host-buffer public entry point, copies inside the timed region
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    Xh, Zh, XXh = pin(cfg["X"]), pin(cfg["Z"]), pin(XXr_np)
    hout = dict(idx=torch.empty((M_rank, n), dtype=torch.int32).pin_memory().numpy(),
                mean=torch.empty(M_rank, dtype=torch.float64).pin_memory().numpy(),
                s2=torch.empty(M_rank, dtype=torch.float64).pin_memory().numpy(),
                var=torch.empty(M_rank, dtype=torch.float64).pin_memory().numpy(),
                flags=torch.empty(M_rank, dtype=torch.int32).pin_memory().numpy().view(np.uint32))
    e2e_ms = 0.0
    e2e_steps = max(1, min(args.steps, 3))
    for _ in range(args.warmup):  # untimed warm-up of the host path, as for every timed form
        lagp.alc_batch_host(Xh, Zh, XXh, d, g, n0, n, Np, form=args.form, out=hout)
    for _ in range(e2e_steps):
        flush.fill_(1.0)
        barrier()
        t0 = time.perf_counter()
        lagp.alc_batch_host(Xh, Zh, XXh, d, g, n0, n, Np, form=args.form, out=hout)
        barrier()
        e2e_ms += (time.perf_counter() - t0) * 1000.0
    te = torch.tensor([e2e_ms / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = M_all / (float(te[0]) / 1000.0)
    h2d = (Xh.nbytes + Zh.nbytes) * world + M_all * XXh.shape[1] * 8  # every rank: X, Z and its XX rows
    d2h = M_all * (n * 4 + 3 * 8 + 4)

    # ---- north_star target shape: C4 (8-d borehole, N = M = 10^6, n = 50, N' = 1000), the
    # whole predictive set split over the ranks (strong scaling; the driver's 1/2/4/8-GPU
    # runs give the 1 -> 8 curve). Same timing rules; fewer steps (1.5 s per step on one GPU).
    north = None
    if not args.no_north_star and args.workload != "C4":
        c4 = make_inputs(1, "C4")
        lo4, m4, mall4 = rank_rows("C4", c4["XX"].shape[0], rank, world)
        X4, Z4 = torch.from_numpy(c4["X"]).to(dev), torch.from_numpy(c4["Z"]).to(dev)
        XX4 = torch.from_numpy(np.ascontiguousarray(c4["XX"][lo4:lo4 + m4])).to(dev)
        h4 = time_form("auto", ClockSampler(local), X4, Z4, XX4, c4, m4, mall4, steps=min(args.steps, 3),
                       workload="C4")
        north = {"workload": WORKLOADS["C4"] + f", d=q10={c4['d']:.4f} g=1e-4", "scaling": "strong",
                 "metric": METRIC, "value": h4["value"], "unit": UNIT, "ms_per_step": h4["ms_step"],
                 "steps": min(args.steps, 3), "warmup": args.warmup,
                 "phase_ms_per_step": {"nn": h4["nn_ms"], "local_design": h4["alc_ms"]},
                 "roofline": h4["roofline"], "nn_roofline": nn_roofline(h4, m4, c4["X"].shape[0], c4["X"].shape[1]),
                 "clocks": h4["clk"], "gpu_launches": h4["launches"],
                 "locations_per_rank": m4, "status": int(h4["res"]["status"])}
        if world == 1 and not args.no_cpu_baseline:
            import oracle

            S4 = 16
            sel4 = np.sort(np.random.default_rng(44).choice(m4, S4, replace=False))
            o4 = oracle.alc_batch(c4["X"], c4["Z"], c4["XX"][lo4 + sel4], c4["d"], c4["g"], c4["n0"], c4["n"],
                                  c4["Nprime"])
            gi4 = h4["res"]["idx"].cpu().numpy()[sel4]
            north["sample_parity"] = {"locations": S4,
                                      "identical_index_sequences": int((gi4 == o4["idx"]).all(1).sum())}
        del X4, Z4, XX4, h4

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.workload == "C2" else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOADS[args.workload] + f", d=q10={d:.4f} g=1e-4",
                   "alc_form": head["form"], "l2": "flushed (256 MiB write) before every timed step",
                   "parallelism": f"dp{world} (XX sharded, X/Z replicated)"},
        "alc_evals_per_sec": M_all * evals / (ms_step / 1000.0),
        # the same numerator over the local-design kernel time (max over ranks),
        # the NN stage and the whole step against the FP64 ALU peak (paper counts)
        "alc_evals_per_sec_kernel": M_all * evals / (head["alc_ms"] / 1000.0),
        "nn_roofline": nn_roofline(head, M_rank, cfg["X"].shape[0], p),
        "end_to_end_paper_count": {
            "frac_fp64_peak": (M_all * (alc_paper_flops_per_location(n0, n, Np) + cfg["X"].shape[0] * 3 * p)
                               / (ms_step / 1000.0) / 1e12 / (world * nominal)),
            "note": "(ALC paper count (N'-j)(2j^2+4j) + NN 3pN) per location / step time / (R x FP64 peak); "
                    "above 1 with the incremental form, which does ~20x less arithmetic than the paper count"},
        "phase_ms_per_step": {"nn": head["nn_ms"], "local_design": head["alc_ms"]},
        "roofline": head["roofline"],
        "forms": others,
        "two_stage": ({k: v for k, v in two.items() if k != "res"} if two else None),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": head["launches"],
        "clocks": head["clk"],
        "status": int(res["status"]),
        "north_star_c4": north,
        "paper_context": PAPER_CONTEXT,
    }
    if world == 1 and not args.no_cpu_baseline:
        o, S, el, used = cpu_baseline(cfg, budget_s=args.cpu_budget, lo=0)
        line["cpu_baseline"] = {"value": S / el, "unit": UNIT, "cores": used, "kind": "oracle", "cpu": cpu_model(),
                                "sample": f"first {S} of the {M_rank} {args.workload} locations of rank 0, "
                                          "OpenMP over locations"}
        gi = res["idx"][:S].cpu().numpy()
        line["sample_parity"] = {"locations": S, "identical_index_sequences": int((gi == o["idx"]).all(1).sum())}
        if two:
            import oracle

            S2 = min(64, M_rank)
            o2 = oracle.local_fit(cfg["X"], cfg["Z"], XXr_np[:S2], d, 1e-3, 10.0, g, n0, n, Np, stages=2)
            g2 = {"idx": two["res"]["idx"][:S2].cpu().numpy(), "theta": two["res"]["theta"][:, :S2].cpu().numpy()}
            same2 = (g2["idx"] == o2["idx"]).all(1)
            th_rel = np.abs(g2["theta"] - o2["theta"]) / o2["theta"]
            line["two_stage"]["sample_parity"] = {
                "locations": S2, "identical_index_sequences": int(same2.sum()),
                "max_rel_theta_diff": float(th_rel[:, same2].max()) if same2.any() else None}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
