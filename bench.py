#!/usr/bin/env python
"""bench.py — B200 benchmark of the wavelength-adaptive 27-point Helmholtz hot path
(arXiv 2108.08730; BASELINE.json `metric`).

One STEP is one pass of the whole north-star hot path (SURVEY.md §8(a) rows a1–a8) over the
N=1 workload, BASELINE configs[1] (config 2: 101³ linear-gradient model, 5 Hz, 4 point sources,
complex64):
    hz_build_weight_table (a1, host C++)  →  hz_assemble_coeffs (a2–a5)  →
    hz_point_sources (a8)  →  hz_solve: batched BiCGSTAB to ‖b−Ax‖/‖b‖ ≤ 1e-6 (a6, a7).

Reported (one JSON line, rank 0):
  value   apply Gpts/s of the whole step = Σ over the step's operator applies of
          (grid points × active RHS) ÷ step time  (the solve's vector kernels, reductions and host
          polls are inside that time; `apply_kernel_gpts_s` is the same count over the apply
          kernels' own CUDA-event time)
  solve_s_per_rhs, iterations, relres       BiCGSTAB part of the metric
  solver_alt  the same step solved with the other Krylov method (BiCGStab(2) beside the default
          BiCGSTAB; `--ell 2` swaps them): ms/step, s/RHS, iterations, relres (min(K, 3) timed
          steps after one warm-up, same timing rules; N = 1 only; `--no-alt` skips it)
  roofline  dominant kernel = the fused coefficient + 27-point apply (apply27_kernel): algorithmic
          bytes of every apply launch (v once + fields per active RHS) ÷ its CUDA-event
          time measured inside the timed steps, against MEASURED_PEAKS.json hbm_gbs
  e2e     same metric through the C ABI with HOST buffers: v (pinned) in, x0 in, x out — the copies
          are inside the timed region
  cpu_baseline  the CPU oracle (scipy CSR BiCGSTAB, complex128, 1 core) on a bounded sample
`--impl reference` times that oracle as the reference arm.

Multi-GPU (torchrun, one rank per GPU): the grid is split in z-slabs (halo planes and dot products
over NCCL inside libhz); total work is fixed → "scaling": "strong".  Timing: W warm-up steps, then
K steps each bracketed by barrier + synchronize, L2 flushed (256 MiB write) before every step, CUDA
events on the launching stream, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "adaptive 27-pt apply Gpts/s & HBM % of peak; BiCGSTAB s/RHS at 1/2/4/8 GPU"
UNIT = "Gpts/s"
TABLE_ARGS = (4.0, 40.0, 0.1, 1e-2)       # G range, ΔG, λ (BASELINE configs[0]; reading A11)


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hz", "reference"], default="hz")
    ap.add_argument("--config", type=int, default=2, help="BASELINE config index 1..5 (default 2 = configs[1])")
    ap.add_argument("--freq", type=float, default=None, help="frequency override (config 4: 5 or 10 Hz)")
    ap.add_argument("--nrhs", type=int, default=None, help="number of sources (default: the config's)")
    ap.add_argument("--dtype", choices=["c64", "c128"], default="c64")
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--max-iter", type=int, default=20000)
    ap.add_argument("--ell", type=int, choices=[1, 2], default=1, help="1: BiCGSTAB (default), 2: BiCGStab(2)")
    ap.add_argument("--replace-every", type=int, default=50,
                    help="residual replacement period")
    ap.add_argument("--stall-window", type=int, default=0,
                    help="iterations without a 10%% residual drop before a RHS is retired (0: max(20 x replace-every, 1000))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="skip the other Krylov method's timing (solver_alt)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=30, help="oracle BiCGSTAB iterations in the cpu_baseline sample")
    ap.add_argument("--ref-iters", type=int, default=4, help="oracle BiCGSTAB iterations per --impl reference step")
    ap.add_argument("--no-large", action="store_true",
                    help="skip the apply-only roofline measurement on the large config (N=1 only)")
    ap.add_argument("--large-config", type=int, default=4, help="config of the apply-only roofline measurement")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(args):
    cfg = synth.get_config(args.config)
    freq = args.freq if args.freq is not None else cfg.freqs[-1] if args.config == 4 else cfg.freq
    nodes = synth.source_nodes(cfg)
    if args.nrhs is not None:
        reps = int(np.ceil(args.nrhs / len(nodes)))
        nodes = np.concatenate([nodes] * reps)[: args.nrhs]
    return cfg, freq, nodes


def workload_name(cfg, freq, nrhs, dtype):
    return (f"config{cfg.index} {cfg.name} {cfg.nx}x{cfg.ny}x{cfg.nz} h={cfg.h:g}m f={freq:g}Hz "
            f"npml={cfg.npml} nrhs={nrhs} {dtype}: table+assemble+sources+BiCGSTAB(rtol)")


def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def read_traffic(workload_key):
    """dram bytes per apply launch from a committed ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        e = d.get(workload_key)
        return None if e is None else float(e["dram_bytes_per_launch"])
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"hz_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        # "under load": samples within the top half of the observed range
        load = [x for x in sm if sm and x >= 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(load) if load else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------------------------------------
def oracle_sample(cfg, freq, nodes, iters, v=None):
    """The CPU oracle as it stands (test infrastructure; bench.py's cpu_baseline / reference leg):
    explicit CSR impedance matrix + scipy-SpMV BiCGSTAB in complex128 on one core."""
    from threadpoolctl import threadpool_limits

    from oracle import operator as op
    from oracle import solvers, weights
    with threadpool_limits(1):
        t0 = time.perf_counter()
        tab = weights.build_adaptive_table(*TABLE_ARGS)
        t1 = time.perf_counter()
        if v is None:
            v = synth.velocity_model(cfg).astype(np.float32).astype(np.float64)
        P = op.Problem(v, cfg.h, freq, cfg.npml, tab)
        A = op.assemble(P)
        b = op.point_sources(P, nodes[:1])[0].ravel()
        t2 = time.perf_counter()
    return {"A": A, "b": b, "t_table": t1 - t0, "t_assemble": t2 - t1, "npts": A.shape[0]}


def oracle_iters(S, iters):
    from threadpoolctl import threadpool_limits

    from oracle import solvers
    with threadpool_limits(1):
        t0 = time.perf_counter()
        _, rel, it = solvers.bicgstab(S["A"], S["b"], rtol=1e-30, max_iter=iters)
        dt = time.perf_counter() - t0
    return dt, it


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg, freq, nodes = workload(args)
    S = oracle_sample(cfg, freq, nodes, args.ref_iters)
    for _ in range(args.warmup):
        oracle_iters(S, args.ref_iters)
    tot, its = 0.0, 0
    for _ in range(args.steps):
        dt, it = oracle_iters(S, args.ref_iters)
        tot += dt
        its += it
    value = S["npts"] * 2 * its / tot / 1e9
    sample = (f"oracle scipy-CSR BiCGSTAB (complex128, 1 thread), {args.ref_iters} iterations (2 SpMV each) of "
              f"RHS 0 per step on the full config-{cfg.index} grid; CSR assembly {S['t_assemble']:.1f}s and "
              f"oracle table {S['t_table']:.1f}s done once outside the timed steps")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
            "dtype": "c128", "data": "synthetic",
            "config": {"workload": workload_name(cfg, freq, len(nodes), args.dtype), "parallelism": "1 CPU core"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
def apply_large(args, hz, ctx, dev, stream, peak):
    """Apply-only roofline on a large BASELINE config (default config 4, 801x801x187, c64, 1 RHS): the
    hot kernel where HBM — not launch latency or the PML share of a small grid — bounds it.  CUDA events
    on the launching stream around each apply, L2 flushed between applies, median of `reps`."""
    import torch
    cfg = synth.get_config(args.large_config)
    freq = cfg.freqs[-1]
    v = synth.velocity_slab(cfg, 0, cfg.nz, device=dev if cfg.index == 5 else None)
    T = hz.hz_build_weight_table(*TABLE_ARGS)
    C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v).to(dev, torch.float32),
                              freq, T, npml=cfg.npml, dtype=hz.HZ_C64)
    del v
    u = C.alloc_field(1)
    u.real.uniform_(-1, 1)
    u.imag.uniform_(-1, 1)
    au = C.alloc_field(1)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def time_apply(Cx, reps=10):
        for _ in range(3):
            hz.hz_apply_impedance(Cx, u, au, stream=stream)
        out = []
        nonlocal_l0[0] = hz.hz_kernel_launch_count()
        for _ in range(reps):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hz.hz_apply_impedance(Cx, u, au, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            out.append(e0.elapsed_time(e1))
        return out

    nonlocal_l0 = [0]
    ts = time_apply(C)
    l0 = nonlocal_l0[0]
    launches = hz.hz_kernel_launch_count() - l0
    ms = statistics.median(ts)
    npts = cfg.nx * cfg.ny * cfg.nz
    # the same apply with non-adaptive weights (a one-row table: the same weights at every point, like the
    # paper's G4 / Gm comparison stencils) — the adaptive lookup costs no bytes and
    # little time ("no overhead")
    v = synth.velocity_slab(cfg, 0, cfg.nz, device=dev if cfg.index == 5 else None)
    Tm = hz.hz_table_import(12.0, 0.1, T.rows5()[80][None])   # the GA row at G = 12, everywhere
    Cm = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v).to(dev, torch.float32),
                               freq, Tm, npml=cfg.npml, dtype=hz.HZ_C64)
    del v
    ms_m = statistics.median(time_apply(Cm))
    del Cm
    # the GAm rule (27-node mean weights stored once, +20 B/pt read per apply, reading A19)
    v = synth.velocity_slab(cfg, 0, cfg.nz, device=dev if cfg.index == 5 else None)
    Cg = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v).to(dev, torch.float32),
                               freq, T, npml=cfg.npml, dtype=hz.HZ_C64, rule=hz.HZ_RULE_GAM)
    del v
    ms_g = statistics.median(time_apply(Cg))
    del Cg
    # GA in record mode (per-point weights stored once, +20 B/pt read per apply)
    v = synth.velocity_slab(cfg, 0, cfg.nz, device=dev if cfg.index == 5 else None)
    Cr = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v).to(dev, torch.float32),
                               freq, T, npml=cfg.npml, dtype=hz.HZ_C64, rule=hz.HZ_RULE_GA_RECORD)
    del v
    ms_r = statistics.median(time_apply(Cr))
    del Cr
    byts = npts * (4 + 16)            # w in, u in, Au out (complex64, 1 RHS): DESIGN.md §5
    achieved = byts / (ms * 1e-3) / 1e9
    return {"workload": f"config{cfg.index} {cfg.name} {cfg.nx}x{cfg.ny}x{cfg.nz} f={freq:g}Hz c64 nrhs=1, "
                        "hz_apply_impedance only", "gpts_s": npts / (ms * 1e-3) / 1e9, "ms": ms,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "algorithmic_bytes_per_launch": byts},
            "gpu_launches": launches, "l2": "flushed before every apply (256 MiB write)",
            "fixed_weights": {"table": "one row (GA weights at G = 12) at every point",
                              "gpts_s": npts / (ms_m * 1e-3) / 1e9, "ms": ms_m, "adaptive_over_fixed_time": ms / ms_m},
            "record_mode": {"gpts_s": npts / (ms_r * 1e-3) / 1e9, "ms": ms_r,
                            "hbm_frac": npts * (4 + 16 + 20) / (ms_r * 1e-3) / 1e9 / peak,
                            "note": "GA weights stored per point, read by the apply (+20 B/pt)"},
            "gam_rule": {"gpts_s": npts / (ms_g * 1e-3) / 1e9, "ms": ms_g,
                         "hbm_frac": npts * (4 + 16 + 20) / (ms_g * 1e-3) / 1e9 / peak,
                         "note": "27-node mean weights read per point (+20 B/pt)"}}


def run_hz(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws != args.gpus:
        args.gpus = ws
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2108_08730_b200 import hz, parallel

    ctx = parallel.make_context(local)      # NCCL communicator over all ranks (uid via torch.distributed)

    cfg, freq, nodes = workload(args)
    nrhs = len(nodes)
    z0, nzl = parallel.slab_partition(cfg.nz, ws, rank)
    rd = torch.float32 if args.dtype == "c64" else torch.float64
    dt_code = hz.HZ_C64 if args.dtype == "c64" else hz.HZ_C128
    v_np = synth.velocity_slab(cfg, z0, nzl, device=dev if cfg.index == 5 else None)
    v_dev = torch.from_numpy(v_np).to(dev, rd).contiguous()
    v_host = torch.from_numpy(v_np).to(rd).contiguous().pin_memory()
    fshape = (nrhs, nzl + 2, cfg.ny, cfg.nx)
    cdt = torch.complex64 if args.dtype == "c64" else torch.complex128
    b = torch.zeros(fshape, dtype=cdt, device=dev)
    x = torch.zeros(fshape, dtype=cdt, device=dev)
    x_host = torch.zeros(fshape, dtype=cdt).pin_memory()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if ws > 1:
            dist.barrier()

    def one_step(v_in, x_out, ell=None):
        T = hz.hz_build_weight_table(*TABLE_ARGS)                                  # a1
        C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_in, freq, T, npml=cfg.npml,
                                  z0=z0, nz_local=nzl, dtype=dt_code)               # a2–a5
        hz.hz_point_sources(C, nodes, b, stream=stream)                             # a8
        if x_out.is_cuda:
            x_out.zero_()
        else:
            x_out.zero_()
        st, rel, its, stt = hz.hz_solve(C, b, x_out, rtol=args.rtol, max_iter=args.max_iter,
                                        replace_every=args.replace_every, timing=True,
                                        ell=args.ell if ell is None else ell,
                                        stall_window=args.stall_window,
                                        stream=stream)                              # a6, a7
        return st, rel, its, stt

    def timed(v_in, x_out, k, ell=None):
        tot_ms, stats, last = 0.0, [], None
        l0 = hz.hz_kernel_launch_count()
        for _ in range(k):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            last = one_step(v_in, x_out, ell)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            tot_ms += e0.elapsed_time(e1)
            stats.append(last[3])
        return tot_ms, stats, last, hz.hz_kernel_launch_count() - l0

    # ---------------- device-resident arm ----------------
    for _ in range(args.warmup):
        one_step(v_dev, x)
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    tot_ms, stats, last, launches = timed(v_dev, x, args.steps)
    clk = clocks.stop()
    st, rel, its, _ = last

    pts = sum(s["apply_points_total"] for s in stats)
    abytes = sum(s["apply_bytes_total"] for s in stats)
    ams = sum(s["apply_ms_total"] for s in stats)
    alaunch = sum(s["apply_launches"] for s in stats)
    (tmax,) = parallel.rank_max([tot_ms], dev)              # the job takes as long as its slowest rank
    pts_all, bytes_all = parallel.rank_sum([pts, abytes], dev)
    (ams_max,) = parallel.rank_max([ams], dev)
    ms_per_step = tmax / args.steps
    value = pts_all / (tmax * 1e-3) / 1e9

    # ---------------- end-to-end arm (host buffers through the C ABI) ----------------
    e2e = None
    if not args.no_e2e:
        for _ in range(max(1, args.warmup)):
            one_step(v_host, x_host)
        tot_e, stats_e, _, _ = timed(v_host, x_host, args.steps)
        pts_e = sum(s["apply_points_total"] for s in stats_e)
        (tmax_e,) = parallel.rank_max([tot_e], dev)
        (pts_e_all,) = parallel.rank_sum([pts_e], dev)
        h2d = v_host.numel() * v_host.element_size() + x_host.numel() * x_host.element_size() + nodes.nbytes
        d2h = x_host.numel() * x_host.element_size()
        e2e = {"value": pts_e_all / (tmax_e * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(h2d) * ws,
               "d2h_bytes_per_step": int(d2h) * ws, "ms_per_step": tmax_e / args.steps}

    # ---------------- the other Krylov method on the same step (time to solution beside it) ----------------
    alt = None
    if not args.no_alt and ws == 1:
        ell_alt = 3 - args.ell
        one_step(v_dev, x, ell_alt)
        tot_a, _, last_a, _ = timed(v_dev, x, min(args.steps, 3), ell_alt)
        (tmax_a,) = parallel.rank_max([tot_a], dev)
        ka = min(args.steps, 3)
        alt = {"solver": "BiCGSTAB" if ell_alt == 1 else "BiCGStab(2)", "ms_per_step": tmax_a / ka,
               "solve_s_per_rhs": tmax_a / ka * 1e-3 / nrhs, "iterations": int(last_a[3]["iterations"]),
               "relres_max": float(np.max(last_a[1])), "status": int(last_a[0]), "steps": ka}

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    peak, peak_src = read_peak()
    achieved = abytes / (ams * 1e-3) / 1e9 if ams > 0 else None
    wkey = f"config{cfg.index}_{args.dtype}_nrhs{nrhs}_f{freq:g}"
    traffic = read_traffic(wkey)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if ws > 1 else "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic",
        "config": {"workload": workload_name(cfg, freq, nrhs, args.dtype), "grid": [cfg.nx, cfg.ny, cfg.nz],
                   "nrhs": nrhs, "rtol": args.rtol, "parallelism": f"z-slab x{ws}",
                   "solver": "BiCGSTAB" if args.ell == 1 else "BiCGStab(2)",
                   "l2": "flushed before every step (256 MiB write); step working set > L2"},
        "solve_s_per_rhs": ms_per_step * 1e-3 / nrhs,
        "solver_alt": alt,
        "iterations": int(stats[-1]["iterations"]),
        "relres_max": float(np.max(rel)),
        "status": int(st),
        "apply_kernel_gpts_s": pts_all / (ams_max * 1e-3) / 1e9 if ams_max > 0 else None,
        "apply_share_of_step": ams / tot_ms if tot_ms > 0 else None,
        "roofline": {"bound": "hbm", "kernel": "apply27_cp (RHS-fused coefficient build + 27-point apply + BiCGSTAB dot epilogues, a2-a6)",
                     "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / peak if achieved else None,
                     "traffic": (traffic if traffic is not None else None),
                     "algorithmic_bytes_per_launch": abytes / alaunch if alaunch else None,
                     "avg_launch_ms": ams / alaunch if alaunch else None},
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": e2e,
    }
    if ws == 1 and not args.no_large:
        line["apply_large"] = apply_large(args, hz, ctx, dev, stream, peak)
    if ws == 1 and not args.no_cpu_baseline:
        S = oracle_sample(cfg, freq, nodes, args.cpu_iters)
        dt, it = oracle_iters(S, args.cpu_iters)
        cv = S["npts"] * 2 * it / dt / 1e9
        line["cpu_baseline"] = {
            "value": cv, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": (f"oracle scipy-CSR BiCGSTAB (complex128, 1 of {os.cpu_count()} cores), {it} iterations "
                       f"(2 SpMV each) of RHS 0 on the full config-{cfg.index} grid in {dt:.1f}s; CSR assembly "
                       f"{S['t_assemble']:.1f}s excluded")}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_hz(args)


if __name__ == "__main__":
    sys.exit(main())
