#!/usr/bin/env python
"""bench.py — B200 benchmark of the wavelength-adaptive 27-point Helmholtz hot path
(arXiv 2108.08730; BASELINE.json `metric`: adaptive 27-pt apply Gpts/s & HBM % of peak; BiCGSTAB
s/RHS at 1/2/4/8 GPU).

Headline workload: BASELINE configs[3] = config 4, the 801×801×187 thrust-belt model (the overthrust
stand-in, Table 1), complex64, f = 10 Hz, z-slab split over the N GPUs (total work
fixed → "scaling": "strong").  One timed STEP = one hz_apply_impedance of a batch of `--nrhs` (8)
fields: the fused per-point coefficient build (G = v/(f h), table lookup + interpolation, PML
stretching; §8(a) a2–a5) and the matrix-free 27-point apply (a6), halo planes over NCCL for N > 1.
  value      Gpts/s = grid points × nrhs ÷ the step's device time (max over ranks)
  roofline   that launch: algorithmic bytes (4 + 16·nrhs per point) ÷ its CUDA-event
             time, against MEASURED_PEAKS.json hbm_gbs; `traffic` = ncu DRAM bytes per launch from
             profiles/ncu_traffic.json (the committed capture of this workload)
  solve      the rest of the hot path on the same workload: weight table (a1) + assemble + point
             sources (a8) + batched solve (a7) of `--solve-nrhs` (2) sources to ‖b−Ax‖/‖b‖ ≤ 1e-6,
             BiCGSTAB (the north star's method) and BiCGStab(2) beside it, each bounded by
             --solve-max-iter; s/RHS, iterations, relres and status reported as they come out
  e2e        the same metric through the C ABI with HOST (pinned) u and Au buffers: the H2D copy of
             the batch and the D2H copy of the result are inside the timed region
  cpu_baseline / --impl reference   the CPU oracle (scipy CSR SpMV, complex128, 1 core) on a
             z-chunk of the same model
  apply_nrhs1, fixed_weights, record_mode, gam_rule, config2_solve   extra measurements (N = 1)
`--weak`: the config-5 weak-scaling series 1201×1201×(50N+1): value = apply
Gpts/s of 1 RHS per GPU's slab, plus the time per BiCGSTAB iteration; "scaling": "weak".

Timing: W warm-up steps, then K steps each bracketed by barrier + synchronize, L2 flushed (256 MiB
write) before every step (the step's working set, ≥ 16 GB, exceeds L2 anyway), CUDA events on the
launching stream, max over ranks; nvidia-smi clocks sampled during the timed steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
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
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hz", "reference"], default="hz")
    ap.add_argument("--config", type=int, default=4, help="BASELINE config index 1..5 (default 4 = configs[3])")
    ap.add_argument("--freq", type=float, default=None, help="frequency (default: the config's highest)")
    ap.add_argument("--nrhs", type=int, default=8, help="fields per apply batch (headline)")
    ap.add_argument("--weak", action="store_true", help="config-5 weak-scaling slab series 1201x1201x(50N+1)")
    ap.add_argument("--solve-nrhs", type=int, default=2, help="sources in the timed solve leg")
    ap.add_argument("--solve-max-iter", type=int, default=12000, help="iteration bound of each solve leg")
    ap.add_argument("--rtol", type=float, default=1e-6)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra measurements (N = 1)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-planes", type=int, default=4, help="z-planes of the oracle's CSR sample")
    ap.add_argument("--cpu-spmv", type=int, default=10, help="oracle SpMVs timed in the cpu_baseline sample")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload(args, ws):
    """(cfg, freq): the headline model, or the weak-scaling slab series of config 5."""
    if args.weak:
        cfg = synth.get_config(5, nz=50 * ws + 1)
        return cfg, cfg.freq
    cfg = synth.get_config(args.config)
    freq = args.freq if args.freq is not None else cfg.freqs[-1]
    return cfg, freq


def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def read_traffic(key):
    """ncu DRAM bytes per launch for a workload key from the committed capture (profiles/), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f).get(key)
        return None if e is None else {"dram_bytes_per_launch": float(e["dram_bytes_per_launch"]),
                                       "source": e.get("source")}
    except Exception:
        return None


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled through NVML every 5 ms on a host thread
    during the timed region (nvidia-smi's query, without its 100 ms+ polling floor)."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index):
        self.index = index
        self.th = None
        self.err = None

    def start(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.dev = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = pynvml.nvmlDeviceGetMaxClockInfo(self.dev, pynvml.NVML_CLOCK_SM)
        except Exception as e:   # noqa: BLE001
            self.err = f"NVML unavailable: {e}"
            return
        self.sm, self.mask, self.stop_ev = [], 0, threading.Event()

        def run():
            nv = self.nv
            while not self.stop_ev.is_set():
                try:
                    self.sm.append(nv.nvmlDeviceGetClockInfo(self.dev, nv.NVML_CLOCK_SM))
                    self.mask |= nv.nvmlDeviceGetCurrentClocksEventReasons(self.dev)
                except Exception:   # noqa: BLE001
                    pass
                self.stop_ev.wait(0.005)
        self.th = threading.Thread(target=run, daemon=True)
        self.th.start()

    def stop(self):
        if self.th is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "not sampled"], "samples": 0}
        self.stop_ev.set()
        self.th.join()
        reasons = sorted(n for n, attr in self.REASONS if self.mask & getattr(self.nv, attr, 0))
        sm = self.sm
        load = [x for x in sm if x >= 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(sm), "source": "NVML, 5 ms period"}


# ------------------------------------------------------------------------------------------------
# CPU oracle (test infrastructure: bench.py's cpu_baseline leg and --impl reference only)
def oracle_chunk(cfg, freq, planes):
    """The oracle's explicit CSR impedance matrix of a `planes`-plane z-chunk of the model (the oracle's
    z-chunked SpMV of SURVEY §8(d)), on one core."""
    from threadpoolctl import threadpool_limits

    from oracle import operator as op
    from oracle import weights
    with threadpool_limits(1):
        z0 = max(0, cfg.nz // 2 - planes // 2)
        v = synth.velocity_slab(cfg, z0, planes).astype(np.float32).astype(np.float64)
        t0 = time.perf_counter()
        tab = weights.build_adaptive_table(*TABLE_ARGS)
        A = op.assemble(op.Problem(v, cfg.h, freq, cfg.npml, tab))
        t1 = time.perf_counter()
    u = synth.random_field((A.shape[0],), seed=99).astype(np.complex128)
    return {"A": A, "u": u, "t_assemble": t1 - t0, "npts": A.shape[0], "planes": planes, "z0": z0}


def oracle_spmv(S, n):
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        t0 = time.perf_counter()
        for _ in range(n):
            S["u"] = S["A"] @ S["u"] * 1e-3
        return time.perf_counter() - t0


def oracle_sample_text(cfg, S, n, dt):
    return (f"oracle scipy CSR SpMV (complex128, 1 of {os.cpu_count()} cores) of a {cfg.nx}x{cfg.ny}x{S['planes']} "
            f"z-chunk (planes {S['z0']}..{S['z0'] + S['planes'] - 1}) of config {cfg.index}, {n} SpMVs in {dt:.2f}s "
            f"(1 RHS); CSR assembly {S['t_assemble']:.1f}s outside the timed region")


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg, freq = workload(args, 1)
    S = oracle_chunk(cfg, freq, args.cpu_planes)
    for _ in range(args.warmup):
        oracle_spmv(S, 1)
    per = []
    for _ in range(args.steps):
        per.append(oracle_spmv(S, 1))
    tot = sum(per)
    value = S["npts"] * args.steps / tot / 1e9
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic",
            "config": {"workload": f"config{cfg.index} {cfg.name} {cfg.nx}x{cfg.ny}x{cfg.nz} f={freq:g}Hz: "
                                   f"27-point impedance apply (oracle CSR SpMV on a {args.cpu_planes}-plane z-chunk)",
                       "parallelism": "1 CPU core"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": oracle_sample_text(cfg, S, args.steps, tot)},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------------------------------------
def run_hz(args):
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    args.gpus = ws
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_2108_08730_b200 import hz, parallel

    ctx = parallel.make_context(local)      # NCCL communicator over all ranks (uid via torch.distributed)
    cfg, freq = workload(args, ws)
    nrhs = 1 if args.weak else args.nrhs
    z0, nzl = parallel.slab_partition(cfg.nz, ws, rank)
    v_np = synth.velocity_slab(cfg, z0, nzl, device=dev if cfg.index == 5 else None)
    v_dev = torch.from_numpy(v_np).to(dev, torch.float32).contiguous()
    del v_np
    T = hz.hz_build_weight_table(*TABLE_ARGS)
    C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_dev, freq, T, npml=cfg.npml, z0=z0,
                              nz_local=nzl, dtype=hz.HZ_C64)
    u = C.alloc_field(nrhs)
    u.real.uniform_(-1, 1)
    u.imag.uniform_(-1, 1)
    au = C.alloc_field(nrhs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    peak, peak_src = read_peak()

    def barrier():
        if ws > 1:
            dist.barrier()

    def time_applies(Cx, uu, aa, k, warm):
        for _ in range(warm):
            hz.hz_apply_impedance(Cx, uu, aa, stream=stream)
        torch.cuda.synchronize(dev)
        out = []
        l0 = hz.hz_kernel_launch_count()
        for _ in range(k):
            flush.fill_(1)
            torch.cuda.synchronize(dev)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hz.hz_apply_impedance(Cx, uu, aa, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            out.append(e0.elapsed_time(e1))
        return out, hz.hz_kernel_launch_count() - l0

    # ---------------- headline: device-resident batched apply ----------------
    torch.cuda.synchronize(dev)
    clocks = ClockSampler(local)
    clocks.start()
    ts, launches = time_applies(C, u, au, args.steps, args.warmup)
    clk = clocks.stop()
    (tot_max,) = parallel.rank_max([sum(ts)], dev)
    npts = cfg.nx * cfg.ny * cfg.nz
    ms_per_step = tot_max / args.steps
    value = npts * nrhs / (ms_per_step * 1e-3) / 1e9
    # dominant kernel = the apply launch itself: rank-0 launch durations (CUDA events on its stream)
    ms_launch = statistics.median(ts)
    pts_local = cfg.nx * cfg.ny * nzl
    byts = pts_local * (4 + 16 * nrhs)
    achieved = byts / (ms_launch * 1e-3) / 1e9
    wkey = f"config{cfg.index}_c64_nrhs{nrhs}_apply_{cfg.nx}x{cfg.ny}x{nzl}"
    traffic = read_traffic(wkey) if ws == 1 else None

    # ---------------- e2e: host (pinned) buffers through the C ABI ----------------
    e2e = None
    if not args.no_e2e:
        uh = C.alloc_field(nrhs, device="cpu", pin_memory=True)
        uh.copy_(u.cpu())
        ah = C.alloc_field(nrhs, device="cpu", pin_memory=True)
        te, _ = time_applies(C, uh, ah, max(2, min(args.steps, 4)), 1)
        (te_max,) = parallel.rank_max([sum(te)], dev)
        ke = max(2, min(args.steps, 4))
        fb = (nzl + 2) * cfg.ny * C.ldx * 8 * nrhs
        e2e = {"value": npts * nrhs / (te_max / ke * 1e-3) / 1e9, "unit": UNIT, "h2d_bytes_per_step": int(fb) * ws,
               "d2h_bytes_per_step": int(fb) * ws, "ms_per_step": te_max / ke, "steps": ke,
               "path": "hz_apply_impedance with pinned host u / Au: the library stages them through device buffers"}
        del uh, ah

    # ---------------- the solve leg: table + assemble + sources + batched solve ----------------
    solve = None
    if not args.no_solve:
        snodes = synth.source_nodes(cfg)
        sn = np.resize(snodes, (min(args.solve_nrhs, len(snodes)) if not args.weak else 1, 3))
        b = None
        solve = {"nrhs": int(len(sn)), "rtol": args.rtol, "max_iter": args.solve_max_iter}
        for ell, name in ((1, "bicgstab"), (2, "bicgstab2")):
            if args.weak and ell == 2:
                break
            torch.cuda.synchronize(dev)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            Ts = hz.hz_build_weight_table(*TABLE_ARGS)                                       # a1
            Cs = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_dev, freq, Ts, npml=cfg.npml,
                                       z0=z0, nz_local=nzl, dtype=hz.HZ_C64)                 # a2-a5 setup
            if b is None:
                b = Cs.alloc_field(len(sn))
                x = Cs.alloc_field(len(sn))
            hz.hz_point_sources(Cs, sn, b, stream=stream)                                   # a8
            x.zero_()
            mi = 100 if args.weak else args.solve_max_iter
            st, rel, its, stt = hz.hz_solve(Cs, b, x, rtol=1e-30 if args.weak else args.rtol, max_iter=mi,
                                            ell=ell, timing=True, stall_window=-1 if args.weak else 0,
                                            stream=stream)                                  # a6, a7
            e1.record(stream)
            torch.cuda.synchronize(dev)
            barrier()
            (tmax,) = parallel.rank_max([e0.elapsed_time(e1)], dev)
            it = int(stt["iterations"])
            solve[name] = {"solver": "BiCGSTAB" if ell == 1 else "BiCGStab(2)", "status": hz.STATUS_NAMES.get(st, st),
                           "converged": bool(st == hz.HZ_OK), "iterations": it,
                           "iterations_per_rhs": [int(i) for i in np.atleast_1d(its)], "relres_max": float(np.max(rel)),
                           "s": tmax * 1e-3, "s_per_rhs": tmax * 1e-3 / len(sn),
                           "ms_per_iteration": tmax / max(1, it),
                           "apply_ms_share": stt["apply_ms_total"] / tmax if tmax > 0 else None,
                           "stagnated": int(stt["stagnated"])}
            del Cs
        if args.weak:
            solve["note"] = "100 BiCGSTAB iterations (rtol 0): t_iter for the weak-scaling efficiency"

    # ---------------- extra measurements (N = 1) ----------------
    extra = {}
    if ws == 1 and not args.no_extra and not args.weak:
        extra = extras(args, hz, ctx, cfg, freq, v_dev, T, C, u, au, time_applies, peak)

    if rank != 0:
        if ws > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic",
        "config": {"workload": (f"config{cfg.index} {cfg.name} {cfg.nx}x{cfg.ny}x{cfg.nz} h={cfg.h:g}m f={freq:g}Hz "
                                f"npml={cfg.npml} c64: hz_apply_impedance of {nrhs} field(s) (fused coefficient build "
                                f"+ 27-point apply, a2-a6)" + (" — weak-scaling slab series 1201x1201x(50N+1)"
                                                              if args.weak else "")),
                   "grid": [cfg.nx, cfg.ny, cfg.nz], "nrhs": nrhs, "parallelism": f"z-slab x{ws}",
                   "l2": "flushed before every step (256 MiB write); the step's working set exceeds L2"},
        "roofline": {"bound": "hbm", "kernel": "apply27_tm (tensor-map TMA tiles: coefficient build + 27-point apply, a2-a6)",
                     "achieved": achieved, "peak": peak, "peak_source": peak_src, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic["dram_bytes_per_launch"] if traffic else None,
                     "traffic_source": traffic["source"] if traffic else None,
                     "algorithmic_bytes_per_launch": byts, "bytes_per_point": 4 + 16 * nrhs,
                     "launch_ms_median": ms_launch},
        "clocks": clk,
        "gpu_launches": int(launches),
        "e2e": e2e,
        "solve": solve,
    }
    if solve and "bicgstab" in solve:
        line["solve_s_per_rhs"] = solve["bicgstab"]["s_per_rhs"]
    line.update(extra)
    if ws == 1 and not args.no_cpu_baseline:
        S = oracle_chunk(cfg, freq, args.cpu_planes)
        dt = oracle_spmv(S, args.cpu_spmv)
        line["cpu_baseline"] = {"value": S["npts"] * args.cpu_spmv / dt / 1e9, "unit": UNIT, "cores": 1,
                                "kind": "oracle", "sample": oracle_sample_text(cfg, S, args.cpu_spmv, dt)}
    print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def extras(args, hz, ctx, cfg, freq, v_dev, T, C, u, au, time_applies, peak):
    """N = 1 extra measurements beside the headline: the 1-RHS apply, non-adaptive weights, the GA
    record mode and the GAm rule on the same model, and the config-2 solve step."""
    import torch
    npts = cfg.nx * cfg.ny * cfg.nz
    out = {}
    u1, a1 = u[:1], au[:1]

    def one(Cx, label, extra_bytes=0):
        ts, _ = time_applies(Cx, u1, a1, 5, 2)
        ms = statistics.median(ts)
        byts = npts * (4 + 16 + extra_bytes)
        return {"gpts_s": npts / (ms * 1e-3) / 1e9, "ms": ms, "hbm_frac": byts / (ms * 1e-3) / 1e9 / peak,
                "note": label}

    out["apply_nrhs1"] = one(C, "the same apply, 1 RHS (20 B/pt)")
    Tm = hz.hz_table_import(12.0, 0.1, T.rows5()[80][None])    # the GA row at G = 12 everywhere
    Cm = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_dev, freq, Tm, npml=cfg.npml, dtype=hz.HZ_C64)
    out["fixed_weights"] = one(Cm, "non-adaptive weights (one-row table: GA at G = 12 everywhere, like the "
                                   "paper's G4/Gm stencils, P:167-170): the adaptive lookup's cost (P:52, P:446)")
    out["fixed_weights"]["adaptive_over_fixed_time"] = out["apply_nrhs1"]["ms"] / out["fixed_weights"]["ms"]
    del Cm
    Cr = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_dev, freq, T, npml=cfg.npml, dtype=hz.HZ_C64,
                               rule=hz.HZ_RULE_GA_RECORD)
    out["record_mode"] = one(Cr, "GA weights stored per point and read by the apply (+20 B/pt)", 20)
    del Cr
    Cg = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v_dev, freq, T, npml=cfg.npml, dtype=hz.HZ_C64,
                               rule=hz.HZ_RULE_GAM)
    out["gam_rule"] = one(Cg, "GAm: 27-node mean weights read per point (+20 B/pt)", 20)
    del Cg
    torch.cuda.empty_cache()
    # config 2 (BASELINE configs[1]): the whole step table + assemble + sources + solve, 4 RHS
    c2 = synth.get_config(2)
    v2 = torch.from_numpy(synth.velocity_model(c2)).cuda().float()
    nodes = synth.source_nodes(c2)
    res = {}
    for ell, name in ((1, "bicgstab"), (2, "bicgstab2")):
        tms = []
        for rep in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            T2 = hz.hz_build_weight_table(*TABLE_ARGS)
            C2 = hz.hz_assemble_coeffs(ctx, c2.nx, c2.ny, c2.nz, c2.h, v2, c2.freq, T2, npml=c2.npml, dtype=hz.HZ_C64)
            b = C2.alloc_field(len(nodes))
            x = C2.alloc_field(len(nodes))
            hz.hz_point_sources(C2, nodes, b)
            st, rel, its, stt = hz.hz_solve(C2, b, x, rtol=args.rtol, ell=ell)
            e1.record()
            torch.cuda.synchronize()
            if rep > 0:
                tms.append(e0.elapsed_time(e1))
        res[name] = {"ms_per_step": statistics.median(tms), "s_per_rhs": statistics.median(tms) * 1e-3 / len(nodes),
                     "iterations": int(stt["iterations"]), "relres_max": float(np.max(rel)),
                     "status": hz.STATUS_NAMES.get(st, st)}
    out["config2_solve"] = {"workload": "config2 gradient 101^3 5 Hz c64, 4 RHS: table + assemble + sources + solve "
                                        "(rtol 1e-6), warm", **res}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_hz(args)


if __name__ == "__main__":
    sys.exit(main())
