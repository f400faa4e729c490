"""Diagnostic: where the BiCGSTAB step time goes on config 2 (timing on/off, poll period)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz
cfg = synth.get_config(2)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = synth.source_nodes(cfg)
b = C.alloc_field(4); hz.hz_point_sources(C, nodes, b)
for timing in (0, 1):
    for ce in (10, 1000):
        for rep in range(2):
            x = C.alloc_field(4)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-6, timing=bool(timing), check_every=ce)
            torch.cuda.synchronize(); dt = time.perf_counter() - t0
        print(f"timing={timing} check_every={ce}: {dt*1e3:.1f} ms, iters {stt['iterations']}, apply ms {stt['apply_ms_total']:.1f}, launches {stt['kernel_launches']}, per-iter {dt*1e3/stt['iterations']:.3f} ms", flush=True)
