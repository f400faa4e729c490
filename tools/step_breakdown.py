"""Wall-time breakdown of the bench step outside the Krylov iterations (config 2 by default):
table build, assemble, sources, and a 1-iteration solve on fresh coefficients (workspace set-up).
Usage: python tools/step_breakdown.py [CFG]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.get_config(ci)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
nodes = synth.source_nodes(cfg)
b = torch.zeros((len(nodes), cfg.nz + 2, cfg.ny, cfg.nx), dtype=torch.complex64, device="cuda")
x = torch.zeros_like(b)


def t(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, r


for rep in range(4):
    t_tab, T = t(lambda: hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2))
    t_asm, C = t(lambda: hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml))
    t_src, _ = t(lambda: hz.hz_point_sources(C, nodes, b))
    t_s1, _ = t(lambda: hz.hz_solve(C, b, x, rtol=1e-14, max_iter=1))
    t_s2, _ = t(lambda: hz.hz_solve(C, b, x, rtol=1e-14, max_iter=1))
    t_del, _ = t(lambda: C.__del__())
    print(f"table {t_tab:.2f} ms  assemble {t_asm:.2f}  sources {t_src:.2f}  solve(1 it, first) {t_s1:.2f}  "
          f"solve(1 it, again) {t_s2:.2f}  destroy {t_del:.2f}", flush=True)
