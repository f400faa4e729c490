"""BASELINE configs[4] on one GPU: the whole 1201x1201x401 grid (5.8e8 points), 10 Hz, 1 point source,
complex64, BiCGStab(2) to rtol 1e-6 with a 5000-iteration stall window (this model plateaus for > 1000
iterations before it converges).  Prints one JSON line.  Usage: python tools/solve_cfg5.py [max_iter]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

max_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 25000
cfg = synth.get_config(5)
dev = torch.device("cuda", 0)
v = torch.from_numpy(synth.velocity_slab(cfg, 0, cfg.nz, device=dev)).to(dev, torch.float32)
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freqs[-1], T, npml=cfg.npml)
nodes = synth.source_nodes(cfg)[:1]
b, x = C.alloc_field(1), C.alloc_field(1)
hz.hz_point_sources(C, nodes, b)
x.zero_()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=max_iter, ell=2, timing=True, stall_window=5000)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
it = int(stats["iterations"])
print(json.dumps({"workload": "config5 1201x1201x401 f=10Hz npml=8 c64, 1 RHS, BiCGStab(2), rtol 1e-6, stall_window 5000",
                  "status": hz.STATUS_NAMES.get(st, st), "iterations": it, "relres": float(np.max(rel)),
                  "s": ms * 1e-3, "ms_per_iteration": ms / max(1, it),
                  "apply_ms_share": stats["apply_ms_total"] / ms, "stagnated": int(stats["stagnated"]),
                  "hbm_gb_allocated": torch.cuda.mem_get_info(dev)[1] / 1e9 - torch.cuda.mem_get_info(dev)[0] / 1e9}))
