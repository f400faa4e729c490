"""Profile target for ncu: the complex64 tensor-map apply on a BASELINE config (default config 4),
nrhs fields, a few launches.  Usage: python tools/prof_tm.py [config] [nrhs] [reps] [npml]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 4
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
npml_override = int(sys.argv[4]) if len(sys.argv) > 4 else None
cfg = synth.get_config(ci)
f = cfg.freqs[-1]
dev = torch.device("cuda", 0)
v = torch.from_numpy(synth.velocity_slab(cfg, 0, cfg.nz, device=dev if ci == 5 else None)).to(dev, torch.float32)
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, f, T,
                          npml=cfg.npml if npml_override is None else npml_override)
u = C.alloc_field(nrhs)
u.real.uniform_(-1, 1)
u.imag.uniform_(-1, 1)
au = C.alloc_field(nrhs)
for _ in range(reps):
    hz.hz_apply_impedance(C, u, au)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hz.hz_apply_impedance(C, u, au)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
npts = cfg.nx * cfg.ny * cfg.nz
ms = sorted(ts)[len(ts) // 2]
print(f"config {ci} nrhs {nrhs} npml {cfg.npml if npml_override is None else npml_override}: {ms:.3f} ms, {npts * nrhs / ms / 1e6:.1f} Gpts/s, "
      f"{npts * (4 + 16 * nrhs) / ms / 1e6:.0f} GB/s")
