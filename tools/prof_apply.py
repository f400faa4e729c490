"""Apply-kernel microbenchmark: hz_apply_impedance on a BASELINE config (random u), CUDA-event timed.
Usage: python tools/prof_apply.py CFG [nrhs] [dtype] [reps]   (CFG 5 = the 1201x1201x51 weak slab)"""
import os
import sys
import json

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
dt = sys.argv[3] if len(sys.argv) > 3 else "c64"
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
npml_override = int(sys.argv[5]) if len(sys.argv) > 5 else None
cfg = synth.get_config(ci)
nz = cfg.nz if ci != 5 else int(os.environ.get("HZ_CFG5_NZ", "51"))
dev = torch.device("cuda", 0)
v = synth.velocity_slab(cfg, 0, nz, device=dev if ci == 5 else None)
rd = torch.float32 if dt == "c64" else torch.float64
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
freq = cfg.freqs[-1]
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, nz, cfg.h, torch.from_numpy(v).to(dev, rd), freq, T,
                          npml=cfg.npml if npml_override is None else npml_override,
                          dtype=hz.HZ_C64 if dt == "c64" else hz.HZ_C128)
u = C.alloc_field(nrhs)
u.real.uniform_(-1, 1)
u.imag.uniform_(-1, 1)
au = C.alloc_field(nrhs)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
for _ in range(3):
    hz.hz_apply_impedance(C, u, au)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    flush.fill_(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    hz.hz_apply_impedance(C, u, au)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
npts = cfg.nx * cfg.ny * nz
esz = 4 if dt == "c64" else 8
byts = npts * (esz + nrhs * 4 * esz)
ms = float(np.median(ts))
print(json.dumps({"cfg": ci, "npml": cfg.npml if npml_override is None else npml_override, "grid": [cfg.nx, cfg.ny, nz], "nrhs": nrhs, "dtype": dt, "ms_median": ms,
                  "ms_min": float(np.min(ts)), "gpts_s": npts * nrhs / ms / 1e6, "GBps": byts / ms / 1e6,
                  "frac_of_6543": byts / ms / 1e6 / 6543.4}))
