"""Per-iteration cost of the batched BiCGSTAB on a BASELINE config: a fixed number of iterations
(rtol unreachable), apply kernels timed with CUDA events inside libhz.
Usage: python tools/solve_iter.py [CFG] [nrhs] [iters] [dtype]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 300
dt = sys.argv[4] if len(sys.argv) > 4 else "c64"
check_every = int(sys.argv[5]) if len(sys.argv) > 5 else 10
cfg = synth.get_config(ci)
rd = np.float32 if dt == "c64" else np.float64
v = torch.from_numpy(synth.velocity_model(cfg).astype(rd)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml,
                          dtype=hz.HZ_C64 if dt == "c64" else hz.HZ_C128)
nodes = np.resize(synth.source_nodes(cfg), (nrhs, 3))
b = C.alloc_field(nrhs)
hz.hz_point_sources(C, nodes, b)
res = []
for timing in (1, 0, 0):
    x = C.alloc_field(nrhs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-14, max_iter=iters, timing=bool(timing), check_every=check_every)
    torch.cuda.synchronize()
    res.append((time.perf_counter() - t0, stt))
wall = min(r[0] for r in res[1:])
stt = res[0][1]
n = stt["iterations"]
print(json.dumps({"cfg": ci, "nrhs": nrhs, "dtype": dt, "iters": n, "ms_per_iter": wall * 1e3 / n,
                  "apply_ms_per_iter": stt["apply_ms_total"] / n,
                  "apply_gpts_s": stt["apply_points_total"] / stt["apply_ms_total"] / 1e6,
                  "apply_frac": stt["apply_bytes_total"] / stt["apply_ms_total"] / 1e6 / 6543.4,
                  "launches_per_iter": stt["kernel_launches"] / n}))
