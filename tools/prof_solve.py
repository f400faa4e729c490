"""Profile target: a few BiCGSTAB iterations on BASELINE config 4 (801x801x187, 10 Hz, 2 RHS, c64), for
the per-kernel launch list of one solve iteration (apply DOT1 / DOT4 epilogues, vector kernels).
Usage: python tools/prof_solve.py [iters] [ell] [nrhs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 1
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 2
cfg = synth.get_config(4)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freqs[-1], T, npml=cfg.npml)
nodes = synth.source_nodes(cfg)[:nrhs]
b, x = C.alloc_field(nrhs), C.alloc_field(nrhs)
hz.hz_point_sources(C, nodes, b)
for rep in range(2):
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-12, max_iter=iters, ell=ell, timing=True)
    e1.record()
    torch.cuda.synchronize()
    print(f"rep {rep}: {iters} it ell {ell} nrhs {nrhs}: {e0.elapsed_time(e1):.1f} ms, "
          f"{e0.elapsed_time(e1) / iters:.3f} ms/it, stats {stats}", flush=True)
