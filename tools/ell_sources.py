"""Per-RHS iteration counts of BiCGSTAB and BiCGStab(2) on a BASELINE config (each source solved in the
batch and alone), to separate method behaviour from rounding-order sensitivity.
Usage: python tools/ell_sources.py [CFG]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = synth.get_config(ci)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = synth.source_nodes(cfg)
for ell in (1, 2):
    b = C.alloc_field(len(nodes))
    hz.hz_point_sources(C, nodes, b)
    x = C.alloc_field(len(nodes))
    st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-6, ell=ell)
    print(f"ell={ell} batch: its {list(its)} restarts {stt['restarts']} replacements {stt['replacements']}", flush=True)
    for r in range(len(nodes)):
        b1 = C.alloc_field(1)
        hz.hz_point_sources(C, nodes[r:r + 1], b1)
        x1 = C.alloc_field(1)
        st, rel, its1, stt = hz.hz_solve(C, b1, x1, rtol=1e-6, ell=ell)
        print(f"   ell={ell} source {r} alone: its {its1[0]} restarts {stt['restarts']} relres {rel[0]:.2e}", flush=True)
