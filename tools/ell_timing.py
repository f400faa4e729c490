"""Wall time per BiCGSTAB-equivalent iteration of hz_solve (fixed iteration count, rtol unreachable)
for ell = 1 / 2, with and without per-apply event timing, and with rare host polls.
Usage: python tools/ell_timing.py [CFG] [nrhs] [iters]"""
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
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 400
cfg = synth.get_config(ci)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = np.resize(synth.source_nodes(cfg), (nrhs, 3))
b = C.alloc_field(nrhs)
hz.hz_point_sources(C, nodes, b)
for ell in (1, 2):
    for timing, check in ((True, 10), (False, 10), (False, 1000)):
        best = 1e9
        for rep in range(3):
            x = C.alloc_field(nrhs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-14, max_iter=iters, timing=timing, check_every=check,
                                            replace_every=50, stall_window=-1, ell=ell)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"ell={ell} timing={int(timing)} check_every={check}: {best / stt['iterations'] * 1e3:.3f} ms/it "
              f"({stt['iterations']} it, apply {stt['apply_ms_total'] / max(1, stt['apply_launches']):.3f} ms/launch, "
              f"launches {stt['kernel_launches']})", flush=True)
