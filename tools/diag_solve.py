"""Diagnostic: BiCGSTAB convergence history on config 1 (GPU c64/c128) vs the oracle."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz
from oracle import weights, operator as op, solvers

cfgi = int(sys.argv[1]) if len(sys.argv) > 1 else 1
cfg = synth.get_config(cfgi)
otab = weights.build_adaptive_table(4.0, 40.0, 0.1, 1e-2)
T = hz.hz_table_import(otab.g_min, otab.dg, otab.u5)
ctx = hz.hz_ctx_create(0)
v = synth.velocity_model(cfg)
nodes = synth.source_nodes(cfg)[:1]
for dt in ("c64", "c128"):
    rd = np.float32 if dt == "c64" else np.float64
    C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v.astype(rd)).cuda(), cfg.freq, T,
                              npml=cfg.npml, dtype=hz.HZ_C64 if dt == "c64" else hz.HZ_C128)
    b = C.alloc_field(1)
    hz.hz_point_sources(C, nodes, b)
    for re in (50, 0):
        for mi in (1, 5, 20, 50, 100, 150, 300, 1000):
            x = C.alloc_field(1)
            st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=mi, replace_every=re, check_every=10)
            print(dt, "replace", re, "max_iter", mi, "status", st, "rel", rel, "its", its, "restarts", stt["restarts"],
                  "repl", stt["replacements"], "xmax", float(x.abs().max()), flush=True)
            if st == 0:
                break
P = op.Problem(v.astype(np.float32).astype(np.float64), cfg.h, cfg.freq, cfg.npml, otab)
A = op.assemble(P)
bo = op.point_sources(P, nodes)[0].ravel()
for mi in (1, 5, 20, 50, 100):
    xo, rr, it = solvers.bicgstab(A, bo, rtol=1e-6, max_iter=mi)
    print("oracle max_iter", mi, "rel", rr, "it", it, flush=True)
# GPU b vs oracle b
bg = b[0, 1:-1].cpu().numpy().ravel()
print("b parity", np.linalg.norm(bg - bo) / np.linalg.norm(bo))
