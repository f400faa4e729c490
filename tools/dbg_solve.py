"""Debug: config-1 solves with growing iteration caps (each step printed and flushed)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz
cfg = synth.get_config(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
ell = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = synth.source_nodes(cfg)
print("setup done", flush=True)
b = C.alloc_field(len(nodes)); hz.hz_point_sources(C, nodes, b)
for mi in (0, 1, 20000):
    x = C.alloc_field(len(nodes))
    t = time.time()
    if mi == 0:
        au = C.alloc_field(len(nodes)); hz.hz_apply_impedance(C, b, au); torch.cuda.synchronize()
        print("apply ok", flush=True); continue
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=mi, ell=ell)
    torch.cuda.synchronize()
    print(f"max_iter {mi}: st {st} its {its} rel {rel} {time.time()-t:.3f}s", flush=True)
