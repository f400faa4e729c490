"""Time of the complex64 solver's fp64-arithmetic residual apply (apply27_v2<double, float>) on a
BASELINE config: hz_solve with max_iter = 1 is two residuals + one iteration; the one-iteration cost is
measured separately and subtracted.  Usage: python tools/prof_resid.py [CFG] [nrhs]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz
ci = int(sys.argv[1]) if len(sys.argv) > 1 else 2
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.get_config(ci)
v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = np.resize(synth.source_nodes(cfg), (nrhs, 3))
b = C.alloc_field(nrhs)
hz.hz_point_sources(C, nodes, b)
def run(iters):
    best = 1e9
    for _ in range(5):
        x = C.alloc_field(nrhs)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        hz.hz_solve(C, b, x, rtol=1e-14, max_iter=iters, replace_every=1000, check_every=1000)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    return best
t1, t11 = run(1), run(11)
per_iter = (t11 - t1) / 10
print(json.dumps({"cfg": ci, "nrhs": nrhs, "resid_ms": (t1 - per_iter) / 2 * 1e3, "iter_ms": per_iter * 1e3}))
