"""BiCGSTAB with and without the shifted-Laplacian multigrid preconditioner (hz_solve_opts.precond) on
a BASELINE config or a crop: iterations, time, relres.  Usage: python tools/precond_cmp.py <cfg|4c5|4c10|5c10> [nrhs] [max_iter]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz

key = sys.argv[1]
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
mi = int(sys.argv[3]) if len(sys.argv) > 3 else 20000
if "c" in key:
    ci, f = key.split("c"); cfg = synth.crop_config(int(ci), float(f))
else:
    cfg = synth.get_config(int(key))
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
if cfg.nx * cfg.ny * cfg.nz > 5e7:
    v = torch.from_numpy(synth.velocity_slab(cfg, 0, cfg.nz)).cuda().float()
else:
    v = torch.from_numpy(synth.velocity_model(cfg).astype(np.float32)).cuda()
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freq, T, npml=cfg.npml)
nodes = np.resize(synth.source_nodes(cfg), (nrhs, 3))
b = C.alloc_field(nrhs); hz.hz_point_sources(C, nodes, b)
res = {}
for pre in (1, 0):
    x = C.alloc_field(nrhs)
    torch.cuda.synchronize(); t = time.time()
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=mi, precond=pre)
    torch.cuda.synchronize(); dt = time.time() - t
    res[pre] = x[:, 1:-1, :, :cfg.nx].cpu().numpy()
    print(f"{key} f={cfg.freq} nrhs={nrhs} precond={pre}: status {st} iterations {list(its)} relres {max(rel):.2e} {dt:.2f} s ({dt/nrhs:.2f} s/RHS)", flush=True)
d = np.linalg.norm(res[1] - res[0]) / np.linalg.norm(res[0])
print(f"  precond vs plain wavefield rel diff {d:.2e}")
