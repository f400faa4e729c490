"""Diagnostic: determinism of the apply and slab-vs-full differences."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz
from oracle import weights
otab = weights.build_adaptive_table(4.0, 40.0, 0.1, 1e-2)
T = hz.hz_table_import(otab.g_min, otab.dg, otab.u5)
ctx = hz.hz_ctx_create(0)
rng = np.random.default_rng(31)
nz, ny, nx, h, f, npml = 23, 21, 45, 25.0, 7.0, 4
v = rng.uniform(1500.0, 4500.0, (nz, ny, nx)).astype(np.float32)
u = synth.random_field((2, nz, ny, nx), seed=6)
def full():
    C = hz.hz_assemble_coeffs(ctx, nx, ny, nz, h, torch.from_numpy(v).cuda(), f, T, npml=npml)
    ud = C.alloc_field(2); ud[:, 1:-1] = torch.from_numpy(u).cuda()
    aud = C.alloc_field(2); hz.hz_apply_impedance(C, ud, aud); torch.cuda.synchronize()
    return aud[:, 1:-1].cpu().numpy()
F = [full() for _ in range(3)]
print("full deterministic:", all(np.array_equal(F[0], g) for g in F[1:]))
def slab(z0, z1):
    nzl = z1 - z0
    vs = np.ones((nzl + 2, ny, nx), np.float32)
    lo, hi = max(z0 - 1, 0), min(z1 + 1, nz)
    vs[lo - (z0 - 1):hi - (z0 - 1)] = v[lo:hi]
    C = hz.hz_assemble_coeffs(ctx, nx, ny, nz, h, torch.from_numpy(vs).cuda(), f, T, npml=npml, z0=z0, nz_local=nzl,
                              v_pml=float(v.max()), v_halo=True)
    ud = C.alloc_field(2)
    for k in range(nzl + 2):
        zg = z0 - 1 + k
        if 0 <= zg < nz:
            ud[:, k] = torch.from_numpy(u[:, zg]).cuda()
    aud = C.alloc_field(2); hz.hz_apply_impedance(C, ud, aud); torch.cuda.synchronize()
    return aud[:, 1:-1].cpu().numpy()
for (z0, z1) in [(0, 1), (9, 16), (0, 23), (12, 23), (0, 12)]:
    S = [slab(z0, z1) for _ in range(2)]
    d = S[0] != F[0][:, z0:z1]
    print((z0, z1), "det", np.array_equal(S[0], S[1]), "ndiff", int(d.sum()), np.argwhere(d)[:4].tolist())
