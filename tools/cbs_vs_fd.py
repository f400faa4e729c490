"""Diagnostic: CBS reference vs the GPU FD (GA) wavefield on a BASELINE config (or a homogeneous /
two-layer variant), err of P:268 (W = distance, PML and a 2-cell ball masked).
Usage: python tools/cbs_vs_fd.py config [variant: model|homog|layer] [source index] [pad] [absorb]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2108_08730_b200 import hz

ci = int(sys.argv[1]); var = sys.argv[2] if len(sys.argv) > 2 else "model"
si = int(sys.argv[3]) if len(sys.argv) > 3 else 0
pad = int(sys.argv[4]) if len(sys.argv) > 4 else -1
absorb = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
cfg = synth.get_config(ci)
if len(sys.argv) > 6:
    import dataclasses
    cfg = dataclasses.replace(cfg, freqs=(float(sys.argv[6]),))
zs = int(sys.argv[7]) if len(sys.argv) > 7 else None
v = synth.velocity_model(cfg).astype(np.float32).astype(np.float64)
if var == "homog":
    v[:] = np.median(v)
elif var == "layer":
    v[:] = 2000.0; v[v.shape[0] // 2:] = 3500.0
node = tuple(int(t) for t in synth.source_nodes(cfg)[si])
if zs is not None:
    node = (node[0], node[1], zs)
ctx = hz.hz_ctx_create(0)
uc = torch.zeros(v.shape, dtype=torch.complex128, device="cuda")
st, stats = hz.hz_cbs_solve(ctx, torch.from_numpy(v).cuda(), cfg.h, cfg.freq, [node], uc, tol=1e-10, pad=pad, absorb=absorb)
ref = uc.cpu().numpy()
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, torch.from_numpy(v.astype(np.float32)).cuda(), cfg.freq, T, npml=cfg.npml)
out = {}
for cons in (False, True):
    b = C.alloc_field(1); hz.hz_point_sources(C, [node], b, consistent=cons)
    x = C.alloc_field(1)
    st2, rel, its, _ = hz.hz_solve(C, b, x, rtol=1e-7, max_iter=20000, ell=2)
    u = x[0, 1:-1, :, :cfg.nx].cpu().numpy().astype(np.complex128)
    nz, ny, nx = v.shape
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    d = np.sqrt((I - node[0]) ** 2 + (J - node[1]) ** 2 + (K - node[2]) ** 2)
    p = cfg.npml
    m = np.zeros(v.shape, bool); m[p:nz - p, p:ny - p, p:nx - p] = True; m &= d > 2
    W = d * cfg.h
    e = lambda a, b: np.abs(W[m] * (a - b)[m]).sum() / np.abs(W[m] * b[m]).sum()
    err = e(u.real, ref.real) + e(u.imag, ref.imag)
    # the ratio of amplitudes and a phase estimate in the interior
    rr = (u[m] * np.conj(ref[m])).sum() / (np.abs(ref[m]) ** 2).sum()
    out["consistent" if cons else "nodal"] = (round(err, 4), complex(np.round(rr, 4)), int(its[0]), st2)
print(f"config {ci} f {cfg.freq} {var} src {node} cbs it {stats['iterations']} be {stats['backward_error']:.1e} box {stats['box']} pad {stats['pad']}: {out}", flush=True)
