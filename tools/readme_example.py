"""The README's Python example, runnable (needs a CUDA device): python tools/readme_example.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2108_08730_b200 import hz

ctx = hz.hz_ctx_create(0)                                   # one per rank (nranks/rank/uid for z-slabs)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)          # G range, dG, Tikhonov lambda
v = torch.full((101, 101, 101), 3000.0, device="cuda")      # [nz][ny][nx] velocity, float32 for c64
C = hz.hz_assemble_coeffs(ctx, 101, 101, 101, 40.0, v, 5.0, T, npml=8)   # h = 40 m, f = 5 Hz

b = C.alloc_field(4)                                        # [nrhs][nz+2][ny][nx] complex64 (halo planes)
hz.hz_point_sources(C, np.array([[50, 50, 10]] * 4), b)     # consistent point sources
x = C.alloc_field(4)                                        # initial guess (zeros)
status, relres, iters, stats = hz.hz_solve(C, b, x, rtol=1e-6, ell=2)   # ell=1: BiCGSTAB

au = C.alloc_field(4)
hz.hz_apply_impedance(C, x, au)                             # matrix-free A·x
print('readme example', status, relres, iters, stats['iterations'])
