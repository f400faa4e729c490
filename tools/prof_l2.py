"""Is the complex64 apply bound inside the SM or by the memory system?  The same launch on a grid whose
whole working set (w, u, Au: 20 B per point) fits the 126 MB L2, timed warm (back to back, L2-resident)
and cold (256 MiB flush before every launch), next to a grid 8x larger in y.
Usage: python tools/prof_l2.py [nx] [ny] [nz] [npml]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2108_08730_b200 import hz

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 801
ny = int(sys.argv[2]) if len(sys.argv) > 2 else 33
nz = int(sys.argv[3]) if len(sys.argv) > 3 else 187
npml = int(sys.argv[4]) if len(sys.argv) > 4 else 0
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
ctx = hz.hz_ctx_create(0)
T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def run(ny_):
    # smooth in x (like the configs' models), 2100-6000 m/s, h = 25 m, f = 10 Hz: G in 8.4 .. 24
    v = (2100.0 + 3900.0 * torch.rand((nz, ny_, 1), device=dev, generator=g)).expand(nz, ny_, nx).contiguous()
    C = hz.hz_assemble_coeffs(ctx, nx, ny_, nz, 25.0, v, 10.0, T, npml=npml)
    u = C.alloc_field(1)
    u.real.uniform_(-1, 1)
    u.imag.uniform_(-1, 1)
    au = C.alloc_field(1)
    out = {}
    for mode in ("warm", "cold"):
        for _ in range(3):
            hz.hz_apply_impedance(C, u, au)
        ts = []
        for _ in range(9):
            if mode == "cold":
                flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hz.hz_apply_impedance(C, u, au)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[mode] = sorted(ts)[len(ts) // 2]
    npts = nx * ny_ * nz
    print(f"{nx}x{ny_}x{nz} npml {npml}: {npts * 20 / 1e6:.0f} MB working set; "
          + "; ".join(f"{m} {t:.4f} ms = {t / npts * 1e9:.3f} ps/pt ({npts * 20 / t / 1e6:.0f} GB/s)" for m, t in out.items()))


run(ny)        # fits L2
run(8 * ny)    # does not
