"""Convergent Born series (CBS) reference wavefields — ORACLE (test infrastructure only).

The paper computes its heterogeneous-model references with "the highly-accurate Convergent Born
Series (CBS) method" (citing Osnabrugge et al. 2016), a volume-integral method built on the
Fourier-domain Green's function of a homogeneous background, "starting from the zero-order term of
the Born series and iteratively recovering the higher-order scattering terms", stopped "according to
a backward error of 1e-12".  Restated here from that published construction, in the sign
convention of this repository (reading A16: (∇² + k²) u = s, outgoing e^{+ikr}):

  k²(r) = k0² + iε + V(r),  V = k² − k0² − iε,  ε ≥ max |k² − k0²|      (background + potential)
  G = (−∇² − k0² − iε)⁻¹, Fourier symbol 1/(|p|² − k0² − iε)              (|G| ≤ 1/ε)
  the equation is u = G(V u − s) (since (∇² + k0² + iε)u = s − V u);
  preconditioner γ = (i/ε) V, iteration u ← u − γ [u − G(V u − s)]        (u₀ = 0: the Born series)

with the spectral Laplacian (symbol −|p|², p = 2π·fftfreq) on a periodic box.  The backward error
‖(∇² + k²)u − s‖ / ‖s‖ is recomputed with that Laplacian.  Reading A26 (the paper is silent on the
CBS box): the model is embedded in a box padded by `pad` cells per side; the padding takes
the velocity of the nearest model node and an absorbing term i·α, α = a·k0²·Σ_axes (d_a / pad)²
(d_a = cells into the padding along axis a); k0² = midpoint of the range of Re k² over the box;
ε = 1.05 × max over the box of |k² − k0²| (at least 1e-3·k0²): strictly above the
maximum, so that V ≠ 0 and γ ≠ 0 everywhere (with ε equal to the maximum, γ vanishes at the most
absorbing box corners, those nodes never update and the iteration stalls at a nonzero backward error).  Point sources: s = amp/h³ at the node.

Plain numpy: every iteration is the formula above with numpy FFTs; no fusion, no reordering.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class CbsBox:
    k2: np.ndarray      # complex128 [Nz][Ny][Nx], the padded box
    pad: int
    h: float
    k0sq: float
    eps: float
    shape: tuple        # model shape (nz, ny, nx)


def box_k2(v, freq, h, pad, absorb=0.5):
    """k² on the padded box (reading A26): nearest model velocity in the padding + i·α absorption."""
    v = np.asarray(v, dtype=np.float64)
    nz, ny, nx = v.shape
    omega = 2.0 * np.pi * freq
    iz = np.clip(np.arange(nz + 2 * pad) - pad, 0, nz - 1)
    iy = np.clip(np.arange(ny + 2 * pad) - pad, 0, ny - 1)
    ix = np.clip(np.arange(nx + 2 * pad) - pad, 0, nx - 1)
    vb = v[np.ix_(iz, iy, ix)]
    k2r = (omega / vb) ** 2
    k0sq = 0.5 * (k2r.min() + k2r.max())

    def dist(n):   # cells into the padding along one axis
        i = np.arange(n + 2 * pad)
        return np.maximum(0, np.maximum(pad - i, i - (pad + n - 1))).astype(np.float64)
    if pad > 0:
        d2 = (dist(nz)[:, None, None] / pad) ** 2 + (dist(ny)[None, :, None] / pad) ** 2 + \
             (dist(nx)[None, None, :] / pad) ** 2
    else:
        d2 = np.zeros(k2r.shape)
    k2 = k2r + 1j * (absorb * k0sq) * d2
    eps = max(1.05 * np.abs(k2 - k0sq).max(), 1e-3 * k0sq)
    return CbsBox(k2=k2, pad=pad, h=h, k0sq=float(k0sq), eps=float(eps), shape=(nz, ny, nx))


def wavenumber2(shape, h):
    """|p|² on the FFT grid of the box (p = 2π·fftfreq(n, h) per axis)."""
    pz, py, px = (2.0 * np.pi * np.fft.fftfreq(n, d=h) for n in shape)
    return pz[:, None, None] ** 2 + py[None, :, None] ** 2 + px[None, None, :] ** 2


def laplacian(u, h):
    """Spectral Laplacian on the periodic box: symbol −|p|²."""
    return np.fft.ifftn(-wavenumber2(u.shape, h) * np.fft.fftn(u))


def point_source_box(box: CbsBox, nodes, amps=None):
    """s = amp/h³ at each model node (x, y, z), placed in the padded box."""
    s = np.zeros(box.k2.shape, dtype=np.complex128)
    amps = np.ones(len(nodes)) if amps is None else np.asarray(amps)
    for (x, y, z), a in zip(nodes, amps):
        s[z + box.pad, y + box.pad, x + box.pad] += a / box.h ** 3
    return s


def backward_error(box: CbsBox, u, s):
    """‖(∇² + k²)u − s‖ / ‖s‖ on the box."""
    r = laplacian(u, box.h) + box.k2 * u - s
    return float(np.linalg.norm(r) / np.linalg.norm(s))


def cbs_solve(box: CbsBox, s, tol=1e-12, max_iter=100000, check_every=10):
    """The preconditioned Born iteration from u₀ = 0 until the backward error ≤ tol.
    Returns (u on the box, backward error, iterations, history of (iteration, backward error))."""
    V = box.k2 - box.k0sq - 1j * box.eps
    gamma = (1j / box.eps) * V
    Gsym = 1.0 / (wavenumber2(box.k2.shape, box.h) - box.k0sq - 1j * box.eps)
    u = np.zeros_like(box.k2)
    hist = []
    be = np.inf
    it = 0
    while it < max_iter:
        t = np.fft.ifftn(Gsym * np.fft.fftn(V * u - s))   # G(V u − s)
        u = u - gamma * (u - t)
        it += 1
        if it % check_every == 0:
            be = backward_error(box, u, s)
            hist.append((it, be))
            if be <= tol:
                break
    return u, be, it, hist


def model_region(box: CbsBox, u):
    """The model nodes of a box field."""
    p = box.pad
    nz, ny, nx = box.shape
    return u[p:p + nz, p:p + ny, p:p + nx]
