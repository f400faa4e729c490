"""Analytic reference wavefields — ORACLE (test infrastructure only).

The paper validates against analytic solutions in a homogeneous medium and in a linear velocity
gradient (the gradient solution is cited to Kuvshinov & Mulder 2006 but not
printed).  Time convention e^{−iωt} so outgoing waves are e^{+ikr}; the operator is
A p = +s (reading A16), hence p = −G_cont where (∇² + k²) G_cont = −δ.
"""
from __future__ import annotations

import numpy as np


def homogeneous(r, k, amp=1.0):
    """p(r) = −amp e^{ikr}/(4π r): solution of ∇²p + k²p = amp δ."""
    r = np.asarray(r, dtype=np.float64)
    return -amp * np.exp(1j * k * r) / (4.0 * np.pi * r)


def gradient(x, y, z, xs, ys, zs, omega, c0, alpha, amp=1.0):
    """Solution of ∇²p + ω²/c(z)² p = amp δ(x − x_s) for c(z) = c0 + α z (z = depth in m).

    With ζ = z + c0/α (so c = α ζ), ν = √((ω/α)² − ¼), R = |x − x_s| and
    σ = 2 asinh(R / (2√(ζ ζ_s))) (the hyperbolic distance, cosh σ = 1 + R²/(2 ζ ζ_s)):
        G_cont = e^{iνσ} / (4π √(ζ ζ_s) sinh σ)        solves (∇² + ω²/c²) G = −δ
    (DESIGN.md App. E; derivation: u = ζ^{-1/2} w maps the operator to the hyperbolic-space
    Helmholtz operator).  Returns p = −amp·G_cont (reading A16).
    """
    zeta = np.asarray(z, dtype=np.float64) + c0 / alpha
    zeta_s = zs + c0 / alpha
    R = np.sqrt((np.asarray(x) - xs) ** 2 + (np.asarray(y) - ys) ** 2 + (np.asarray(z) - zs) ** 2)
    nu = np.sqrt((omega / alpha) ** 2 - 0.25)
    sig = 2.0 * np.arcsinh(R / (2.0 * np.sqrt(zeta * zeta_s)))
    G = np.exp(1j * nu * sig) / (4.0 * np.pi * np.sqrt(zeta * zeta_s) * np.sinh(sig))
    return -amp * G
