"""Plane-wave dispersion of the 27-point stencil — ORACLE (test infrastructure only).

Follows PAPER.md §2.2 "Numerical dispersion analysis for adaptive mass and stiffness
weights".

Weight conventions (reading A2):
  * class weights  w7 = (ws1, ws2, ws3, wm0, wm1, wm2, wm3) with ws1+ws2+ws3 = 1 and
    wm0+wm1+wm2+wm3 = 1 — the weights of the stiffness sum and of Eq. 8;
  * per-point mass weights  mu = (wm0, wm1/6, wm2/12, wm3/8) — the weights that actually
    multiply one neighbour in Eq. 8.  J and H3..H5 are written in these
    per-point units, so the five LS unknowns "[w_s1, w_s2, w_m0, w_m1, w_m2]" are
    (ws1, ws2, mu0, mu1, mu2).
"""
from __future__ import annotations

import numpy as np


def abc(G, theta, phi):
    """A, B, C of P:136-143 (a = 2π cosφ cosθ/G, b = 2π cosφ sinθ/G, c = 2π sinφ/G)."""
    G = np.asarray(G, dtype=np.float64)
    a = 2.0 * np.pi * np.cos(phi) * np.cos(theta) / G
    b = 2.0 * np.pi * np.cos(phi) * np.sin(theta) / G
    c = 2.0 * np.pi * np.sin(phi) / G
    ca, cb, cc = np.cos(a), np.cos(b), np.cos(c)
    A = ca * cb * cc
    B = ca * cb + ca * cc + cb * cc
    C = ca + cb + cc
    return A, B, C


def per_point_mass(w7):
    """(mu0, mu1, mu2, mu3) = (wm0, wm1/6, wm2/12, wm3/8)  (Eq. 8; reading A2)."""
    ws1, ws2, ws3, wm0, wm1, wm2, wm3 = w7
    return wm0, wm1 / 6.0, wm2 / 12.0, wm3 / 8.0


def radicand(w7, G, theta, phi):
    """R = ws1(3−C) + (ws2/3)(6−C−B) + (2 ws3/4)(3−3A+B−C)."""
    A, B, C = abc(G, theta, phi)
    ws1, ws2, ws3 = w7[0], w7[1], w7[2]
    return ws1 * (3.0 - C) + ws2 / 3.0 * (6.0 - C - B) + 2.0 * ws3 / 4.0 * (3.0 - 3.0 * A + B - C)


def J_factor(w7, G, theta, phi):
    """J = mu0 + 2 mu1 C + 4 mu2 B + 8 mu3 A with per-point mass weights (reading A2)."""
    A, B, C = abc(G, theta, phi)
    mu0, mu1, mu2, mu3 = per_point_mass(w7)
    return mu0 + 2.0 * mu1 * C + 4.0 * mu2 * B + 8.0 * mu3 * A


def vtilde(w7, G, theta, phi):
    """Normalised numerical phase velocity ṽ = G/(√(2J) π) · √R   (Eq. `vtilde`)."""
    G = np.asarray(G, dtype=np.float64)
    R = radicand(w7, G, theta, phi)
    J = J_factor(w7, G, theta, phi)
    return G / (np.sqrt(2.0 * J) * np.pi) * np.sqrt(R)


def h_row(G, theta, phi):
    """Linearised ṽ = 1 condition Σ H_l w_l = g  (Eq. `linear_basic`).

    Returns (H1, H2, H3, H4, H5, g) for unknowns (ws1, ws2, mu0, mu1, mu2).
    H2 carries the "+1" missing from the printed P:155 (reading A1):
        H2 = ½(1 + 3A − 5B/3 + C/3);
    all other entries are exactly as printed.
    """
    A, B, C = abc(G, theta, phi)
    G = np.asarray(G, dtype=np.float64)
    k = 2.0 * np.pi ** 2 / G ** 2
    H1 = 0.5 * (3.0 + 3.0 * A - B - C)
    H2 = 0.5 * (1.0 + 3.0 * A - 5.0 / 3.0 * B + 1.0 / 3.0 * C)
    H3 = k * (A - 1.0)
    H4 = k * (6.0 * A - 2.0 * C)
    H5 = k * (12.0 * A - 4.0 * B)
    g = 0.5 * ((4.0 * np.pi ** 2 / G ** 2 + 3.0) * A - B + C - 3.0)
    return H1, H2, H3, H4, H5, g


def angle_grid(thetas_deg=None, phis_deg=None):
    """LS angle grid, φ outer and θ inner; default {0,10,20,30,40}° each (reading A10,
    Fig. 2 caption P:244 "between 0 and 45° with a step of 10°")."""
    if thetas_deg is None:
        thetas_deg = [0.0, 10.0, 20.0, 30.0, 40.0]
    if phis_deg is None:
        phis_deg = [0.0, 10.0, 20.0, 30.0, 40.0]
    th, ph = [], []
    for p in phis_deg:          # outer
        for t in thetas_deg:    # inner
            th.append(np.deg2rad(t))
            ph.append(np.deg2rad(p))
    return np.array(th), np.array(ph)


def max_dispersion_error(w7, G, n_theta=19, n_phi=10):
    """max over θ ∈ [0, 90°], φ ∈ [0, 45°] of |ṽ − 1| (evaluation grid finer than the LS grid,
    reading A10: the text's θ ∈ [0, π/2], φ ∈ [0, π/4])."""
    th = np.deg2rad(np.linspace(0.0, 90.0, n_theta))
    ph = np.deg2rad(np.linspace(0.0, 45.0, n_phi))
    T, P = np.meshgrid(th, ph, indexing="ij")
    return float(np.max(np.abs(vtilde(w7, G, T, P) - 1.0)))
