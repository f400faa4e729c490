"""Per-point coefficients, PML, explicit impedance matrix and RHS — ORACLE (test infrastructure).

Follows PAPER.md §2.1 and the adaptive rule of P:36/P:51/P:273/P:446:

  [M + S] p = s
  S = ws1 S1 + (ws2/3) Σ S2,i + (ws3/4) Σ S3,i
  M: ω²/κ p ⟹ ω² (wm0 p0/κ0 + wm1/6 Σ6 p/κ + wm2/12 Σ12 p/κ + wm3/8 Σ8 p/κ)   (Eq. 8)
  GA: each row uses the weights tabulated at its local G = v/(f h)
  GAm: each row uses the mean of the weights tabulated at its 27 stencil nodes (reading A19)

with κ = v² (ρ = 1; reading A17) and the PML stretching ∂x̃ = ξx⁻¹ ∂x, ξ = 1 + iγ/ω.

Visco-acoustic, variable density (NEXT-2; Eqs. 1.1-1.4 and 2): Problem(b=…, Q=…) gives
  ω²/κ p + Σ_a ∂_a b ∂_a p = s,   κ = v_c²/b,  v_c = v (1 − i/(2Q))            (reading A24)
with the per-axis D_a b-weighted at the staggered midpoints: on the stencil line through the
transverse neighbour (p, q) of row n the edge buoyancy is the mean of the row line's and that line's
edge values, each the mean of its two end nodes (reading A25).  b = None, Q = None is the ρ = 1
elastic operator above, computed by the original expressions.

Readings: A4 (Eq. 8's p0 is p0/κ0), A5 (Eq. 8 is the default mass;
Eq. "10" collocation mass available as mass="colloc"), A6 (stiffness in per-axis form
S = Σ_a D2_a ⊗ T_a with t0 = ws1 + ⅔ws2 + ½ws3, t1 = ws2/12, t2 = ws3/8 — the unique
cubic-symmetric 27-point stencil whose symbol is the radicand of P:133), A7 (γ profile),
A8 (PML stretches only the 1-D second difference along each axis; T and the mass are not
stretched), A9 (Dirichlet behind the PML), A13 (lookup = clamped linear interpolation in G),
A15 (consistent point source), A16 (A p = +s), A18 (dims include the PML).

The matrix is assembled explicitly, entry by entry over the 27 offsets: no class sums, no
factorisation, no fusion.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp

from .weights import WeightTable, lookup, u5_to_w7

OFFSETS = [(dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]


def mass_class(d):
    """Class of an offset: number of non-zero components (0 centre, 1 face, 2 edge, 3 corner),
    Fig. 1d."""
    return sum(1 for c in d if c != 0)


def T_weight(p, q, t0, t1, t2):
    """Transverse weight T(p, q) of the per-axis stiffness form (reading A6):
    t0 at the centre, t1 on the 4 transverse faces, t2 on the 4 transverse corners."""
    if p == 0 and q == 0:
        return t0
    if abs(p) + abs(q) == 1:
        return t1
    return t2


@dataclass
class PointCoefficients:
    G: np.ndarray
    clamped: np.ndarray
    w7: np.ndarray           # [..., 7] class weights at each point
    t0: np.ndarray
    t1: np.ndarray
    t2: np.ndarray
    mu: np.ndarray           # [..., 4] per-point mass weights (wm0, wm1/6, wm2/12, wm3/8)
    k2: np.ndarray           # (ω / v)²


def average_27(u5):
    """GAm ("average weights, the averaging being performed over the 27 points"; reading A19):
    the weight vector of row n is the arithmetic mean of the weight vectors looked up at the row's
    27 stencil nodes, over the nodes that lie inside the grid (a node on a face / edge / corner of the
    grid averages 18 / 12 / 8 vectors).  The free weights (ws1, ws2, μ0, μ1, μ2) are averaged; the
    dependent ones follow from the sum constraints, so the mean satisfies them exactly (the
    renormalisation of SPEC S:280 is then the identity)."""
    nz, ny, nx = u5.shape[:3]
    acc = np.zeros_like(u5)
    cnt = np.zeros((nz, ny, nx))
    for dz, dy, dx in OFFSETS:
        # rows n whose neighbour n + d is in the grid
        zs = slice(max(0, -dz), nz - max(0, dz))
        ys = slice(max(0, -dy), ny - max(0, dy))
        xs = slice(max(0, -dx), nx - max(0, dx))
        zn = slice(max(0, dz), nz - max(0, -dz))
        yn = slice(max(0, dy), ny - max(0, -dy))
        xn = slice(max(0, dx), nx - max(0, -dx))
        acc[zs, ys, xs] += u5[zn, yn, xn]
        cnt[zs, ys, xs] += 1.0
    return acc / cnt[..., None]


def point_coefficients(v, freq, h, table: WeightTable, rule: str = "GA") -> PointCoefficients:
    """a2–a5: local G = v/(f h) (Table 1), clamped lookup + linear
    interpolation of the adaptive weights (A13) — per point ("GA") or averaged over the
    row's 27 stencil nodes ("GAm", `average_27`) — stiffness transverse weights t0, t1, t2
    (A6), per-point mass weights (A2) and k² = (2πf/v)²."""
    v = np.asarray(v, dtype=np.float64)
    G = v / (freq * h)
    u5, clamped = lookup(table, G)
    if rule == "GAm":
        u5 = average_27(u5)
    elif rule != "GA":
        raise ValueError(f"unknown weight rule {rule!r}")
    w7 = u5_to_w7(u5)
    ws1, ws2, ws3 = w7[..., 0], w7[..., 1], w7[..., 2]
    t0 = ws1 + 2.0 / 3.0 * ws2 + 0.5 * ws3
    t1 = ws2 / 12.0
    t2 = ws3 / 8.0
    mu = np.stack([w7[..., 3], w7[..., 4] / 6.0, w7[..., 5] / 12.0, w7[..., 6] / 8.0], axis=-1)
    k2 = (2.0 * np.pi * freq / v) ** 2
    return PointCoefficients(G, clamped, w7, t0, t1, t2, mu, k2)


def pml_gamma(s, n, npml, h, v_pml, r_coeff=1e-3):
    """Damping γ at continuous index s along an axis of n nodes (reading A7):
    γ(d) = (3 v_pml / (2L)) ln(1/R) (d/L)², L = npml h, d = h·max(0, npml − s, s − (n−1−npml))."""
    s = np.asarray(s, dtype=np.float64)
    if npml <= 0:
        return np.zeros_like(s)
    L = npml * h
    d = h * np.maximum(0.0, np.maximum(npml - s, s - (n - 1 - npml)))
    return 1.5 * v_pml / L * np.log(1.0 / r_coeff) * (d / L) ** 2


def pml_axis(n, npml, h, omega, v_pml, r_coeff=1e-3):
    """1-D stretched second-difference coefficients of one axis (readings A7, A8):
    ξ(s) = 1 + iγ(s)/ω;  a⁻(i) = 1/(h² ξ(i) ξ(i−½)),  a⁺(i) = 1/(h² ξ(i) ξ(i+½))."""
    i = np.arange(n, dtype=np.float64)
    xi = lambda s: 1.0 + 1j * pml_gamma(s, n, npml, h, v_pml, r_coeff) / omega  # noqa: E731
    am = 1.0 / (h * h * xi(i) * xi(i - 0.5))
    ap = 1.0 / (h * h * xi(i) * xi(i + 0.5))
    return am, ap


@dataclass
class Problem:
    v: np.ndarray            # [nz][ny][nx] velocity (m/s), including the PML pad (A18)
    h: float
    freq: float
    npml: int
    table: WeightTable
    r_coeff: float = 1e-3
    v_pml: Optional[float] = None     # None → max(v) (reading A7)
    mass: str = "eq8"                 # "eq8" (default A5) | "colloc"
    rule: str = "GA"                  # "GA" (row's own weights) | "GAm" (27-point mean, A19)
    b: Optional[np.ndarray] = None    # buoyancy 1/ρ per node (Eq. 2), None → 1 (A17)
    Q: Optional[object] = None        # quality factor per node or scalar (visco-acoustic κ, A24), None → ∞

    @property
    def omega(self):
        return 2.0 * np.pi * self.freq

    @property
    def shape(self):
        return self.v.shape

    def coefficients(self) -> PointCoefficients:
        return point_coefficients(self.v, self.freq, self.h, self.table, self.rule)

    def kappa(self):
        """Bulk modulus per node: v² (b = None, Q = None: the ρ = 1 operator, A17), else
        κ = v_c²/b with the complex velocity v_c = v (1 − i/(2Q)) (reading A24; e^{−iωt}, so
        Im k = Im(ω/v_c) > 0 attenuates)."""
        if self.b is None and self.Q is None:
            return self.v ** 2
        vc = self.v if self.Q is None else self.v * (1.0 - 0.5j / np.asarray(self.Q, dtype=np.float64))
        kap = vc ** 2 / (1.0 if self.b is None else self.b)
        if np.iscomplexobj(kap) and not np.any(kap.imag):   # Q = ∞ everywhere: κ is real
            kap = kap.real
        return kap

    def pml(self):
        vp = float(np.max(self.v)) if self.v_pml is None else float(self.v_pml)
        nz, ny, nx = self.v.shape
        return (pml_axis(nx, self.npml, self.h, self.omega, vp, self.r_coeff),
                pml_axis(ny, self.npml, self.h, self.omega, vp, self.r_coeff),
                pml_axis(nz, self.npml, self.h, self.omega, vp, self.r_coeff))


def _entry(prob: Problem, coef: PointCoefficients, pml, K, J, I, d):
    """Value of A[n, n+d] for the nodes n = (K, J, I) (arrays) and one offset d = (dz, dy, dx):
         ω² mu_{class(d)}(w_n) / v²_{n+d}                                   (Eq. 8)
       + Σ_a D_a(n_a, d_a) · T(d_⊥1, d_⊥2; t(w_n))                          (readings A6, A8)
    with D_a(i, −1) = a⁻_a(i), D_a(i, +1) = a⁺_a(i), D_a(i, 0) = −a⁻_a(i) − a⁺_a(i).
    `coef` holds the row coefficients at the same nodes.  Also returns the in-grid mask."""
    dz, dy, dx = d
    v = prob.v
    nz, ny, nx = v.shape
    (amx, apx), (amy, apy), (amz, apz) = pml
    Dx = {-1: amx, 1: apx, 0: -amx - apx}
    Dy = {-1: amy, 1: apy, 0: -amy - apy}
    Dz = {-1: amz, 1: apz, 0: -amz - apz}
    kk, jj, ii = K + dz, J + dy, I + dx
    ok = (kk >= 0) & (kk < nz) & (jj >= 0) & (jj < ny) & (ii >= 0) & (ii < nx)
    c = mass_class(d)
    kk_c, jj_c, ii_c = np.clip(kk, 0, nz - 1), np.clip(jj, 0, ny - 1), np.clip(ii, 0, nx - 1)
    w2 = prob.omega ** 2
    kap = prob.kappa()
    if prob.mass == "eq8":
        mass = w2 * coef.mu[..., c] / kap[kk_c, jj_c, ii_c]
    elif prob.mass == "colloc":
        mass = w2 * coef.mu[..., c] / kap[K, J, I]          # Eq. "10", κ0 for all 27
    else:
        raise ValueError(prob.mass)
    if prob.b is None:
        stiff = (Dx[dx][I] * T_weight(dy, dz, coef.t0, coef.t1, coef.t2)
                 + Dy[dy][J] * T_weight(dx, dz, coef.t0, coef.t1, coef.t2)
                 + Dz[dz][K] * T_weight(dx, dy, coef.t0, coef.t1, coef.t2))
    else:
        bz = _b_weighted(prob, K, J, I, dz, (dz, dy, dx), 0, amz, apz)
        by = _b_weighted(prob, K, J, I, dy, (dz, dy, dx), 1, amy, apy)
        bx = _b_weighted(prob, K, J, I, dx, (dz, dy, dx), 2, amx, apx)
        stiff = (bx * T_weight(dy, dz, coef.t0, coef.t1, coef.t2)
                 + by * T_weight(dx, dz, coef.t0, coef.t1, coef.t2)
                 + bz * T_weight(dx, dy, coef.t0, coef.t1, coef.t2))
    return mass + stiff, ok, (kk, jj, ii)


def _b_at(b, K, J, I):
    """b at nodes (K, J, I), indices clamped into the grid (out-of-grid buoyancy = the nearest
    node's; only the centre coefficients of lines at the grid edge use it, reading A25)."""
    nz, ny, nx = b.shape
    return b[np.clip(K, 0, nz - 1), np.clip(J, 0, ny - 1), np.clip(I, 0, nx - 1)]


def _b_weighted(prob, K, J, I, da, d, axis, am, ap):
    """D_a(n, d_a) of the b-weighted second difference along axis a (0 = z, 1 = y, 2 = x) on the
    stencil line through the transverse neighbour n + d⊥ of row n (reading A25, Eq. 2):
        edge buoyancy of a line at node m:  b±(m) = (b(m) + b(m ± e_a)) / 2   (staggered midpoint)
        β± = (b±(n) + b±(n + d⊥)) / 2        (row line and transverse line averaged: A symmetric)
        D_a(n, −1) = β⁻ a⁻_a(n_a),  D_a(n, +1) = β⁺ a⁺_a(n_a),  D_a(n, 0) = −(β⁻ a⁻ + β⁺ a⁺)."""
    b = prob.b
    e = [0, 0, 0]
    e[axis] = 1
    t = list(d)
    t[axis] = 0                                        # transverse neighbour offset d⊥
    n_a = (K, J, I)[axis]

    def edge(sign, k, j, i):
        return 0.5 * (_b_at(b, k, j, i) + _b_at(b, k + sign * e[0], j + sign * e[1], i + sign * e[2]))
    beta_p = 0.5 * (edge(+1, K, J, I) + edge(+1, K + t[0], J + t[1], I + t[2]))
    beta_m = 0.5 * (edge(-1, K, J, I) + edge(-1, K + t[0], J + t[1], I + t[2]))
    if da == 1:
        return beta_p * ap[n_a]
    if da == -1:
        return beta_m * am[n_a]
    return -(beta_m * am[n_a] + beta_p * ap[n_a])


def assemble(prob: Problem, coef: Optional[PointCoefficients] = None) -> sp.csr_matrix:
    """Explicit sparse impedance matrix A = M + S, one row per node, ≤ 27 entries
    (values from `_entry`).  Out-of-grid neighbours are dropped (Dirichlet, A9).
    Node index n = (z·ny + y)·nx + x."""
    if coef is None:
        coef = prob.coefficients()
    nz, ny, nx = prob.v.shape
    N = nx * ny * nz
    pml = prob.pml()
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    rows_all, cols_all, vals_all = [], [], []
    n_idx = (K * ny + J) * nx + I
    for d in OFFSETS:
        val, ok, (kk, jj, ii) = _entry(prob, coef, pml, K, J, I, d)
        rows_all.append(n_idx[ok])
        cols_all.append(((kk * ny + jj) * nx + ii)[ok])
        vals_all.append(np.asarray(val)[ok])
    rows = np.concatenate(rows_all)
    cols = np.concatenate(cols_all)
    vals = np.concatenate(vals_all).astype(np.complex128)
    idx_t = np.int32 if len(vals) < 2 ** 31 - 1 else np.int64
    A = sp.csr_matrix((vals, (rows.astype(idx_t), cols.astype(idx_t))), shape=(N, N))
    A.sort_indices()
    return A


def apply_rows(prob: Problem, u: np.ndarray, nodes) -> np.ndarray:
    """(Au)_n for selected nodes only (sampled parity at sizes where the full matrix is too big):
    the same row entries as `assemble`, evaluated row by row.  u: [nz][ny][nx]; nodes: [m][3] as
    (x, y, z).  Returns [m] complex128."""
    nodes = np.asarray(nodes, dtype=np.int64).reshape(-1, 3)
    I, J, K = nodes[:, 0], nodes[:, 1], nodes[:, 2]
    coef = point_coefficients(prob.v[K, J, I], prob.freq, prob.h, prob.table)
    if prob.rule == "GAm":   # the 27-node mean at the selected rows only (same rule as average_27)
        nz, ny, nx = prob.v.shape
        acc = np.zeros((len(nodes), 5))
        cnt = np.zeros(len(nodes))
        for dz, dy, dx in OFFSETS:
            kk, jj, ii = K + dz, J + dy, I + dx
            ok = (kk >= 0) & (kk < nz) & (jj >= 0) & (jj < ny) & (ii >= 0) & (ii < nx)
            vv = prob.v[np.clip(kk, 0, nz - 1), np.clip(jj, 0, ny - 1), np.clip(ii, 0, nx - 1)]
            u5, _ = lookup(prob.table, vv / (prob.freq * prob.h))
            acc += np.where(ok[:, None], u5, 0.0)
            cnt += ok
        w7 = u5_to_w7(acc / cnt[:, None])
        coef.w7 = w7
        coef.t0 = w7[:, 0] + 2.0 / 3.0 * w7[:, 1] + 0.5 * w7[:, 2]
        coef.t1 = w7[:, 1] / 12.0
        coef.t2 = w7[:, 2] / 8.0
        coef.mu = np.stack([w7[:, 3], w7[:, 4] / 6.0, w7[:, 5] / 12.0, w7[:, 6] / 8.0], axis=-1)
    pml = prob.pml()
    nz, ny, nx = prob.v.shape
    out = np.zeros(len(nodes), dtype=np.complex128)
    for d in OFFSETS:
        val, ok, (kk, jj, ii) = _entry(prob, coef, pml, K, J, I, d)
        uu = u[np.clip(kk, 0, nz - 1), np.clip(jj, 0, ny - 1), np.clip(ii, 0, nx - 1)].astype(np.complex128)
        out += np.where(ok, val * uu, 0.0)
    return out


def apply(A: sp.csr_matrix, u: np.ndarray) -> np.ndarray:
    """Au for a field u [..., nz, ny, nx] (complex), by the explicit matrix."""
    shp = u.shape
    U = np.asarray(u, dtype=np.complex128).reshape(-1, A.shape[0])
    out = np.stack([A @ U[r] for r in range(U.shape[0])])
    return out.reshape(shp)


def point_sources(prob: Problem, nodes, amps=None, consistent=True, coef=None) -> np.ndarray:
    """RHS for point sources on grid nodes, s = Σ amp δ(x − x_s).

    consistent=True (reading A15): b_n = amp · mu_{class(n−s)}(w_n) / h³ for ‖n − s‖∞ ≤ 1,
    i.e. row n of the κ-free consistent-mass stencil applied to the nodal delta.
    consistent=False: the nodal delta amp/h³ at the source node (diagnostic).
    A source inside the PML is an error.  Returns [nsrc][nz][ny][nx].
    """
    nodes = np.asarray(nodes, dtype=np.int64).reshape(-1, 3)
    nsrc = len(nodes)
    if amps is None:
        amps = np.ones(nsrc, dtype=np.complex128)
    if coef is None and consistent:
        coef = prob.coefficients()
    nz, ny, nx = prob.v.shape
    p = prob.npml
    b = np.zeros((nsrc, nz, ny, nx), dtype=np.complex128)
    h3 = prob.h ** 3
    for s, ((x, y, z), a) in enumerate(zip(nodes, amps)):
        if not (p <= x < nx - p and p <= y < ny - p and p <= z < nz - p):
            raise ValueError(f"source {(x, y, z)} lies inside the PML")
        if not consistent:
            b[s, z, y, x] = a / h3
            continue
        for (dz, dy, dx) in OFFSETS:
            n = (z + dz, y + dy, x + dx)
            if 0 <= n[0] < nz and 0 <= n[1] < ny and 0 <= n[2] < nx:
                # row n, column s: offset from n to s is −d → same class
                b[s][n] = a * coef.mu[n][mass_class((dz, dy, dx))] / h3
    return b
