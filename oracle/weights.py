"""Weight estimation by dispersion minimisation — ORACLE (test infrastructure only).

Follows PAPER.md P:161-237:
  * `eq_cost`: one weight vector for a set of G values — N_G = 1 gives the paper's
    "G4" weights, N_G = 4 with G = 4, 6, 8, 10 gives "Gm";
  * `eq_cost_fun` with the Tikhonov-regularised block problem
    min ‖H w − g‖² + λ‖L w‖², L = D P: the adaptive table.

Readings: A1 (H2 corrected, via dispersion.h_row), A2 (unknowns are
(ws1, ws2, mu0, mu1, mu2) with per-point mass weights), A10 (angles {0..40°}², φ outer),
A11 (λ = 1e-2, D = first differences with no boundary rows), A12 (G ∈ [4, 40], ΔG = 0.1),
A14 (a single-G block has rank 3: G4 is the minimum-norm LS solution).

The least-squares solves are plain `numpy.linalg.lstsq` on the explicitly stacked matrix — no
normal equations, no block elimination.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dispersion import angle_grid, h_row


def u5_to_w7(u5):
    """(ws1, ws2, mu0, mu1, mu2) → class weights (ws1, ws2, ws3, wm0, wm1, wm2, wm3).

    ws3 = 1 − ws1 − ws2, wm0 = mu0, wm1 = 6 mu1, wm2 = 12 mu2 (reading A2),
    wm3 = 1 − wm0 − wm1 − wm2.  Works on [..., 5] arrays.
    """
    u5 = np.asarray(u5, dtype=np.float64)
    ws1, ws2, mu0, mu1, mu2 = (u5[..., i] for i in range(5))
    ws3 = 1.0 - ws1 - ws2
    wm0, wm1, wm2 = mu0, 6.0 * mu1, 12.0 * mu2
    wm3 = 1.0 - wm0 - wm1 - wm2
    return np.stack([ws1, ws2, ws3, wm0, wm1, wm2, wm3], axis=-1)


def block(G, thetas=None, phis=None):
    """H^(i) (n_angles × 5) and g^(i) for one G, rows ordered φ outer / θ inner."""
    if thetas is None:
        thetas, phis = angle_grid()
    rows = np.array(h_row(G, thetas, phis))        # 6 × n_angles
    return rows[:5].T.copy(), rows[5].copy()


@dataclass
class WeightTable:
    g_min: float
    dg: float
    G: np.ndarray        # [n_g]
    u5: np.ndarray       # [n_g][5]  (ws1, ws2, mu0, mu1, mu2)
    lam: float

    @property
    def n_g(self):
        return len(self.G)

    @property
    def w7(self):
        return u5_to_w7(self.u5)


def n_table(g_min, g_max, dg):
    return int(round((g_max - g_min) / dg)) + 1


def build_adaptive_table(g_min=4.0, g_max=40.0, dg=0.1, lam=1e-2, thetas=None, phis=None):
    """The adaptive (GA) table: stacked block-diagonal H over N_G tabulated G,
    augmented with √λ·L, L = D P, solved as one least-squares problem."""
    n_g = n_table(g_min, g_max, dg)
    Gs = g_min + dg * np.arange(n_g)
    blocks = [block(G, thetas, phis) for G in Gs]
    na = blocks[0][0].shape[0]
    nw = 5
    H = np.zeros((n_g * na, n_g * nw))
    g = np.zeros(n_g * na)
    for i, (Hi, gi) in enumerate(blocks):
        H[i * na:(i + 1) * na, i * nw:(i + 1) * nw] = Hi
        g[i * na:(i + 1) * na] = gi
    # L = D P: P gathers weight l over all G contiguously; D = first differences
    # along G with no boundary rows (reading A11).  Row (l, r): −w_l^(r) + w_l^(r+1).
    L = np.zeros((nw * (n_g - 1), n_g * nw))
    for l in range(nw):
        for r in range(n_g - 1):
            L[l * (n_g - 1) + r, r * nw + l] = -1.0
            L[l * (n_g - 1) + r, (r + 1) * nw + l] = 1.0
    M = np.vstack([H, np.sqrt(lam) * L])
    rhs = np.concatenate([g, np.zeros(L.shape[0])])
    w, *_ = np.linalg.lstsq(M, rhs, rcond=None)
    return WeightTable(float(g_min), float(dg), Gs, w.reshape(n_g, nw), float(lam))


def solve_joint(Gs, thetas=None, phis=None):
    """One weight vector minimising `eq_cost` over the listed G values.

    N_G = 1 at G = 4 is rank-deficient (rank 3, reading A14): numpy's lstsq returns the
    minimum-norm minimiser, which is the convention adopted for "G4".
    """
    Hs, gs = zip(*[block(G, thetas, phis) for G in Gs])
    H = np.vstack(Hs)
    g = np.concatenate(gs)
    w, *_ = np.linalg.lstsq(H, g, rcond=None)
    return w


def g4_weights():
    """Non-adaptive "G4" weights: eq_cost with N_G = 1, G = 4, min-norm (A14)."""
    return solve_joint([4.0])


def gm_weights():
    """Non-adaptive "Gm" weights: eq_cost with N_G = 4, G = 4, 6, 8, 10."""
    return solve_joint([4.0, 6.0, 8.0, 10.0])


def lookup(table: WeightTable, G):
    """Weights at local G: clamp to [g_min, g_max], linear interpolation in G between
    tabulated rows (north star "lookup and interpolation"; reading A13).  Returns
    (u5 [..., 5], clamped mask).  A 1-row table returns its row everywhere."""
    G = np.asarray(G, dtype=np.float64)
    if table.n_g == 1:
        u = np.broadcast_to(table.u5[0], G.shape + (5,)).copy()
        return u, np.zeros(G.shape, dtype=bool)
    g_max = table.g_min + table.dg * (table.n_g - 1)
    clamped = (G < table.g_min) | (G > g_max)
    Gc = np.clip(G, table.g_min, g_max)
    s = (Gc - table.g_min) / table.dg
    i = np.minimum(np.floor(s).astype(np.int64), table.n_g - 2)
    tau = s - i
    u = (1.0 - tau)[..., None] * table.u5[i] + tau[..., None] * table.u5[i + 1]
    return u, clamped
