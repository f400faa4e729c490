"""Linear solves of A p = s — ORACLE (test infrastructure only).

The paper factorises A with the MUMPS multifrontal LU.  The north star replaces that by
a batched BiCGSTAB (BASELINE.json north_star (3)); the oracle provides:
  * dense LAPACK solve for tiny grids (brute force, ≤ 9³),
  * scipy SuperLU (a sparse direct solve, the paper's setting in spirit),
  * a plain complex128 BiCGSTAB written out step by step (van der Vorst 1992),
    with the convergence test on the recomputed true residual ‖b − Ax‖/‖b‖.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def solve_dense(A: sp.spmatrix, b: np.ndarray) -> np.ndarray:
    return np.linalg.solve(A.toarray(), b)


def solve_splu(A: sp.spmatrix, b: np.ndarray) -> np.ndarray:
    lu = spla.splu(sp.csc_matrix(A))
    return lu.solve(b)


def bicgstab(A, b, x0=None, rtol=1e-10, max_iter=20000, replace_every=50):
    """Unpreconditioned BiCGSTAB, complex128, inner product (a, b) = aᴴ b.

    Per iteration:
      v = A p;  α = ρ / (r̂0, v);  s = r − α v;  t = A s;  ω = (t, s)/(t, t);
      x ← x + α p + ω s;  r ← s − ω t;  ρ' = (r̂0, r);  β = (ρ'/ρ)(α/ω);  p ← r + β (p − ω v).
    Every `replace_every` iterations r is replaced by b − A x (residual replacement).
    Converged when the TRUE relative residual ‖b − Ax‖/‖b‖ ≤ rtol.
    Returns (x, relres_true, iterations).
    """
    b = np.asarray(b, dtype=np.complex128)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.complex128)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b), 0.0, 0
    r = b - A @ x
    rhat = r.copy()
    p = r.copy()
    rho = np.vdot(rhat, r)
    it = 0
    while it < max_iter:
        v = A @ p
        den = np.vdot(rhat, v)
        if den == 0:
            break
        alpha = rho / den
        s = r - alpha * v
        t = A @ s
        tt = np.vdot(t, t)
        omega = np.vdot(t, s) / tt if tt != 0 else 0.0
        x = x + alpha * p + omega * s
        r = s - omega * t
        it += 1
        if it % replace_every == 0:
            r = b - A @ x
        rn = np.linalg.norm(r) / nb
        if rn <= rtol:
            true = np.linalg.norm(b - A @ x) / nb
            if true <= rtol:
                return x, true, it
            r = b - A @ x
        rho_new = np.vdot(rhat, r)
        if rho_new == 0 or omega == 0:
            # breakdown: restart with r̂0 = r
            rhat = r.copy()
            p = r.copy()
            rho = np.vdot(rhat, r)
            continue
        beta = (rho_new / rho) * (alpha / omega)
        p = r + beta * (p - omega * v)
        rho = rho_new
    return x, np.linalg.norm(b - A @ x) / nb, it


def bicgstab_l(A, b, ell=2, x0=None, rtol=1e-10, max_iter=20000):
    """Unpreconditioned BiCGStab(ℓ) (Sleijpen & Fokkema 1993), complex128, (a, b) = aᴴ b — the
    algorithm of hz_solve_opts.ell = 2 (reading A23), written out for any ℓ ≥ 1.

    Per outer step (r̂0 = r at the start; ρ0 = α = ω = 1, α = 0 initially):
      ρ0 ← −ω ρ0
      for j = 0..ℓ−1 (BiCG part):
        ρ1 = (r̂0, r_j);  β = α ρ1/ρ0;  ρ0 ← ρ1
        u_i ← r_i − β u_i  (i = 0..j);   u_{j+1} = A u_j
        α = ρ0 / (r̂0, u_{j+1})
        r_i ← r_i − α u_{i+1}  (i = 0..j);   r_{j+1} = A r_j;   x ← x + α u_0
      MR part: γ = argmin ‖r_0 − Σ_{k=1..ℓ} γ_k r_k‖ (normal equations, lstsq here);
        x ← x + Σ γ_k r_{k−1};  r_0 ← r_0 − Σ γ_k r_k;  u_0 ← u_0 − Σ γ_k u_k;  ω = γ_ℓ.
    One outer step applies A 2ℓ times and counts as ℓ BiCGSTAB iterations.  Converged when the TRUE
    relative residual ‖b − Ax‖/‖b‖ ≤ rtol (checked after every outer step).
    Returns (x, relres_true, iterations).
    """
    b = np.asarray(b, dtype=np.complex128)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.complex128)
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return np.zeros_like(b), 0.0, 0
    r = [b - A @ x] + [None] * ell
    u = [np.zeros_like(b)] + [None] * ell
    rhat = r[0].copy()
    rho0, alpha, omega = 1.0 + 0j, 0.0 + 0j, 1.0 + 0j
    it = 0
    while it < max_iter:
        rho0 = -omega * rho0
        for j in range(ell):
            rho1 = np.vdot(rhat, r[j])
            beta = alpha * rho1 / rho0
            rho0 = rho1
            for i in range(j + 1):
                u[i] = r[i] - beta * u[i]
            u[j + 1] = A @ u[j]
            alpha = rho0 / np.vdot(rhat, u[j + 1])
            for i in range(j + 1):
                r[i] = r[i] - alpha * u[i + 1]
            r[j + 1] = A @ r[j]
            x = x + alpha * u[0]
        R = np.stack(r[1:], axis=1)
        gamma = np.linalg.lstsq(R, r[0], rcond=None)[0]
        for k in range(1, ell + 1):
            x = x + gamma[k - 1] * r[k - 1]
        r[0] = r[0] - R @ gamma
        u[0] = u[0] - np.stack(u[1:], axis=1) @ gamma
        omega = gamma[-1]
        it += ell
        true = np.linalg.norm(b - A @ x) / nb
        if true <= rtol:
            return x, true, it
    return x, np.linalg.norm(b - A @ x) / nb, it
