"""Pins for the oracle's solves against analytic wavefields (north-star checks 1 and 2) and for the
analytic formulas and the `eqerror` metric themselves."""
import numpy as np
import pytest

import synth
from oracle import analytic, dispersion as d, metrics, operator as op, solvers, weights


def grid_xyz(shape, npml, h):
    nz, ny, nx = shape
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return (I - npml) * h, (J - npml) * h, (K - npml) * h


def test_eqerror_properties(rng):
    """err(u, u) = 0, err(2u, u) = 2, invariant to a common positive scale and to the
    gain units."""
    u = rng.normal(size=(6, 7, 8)) + 1j * rng.normal(size=(6, 7, 8))
    W = rng.uniform(0.1, 3.0, size=u.shape)
    assert metrics.eqerror(u, u, W) == 0.0
    assert abs(metrics.eqerror(u, 2 * u, W) - 2.0) < 1e-14
    v = u + 0.1 * (rng.normal(size=u.shape) + 1j * rng.normal(size=u.shape))
    e = metrics.eqerror(u, v, W)
    assert abs(metrics.eqerror(3.7 * u, 3.7 * v, W) - e) < 1e-13
    assert abs(metrics.eqerror(u, v, 1000 * W) - e) < 1e-13


def test_gradient_formula_solves_the_pde():
    """App. E closed form: a 4th-order finite-difference Laplacian of the formula satisfies
    ∇²p + ω²/c(z)² p = 0 away from the source, and α → 0 recovers −e^{ikR}/(4πR)."""
    c0, alpha, omega = 1500.0, 0.7, 2 * np.pi * 5.0
    xs, ys, zs = 0.0, 0.0, 300.0
    e = 1.0
    for (x, y, z) in [(400.0, 100.0, 600.0), (-700.0, 250.0, 1500.0), (50.0, -900.0, 200.0)]:
        f = lambda X, Y, Z: analytic.gradient(X, Y, Z, xs, ys, zs, omega, c0, alpha)  # noqa
        lap = 0
        for dvec in [(1, 0, 0), (0, 1, 0), (0, 0, 1)]:
            pts = [f(x + k * e * dvec[0], y + k * e * dvec[1], z + k * e * dvec[2]) for k in (-2, -1, 0, 1, 2)]
            lap += (-pts[0] + 16 * pts[1] - 30 * pts[2] + 16 * pts[3] - pts[4]) / (12 * e * e)
        p = f(x, y, z)
        c = c0 + alpha * z
        res = lap + omega ** 2 / c ** 2 * p
        assert abs(res) <= 1e-6 * omega ** 2 / c ** 2 * abs(p)
    R = np.array([300.0, 1234.0])
    g = analytic.gradient(R, 0 * R, zs + 0 * R, xs, ys, zs, omega, 3000.0, 1e-6)
    h = analytic.homogeneous(R, omega / 3000.0)
    assert np.max(np.abs(g - h) / np.abs(h)) < 1e-5


def test_homogeneous_analytic_config1(ga_table):
    """North-star check 1 on BASELINE config 1 (41³, G = 12, consistent source, A15): GA err
    ≤ 5e-3 and GA err < Gm err / 5; the nodal-source diagnostic has amplitude ≈ 1/J(k0)."""
    c = synth.get_config(1)
    v = synth.velocity_model(c)
    src = synth.source_nodes(c)[0]
    D = metrics.distance(v.shape, src, c.h)
    m = metrics.interior_mask(v.shape, c.npml, src)
    k = 2 * np.pi * c.freq / 3000.0
    ref = analytic.homogeneous(np.where(D > 0, D, 1.0), k)
    errs = {}
    for name, tab in [("GA", ga_table),
                      ("Gm", weights.WeightTable(4.0, 0.1, np.array([4.0]), weights.gm_weights()[None], 0))]:
        P = op.Problem(v, c.h, c.freq, c.npml, tab)
        A = op.assemble(P)
        b = op.point_sources(P, [src])[0].ravel()
        x, rr, it = solvers.bicgstab(A, b, rtol=1e-8)
        assert rr <= 1e-8
        u = x.reshape(v.shape)
        errs[name] = metrics.eqerror(ref, u, D, m)
        if name == "GA":
            assert np.linalg.norm((ref - u)[m]) / np.linalg.norm(ref[m]) <= 5e-3
            bn = op.point_sources(P, [src], consistent=False)[0].ravel()
            xn, _, _ = solvers.bicgstab(A, bn, rtol=1e-8)
            ratio = np.median(np.abs(xn.reshape(v.shape)[m]) / np.abs(ref[m]))
            J = d.J_factor(tab.w7[int(round((12.0 - 4.0) / 0.1))], 12.0, 0.0, 0.0)
            assert abs(ratio * J - 1.0) <= 5e-3
    assert errs["GA"] <= 5e-3
    assert errs["GA"] < errs["Gm"] / 5


def _gradient_case(n, table):
    c = synth.get_config(2, nx=n, ny=n, nz=n)
    v = synth.velocity_model(c)
    src = np.array([n // 2, n // 2, c.npml + 2])
    P = op.Problem(v, c.h, c.freq, c.npml, table)
    A = op.assemble(P)
    b = op.point_sources(P, [src])[0].ravel()
    x, rr, it = solvers.bicgstab(A, b, rtol=1e-8)
    X, Y, Z = grid_xyz(v.shape, c.npml, c.h)
    xs, ys, zs = [(s - c.npml) * c.h for s in src]
    D = metrics.distance(v.shape, src, c.h)
    m = metrics.interior_mask(v.shape, c.npml, src)
    Xs = np.where(D > 0, X, X + 1.0)
    ref = analytic.gradient(Xs, Y, Z, xs, ys, zs, 2 * np.pi * c.freq, 1500.0, 0.7)
    return metrics.eqerror(ref, x.reshape(v.shape), D, m)


def test_gradient_analytic_reduced(ga_table):
    """North-star check 2 on a reduced config-2 analog (61³, same h, f and v(z) = 1500 + 0.7 z)."""
    assert _gradient_case(61, ga_table) <= 0.02


def test_gradient_ordering_ga_gm(ga_table):
    """Paper's Linear row ordering GA < Gm (Table 2), shrunk to a 31³ analog of config 2 (same
    h, f and v(z)) so that it runs in the default suite (~25 s): measured err 2.5e-3 (GA) vs 1.3e-2
    (Gm); the margin asserted is 3×."""
    gm = weights.WeightTable(4.0, 0.1, np.array([4.0]), weights.gm_weights()[None], 0)
    assert 3.0 * _gradient_case(31, ga_table) < _gradient_case(31, gm)


def _small_helmholtz(ga_table, seed=5, n=(12, 11, 10)):
    rng = np.random.default_rng(seed)
    v = rng.uniform(1500.0, 3500.0, n)
    P = op.Problem(v, 25.0, 5.0, 3, ga_table)
    A = op.assemble(P)
    b = op.point_sources(P, np.array([[5, 5, 4]]))[0].ravel()
    return A, b


def test_bicgstab_l1_is_bicgstab(ga_table):
    """BiCGStab(1) is BiCGSTAB (Sleijpen & Fokkema 1993, §3): the oracle's two independently written
    recurrences give the same iterates after 8 iterations (no residual replacement)."""
    A, b = _small_helmholtz(ga_table)
    x1, _, it1 = solvers.bicgstab(A, b, rtol=0.0, max_iter=8, replace_every=10 ** 9)
    xl, _, itl = solvers.bicgstab_l(A, b, ell=1, rtol=0.0, max_iter=8)
    assert it1 == itl == 8
    assert np.linalg.norm(x1 - xl) <= 1e-9 * np.linalg.norm(x1)


def test_bicgstab_l2_reaches_the_direct_solution(ga_table):
    """BiCGStab(2) converges to the sparse direct (LU) solution of a complex-symmetric, indefinite
    Helmholtz system with PML (random velocities)."""
    A, b = _small_helmholtz(ga_table)
    xd = solvers.solve_splu(A, b)
    x2, rel, it = solvers.bicgstab_l(A, b, ell=2, rtol=1e-10)
    assert rel <= 1e-10 and it % 2 == 0
    assert np.linalg.norm(x2 - xd) <= 1e-7 * np.linalg.norm(xd)
