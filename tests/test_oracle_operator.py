"""Pins for oracle/operator.py: plane-wave symbol equivalence with Eq. vtilde, textbook reductions,
structure (symmetry, reciprocity), brute force, the per-type stiffness decomposition, RHS and PML."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import dispersion as d
from oracle import operator as op
from oracle import solvers, weights


def one_row_table(u5):
    return weights.WeightTable(4.0, 0.1, np.array([4.0]), np.asarray(u5, float)[None, :], 0.0)


def homog_problem(n, u5, v=2000.0, f=5.0, h=20.0, npml=0, r_coeff=1e-3):
    return op.Problem(np.full((n, n, n), v), h, f, npml, one_row_table(u5), r_coeff=r_coeff)


def test_table1_local_G():
    """G = c/(f h) reproduces Table 1's G columns."""
    for name, cm, cM, f, h, gm, gM in read_golden("table1_G.txt"):
        Gm = float(cm) / (float(f) * float(h))
        GM = float(cM) / (float(f) * float(h))
        assert abs(Gm - float(gm)) <= 0.05 * float(gm), name
        assert abs(GM - float(gM)) <= 0.05 * float(gM), name
    c = op.point_coefficients(np.array([1500.0]), 7.5, 50.0, one_row_table([1, 0, 1, 0, 0]))
    assert c.G[0] == 4.0


def test_symbol_equivalence(rng):
    """Interior row on a plane wave: (Au)/u = (ω²/v²) J(k) − (2/h²) R(k) with J, R of P:133-135
    (SPEC S:269/S:490).  Ties the assembled matrix to the ṽ formula with no shared code."""
    n = 5
    for _ in range(25):
        u5 = rng.uniform(-0.5, 1.0, 5) * np.array([1, 1, 1, 0.2, 0.1])
        P = homog_problem(n, u5, v=rng.uniform(1500, 4000), f=rng.uniform(2, 10), h=25.0)
        A = op.assemble(P)
        G = rng.uniform(2.5, 30.0)
        th, ph = rng.uniform(0, np.pi / 2), rng.uniform(0, np.pi / 4)
        kx = 2 * np.pi * np.cos(ph) * np.cos(th) / (G * P.h)
        ky = 2 * np.pi * np.cos(ph) * np.sin(th) / (G * P.h)
        kz = 2 * np.pi * np.sin(ph) / (G * P.h)
        K, J, I = np.meshgrid(*(np.arange(n),) * 3, indexing="ij")
        u = np.exp(1j * P.h * (kx * I + ky * J + kz * K))
        Au = (A @ u.ravel()).reshape(u.shape)
        sym = Au[2, 2, 2] / u[2, 2, 2]
        w7 = weights.u5_to_w7(u5)
        ref = P.omega ** 2 / P.v[0, 0, 0] ** 2 * d.J_factor(w7, G, th, ph) \
            - 2.0 / P.h ** 2 * d.radicand(w7, G, th, ph)
        assert abs(sym - ref) <= 1e-12 * (abs(ref) + P.omega ** 2 / P.v[0, 0, 0] ** 2 + 6 / P.h ** 2)


def test_seven_point_reduction():
    """w = (1,0,0 | 1,0,0,0): the lumped 7-point Helmholtz row."""
    P = homog_problem(5, [1.0, 0.0, 1.0, 0.0, 0.0], v=2500.0, f=4.0, h=30.0)
    A = op.assemble(P).toarray()
    n = (2 * 5 + 2) * 5 + 2
    row = A[n].reshape(5, 5, 5)
    k2 = P.omega ** 2 / 2500.0 ** 2
    ref = np.zeros((5, 5, 5), complex)
    ref[2, 2, 2] = -6 / 30.0 ** 2 + k2
    for dz, dy, dx in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
        ref[2 + dz, 2 + dy, 2 + dx] = 1 / 30.0 ** 2
    assert np.max(np.abs(row - ref)) < 1e-15


def test_per_type_stiffness_decomposition(rng):
    """Interior class coefficients equal ws1·S1 + ws2·(⅓ΣS2) + ws3·(¼ΣS3).  S1 is the
    7-point cross; S2,x is the 11-point stencil of the 45° rotation about x: the x second
    difference plus the two (y,z) diagonal second differences at spacing h√2 (Fig. 1b);
    ¼ΣS3 is fixed by its symbol −(3 − 3A + B − C) (reading A6)."""
    h = 10.0
    S1 = np.zeros((3, 3, 3))
    for a in range(3):
        for s in (-1, 1):
            idx = [1, 1, 1]
            idx[a] += s
            S1[tuple(idx)] += 1
    S1[1, 1, 1] = -6
    S2 = np.zeros((3, 3, 3))
    for a in range(3):       # rotation about axis a
        b, c = [x for x in range(3) if x != a]
        for s in (-1, 1):
            idx = [1, 1, 1]
            idx[a] += s
            S2[tuple(idx)] += 1
        S2[1, 1, 1] -= 2
        for sb, sc in [(1, 1), (-1, -1), (1, -1), (-1, 1)]:
            idx = [1, 1, 1]
            idx[b] += sb
            idx[c] += sc
            S2[tuple(idx)] += 0.5   # diagonal spacing h√2 → 1/(2h²)
        S2[1, 1, 1] -= 2
    S2 /= 3.0
    S3 = np.zeros((3, 3, 3))
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                S3[dz + 1, dy + 1, dx + 1] = [-3.0, 0.5, -0.25, 0.375][op.mass_class((dz, dy, dx))]
    for _ in range(5):
        u5 = np.array([rng.uniform(-1, 1), rng.uniform(-1, 1), 1.0, 0.0, 0.0])
        P = homog_problem(5, u5, v=1e30, f=1.0, h=h)      # ω²/v² ≈ 0: stiffness only
        A = op.assemble(P).toarray()
        row = A[(2 * 5 + 2) * 5 + 2].reshape(5, 5, 5)[1:4, 1:4, 1:4].real
        w7 = weights.u5_to_w7(u5)
        ref = (w7[0] * S1 + w7[1] * S2 + w7[2] * S3) / h ** 2
        assert np.max(np.abs(row - ref)) < 1e-15


def test_constants_and_mass_sum(rng):
    """Stiffness annihilates constants and the mass weights sum to 1: on a
    homogeneous no-PML grid, interior rows of A·1 equal ω²/v²."""
    u5 = rng.uniform(-0.5, 1.0, 5) * np.array([1, 1, 1, 0.2, 0.1])
    P = homog_problem(6, u5, v=1800.0, f=3.0, h=15.0)
    A = op.assemble(P)
    r = (A @ np.ones(6 ** 3)).reshape(6, 6, 6)[1:5, 1:5, 1:5]
    assert np.max(np.abs(r - P.omega ** 2 / 1800.0 ** 2)) < 1e-15 + 1e-12 * P.omega ** 2 / 1800.0 ** 2


def test_pml_transparency_and_profile():
    """γ ≡ 0 (R = 1 ⇒ ln(1/R) = 0) gives a bit-identical matrix to the no-PML one; the
    profile vanishes in the interior and grows monotonically into the layer (reading A7)."""
    u5 = [0.2, 0.7, 0.65, 0.02, 0.012]
    A0 = op.assemble(homog_problem(7, u5, npml=0))
    A1 = op.assemble(homog_problem(7, u5, npml=2, r_coeff=1.0))
    assert (A0 != A1).nnz == 0
    g = op.pml_gamma(np.arange(0, 20, 0.5), 20, 5, 10.0, 3000.0)
    s = np.arange(0, 20, 0.5)
    assert np.all(g[(s >= 5) & (s <= 14)] == 0)
    assert np.all(np.diff(g[s <= 5]) < 0) and np.all(np.diff(g[s >= 14]) > 0)
    L = 50.0
    assert abs(g[0] - 1.5 * 3000.0 / L * np.log(1e3)) < 1e-9


def test_symmetry_no_pml_constant_v(rng):
    """North-star check 4a: without PML and with constant v, A = Aᵀ exactly."""
    u5 = rng.uniform(-0.5, 1.0, 5) * np.array([1, 1, 1, 0.2, 0.1])
    A = op.assemble(homog_problem(6, u5))
    assert abs(A - A.T).max() == 0


def test_reciprocity_homogeneous_with_pml(ga_table):
    """North-star check 4b: u_s(r) = u_r(s) for a homogeneous model with PML (GA weights)."""
    n = 25
    P = op.Problem(np.full((n, n, n), 3000.0), 50.0, 5.0, 8, ga_table)
    A = op.assemble(P)
    s, r = (9, 12, 10), (15, 11, 14)
    bs = op.point_sources(P, [s], consistent=False)[0].ravel()
    br = op.point_sources(P, [r], consistent=False)[0].ravel()
    us = solvers.solve_splu(A, bs).reshape(n, n, n)
    ur = solvers.solve_splu(A, br).reshape(n, n, n)
    a, b = us[r[2], r[1], r[0]], ur[s[2], s[1], s[0]]
    assert abs(a - b) / abs(a) <= 1e-5


def test_brute_force_dense_vs_sparse(ga_table):
    """North-star check 4c: on a 9³ grid the dense LAPACK solve, SuperLU and the oracle's BiCGSTAB agree."""
    n = 9
    rng = np.random.default_rng(7)
    v = rng.uniform(1500, 4000, (n, n, n))
    P = op.Problem(v, 20.0, 12.0, 2, ga_table)
    A = op.assemble(P)
    b = op.point_sources(P, [(4, 4, 4)])[0].ravel()
    xd = solvers.solve_dense(A, b)
    xs = solvers.solve_splu(A, b)
    xb, rr, it = solvers.bicgstab(A, b, rtol=1e-12)
    assert np.linalg.norm(xd - xs) / np.linalg.norm(xd) <= 1e-12
    assert np.linalg.norm(xd - xb) / np.linalg.norm(xd) <= 1e-9
    assert np.linalg.norm(A @ xd - b) / np.linalg.norm(b) <= 1e-12


def test_rhs_entries(ga_table):
    """Nodal source entry amp/h³ (1/50³ = 8e-6); the consistent source spreads
    mu_c(w_n)/h³ over the 27 neighbours so that its entries sum to amp/h³ on a homogeneous
    model (mass weights sum to 1); a source in the PML is rejected."""
    n = 21
    P = op.Problem(np.full((n, n, n), 3000.0), 50.0, 5.0, 8, ga_table)
    bn = op.point_sources(P, [(10, 10, 10)], consistent=False)[0]
    assert bn[10, 10, 10] == 8e-6 and np.count_nonzero(bn) == 1
    bc = op.point_sources(P, [(10, 10, 10)])[0]
    assert np.count_nonzero(bc) == 27
    assert abs(bc.sum() - 8e-6) < 1e-19
    with pytest.raises(ValueError):
        op.point_sources(P, [(3, 10, 10)])


def test_coefficient_identities(ga_table, rng):
    """t0 + 4 t1 + 4 t2 = ws1 + ws2 + ws3 = 1 and Σ_c N_c mu_c = 1 at every point (A2, A6)."""
    v = rng.uniform(1200.0, 9000.0, (4, 5, 6))
    c = op.point_coefficients(v, 6.0, 25.0, ga_table)
    assert np.max(np.abs(c.t0 + 4 * c.t1 + 4 * c.t2 - 1)) < 1e-14
    assert np.max(np.abs(c.mu @ np.array([1, 6, 12, 8]) - 1)) < 1e-14
    assert np.array_equal(c.clamped, (c.G < 4.0) | (c.G > 40.0 + 1e-9))


# ---- GAm: weights averaged over the 27 stencil points (reading A19) -------
def test_gam_equals_ga_on_homogeneous_models(ga_table):
    """all 27 local G are equal on a homogeneous model, so GAm = GA (to the rounding of a mean
    of 8–27 equal numbers), with and without PML."""
    v = np.full((7, 6, 8), 2600.0)
    for npml in (0, 2):
        A = op.assemble(op.Problem(v, 25.0, 7.0, npml, ga_table))
        B = op.assemble(op.Problem(v, 25.0, 7.0, npml, ga_table, rule="GAm"))
        assert abs(A - B).max() <= 1e-14 * abs(A).max()


def test_gam_of_affine_model_inside_one_table_interval(ga_table):
    """Closed form: within one table interval the interpolated weights are affine in G; for v affine
    in x, y and z the mean of an affine function over the symmetric 27-point neighbourhood is its
    value at the centre, so interior rows of GAm equal GA rows exactly (to rounding), while rows on the
    grid boundary (one-sided neighbourhoods) must differ."""
    nz, ny, nx = 6, 5, 7
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    h, f = 25.0, 7.0
    G0 = 12.03                                  # G range 12.03 .. 12.09: inside [12.0, 12.1]
    v = (G0 + 0.002 * x + 0.003 * y + 0.004 * z) * f * h
    cga = op.point_coefficients(v, f, h, ga_table, "GA")
    cgm = op.point_coefficients(v, f, h, ga_table, "GAm")
    inner = (slice(1, -1), slice(1, -1), slice(1, -1))
    assert np.allclose(cgm.w7[inner], cga.w7[inner], rtol=0, atol=1e-14)
    # boundary rows: the one-sided mean is the weight at the neighbourhood's centroid, not the node
    assert np.abs(cgm.w7[0, 2, 3] - cga.w7[0, 2, 3]).max() > 1e-7


def test_gam_sum_constraints_and_counts(ga_table, rng):
    """The mean keeps ws1+ws2+ws3 = 1 and Σwm = 1; a corner row averages its 8 in-grid
    nodes: on a model that is v1 at one corner node and v2 elsewhere, the corner row's weights are
    (w(v1) + 7 w(v2))/8 and the far corner's are w(v2)."""
    v = rng.uniform(1500.0, 4500.0, (5, 6, 7))
    c = op.point_coefficients(v, 7.0, 25.0, ga_table, "GAm")
    assert np.allclose(c.w7[..., :3].sum(-1), 1.0, atol=1e-14)
    assert np.allclose(c.w7[..., 3:].sum(-1), 1.0, atol=1e-14)
    v = np.full((4, 4, 4), 3000.0)
    v[0, 0, 0] = 2000.0
    c = op.point_coefficients(v, 7.0, 25.0, ga_table, "GAm")
    w1, _ = weights.lookup(ga_table, 2000.0 / 175.0)
    w2, _ = weights.lookup(ga_table, 3000.0 / 175.0)
    assert np.allclose(c.w7[0, 0, 0], weights.u5_to_w7((w1 + 7 * w2) / 8), atol=1e-14)
    assert np.allclose(c.w7[3, 3, 3], weights.u5_to_w7(w2), atol=1e-14)


def test_gam_row_evaluation_matches_assembly(ga_table, rng):
    """apply_rows (row-by-row, used for sampled parity) and the assembled GAm matrix agree."""
    v = rng.uniform(1500.0, 4500.0, (6, 7, 8))
    P = op.Problem(v, 25.0, 7.0, 2, ga_table, rule="GAm")
    u = rng.standard_normal(v.shape) + 1j * rng.standard_normal(v.shape)
    full = op.apply(op.assemble(P), u[None])[0]
    nodes = np.array([[0, 0, 0], [3, 4, 2], [7, 6, 5], [1, 6, 0], [4, 0, 3]])
    rows = op.apply_rows(P, u, nodes)
    assert np.allclose(rows, full[nodes[:, 2], nodes[:, 1], nodes[:, 0]], rtol=1e-13, atol=0)
