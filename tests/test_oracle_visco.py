"""Pins of the oracle's visco-acoustic, variable-density operator (NEXT-2; Eqs. 1.1-1.4 and 2,
P:64-78; readings A24, A25), each independent of the code it checks:

  * reductions: b ≡ 1 and Q = ∞ give the ρ = 1 elastic matrix BITWISE (the original expressions);
  * scaling: a constant b multiplies the whole operator (ω² b/v² and ∇·b∇) — exactly for b = 2;
  * symbol: on a homogeneous model with constant complex κ and constant b, A applied to a discrete
    plane wave is the closed-form symbol ω²/κ·M̂(k) + b·Σ_a (2cos k_a h − 2)/h² T̂_a(k) times the wave,
    written here from the stencil's definition (Eq. 8 classes, the per-axis form A6);
  * consistency: for smooth variable b the b-weighted stiffness converges to ∂_a(b ∂_a u) at second
    order (a staggered-midpoint slip — b at a node, a wrong line — drops the order to 1);
  * reciprocity: with constant weights and no PML the b-weighted stiffness is symmetric;
  * attenuation: the solved field of a homogeneous model with Q = 30 matches the analytic
    −e^{i k_c r}/(4π b r), k_c = ω/v_c, v_c = v(1 − i/(2Q)) (P:265's check with a complex velocity).
"""
import numpy as np
import pytest

import synth
from oracle import analytic, metrics, operator as op, solvers, weights


def one_row(table_u5):
    return weights.WeightTable(4.0, 0.1, np.array([4.0]), table_u5[None], 0)


@pytest.fixture(scope="module")
def model():
    rng = np.random.default_rng(2108)
    v = rng.uniform(1500.0, 4000.0, (9, 10, 11))
    b = rng.uniform(0.4, 1.1, v.shape)
    Q = rng.uniform(20.0, 200.0, v.shape)
    return v, b, Q


@pytest.mark.parametrize("mass", ["eq8", "colloc"])
def test_unit_buoyancy_and_infinite_q_are_the_elastic_matrix_bitwise(ga_table, model, mass):
    v, _, _ = model
    A0 = op.assemble(op.Problem(v, 25.0, 6.0, 3, ga_table, mass=mass))
    for kw in ({"b": np.ones_like(v)}, {"Q": np.inf}, {"b": np.ones_like(v), "Q": np.full(v.shape, np.inf)}):
        A = op.assemble(op.Problem(v, 25.0, 6.0, 3, ga_table, mass=mass, **kw))
        assert (A.indptr == A0.indptr).all() and (A.indices == A0.indices).all()
        assert np.array_equal(A.data, A0.data), kw


def test_constant_buoyancy_scales_the_operator(ga_table, model):
    v, _, Q = model
    A1 = op.assemble(op.Problem(v, 25.0, 6.0, 3, ga_table, b=np.ones_like(v), Q=Q))
    A2 = op.assemble(op.Problem(v, 25.0, 6.0, 3, ga_table, b=np.full(v.shape, 2.0), Q=Q))
    assert np.array_equal(A2.data, 2.0 * A1.data)                   # power of two: exact
    Ac = op.assemble(op.Problem(v, 25.0, 6.0, 3, ga_table, b=np.full(v.shape, 0.37), Q=Q))
    assert np.max(np.abs(Ac.data - 0.37 * A1.data)) <= 1e-15 * np.max(np.abs(A1.data))


def test_plane_wave_symbol_constant_complex_kappa(ga_table):
    """A e^{ik·x} = [ω²/κ M̂(k) + b Ŝ(k)] e^{ik·x} at rows whose 27 nodes are inside (npml = 0):
    M̂ = μ0 + 2μ1 Σc + 4μ2 Σcc + 8μ3 cx cy cz (Eq. 8 classes with μ = wm/(1, 6, 12, 8)),
    Ŝ = Σ_a (2c_a − 2)/h² (t0 + 2t1 (c_b + c_c) + 4t2 c_b c_c),  c_a = cos(k_a h)."""
    n, h, f, v0, Q0, b0 = 9, 20.0, 8.0, 2500.0, 25.0, 0.8
    v = np.full((n, n, n), v0)
    P = op.Problem(v, h, f, 0, ga_table, b=np.full(v.shape, b0), Q=Q0)
    A = op.assemble(P)
    coef = op.point_coefficients(np.array([v0]), f, h, ga_table)
    t0, t1, t2 = coef.t0[0], coef.t1[0], coef.t2[0]
    mu = coef.mu[0]
    mu3 = mu[3]
    kap = (v0 * (1 - 0.5j / Q0)) ** 2 / b0
    w = 2 * np.pi * f
    K, J, I = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    inner = (K > 0) & (K < n - 1) & (J > 0) & (J < n - 1) & (I > 0) & (I < n - 1)
    rng = np.random.default_rng(3)
    for _ in range(4):
        kx, ky, kz = rng.uniform(-np.pi / h, np.pi / h, 3)
        u = np.exp(1j * (kx * I + ky * J + kz * K) * h)
        cx, cy, cz = np.cos(kx * h), np.cos(ky * h), np.cos(kz * h)
        M = mu[0] + 2 * mu[1] * (cx + cy + cz) + 4 * mu[2] * (cx * cy + cy * cz + cx * cz) + 8 * mu3 * cx * cy * cz
        T = lambda a, c: t0 + 2 * t1 * (a + c) + 4 * t2 * a * c  # noqa: E731
        S = ((2 * cx - 2) * T(cy, cz) + (2 * cy - 2) * T(cx, cz) + (2 * cz - 2) * T(cx, cy)) / h ** 2
        sym = w ** 2 / kap * M + b0 * S
        Au = (A @ u.ravel()).reshape(u.shape)
        assert np.max(np.abs(Au[inner] - sym * u[inner])) <= 1e-12 * np.max(np.abs(sym * u[inner])) + 1e-18


def _stiffness(Pf1, Pf2, f1, f2):
    """S = A − M from two frequencies with a one-row table and npml = 0 (M ∝ ω², S ω-free)."""
    A1, A2 = op.assemble(Pf1), op.assemble(Pf2)
    return (f2 ** 2 * A1 - f1 ** 2 * A2) / (f2 ** 2 - f1 ** 2)


def test_variable_buoyancy_stiffness_is_second_order():
    """(S u)(n) → Σ_a ∂_a(b ∂_a u) at O(h²) for smooth b and u (Σ T(p, q) = 1): halving h divides the
    interior error by ≈ 4."""
    tab = one_row(weights.gm_weights())
    L = 1.0
    ub = lambda x, y, z: np.sin(2.1 * x + 0.3) * np.cos(1.7 * y) * np.sin(1.3 * z + 0.5)  # noqa: E731
    bb = lambda x, y, z: 1.0 + 0.4 * np.sin(1.9 * x + 0.7 * y) * np.cos(1.1 * z)         # noqa: E731

    def div_b_grad(x, y, z, e=1e-4):
        tot = 0.0
        for a in range(3):
            d = np.zeros(3)
            d[a] = e
            g = lambda X, Y, Z: bb(X, Y, Z) * (ub(X + d[0] / 2, Y + d[1] / 2, Z + d[2] / 2)  # noqa: E731
                                               - ub(X - d[0] / 2, Y - d[1] / 2, Z - d[2] / 2)) / e
            tot = tot + (g(x + d[0] / 2, y + d[1] / 2, z + d[2] / 2) - g(x - d[0] / 2, y - d[1] / 2, z - d[2] / 2)) / e
        return tot

    errs = []
    for n in (9, 17):
        h = L / (n - 1)
        K, J, I = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
        x, y, z = I * h, J * h, K * h
        v = np.full((n, n, n), 1.0)
        b = bb(x, y, z)
        S = _stiffness(op.Problem(v, h, 0.05, 0, tab, b=b), op.Problem(v, h, 0.1, 0, tab, b=b), 0.05, 0.1)
        Su = (S @ ub(x, y, z).ravel()).reshape(v.shape)
        m = (K >= 2) & (K <= n - 3) & (J >= 2) & (J <= n - 3) & (I >= 2) & (I <= n - 3)
        ex = div_b_grad(x, y, z)
        ctr = (np.abs(x - 0.5) < 1e-9) & (np.abs(y - 0.5) < 1e-9) & (np.abs(z - 0.5) < 1e-9)
        assert ctr.sum() == 1 and m[ctr].all()
        errs.append(np.max(np.abs(Su - ex)[ctr]))
    assert errs[0] / errs[1] > 3.3, errs


def test_variable_buoyancy_stiffness_is_symmetric(model):
    v, b, _ = model
    tab = one_row(weights.gm_weights())
    S = _stiffness(op.Problem(v, 25.0, 3.0, 0, tab, b=b), op.Problem(v, 25.0, 7.0, 0, tab, b=b), 3.0, 7.0)
    D = (S - S.T).tocoo()
    assert np.max(np.abs(D.data), initial=0.0) <= 1e-12 * np.max(np.abs(S.data))
    # the ρ = 1 part alone is symmetric too, and b enters: S(b) ≠ S(1)
    S1 = _stiffness(op.Problem(v, 25.0, 3.0, 0, tab), op.Problem(v, 25.0, 7.0, 0, tab), 3.0, 7.0)
    assert np.max(np.abs((S - S1).data)) > 1e-3 * np.max(np.abs(S1.data))


def test_attenuating_homogeneous_green_function(ga_table):
    """Config-1 model (41³, G = 12, 8-point PML) with Q = 30 and b = 0.5: the solved field matches
    −e^{i k_c r}/(4π b r), k_c = ω / (v (1 − i/(2Q))), within the elastic check's 5e-3 (relative L2
    outside the PML and a 2-cell source ball); a sign slip in Im κ or a dropped b fails it."""
    c = synth.get_config(1)
    v = synth.velocity_model(c)
    src = synth.source_nodes(c)[0]
    Q, b0 = 30.0, 0.5
    P = op.Problem(v, c.h, c.freq, c.npml, ga_table, b=np.full(v.shape, b0), Q=Q)
    A = op.assemble(P)
    rhs = op.point_sources(P, [src])[0].ravel()
    x, rr, it = solvers.bicgstab(A, rhs, rtol=1e-9)
    assert rr <= 1e-9
    u = x.reshape(v.shape)
    D = metrics.distance(v.shape, src, c.h)
    m = metrics.interior_mask(v.shape, c.npml, src)
    kc = 2 * np.pi * c.freq / (3000.0 * (1 - 0.5j / Q))
    ref = analytic.homogeneous(np.where(D > 0, D, 1.0), kc) / b0
    assert np.linalg.norm((ref - u)[m]) / np.linalg.norm(ref[m]) <= 5e-3
    # the attenuation is resolved by this check: the Q = ∞ field is 5e-3 away many times over
    ref_el = analytic.homogeneous(np.where(D > 0, D, 1.0), 2 * np.pi * c.freq / 3000.0) / b0
    assert np.linalg.norm((ref_el - u)[m]) / np.linalg.norm(ref_el[m]) > 4e-2
