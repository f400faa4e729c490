"""Pins for oracle/dispersion.py against closed forms, worked examples and invariants."""
import numpy as np
import pytest

from conftest import read_golden
from oracle import dispersion as d
from oracle import weights

W7_7PT = (1.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0)


def random_w7(rng, n=1):
    u5 = rng.uniform(-0.5, 1.0, size=(n, 5)) * np.array([1, 1, 1, 0.2, 0.1])
    return weights.u5_to_w7(u5)


def test_abc_worked_examples():
    # P:136-143 at G=4, theta=phi=0: cos(pi/2)=0, cos 0 = 1
    A, B, C = d.abc(4.0, 0.0, 0.0)
    assert abs(A) < 1e-15 and abs(B - 1) < 1e-15 and abs(C - 2) < 1e-15
    A, B, C = d.abc(4.0, np.pi / 2, 0.0)          # axis permutation
    assert abs(A) < 1e-15 and abs(B - 1) < 1e-15 and abs(C - 2) < 1e-15
    A, B, C = d.abc(1e12, 0.3, 0.2)               # 1/G -> 0 limit
    assert np.allclose([A, B, C], [1, 3, 3], atol=1e-12)


def test_vtilde_7pt_closed_form():
    for G, ref in read_golden("vtilde_7pt.txt"):
        G, ref = float(G), float(ref)
        assert abs(d.vtilde(W7_7PT, G, 0.0, 0.0) - ref) < 1e-13
        # the closed form itself, independent of the golden file
        assert abs(ref - G / np.pi * np.sin(np.pi / G)) < 1e-13


def test_vtilde_continuum_limit_and_symmetry(rng):
    for w7 in random_w7(rng, 20):
        th, ph = d.angle_grid()
        assert np.max(np.abs(d.vtilde(w7, 1e4, th, ph) - 1.0)) < 1e-6
        t = rng.uniform(0, np.pi / 2, 7)
        a = d.vtilde(w7, 7.3, t, 0.0)
        b = d.vtilde(w7, 7.3, np.pi / 2 - t, 0.0)
        assert np.max(np.abs(a - b)) < 1e-12


def test_h_row_worked_example():
    for row in read_golden("h_row_worked.txt"):
        G, th, ph = (float(x) for x in row[:3])
        ref = np.array([float(x) for x in row[3:]])
        got = np.array(d.h_row(G, np.deg2rad(th), np.deg2rad(ph)))
        assert np.max(np.abs(got - ref)) < 1e-12


def test_h_row_is_the_linearisation_of_vtilde(rng):
    """Σ H_l w_l − g must equal R(w) − (2π²/G²) J(w) for EVERY weight vector (the derivation of
    P:146: ṽ = 1 ⇔ R = 2π²J/G², with ws3 and wm3 eliminated).  This pins all five H columns and g
    against the ṽ formula of P:133-135 (whose pieces are pinned by the assembly symbol test).
    The printed H2 of P:155 (without +1) fails this identity (reading A1)."""
    for _ in range(50):
        G = rng.uniform(3.0, 40.0)
        th, ph = rng.uniform(0, np.pi / 2), rng.uniform(0, np.pi / 4)
        u5 = rng.normal(size=5)
        w7 = weights.u5_to_w7(u5)
        H1, H2, H3, H4, H5, g = d.h_row(G, th, ph)
        lhs = H1 * u5[0] + H2 * u5[1] + H3 * u5[2] + H4 * u5[3] + H5 * u5[4] - g
        rhs = d.radicand(w7, G, th, ph) - 2 * np.pi ** 2 / G ** 2 * d.J_factor(w7, G, th, ph)
        assert abs(lhs - rhs) < 1e-12 * (1 + np.abs(u5).sum())
        A, B, C = d.abc(G, th, ph)
        H2_printed = 0.5 * (3 * A - 5 * B / 3 + C / 3)
        lhs_printed = lhs - H2 * u5[1] + H2_printed * u5[1]
        assert abs(u5[1]) < 1e-3 or abs(lhs_printed - rhs) > 1e-6


def test_vtilde_equals_one_iff_linear_row_satisfied(rng):
    """Choose ws2 so that the single row is satisfied; ṽ must then be exactly 1."""
    for _ in range(20):
        G = rng.uniform(4.0, 30.0)
        th, ph = rng.uniform(0, np.pi / 2), rng.uniform(0, np.pi / 4)
        u5 = rng.uniform(0.0, 0.2, size=5)
        H1, H2, H3, H4, H5, g = d.h_row(G, th, ph)
        u5[1] = (g - H1 * u5[0] - H3 * u5[2] - H4 * u5[3] - H5 * u5[4]) / H2
        assert abs(d.vtilde(weights.u5_to_w7(u5), G, th, ph) - 1.0) < 1e-10
