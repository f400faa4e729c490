"""Pins of the CBS reference oracle (oracle/cbs.py, reading A26) against what the
mathematics fixes, independent of the oracle's own iteration:

* its fixed point equals a dense direct solve of the same spectral system (brute force, tiny box);
* in a homogeneous medium it reproduces the outgoing free-space Green's function −e^{ikr}/(4πr)
  (reading A16) away from the source, and not the incoming one;
* source/receiver reciprocity (the spectral Laplacian + diag(k²) is complex symmetric);
* the recomputed backward error reaches the paper's 1e-12 on a sharp two-layer contrast.
"""
import numpy as np
import pytest

from oracle import cbs


def dense_operator(box):
    """(∇²_spectral + diag(k²)) as a dense matrix, column by column from unit vectors."""
    shp = box.k2.shape
    N = box.k2.size
    L = np.zeros((N, N), dtype=np.complex128)
    for j in range(N):
        e = np.zeros(N, dtype=np.complex128)
        e[j] = 1.0
        L[:, j] = cbs.laplacian(e.reshape(shp), box.h).ravel()
    return L + np.diag(box.k2.ravel())


def test_fixed_point_equals_dense_solve():
    rng = np.random.default_rng(3)
    v = rng.uniform(1500.0, 3000.0, (4, 5, 3))
    box = cbs.box_k2(v, 7.0, 25.0, pad=2, absorb=1.0)
    s = cbs.point_source_box(box, [(1, 2, 1)])
    u, be, it, _ = cbs.cbs_solve(box, s, tol=1e-13, check_every=5)
    assert be <= 1e-13
    ud = np.linalg.solve(dense_operator(box), s.ravel()).reshape(box.k2.shape)
    assert np.linalg.norm(u - ud) / np.linalg.norm(ud) <= 1e-11


def homogeneous(n=16, pad=24):
    v = np.full((n, n, n), 3000.0)
    h, f = 50.0, 5.0                    # G = 12
    box = cbs.box_k2(v, f, h, pad=pad, absorb=1.0)
    src = (n // 2, n // 2, n // 2)
    u, be, it, _ = cbs.cbs_solve(box, cbs.point_source_box(box, [src]), tol=1e-10, check_every=25)
    um = cbs.model_region(box, u)
    K, J, I = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    r = h * np.sqrt((I - src[0]) ** 2 + (J - src[1]) ** 2 + (K - src[2]) ** 2)
    k = 2 * np.pi * f / 3000.0
    return um, r, k, h, be


def test_homogeneous_outgoing_greens_function():
    um, r, k, h, be = homogeneous()
    assert be <= 1e-10
    m = (r >= 4 * h) & (r <= 7 * h)
    out = -np.exp(1j * k * r[m]) / (4 * np.pi * r[m])
    inc = -np.exp(-1j * k * r[m]) / (4 * np.pi * r[m])
    e_out = np.linalg.norm(um[m] - out) / np.linalg.norm(out)
    e_inc = np.linalg.norm(um[m] - inc) / np.linalg.norm(inc)
    # band-limited point source + absorbing box: ~5e-3 measured (A26)
    assert e_out <= 1.5e-2, e_out
    assert e_inc >= 0.5, e_inc


def test_reciprocity():
    rng = np.random.default_rng(11)
    v = rng.uniform(1500.0, 4000.0, (8, 9, 7))
    box = cbs.box_k2(v, 6.0, 30.0, pad=6, absorb=1.0)
    a, b = (1, 2, 3), (6, 5, 1)
    ua, _, _, _ = cbs.cbs_solve(box, cbs.point_source_box(box, [a]), tol=1e-12)
    ub, _, _, _ = cbs.cbs_solve(box, cbs.point_source_box(box, [b]), tol=1e-12)
    va = cbs.model_region(box, ua)[b[2], b[1], b[0]]
    vb = cbs.model_region(box, ub)[a[2], a[1], a[0]]
    assert abs(va - vb) <= 1e-9 * abs(va)


def test_backward_error_reaches_paper_tolerance_on_sharp_contrast():
    v = np.full((16, 16, 16), 1500.0)
    v[8:] = 4500.0                     # two layers, contrast 3
    box = cbs.box_k2(v, 6.0, 25.0, pad=12, absorb=1.0)
    s = cbs.point_source_box(box, [(8, 8, 5)])
    u, be, it, hist = cbs.cbs_solve(box, s, tol=1e-12, check_every=20)
    assert be <= 1e-12, (be, it)
    assert abs(cbs.backward_error(box, u, s) - be) <= 1e-14
    bes = np.array([h[1] for h in hist])
    half = len(bes) // 2
    assert np.all(np.diff(np.log(bes[half:])) <= 0.5)   # decreasing after the transient
