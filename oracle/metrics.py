"""Accuracy metric — ORACLE (test infrastructure only).

`eqerror`: err = |W Re(u_ref − u)|₁ / |W Re(u_ref)|₁ + |W Im(u_ref − u)|₁ / |W Im(u_ref)|₁
with W a diagonal linear gain with distance from the source.  Reading A20: W = distance in
metres, the PML and a 2-cell ball around the source are masked out (the paper is silent).
"""
from __future__ import annotations

import numpy as np


def interior_mask(shape, npml, src=None, h=1.0, ball_cells=2.0):
    nz, ny, nx = shape
    m = np.zeros(shape, dtype=bool)
    m[npml:nz - npml, npml:ny - npml, npml:nx - npml] = True
    if src is not None:
        K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
        d = np.sqrt((I - src[0]) ** 2 + (J - src[1]) ** 2 + (K - src[2]) ** 2)
        m &= d > ball_cells
    return m


def distance(shape, src, h):
    nz, ny, nx = shape
    K, J, I = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return h * np.sqrt((I - src[0]) ** 2 + (J - src[1]) ** 2 + (K - src[2]) ** 2)


def eqerror(u_ref, u, W, mask=None):
    """err of P:268 with weights W (same shape) restricted to `mask`."""
    u_ref = np.asarray(u_ref)
    u = np.asarray(u)
    if mask is None:
        mask = np.ones(u_ref.shape, dtype=bool)
    W = np.asarray(W)[mask]
    dr = np.sum(np.abs(W * (u_ref.real[mask] - u.real[mask])))
    di = np.sum(np.abs(W * (u_ref.imag[mask] - u.imag[mask])))
    nr = np.sum(np.abs(W * u_ref.real[mask]))
    ni = np.sum(np.abs(W * u_ref.imag[mask]))
    if nr == 0 or ni == 0:
        raise ZeroDivisionError("degenerate reference field")
    return dr / nr + di / ni
