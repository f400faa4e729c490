"""CPU checks of the complex64 apply's tile planner (host logic in libhz, include/hz_debug.h): for many
plane sizes and PML widths every point of the plane is stored by exactly one tile, every tile respects
the kernel's shape limits, and a tile runs the x/y-PML body exactly when its stored points are PML points
(a tile is wholly inside or outside the x/y-PML)."""
import ctypes

import numpy as np
import pytest

hz = pytest.importorskip("paper_2108_08730_b200.hz", reason="libhz.so not built")

CP_HALO = 768


def plan(nx, ny, lo_x, hi_x, lo_y, hi_y, ny_rows):
    lib = ctypes.CDLL(hz._LIBPATH)
    f = lib.hz_debug_plan_tiles
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int] * 7 + [ctypes.POINTER(ctypes.c_int), ctypes.c_int]
    n = f(nx, ny, lo_x, hi_x, lo_y, hi_y, ny_rows, None, 0)
    assert n > 0
    buf = (ctypes.c_int * (9 * n))()
    assert f(nx, ny, lo_x, hi_x, lo_y, hi_y, ny_rows, buf, n) == n
    return np.frombuffer(buf, dtype=np.int32).reshape(n, 9).copy()


CASES = [(101, 101, 8), (41, 41, 8), (801, 801, 8), (201, 201, 10), (45, 21, 4), (301, 27, 4), (3, 3, 1),
         (7, 5, 0), (64, 66, 0), (65, 3, 1), (130, 129, 2), (17, 250, 5), (5, 9, 3)]


@pytest.mark.parametrize("rows", [1, 2])
@pytest.mark.parametrize("nx,ny,npml", CASES)
def test_tiles_partition_the_plane(nx, ny, npml, rows):
    # PML-free range of an axis as libhz derives it from the profile: (npml, n-1-npml) exclusive of the
    # half-step stretch at the boundary node (lo = npml + 1, hi = n - 2 - npml); no PML: [0, n-1]
    def rng(n):
        if npml == 0:
            return 0, n - 1
        return npml + 1, n - 2 - npml
    lo_x, hi_x = rng(nx)
    lo_y, hi_y = rng(ny)
    T = plan(nx, ny, lo_x, hi_x, lo_y, hi_y, rows)
    count = np.zeros((ny, nx), np.int32)
    in_pml_x = np.ones(nx, bool) if hi_x < lo_x else ~((np.arange(nx) >= lo_x) & (np.arange(nx) <= hi_x))
    in_pml_y = np.ones(ny, bool) if hi_y < lo_y else ~((np.arange(ny) >= lo_y) & (np.arange(ny) <= hi_y))
    for x0, y0, tx, ty, xs, ys, xe, ye, pml in T:
        assert 1 <= tx <= 64 and ty >= 2 and ty % 2 == 0
        assert tx * ty <= 256 * rows and (tx + 2) * (ty + 2) <= CP_HALO
        assert 0 <= x0 <= xs < xe <= x0 + tx <= nx and 0 <= y0 <= ys < ye <= y0 + ty <= ny
        count[ys:ye, xs:xe] += 1
        stored_pml = in_pml_x[xs:xe][None, :] | in_pml_y[ys:ye][:, None]
        assert stored_pml.all() if pml else not stored_pml.any()
    assert (count == 1).all(), np.argwhere(count != 1)[:5]
