"""CPU checks of the complex64 tensor-map apply's work-list planner (host logic in libhz,
include/hz_debug.h): for many grid sizes and PML widths every (point, plane) of the slab — pad columns
included — is computed by exactly one work item (tile x0 computes the columns [x0 − 1, x0 + tx − 1)),
the tile shape respects the kernel's limits (tx ∈ {32, 64}, ty·tx/2 = 352 consumer threads), and the
item's mode bits match the PML it
touches: TM_PMLXY exactly on tiles holding x/y-PML points, TM_PMLZ exactly on chunks
holding z-PML planes."""
import ctypes

import numpy as np
import pytest

hz = pytest.importorskip("paper_2108_08730_b200.hz", reason="libhz.so not built")


def plan(nx, ny, nz, lo, hi, slots=148, nrhs=1):
    lib = ctypes.CDLL(hz._LIBPATH)
    f = lib.hz_debug_plan_tiles
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_int] * 11 + [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_int)]
    args = [nx, ny, nz, lo[0], hi[0], lo[1], hi[1], lo[2], hi[2], slots, nrhs]
    n = f(*args, None, 0, None)
    assert n > 0
    buf = (ctypes.c_int * (5 * n))()
    wh = (ctypes.c_int * 2)()
    assert f(*args, buf, n, wh) == n
    return np.frombuffer(buf, dtype=np.int32).reshape(n, 5).copy(), wh[0], wh[1]


CASES = [(101, 101, 101, 8), (41, 41, 41, 8), (801, 801, 19, 8), (201, 201, 101, 10), (45, 21, 9, 4),
         (301, 27, 12, 4), (3, 3, 3, 1), (7, 5, 4, 0), (64, 66, 5, 0), (65, 3, 3, 1), (130, 129, 7, 2),
         (17, 250, 6, 5), (5, 9, 3, 3), (1201, 40, 6, 8)]


def pml_range(n, npml):
    # PML-free range as libhz derives it from the profile: lo = npml + 1, hi = n - 2 - npml; no PML: [0, n-1]
    if npml == 0:
        return 0, n - 1
    return npml + 1, n - 2 - npml


@pytest.mark.parametrize("nrhs", [1, 3])
@pytest.mark.parametrize("nx,ny,nz,npml", CASES)
def test_items_partition_the_slab(nx, ny, nz, npml, nrhs):
    lo, hi = zip(*[pml_range(n, npml) for n in (nx, ny, nz)])
    items, tx, ty = plan(nx, ny, nz, lo, hi, nrhs=nrhs)
    ldx = hz.hz_field_ldx(nx)
    assert ldx % 4 == 0 and ldx >= nx > ldx - 4
    assert tx in (32, 64) and ty * (tx // 2) == 352     # 11 consumer warps of whole tile rows
    ntx = -(-(ldx + 1) // tx)
    assert (ntx - 1) * tx - 1 < ldx                     # no tile wholly outside the pitched row
    count = np.zeros((nz, ny, ntx * tx + 1), np.int32)  # column c + 1 ↔ x = c (x = −1 first)

    def in_pml(n, a, b):
        idx = np.arange(n)
        return np.ones(n, bool) if b < a else ~((idx >= a) & (idx <= b))
    px, py, pz = in_pml(nx, lo[0], hi[0]), in_pml(ny, lo[1], hi[1]), in_pml(nz, lo[2], hi[2])
    for x0, y0, z0, z1, mode in items:
        assert x0 % tx == 0 and y0 % ty == 0 and 0 <= z0 < z1 <= nz
        count[z0:z1, y0:y0 + ty, x0:x0 + tx] += 1          # x ∈ [x0 − 1, x0 + tx − 1)
        xs, ys = slice(max(x0 - 1, 0), min(x0 + tx - 1, nx)), slice(y0, min(y0 + ty, ny))
        xy_pml = px[xs].any() or py[ys].any()
        assert bool(mode & 2) == xy_pml                       # TM_PMLXY: the tile holds x/y-PML points
        assert bool(mode & 1) == bool(pz[z0:z1].any())       # TM_PMLZ: the chunk holds z-PML planes
    assert (count[:, :ny, 1:ldx + 1] == 1).all()
    # within a z-chunk, x/y-PML tiles first (heavier, scheduled first)
    for z0 in np.unique(items[:, 2]):
        sel = items[items[:, 2] == z0]
        xyi = (sel[:, 4] & 2) != 0
        if xyi.any() and (~xyi).any():
            assert np.max(np.nonzero(xyi)) < np.min(np.nonzero(~xyi))
