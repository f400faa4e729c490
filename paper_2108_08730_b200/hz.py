"""Thin ctypes binding of libhz (include/hz.h) — argument marshalling only.

Every step of the hot path runs in libhz's CUDA kernels; this module only converts Python / torch /
numpy arguments into the C ABI's plain pointers and sizes.  There is no CPU fallback: if
`libhz.so` is missing or cannot be loaded, importing this module raises.
"""
from __future__ import annotations

import ctypes as ct
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIBPATH = os.environ.get("HZ_LIB") or os.path.join(_HERE, "libhz.so")   # HZ_LIB: tuning-sweep builds
if not os.path.exists(_LIBPATH):
    raise ImportError(
        f"libhz.so not found at {_LIBPATH}: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")
_lib = ct.CDLL(_LIBPATH)

HZ_OK, HZ_NOT_CONVERGED, HZ_BREAKDOWN, HZ_WARN_CLAMPED = 0, 1, 2, 3
HZ_C64, HZ_C128 = 0, 1
HZ_MASS_EQ8, HZ_MASS_COLLOC = 0, 1
HZ_RULE_GA, HZ_RULE_GAM, HZ_RULE_GA_RECORD = 0, 1, 2
STATUS_NAMES = {0: "HZ_OK", 1: "HZ_NOT_CONVERGED", 2: "HZ_BREAKDOWN", 3: "HZ_WARN_CLAMPED",
                -1: "HZ_ERR_INVALID_ARG", -2: "HZ_ERR_DOMAIN", -3: "HZ_ERR_RANK", -4: "HZ_ERR_OOM",
                -5: "HZ_ERR_CUDA", -6: "HZ_ERR_NCCL", -7: "HZ_ERR_SOURCE_IN_PML"}


class HzError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.hz_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")


class hz_angles(ct.Structure):
    _fields_ = [("n_theta", ct.c_int), ("n_phi", ct.c_int),
                ("theta_rad", ct.POINTER(ct.c_double)), ("phi_rad", ct.POINTER(ct.c_double))]


class hz_grid(ct.Structure):
    _fields_ = [("nx", ct.c_int), ("ny", ct.c_int), ("nz_global", ct.c_int),
                ("z0", ct.c_int), ("nz_local", ct.c_int), ("h", ct.c_double), ("v_halo", ct.c_int)]


class hz_pml(ct.Structure):
    _fields_ = [("npml", ct.c_int), ("r_coeff", ct.c_double), ("v_pml", ct.c_double)]


class hz_solve_opts(ct.Structure):
    _fields_ = [("rtol", ct.c_double), ("max_iter", ct.c_int), ("replace_every", ct.c_int),
                ("check_every", ct.c_int), ("timing", ct.c_int), ("ell", ct.c_int),
                ("stall_window", ct.c_int), ("precond", ct.c_int)]


class hz_solve_stats(ct.Structure):
    _fields_ = [("apply_ms_total", ct.c_double), ("apply_launches", ct.c_longlong),
                ("kernel_launches", ct.c_longlong), ("apply_bytes_total", ct.c_double),
                ("apply_points_total", ct.c_double),
                ("replacements", ct.c_int), ("restarts", ct.c_int), ("iterations", ct.c_int),
                ("stagnated", ct.c_int)]


class hz_cbs_opts(ct.Structure):
    _fields_ = [("pad", ct.c_int), ("absorb", ct.c_double), ("tol", ct.c_double), ("max_iter", ct.c_int),
                ("check_every", ct.c_int)]


class hz_cbs_stats(ct.Structure):
    _fields_ = [("iterations", ct.c_int), ("backward_error", ct.c_double), ("k0sq", ct.c_double),
                ("eps", ct.c_double), ("box", ct.c_int * 3), ("pad", ct.c_int), ("seconds", ct.c_double)]


_vp = ct.c_void_p
_P = ct.POINTER
_sigs = {
    "hz_last_error": (ct.c_char_p, []),
    "hz_version": (ct.c_char_p, []),
    "hz_field_ldx": (ct.c_int, [ct.c_int]),
    "hz_ctx_create_loopback": (ct.c_int, [ct.c_int, ct.c_int, _P(_vp)]),
    "hz_solve_opts_default": (hz_solve_opts, []),
    "hz_kernel_launch_count": (ct.c_longlong, []),
    "hz_trim_memory": (None, []),
    "hz_get_unique_id": (ct.c_int, [ct.c_char_p]),
    "hz_ctx_create": (ct.c_int, [ct.c_int, ct.c_int, ct.c_int, ct.c_char_p, _P(_vp)]),
    "hz_ctx_destroy": (None, [_vp]),
    "hz_build_weight_table": (ct.c_int, [ct.c_double, ct.c_double, ct.c_double, ct.c_double,
                                         _P(hz_angles), _P(_vp)]),
    "hz_table_import": (ct.c_int, [ct.c_double, ct.c_double, ct.c_int, _P(ct.c_double), _P(_vp)]),
    "hz_table_rows": (ct.c_int, [_vp, _P(ct.c_int), _P(ct.c_double), _P(ct.c_double)]),
    "hz_table_destroy": (None, [_vp]),
    "hz_assemble_coeffs": (ct.c_int, [_vp, _P(hz_grid), ct.c_int, _vp, ct.c_double, _P(hz_pml), _vp,
                                      ct.c_int, ct.c_int, _P(_vp), _P(ct.c_longlong)]),
    "hz_coeffs_export": (ct.c_int, [_vp, _vp, _vp, ct.c_int]),
    "hz_coeffs_destroy": (None, [_vp]),
    "hz_coeffs_set_medium": (ct.c_int, [_vp, _vp, _vp, _vp]),
    "hz_apply_impedance": (ct.c_int, [_vp, _vp, _vp, ct.c_int, _vp]),
    "hz_solve": (ct.c_int, [_vp, _vp, _vp, ct.c_int, _P(hz_solve_opts), _P(ct.c_double),
                            _P(ct.c_int), _P(hz_solve_stats), _vp]),
    "hz_point_sources": (ct.c_int, [_vp, ct.c_int, _P(ct.c_longlong), _P(ct.c_double), ct.c_int, _vp, _vp]),
    "hz_export_matrix": (ct.c_int, [_vp, _P(ct.c_longlong), _vp, _vp]),
    "hz_eqerror": (ct.c_int, [_vp, _vp, _vp, _P(ct.c_longlong), ct.c_int, ct.c_double, _P(ct.c_double), _vp]),
    "hz_table_dispersion": (ct.c_int, [_vp, ct.c_int, _P(ct.c_double), ct.c_int, _P(ct.c_double), _P(ct.c_double),
                                       _P(ct.c_double), _vp]),
    "hz_cbs_opts_default": (hz_cbs_opts, []),
    "hz_cbs_solve": (ct.c_int, [_vp, ct.c_int, ct.c_int, ct.c_int, ct.c_double, _vp, ct.c_double, ct.c_int,
                                _P(ct.c_longlong), _P(ct.c_double), _P(hz_cbs_opts), _vp, _P(hz_cbs_stats), _vp]),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


def _check(status, where):
    if status < 0:
        raise HzError(status, where)
    return status


def _ptr(a):
    """Raw address of a torch tensor (device or host) or a numpy array (host)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return a.data_ptr()
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    raise TypeError(type(a))


def _strides_elems(a):
    if hasattr(a, "data_ptr"):
        return tuple(a.stride()), a.shape
    return tuple(st // a.itemsize for st in a.strides), a.shape


def _fptr(c, a, what="field"):
    """Address of a field buffer in the ABI layout [nrhs][nz_local+2][ny][ldx] (include/hz.h): the
    [..][nx] view that Coeffs.alloc_field returns, or a dense tensor / array whose last dim is ldx."""
    if a is None:
        return None
    g = c.grid
    ldx = c.ldx
    st, shp = _strides_elems(a)
    if len(shp) not in (3, 4) or tuple(shp[-3:-1]) != (g.nz_local + 2, g.ny) or shp[-1] not in (g.nx, ldx):
        raise ValueError(f"{what}: shape {tuple(shp)} is not [nrhs][{g.nz_local + 2}][{g.ny}][{g.nx} or {ldx}]")
    fstride = ldx * g.ny * (g.nz_local + 2)
    ok = tuple(st[-3:]) == (ldx * g.ny, ldx, 1) and (len(shp) == 3 or shp[0] == 1 or st[0] == fstride)
    if not ok:
        raise ValueError(f"{what}: strides {tuple(st)} are not the padded field layout (row pitch {ldx}); "
                         "allocate it with Coeffs.alloc_field")
    return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data


def _stream_ptr(stream):
    if stream is None:
        return None
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def hz_version() -> str:
    return _lib.hz_version().decode()


def hz_field_ldx(nx: int) -> int:
    """Row pitch of every field buffer (include/hz.h): nx rounded up to a multiple of 4."""
    return int(_lib.hz_field_ldx(nx))


def hz_kernel_launch_count() -> int:
    return int(_lib.hz_kernel_launch_count())


def hz_trim_memory() -> None:
    _lib.hz_trim_memory()


# ------------------------------------------------------------------------------------------------
class Ctx:
    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.hz_ctx_destroy(self._h)
            except Exception:   # interpreter shutdown
                pass
            self._h = None


def hz_get_unique_id() -> bytes:
    buf = ct.create_string_buffer(128)
    _check(_lib.hz_get_unique_id(buf), "hz_get_unique_id")
    return buf.raw


def hz_ctx_create(device: int = 0, nranks: int = 1, rank: int = 0, uid: Optional[bytes] = None) -> Ctx:
    h = _vp()
    _check(_lib.hz_ctx_create(device, nranks, rank, uid, ct.byref(h)), "hz_ctx_create")
    return Ctx(h)


def hz_ctx_create_loopback(device: int, nranks: int):
    """nranks contexts of one loopback group on one device (include/hz.h): call each rank's functions
    from its own thread."""
    arr = (_vp * nranks)()
    _check(_lib.hz_ctx_create_loopback(device, nranks, arr), "hz_ctx_create_loopback")
    return [Ctx(_vp(arr[r])) for r in range(nranks)]


# ------------------------------------------------------------------------------------------------
class Table:
    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.hz_table_destroy(self._h)
            except Exception:   # interpreter shutdown
                pass
            self._h = None

    @property
    def n_g(self) -> int:
        n = ct.c_int()
        _check(_lib.hz_table_rows(self._h, ct.byref(n), None, None), "hz_table_rows")
        return n.value

    def rows5(self) -> np.ndarray:
        out = np.zeros((self.n_g, 5))
        _check(_lib.hz_table_rows(self._h, None, out.ctypes.data_as(_P(ct.c_double)), None), "hz_table_rows")
        return out

    def rows7(self) -> np.ndarray:
        out = np.zeros((self.n_g, 7))
        _check(_lib.hz_table_rows(self._h, None, None, out.ctypes.data_as(_P(ct.c_double))), "hz_table_rows")
        return out


def hz_build_weight_table(g_min=4.0, g_max=40.0, dg=0.1, lam=1e-2,
                          thetas: Optional[Sequence[float]] = None,
                          phis: Optional[Sequence[float]] = None) -> Table:
    h = _vp()
    ang = None
    if thetas is not None or phis is not None:
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        ph = np.ascontiguousarray(phis, dtype=np.float64)
        ang = hz_angles(len(th), len(ph), th.ctypes.data_as(_P(ct.c_double)), ph.ctypes.data_as(_P(ct.c_double)))
        ang._keep = (th, ph)
    _check(_lib.hz_build_weight_table(g_min, g_max, dg, lam, ct.byref(ang) if ang else None, ct.byref(h)),
           "hz_build_weight_table")
    return Table(h)


def hz_table_import(g_min: float, dg: float, rows5) -> Table:
    r = np.ascontiguousarray(rows5, dtype=np.float64).reshape(-1, 5)
    h = _vp()
    _check(_lib.hz_table_import(g_min, dg, r.shape[0], r.ctypes.data_as(_P(ct.c_double)), ct.byref(h)),
           "hz_table_import")
    return Table(h)


# ------------------------------------------------------------------------------------------------
class Coeffs:
    def __init__(self, handle, grid: hz_grid, dtype: int, status: int, n_clamped: int, ctx: Ctx):
        self._h = handle
        self.grid = grid
        self.dtype = dtype
        self.status = status
        self.n_clamped = n_clamped
        self._ctx = ctx   # keep the context alive

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            try:
                _lib.hz_coeffs_destroy(self._h)
            except Exception:   # interpreter shutdown
                pass
            self._h = None

    @property
    def ldx(self) -> int:
        return hz_field_ldx(self.grid.nx)

    @property
    def field_shape(self):
        g = self.grid
        return (g.nz_local + 2, g.ny, g.nx)

    def alloc_field(self, nrhs: int, device="cuda", pin_memory: bool = False):
        """Zeroed field buffer in the ABI layout [nrhs][nz_local+2][ny][ldx], returned as its
        [nrhs][nz_local+2][ny][nx] view (the pad columns are not part of the field)."""
        import torch
        dt = torch.complex64 if self.dtype == HZ_C64 else torch.complex128
        g = self.grid
        full = torch.zeros((nrhs, g.nz_local + 2, g.ny, self.ldx), dtype=dt, device=device,
                           pin_memory=pin_memory and str(device) == "cpu")
        return full[..., :g.nx]


def hz_assemble_coeffs(ctx: Ctx, nx: int, ny: int, nz_global: int, h: float, v, freq: float, table: Table,
                       npml: int = 8, r_coeff: float = 1e-3, v_pml: float = 0.0, z0: int = 0,
                       nz_local: Optional[int] = None, dtype: int = HZ_C64, mass: int = HZ_MASS_EQ8,
                       v_halo: bool = False, rule: int = HZ_RULE_GA) -> Coeffs:
    if nz_local is None:
        nz_local = nz_global - z0
    g = hz_grid(nx, ny, nz_global, z0, nz_local, h, 1 if v_halo else 0)
    p = hz_pml(npml, r_coeff, v_pml)
    out = _vp()
    ncl = ct.c_longlong(0)
    st = _check(_lib.hz_assemble_coeffs(ctx._h, ct.byref(g), dtype, _ptr(v), freq, ct.byref(p), table._h, mass,
                                        rule, ct.byref(out), ct.byref(ncl)), "hz_assemble_coeffs")
    return Coeffs(out, g, dtype, st, ncl.value, ctx)


def hz_coeffs_export(c: Coeffs, record=None, pml=None) -> None:
    nmax = 0 if pml is None else pml.shape[-1]
    _check(_lib.hz_coeffs_export(c._h, _ptr(record), _ptr(pml), nmax), "hz_coeffs_export")


def hz_coeffs_set_medium(c: Coeffs, b=None, q=None, stream=None) -> None:
    """Buoyancy b = 1/ρ and quality factor Q (arrays of the coeffs' real dtype in v's layout, or None
    for b = 1 / Q = ∞) for every later apply and solve of c (include/hz.h)."""
    _check(_lib.hz_coeffs_set_medium(c._h, _ptr(b), _ptr(q), _stream_ptr(stream)), "hz_coeffs_set_medium")


def hz_apply_impedance(c: Coeffs, u, au, nrhs: Optional[int] = None, stream=None) -> None:
    if nrhs is None:
        nrhs = u.shape[0]
    _check(_lib.hz_apply_impedance(c._h, _fptr(c, u, "u"), _fptr(c, au, "au"), nrhs, _stream_ptr(stream)),
           "hz_apply_impedance")


def hz_solve(c: Coeffs, b, x, nrhs: Optional[int] = None, rtol=1e-6, max_iter=20000, replace_every=50,
             check_every=10, timing=False, ell=1, stall_window=0, precond=0, stream=None):
    """Zero for rtol / max_iter / replace_every / check_every / ell / stall_window selects the default
    (include/hz.h); replace_every < 0 turns residual replacement off."""
    """Returns (status, relres[nrhs], iters[nrhs], stats dict).  ell = 1: BiCGSTAB; 2: BiCGStab(2)."""
    if nrhs is None:
        nrhs = b.shape[0]
    o = hz_solve_opts(rtol, max_iter, replace_every, check_every, 1 if timing else 0, ell, stall_window, precond)
    rel = (ct.c_double * nrhs)()
    its = (ct.c_int * nrhs)()
    stt = hz_solve_stats()
    st = _check(_lib.hz_solve(c._h, _fptr(c, b, "b"), _fptr(c, x, "x"), nrhs, ct.byref(o), rel, its, ct.byref(stt),
                              _stream_ptr(stream)), "hz_solve")
    stats = {k: getattr(stt, k) for k, _ in hz_solve_stats._fields_}
    return st, np.array(rel[:]), np.array(its[:]), stats


def hz_point_sources(c: Coeffs, nodes, b, amps=None, consistent=True, stream=None) -> None:
    n = np.ascontiguousarray(nodes, dtype=np.int64).reshape(-1, 3)
    a = None
    if amps is not None:
        av = np.asarray(amps, dtype=np.complex128).reshape(-1)
        a = np.ascontiguousarray(np.stack([av.real, av.imag], axis=1))
    _check(_lib.hz_point_sources(c._h, n.shape[0], n.ctypes.data_as(_P(ct.c_longlong)),
                                 a.ctypes.data_as(_P(ct.c_double)) if a is not None else None,
                                 1 if consistent else 0, _fptr(c, b, "b"), _stream_ptr(stream)), "hz_point_sources")


def hz_eqerror(c: Coeffs, u_ref, u, src_xyz, npml_mask: int, ball_cells: float = 2.0, stream=None) -> float:
    """The paper's err (reading A20) between two slab wavefields (see include/hz.h)."""
    src = (ct.c_longlong * 3)(*[int(t) for t in src_xyz])
    out = ct.c_double()
    _check(_lib.hz_eqerror(c._h, _fptr(c, u_ref, "u_ref"), _fptr(c, u, "u"), src, npml_mask, ball_cells, ct.byref(out),
                           _stream_ptr(stream)),
           "hz_eqerror")
    return out.value


def hz_cbs_solve(ctx: Ctx, v, h: float, freq: float, src_xyz, u, amps=None, pad=-1, absorb=1.0, tol=1e-12,
                 max_iter=200000, check_every=20, stream=None):
    """Convergent Born series reference (NEXT-3, see include/hz.h): v is a dense [nz][ny][nx] float64
    array (numpy or torch, host or device), u a caller-owned complex128 [nz][ny][nx] array of the same
    placement.  Returns (status, stats dict)."""
    nz, ny, nx = (int(t) for t in v.shape)
    if tuple(u.shape) != (nz, ny, nx):
        raise ValueError("u must have the model's shape")
    src = np.ascontiguousarray(src_xyz, dtype=np.int64).reshape(-1, 3)
    a = None
    if amps is not None:
        av = np.asarray(amps, dtype=np.complex128).reshape(-1)
        a = np.ascontiguousarray(np.stack([av.real, av.imag], axis=1))

    def ptr(x, dt):
        if hasattr(x, "data_ptr"):
            if str(x.dtype) != dt or not x.is_contiguous():
                raise ValueError(f"expected a contiguous {dt} tensor")
            return ct.c_void_p(x.data_ptr())
        if x.dtype != np.dtype(dt.replace("torch.", "")) or not x.flags.c_contiguous:
            raise ValueError(f"expected a contiguous {dt} array")
        return ct.c_void_p(x.ctypes.data)
    o = hz_cbs_opts(pad, absorb, tol, max_iter, check_every)
    st = hz_cbs_stats()
    status = _check(_lib.hz_cbs_solve(ctx._h, nx, ny, nz, float(h), ptr(v, "torch.float64"), float(freq), src.shape[0],
                                      src.ctypes.data_as(_P(ct.c_longlong)),
                                      a.ctypes.data_as(_P(ct.c_double)) if a is not None else None, ct.byref(o),
                                      ptr(u, "torch.complex128"), ct.byref(st), _stream_ptr(stream)), "hz_cbs_solve")
    stats = {k: getattr(st, k) for k, _ in hz_cbs_stats._fields_}
    stats["box"] = tuple(st.box)
    return status, stats


def hz_table_dispersion(table: Table, G, theta, phi, stream=None) -> np.ndarray:
    """vtilde[len(G)][len(theta)] of the table's stencil at the given G and angles (radians), on the device."""
    G = np.ascontiguousarray(G, dtype=np.float64).ravel()
    th = np.ascontiguousarray(theta, dtype=np.float64).ravel()
    ph = np.ascontiguousarray(phi, dtype=np.float64).ravel()
    if th.shape != ph.shape:
        raise ValueError("theta and phi must have the same length")
    out = np.zeros((G.size, th.size))
    _check(_lib.hz_table_dispersion(table._h, G.size, G.ctypes.data_as(_P(ct.c_double)), th.size,
                                    th.ctypes.data_as(_P(ct.c_double)), ph.ctypes.data_as(_P(ct.c_double)),
                                    out.ctypes.data_as(_P(ct.c_double)), _stream_ptr(stream)), "hz_table_dispersion")
    return out


def hz_export_matrix(c: Coeffs, stream=None):
    """(cols [n][27] int64, vals [n][27] complex) of this rank's rows (see include/hz.h)."""
    g = c.grid
    n = g.nz_local * g.ny * g.nx
    cols = np.empty((n, 27), dtype=np.int64)
    vals = np.empty((n, 27), dtype=np.complex64 if c.dtype == HZ_C64 else np.complex128)
    _check(_lib.hz_export_matrix(c._h, cols.ctypes.data_as(_P(ct.c_longlong)), vals.ctypes.data_as(_vp),
                                 _stream_ptr(stream)), "hz_export_matrix")
    return cols, vals
