"""Seeded synthetic workloads standing in for the paper's benchmarks.

The paper's models (SEG/EAGE overthrust and salt, GO_3D_OBS; PAPER.md P:315, P:329,
P:359, Table 1) are not available, so BASELINE.json `configs` defines five
synthetic stand-ins with the same shapes, value ranges and structure.  The recipes
below follow SURVEY.md §8(d) (base seed S = 210808730, config i draws from
numpy Generator(Philox(S + i))).

Conventions: grid dimensions INCLUDE the PML pad; physical
depth is measured from the first interior node, z_phys = (k - npml) * h; model values
inside the PML come from evaluating the generator there (no edge replication is
needed because every generator is a closed-form function of position).

Arrays are C-ordered [z][y][x] (x fastest).  Every generator is a pure function of
GLOBAL node coordinates plus draws made once per config, so any z-slab can be
generated independently of the partition (needed for the multi-GPU z-slab runs).

This module contains no part of the method (no weights, coefficients or operator).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Tuple

import numpy as np

BASE_SEED = 210808730


def rng_for(config_index: int, counter: Optional[int] = None) -> np.random.Generator:
    """Generator(Philox(S + i)); `counter` selects an independent stream (per z-plane)."""
    if counter is None:
        return np.random.Generator(np.random.Philox(BASE_SEED + config_index))
    return np.random.Generator(
        np.random.Philox(key=BASE_SEED + config_index, counter=int(counter) & ((1 << 256) - 1)))


@dataclass
class Config:
    index: int
    name: str
    nx: int
    ny: int
    nz: int
    h: float
    freqs: Tuple[float, ...]
    npml: int
    dtype: str                     # "c64" | "c128" (the BASELINE config's compute type)
    nsrc: int
    description: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def freq(self) -> float:
        return self.freqs[0]

    @property
    def npoints(self) -> int:
        return self.nx * self.ny * self.nz

    @property
    def shape(self) -> Tuple[int, int, int]:
        return (self.nz, self.ny, self.nx)


CONFIGS = {
    1: Config(1, "homogeneous", 41, 41, 41, 50.0, (5.0,), 8, "c64", 1,
              "BASELINE configs[0]: 41^3, h=50 m, v=3000 m/s (G=12 at 5 Hz), 8-pt PML, "
              "one unit source at the grid centre"),
    2: Config(2, "gradient", 101, 101, 101, 40.0, (5.0,), 8, "c64", 4,
              "BASELINE configs[1]: 101^3, h=40 m, v(z)=1500+0.7 z, 5 Hz, 8-pt PML, "
              "4 sources at 80 m depth on a seeded uniform random layout"),
    3: Config(3, "blocky", 201, 201, 101, 25.0, (7.0,), 10, "c64", 16,
              "BASELINE configs[2]: 201x201x101, h=25 m, 6 layers + random boxes, "
              "1500-4500 m/s, 7 Hz, 10-pt PML, 16 sources at 25 m on a 4x4 grid"),
    4: Config(4, "thrust", 801, 801, 187, 25.0, (5.0, 10.0), 8, "c64", 64,
              "BASELINE configs[3]: 801x801x187, h=25 m, folded/faulted layers 2100-6000 m/s, "
              "5 and 10 Hz, 64 sources at 25 m on an 8x8 grid"),
    5: Config(5, "large", 1201, 1201, 401, 20.0, (10.0,), 8, "c64", 32,
              "BASELINE configs[4]: 1201x1201x401, h=20 m, Gaussian random field "
              "(l=500 m, mean 3000, std 600, clip 1500-5500) + 3 interfaces, 10 Hz"),
}


def get_config(i: int, **overrides) -> Config:
    c = CONFIGS[int(i)]
    if overrides:
        d = dict(c.__dict__)
        d.update(overrides)
        c = Config(**d)
    return c


# ----------------------------------------------------------------------------------------
# velocity generators: v(k, j, i) for global node indices (z, y, x); all return float64
# ----------------------------------------------------------------------------------------

def _cfg3_draws(cfg: Config):
    """Blocky sharp-contrast model (salt stand-in)."""
    rng = rng_for(3)
    nz, ny, nx, npml = cfg.nz, cfg.ny, cfg.nx, cfg.npml
    depths = np.round(np.sort(rng.uniform(npml + 2, nz - npml - 2, 5))).astype(np.int64)
    vel = []
    prev = None
    for _ in range(6):
        while True:
            v = float(rng.uniform(1500.0, 4500.0))
            if prev is None or max(v, prev) / min(v, prev) <= 2.0:
                break
        vel.append(v)
        prev = v
    tops = np.concatenate([[0], depths])
    bots = np.concatenate([depths, [nz]])
    boxes = []  # (layer, x0, x1, y0, y1, z0, z1, v)
    for l in range(6):
        for _ in range(3):
            ex = int(rng.integers(10, 61))
            ey = int(rng.integers(10, 61))
            x0 = int(rng.integers(npml, max(npml + 1, nx - npml - ex)))
            y0 = int(rng.integers(npml, max(npml + 1, ny - npml - ey)))
            zt, zb = int(tops[l]), int(bots[l])
            za = int(rng.integers(zt, max(zt + 1, zb)))
            zb2 = int(rng.integers(za + 1, max(za + 2, zb + 1)))
            fac = float(rng.uniform(0.5, 2.0))
            vb = float(np.clip(vel[l] * fac, 1500.0, 4500.0))
            boxes.append((l, x0, x0 + ex, y0, y0 + ey, za, min(zb2, zb), vb))
    return depths, np.array(vel), boxes


def _cfg4_draws(cfg: Config):
    """Thrust-belt-shaped model (overthrust stand-in)."""
    rng = rng_for(4)
    nz, h, npml = cfg.nz, cfg.h, cfg.npml
    folds = []  # (A [m], Lambda [m], beta, phase)
    for _ in range(4):
        folds.append((float(rng.uniform(50.0, 300.0)), float(rng.uniform(2000.0, 10000.0)),
                      float(rng.uniform(0.0, np.pi)), float(rng.uniform(0.0, 2 * np.pi))))
    nlay = 8
    depth_int = (nz - 2 * npml) * h
    zbar = [depth_int * (l + 1) / nlay for l in range(nlay - 1)]  # 7 interfaces
    vel = np.linspace(2100.0, 6000.0, nlay) * rng.uniform(0.95, 1.05, nlay)
    vel = np.clip(np.sort(vel), 2100.0, 6000.0)
    faults = []  # (xf, yf, zf, strike, dip, throw)
    Lx, Ly = (cfg.nx - 2 * npml) * h, (cfg.ny - 2 * npml) * h
    for _ in range(3):
        faults.append((float(rng.uniform(0, Lx)), float(rng.uniform(0, Ly)),
                       float(rng.uniform(0, depth_int)), float(rng.uniform(0, np.pi)),
                       float(np.deg2rad(rng.uniform(20.0, 40.0))), float(rng.uniform(200.0, 600.0))))
    return folds, zbar, vel, faults


def _cfg5_draws(cfg: Config):
    rng = rng_for(5)
    nz, h, npml = cfg.nz, cfg.h, cfg.npml
    depth_int = (nz - 2 * npml) * h
    Lx, Ly = (cfg.nx - 2 * npml) * h, (cfg.ny - 2 * npml) * h
    planes = []
    tmax = np.tan(np.deg2rad(5.0))
    for _ in range(3):
        zi = float(rng.uniform(0.1 * depth_int, 0.9 * depth_int))
        ang = float(rng.uniform(0, 2 * np.pi))
        mag = float(rng.uniform(0, tmax))
        planes.append((zi, mag * np.cos(ang), mag * np.sin(ang), float(rng.uniform(300.0, 800.0)),
                       Lx / 2, Ly / 2))
    return planes


def _grf_kernel(h: float, ell: float = 500.0):
    half = int(round(2 * ell / h))
    xs = np.arange(-half, half + 1) * h
    k = np.exp(-2.0 * xs ** 2 / ell ** 2)
    return k


def velocity_slab(cfg: Config, z0: int = 0, nz_local: Optional[int] = None,
                  device=None) -> np.ndarray:
    """Velocity [nz_local][ny][nx] (float64) for global planes z0 .. z0+nz_local-1.

    `device` is only used by config 5 (its Gaussian-random-field convolution is run with
    torch on that device when given; the result is identical up to float rounding).
    """
    if nz_local is None:
        nz_local = cfg.nz - z0
    if "origin" in cfg.extra:
        return _crop_slab(cfg, z0, nz_local, device)
    nx, ny, h, npml = cfg.nx, cfg.ny, cfg.h, cfg.npml
    k = np.arange(z0, z0 + nz_local, dtype=np.float64)
    if cfg.index == 1:
        return np.full((nz_local, ny, nx), 3000.0)
    if cfg.index == 2:
        zphys = (k - npml) * h
        v = 1500.0 + 0.7 * zphys
        return np.broadcast_to(v[:, None, None], (nz_local, ny, nx)).copy()
    if cfg.index == 3:
        depths, vel, boxes = _cfg3_draws(cfg)
        kk = np.arange(z0, z0 + nz_local)
        layer = np.searchsorted(depths, kk, side="right")  # interfaces at node depths
        v = np.broadcast_to(vel[layer][:, None, None], (nz_local, ny, nx)).copy()
        for (l, x0, x1, y0, y1, za, zb, vb) in boxes:
            lo, hi = max(za, z0), min(zb, z0 + nz_local)
            if lo < hi:
                v[lo - z0:hi - z0, y0:y1, x0:x1] = vb
        return v
    if cfg.index == 4:
        draws = _cfg4_draws(cfg)
        out = np.empty((nz_local, ny, nx))
        for a in range(0, nz_local, 8):       # z-chunks bound the temporary memory
            b = min(nz_local, a + 8)
            out[a:b] = _cfg4_eval(cfg, draws, k[a:b])
        return out
    if cfg.index == 5:
        return _cfg5_slab(cfg, z0, nz_local, device)
    raise ValueError(cfg.index)


# ----------------------------------------------------------------------------------------
# seeded crops of configs 4-5 (SURVEY §8(d) "Oracle timing": solve parity of the large models on a
# 201×201×101 window of the same generated model, with its own npml = 8 PML, same f and h, 1 source)
# ----------------------------------------------------------------------------------------

CROP_SHAPE = (101, 201, 201)   # (nz, ny, nx)


def crop_config(ci: int, freq: Optional[float] = None) -> Config:
    """The seeded 201×201×101 crop of config 4 or 5: a Config whose velocity is the parent model's
    on the window at extra["origin"] = (x0, y0, z0) (global node indices), npml = 8, the parent's h
    and frequency (config 4: 5 or 10 Hz), one source (see source_nodes)."""
    parent = get_config(ci)
    if ci not in (4, 5):
        raise ValueError("crops are defined for configs 4 and 5")
    nz, ny, nx = CROP_SHAPE
    rng = rng_for(ci, counter=9001)
    x0 = int(rng.integers(0, parent.nx - nx + 1))
    y0 = int(rng.integers(0, parent.ny - ny + 1))
    z0 = int(rng.integers(0, parent.nz - nz + 1))
    f = parent.freq if freq is None else float(freq)
    if f not in parent.freqs:
        raise ValueError(f"config {ci} is defined at {parent.freqs} Hz")
    return Config(ci, parent.name + "-crop", nx, ny, nz, parent.h, (f,), 8, "c64", 1,
                  f"seeded {nx}x{ny}x{nz} crop of BASELINE config {ci} at origin {(x0, y0, z0)}, {f} Hz",
                  extra={"origin": (x0, y0, z0), "parent": parent})


def _crop_slab(cfg: Config, z0: int, nz_local: int, device=None) -> np.ndarray:
    parent = cfg.extra["parent"]
    gx0, gy0, gz0 = cfg.extra["origin"]
    if cfg.index == 4:
        draws = _cfg4_draws(parent)
        k = np.arange(gz0 + z0, gz0 + z0 + nz_local, dtype=np.float64)
        win = Config(**{**parent.__dict__, "nx": cfg.nx, "ny": cfg.ny})
        out = np.empty((nz_local, cfg.ny, cfg.nx))
        for a in range(0, nz_local, 8):
            b = min(nz_local, a + 8)
            out[a:b] = _cfg4_eval(win, draws, k[a:b], gx0, gy0)
        return out
    return _cfg5_slab(parent, gz0 + z0, nz_local, device, gx0, gy0, cfg.nx, cfg.ny)


def _cfg4_eval(cfg: Config, draws, k, x0: int = 0, y0: int = 0) -> np.ndarray:
    """Model at global planes k, columns x0 .. x0+cfg.nx-1, rows y0 .. y0+cfg.ny-1."""
    folds, zbar, vel, faults = draws
    nx, ny, h, npml = cfg.nx, cfg.ny, cfg.h, cfg.npml
    x = (np.arange(x0, x0 + nx) - npml) * h
    y = (np.arange(y0, y0 + ny) - npml) * h
    z = (np.asarray(k, dtype=np.float64) - npml) * h
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    for (xf, yf, zf, strike, dip, throw) in faults:
        dh = np.array([-np.sin(strike), np.cos(strike)])
        dist_h = (X - xf) * dh[0] + (Y - yf) * dh[1]
        hanging = Z < zf + np.tan(dip) * dist_h
        # hanging-wall nodes take the layer index of the point displaced by -throw along dip
        X = np.where(hanging, X - throw * np.cos(dip) * dh[0], X)
        Y = np.where(hanging, Y - throw * np.cos(dip) * dh[1], Y)
        Z = np.where(hanging, Z - throw * np.sin(dip), Z)
    fold = np.zeros_like(X)
    for (A, Lam, beta, ph) in folds:
        fold += A * np.sin(2 * np.pi * (X * np.cos(beta) + Y * np.sin(beta)) / Lam + ph)
    layer = np.zeros(X.shape, dtype=np.int64)
    for l, zb in enumerate(zbar):
        taper = 1.0 - 0.5 * (l + 1) / 8.0
        layer += (Z > zb + taper * fold).astype(np.int64)
    return vel[layer]


def _cfg5_slab(cfg: Config, z0: int, nz_local: int, device=None, x0: int = 0, y0: int = 0,
               nxw: Optional[int] = None, nyw: Optional[int] = None) -> np.ndarray:
    """Config-5 model at global planes z0 .. z0+nz_local-1 over the window of nxw × nyw nodes at
    (x0, y0) (default: the whole plane).  The noise of a plane is drawn for the whole grid (one
    Philox stream per plane), so a window equals the same window of the full model."""
    nx, ny, h, npml = cfg.nx, cfg.ny, cfg.h, cfg.npml
    nxw = nx if nxw is None else nxw
    nyw = ny if nyw is None else nyw
    ker = _grf_kernel(h)
    half = (len(ker) - 1) // 2
    planes = list(range(z0 - half, z0 + nz_local + half))
    noise = np.empty((len(planes), nyw + 2 * half, nxw + 2 * half), dtype=np.float32)
    for n, p in enumerate(planes):
        full = rng_for(5, counter=p + (1 << 40)).standard_normal(
            (ny + 2 * half, nx + 2 * half), dtype=np.float32)
        noise[n] = full[y0:y0 + nyw + 2 * half, x0:x0 + nxw + 2 * half]
    nx, ny = nxw, nyw
    norm = float(np.sqrt(np.sum(ker ** 2)) ** 3)
    if device is not None:
        import torch
        t = torch.from_numpy(noise).to(device)
        kt = torch.from_numpy(ker.astype(np.float32)).to(device)
        # separable valid convolution along x, y, z
        t = torch.nn.functional.conv1d(t.reshape(-1, 1, t.shape[-1]), kt.view(1, 1, -1)).reshape(
            len(planes), ny + 2 * half, nx)
        t = t.transpose(1, 2).contiguous()
        t = torch.nn.functional.conv1d(t.reshape(-1, 1, t.shape[-1]), kt.view(1, 1, -1)).reshape(
            len(planes), nx, ny).transpose(1, 2).contiguous()
        t = t.permute(1, 2, 0).contiguous()
        t = torch.nn.functional.conv1d(t.reshape(-1, 1, t.shape[-1]), kt.view(1, 1, -1)).reshape(
            ny, nx, nz_local).permute(2, 0, 1).contiguous()
        g = t.double().cpu().numpy()
    else:
        from numpy.lib.stride_tricks import sliding_window_view as sw
        g = noise.astype(np.float64)
        g = np.tensordot(sw(g, len(ker), axis=2), ker, axes=([3], [0]))
        g = np.tensordot(sw(g, len(ker), axis=1), ker, axes=([3], [0]))
        g = np.tensordot(sw(g, len(ker), axis=0), ker, axes=([3], [0]))
    g = g / norm
    v = 3000.0 + 600.0 * g
    x = (np.arange(x0, x0 + nx) - npml) * h
    y = (np.arange(y0, y0 + ny) - npml) * h
    z = (np.arange(z0, z0 + nz_local) - npml) * h
    for (zi, a, b, dv, xc, yc) in _cfg5_draws(cfg):
        surf = zi + a * (x[None, :] - xc) + b * (y[:, None] - yc)
        v = v + dv * (z[:, None, None] > surf[None, :, :])
    return np.clip(v, 1500.0, 5500.0)


def velocity_model(cfg: Config) -> np.ndarray:
    return velocity_slab(cfg, 0, cfg.nz)


def source_nodes(cfg: Config) -> np.ndarray:
    """Global (x, y, z) node indices of the config's point sources, int64 [nsrc][3]."""
    n, npml = cfg.nx, cfg.npml
    if "origin" in cfg.extra:   # crop: one source at the window's centre column, one node below its PML
        return np.array([[cfg.nx // 2, cfg.ny // 2, npml + 1]], dtype=np.int64)
    if cfg.index == 1:
        return np.array([[cfg.nx // 2, cfg.ny // 2, cfg.nz // 2]], dtype=np.int64)
    if cfg.index == 2:
        rng = rng_for(2)
        xy = rng.integers(npml + 2, n - npml - 2, size=(4, 2))
        kz = npml + int(round(80.0 / cfg.h))
        return np.array([[a, b, kz] for a, b in xy], dtype=np.int64)
    if cfg.index in (3, 4):
        m = 4 if cfg.index == 3 else 8
        kz = npml + int(round(25.0 / cfg.h))
        xs = np.round(np.linspace(npml + 20, cfg.nx - npml - 21, m)).astype(np.int64)
        ys = np.round(np.linspace(npml + 20, cfg.ny - npml - 21, m)).astype(np.int64)
        return np.array([[a, b, kz] for b in ys for a in xs], dtype=np.int64)
    if cfg.index == 5:
        rng = rng_for(5, counter=7)
        xy = rng.integers(npml + 2, cfg.nx - npml - 2, size=(cfg.nsrc, 2))
        return np.array([[a, b, npml + 1] for a, b in xy], dtype=np.int64)
    raise ValueError(cfg.index)


def random_field(shape, seed: int, dtype=np.complex64) -> np.ndarray:
    """Seeded complex field with Re, Im ~ U(-1, 1) (apply-parity inputs)."""
    rng = np.random.Generator(np.random.Philox(BASE_SEED + 1000 + int(seed)))
    re = rng.uniform(-1.0, 1.0, size=shape)
    im = rng.uniform(-1.0, 1.0, size=shape)
    return (re + 1j * im).astype(dtype)
