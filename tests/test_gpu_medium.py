"""GPU parity of the visco-acoustic, variable-density path (NEXT-2; hz_coeffs_set_medium,
csrc/apply_medium.cu; readings A24, A25) against the oracle's explicit matrix (oracle/operator.py
with Problem(b=…, Q=…)), on seeded random models with PML, ragged sizes and every row rule:

  * apply: relative L2 ≤ 1e-5 (complex64) / 1e-12 (complex128), Eq. 8 and collocation mass, GA and GAm;
  * b ≡ 1 with Q = ∞ through the medium kernel reproduces the class-sum kernels' apply;
  * emulated z-slabs (caller-supplied halo planes) are bitwise the single-domain apply;
  * the loopback communicator's slabs (b / Q halo planes exchanged by the library) likewise;
  * batched solves (BiCGSTAB and BiCGStab(2), both precisions) match the oracle's direct solve ≤ 1e-4.
"""
import threading

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import synth
from oracle import operator as op
from paper_2108_08730_b200 import parallel

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2108_08730_b200 import hz as _hz
    return _hz


@pytest.fixture(scope="module")
def ctx(hz):
    return hz.hz_ctx_create(0)


@pytest.fixture(scope="module")
def table(hz, ga_table):
    return hz.hz_table_import(ga_table.g_min, ga_table.dg, ga_table.u5)


def rdt(dtype):
    return np.float32 if dtype == "c64" else np.float64


def medium_model(shape, seed):
    rng = np.random.default_rng(seed)
    v = rng.uniform(1500.0, 4500.0, shape)
    b = rng.uniform(0.35, 1.2, shape)          # ρ from 0.83 to 2.9 g/cc
    Q = rng.uniform(15.0, 300.0, shape)
    return v, b, Q


def gpu_coeffs(hz, ctx, table, v, b, Q, h, f, npml, dtype, mass="eq8", rule="GA", **kw):
    t = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a.astype(rdt(dtype)))).cuda()  # noqa
    nzg = kw.pop("nz_global", v.shape[0])
    C = hz.hz_assemble_coeffs(ctx, v.shape[-1], v.shape[-2], nzg, h, t(v), f, table, npml=npml,
                              dtype=hz.HZ_C64 if dtype == "c64" else hz.HZ_C128,
                              mass=hz.HZ_MASS_EQ8 if mass == "eq8" else hz.HZ_MASS_COLLOC,
                              rule=hz.HZ_RULE_GA if rule == "GA" else hz.HZ_RULE_GAM, **kw)
    hz.hz_coeffs_set_medium(C, t(b), t(Q))
    return C


def oracle_problem(v, b, Q, h, f, npml, ga_table, dtype, mass="eq8", rule="GA"):
    c = lambda a: None if a is None else a.astype(rdt(dtype)).astype(np.float64)  # noqa: E731
    return op.Problem(c(v), h, f, npml, ga_table, mass=mass, rule=rule, b=c(b), Q=c(Q))


def gpu_apply(hz, C, u):
    ud = C.alloc_field(u.shape[0])
    ud[:, 1:-1] = torch.from_numpy(u).cuda()
    aud = C.alloc_field(u.shape[0])
    hz.hz_apply_impedance(C, ud, aud)
    torch.cuda.synchronize()
    return aud[:, 1:-1].cpu().numpy()


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


TOL = {"c64": 1e-5, "c128": 1e-12}


@pytest.mark.parametrize("dtype", ["c64", "c128"])
@pytest.mark.parametrize("mass,rule", [("eq8", "GA"), ("colloc", "GA"), ("eq8", "GAm")])
@pytest.mark.parametrize("shape,npml", [((13, 19, 37), 3), ((9, 8, 33), 2), ((6, 11, 7), 0)])
def test_medium_apply_parity(hz, ctx, table, ga_table, dtype, mass, rule, shape, npml):
    v, b, Q = medium_model(shape, seed=sum(shape) + npml)
    h, f = 25.0, 7.0
    C = gpu_coeffs(hz, ctx, table, v, b, Q, h, f, npml, dtype, mass, rule)
    u = synth.random_field((2,) + shape, seed=5).astype(np.complex64 if dtype == "c64" else np.complex128)
    got = gpu_apply(hz, C, u)
    A = op.assemble(oracle_problem(v, b, Q, h, f, npml, ga_table, dtype, mass, rule))
    ref = op.apply(A, u.astype(np.complex128))
    assert rel(got, ref) <= TOL[dtype], rel(got, ref)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_medium_b_only_and_q_only(hz, ctx, table, ga_table, dtype):
    v, b, Q = medium_model((10, 12, 21), seed=8)
    u = synth.random_field((1, 10, 12, 21), seed=2).astype(np.complex64 if dtype == "c64" else np.complex128)
    for bb, qq in ((b, None), (None, Q)):
        C = gpu_coeffs(hz, ctx, table, v, bb, qq, 20.0, 9.0, 3, dtype)
        ref = op.apply(op.assemble(oracle_problem(v, bb, qq, 20.0, 9.0, 3, ga_table, dtype)), u.astype(np.complex128))
        assert rel(gpu_apply(hz, C, u), ref) <= TOL[dtype]


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_unit_medium_matches_class_sum_kernels(hz, ctx, table, dtype):
    v, _, _ = medium_model((11, 14, 29), seed=4)
    u = synth.random_field((2, 11, 14, 29), seed=7).astype(np.complex64 if dtype == "c64" else np.complex128)
    vt = torch.from_numpy(v.astype(rdt(dtype))).cuda()
    dt = hz.HZ_C64 if dtype == "c64" else hz.HZ_C128
    C0 = hz.hz_assemble_coeffs(ctx, 29, 14, 11, 25.0, vt, 6.0, table, npml=3, dtype=dt)
    ref = gpu_apply(hz, C0, u)
    C1 = hz.hz_assemble_coeffs(ctx, 29, 14, 11, 25.0, vt, 6.0, table, npml=3, dtype=dt)
    ones = torch.ones_like(vt)
    hz.hz_coeffs_set_medium(C1, ones, torch.full_like(vt, float("inf")))
    assert rel(gpu_apply(hz, C1, u), ref) <= (2e-6 if dtype == "c64" else 1e-13)
    hz.hz_coeffs_set_medium(C1, None, None)          # back to the class-sum kernels: bitwise
    assert np.array_equal(gpu_apply(hz, C1, u), ref)


def test_medium_domain_errors(hz, ctx, table):
    v, b, Q = medium_model((6, 7, 8), seed=1)
    C = hz.hz_assemble_coeffs(ctx, 8, 7, 6, 25.0, torch.from_numpy(v.astype(np.float32)).cuda(), 6.0, table, npml=1)
    bad = b.astype(np.float32).copy()
    bad[3, 2, 1] = -1.0
    with pytest.raises(hz.HzError):
        hz.hz_coeffs_set_medium(C, torch.from_numpy(bad).cuda(), None)
    badq = Q.astype(np.float32).copy()
    badq[0, 0, 0] = np.nan
    with pytest.raises(hz.HzError):
        hz.hz_coeffs_set_medium(C, None, torch.from_numpy(badq).cuda())


def test_medium_emulated_slabs_bitwise(hz, ctx, table):
    nz, ny, nx, h, f, npml = 17, 13, 35, 25.0, 7.0, 3
    v, b, Q = medium_model((nz, ny, nx), seed=12)
    u = synth.random_field((2, nz, ny, nx), seed=3)
    full = gpu_apply(hz, gpu_coeffs(hz, ctx, table, v, b, Q, h, f, npml, "c64", v_pml=float(v.max())), u)
    for cuts in ([0, 8, 17], [0, 1, 5, 12, 17]):
        out = np.zeros_like(full)
        for z0, z1 in zip(cuts[:-1], cuts[1:]):
            nzl = z1 - z0

            def halo(a):
                s = np.ones((nzl + 2, ny, nx))
                lo, hi = max(z0 - 1, 0), min(z1 + 1, nz)
                s[lo - (z0 - 1):hi - (z0 - 1)] = a[lo:hi]
                return s
            C = gpu_coeffs(hz, ctx, table, halo(v), halo(b), halo(Q), h, f, npml, "c64", z0=z0, nz_local=nzl,
                           nz_global=nz, v_pml=float(v.max()), v_halo=True)
            ud = C.alloc_field(2)
            for k in range(nzl + 2):
                zg = z0 - 1 + k
                if 0 <= zg < nz:
                    ud[:, k] = torch.from_numpy(u[:, zg]).cuda()
            aud = C.alloc_field(2)
            hz.hz_apply_impedance(C, ud, aud)
            torch.cuda.synchronize()
            out[:, z0:z1] = aud[:, 1:-1].cpu().numpy()
        assert np.array_equal(out, full), cuts


def run_ranks(P, fn):
    out, err = [None] * P, []

    def wrap(r):
        try:
            out[r] = fn(r)
        except BaseException as e:   # noqa: BLE001
            err.append(e)
    th = [threading.Thread(target=wrap, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


@pytest.mark.parametrize("P", [2, 3])
def test_medium_loopback_apply_and_solve(hz, table, ga_table, P):
    """Library-exchanged b / Q halo planes: the P-slab apply is bitwise the single-domain apply, and
    the P-slab c64 solve matches the single-domain one within 1e-4."""
    nz, ny, nx, h, f, npml = 24, 21, 27, 25.0, 6.0, 3
    v, b, Q = medium_model((nz, ny, nx), seed=40 + P)
    u = synth.random_field((1, nz, ny, nx), seed=11)
    ctx1 = hz.hz_ctx_create(0)
    C1 = gpu_coeffs(hz, ctx1, table, v, b, Q, h, f, npml, "c64")
    full = gpu_apply(hz, C1, u)
    nodes = np.array([[13, 10, 8], [7, 15, 17]], dtype=np.int64)
    b1, x1 = C1.alloc_field(2), C1.alloc_field(2)
    hz.hz_point_sources(C1, nodes, b1)
    st1, _, its1, _ = hz.hz_solve(C1, b1, x1, rtol=1e-6)
    assert st1 == hz.HZ_OK
    ref = x1[:, 1:-1].cpu().numpy()
    ctxs = hz.hz_ctx_create_loopback(0, P)

    def rank(r):
        torch.cuda.set_device(0)
        z0, nzl = parallel.slab_partition(nz, P, r)
        sl = slice(z0, z0 + nzl)
        C = gpu_coeffs(hz, ctxs[r], table, v[sl], b[sl], Q[sl], h, f, npml, "c64", z0=z0, nz_local=nzl, nz_global=nz)
        s = torch.cuda.Stream()
        us, as_ = C.alloc_field(1), C.alloc_field(1)
        us[:, 1:-1] = torch.from_numpy(u[:, sl]).cuda()
        torch.cuda.synchronize()
        hz.hz_apply_impedance(C, us, as_, stream=s)
        bb, xx = C.alloc_field(2), C.alloc_field(2)
        hz.hz_point_sources(C, nodes, bb, stream=s)
        st, rl, its, _ = hz.hz_solve(C, bb, xx, rtol=1e-6, stream=s)
        s.synchronize()
        return z0, nzl, as_[:, 1:-1].cpu().numpy(), st, xx[:, 1:-1].cpu().numpy()
    out = np.zeros_like(full)
    xo = np.zeros_like(ref)
    for z0, nzl, a, st, xs in run_ranks(P, rank):
        assert st == hz.HZ_OK
        out[:, z0:z0 + nzl] = a
        xo[:, z0:z0 + nzl] = xs
    assert np.array_equal(out, full)
    for k in range(2):
        assert np.linalg.norm(xo[k] - ref[k]) / np.linalg.norm(ref[k]) <= 1e-4


@pytest.mark.parametrize("dtype,ell", [("c64", 1), ("c64", 2), ("c128", 1)])
def test_medium_solve_parity(hz, ctx, table, ga_table, dtype, ell):
    """Batched solve of 2 point sources on a visco-acoustic variable-density model with PML against
    the oracle's sparse direct solve: wavefield relative L2 ≤ 1e-4 at rtol 1e-6."""
    nz, ny, nx, h, f, npml = 22, 25, 31, 25.0, 6.0, 4
    v, b, Q = medium_model((nz, ny, nx), seed=77)
    C = gpu_coeffs(hz, ctx, table, v, b, Q, h, f, npml, dtype)
    nodes = np.array([[15, 12, 9], [9, 17, 14]], dtype=np.int64)
    bd, xd = C.alloc_field(2), C.alloc_field(2)
    hz.hz_point_sources(C, nodes, bd)
    st, rl, its, _ = hz.hz_solve(C, bd, xd, rtol=1e-6, ell=ell)
    assert st == hz.HZ_OK and np.all(rl <= 1e-6)
    got = xd[:, 1:-1].cpu().numpy()
    P = oracle_problem(v, b, Q, h, f, npml, ga_table, dtype)
    A = op.assemble(P).tocsc()
    rhs = op.point_sources(P, nodes)
    lu = spla.splu(A)
    for k in range(2):
        ref = lu.solve(rhs[k].ravel()).reshape(v.shape)
        assert rel(got[k], ref) <= 1e-4, (k, rel(got[k], ref))
