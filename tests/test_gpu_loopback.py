"""The multi-slab data path on one GPU: P z-slab ranks of one process (include/hz.h
hz_ctx_create_loopback), one host thread per rank, going through the same halo-exchange / allreduce /
broadcast call sites as the NCCL path (halo planes by cudaMemcpyAsync, dot products summed by a device
kernel in rank order) — SURVEY §4 item 4, §8(e).

  * apply: the slabs' halo planes come from the library's exchange (not from the caller), overlapped
    with the interior planes' items (the boundary planes' one-plane items run after the join; slabs
    too thin for an interior run everything after the exchange, P = 16): the gathered result is
    bitwise the single-domain apply (per-point arithmetic identical, halos are copies);
  * solve: decomposition invariance at P = 2, 4, 8 — wavefields within 1e-4 of the single-domain solve
    and iteration counts within a few percent (the dot products' summation order changes with P);
  * BiCGStab(2) and the complex64 compensated iterate (whose x_lo halo planes are exchanged too).
"""
import threading

import numpy as np
import pytest

import synth
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
def table(hz, ga_table):
    return hz.hz_table_import(ga_table.g_min, ga_table.dg, ga_table.u5)


NX, NY, NZ, H, F, NPML = 45, 41, 40, 25.0, 6.0, 4


@pytest.fixture(scope="module")
def model():
    rng = np.random.default_rng(2024)
    v = np.empty((NZ, NY, NX))
    v[:] = np.linspace(1600.0, 3800.0, NZ)[:, None, None]
    v += rng.uniform(-150.0, 150.0, v.shape)          # heterogeneous: Eq. 8 couples neighbouring slabs
    return v.astype(np.float32)


def run_ranks(P, fn):
    """fn(rank) on P threads; re-raises the first failure."""
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
    assert not any(t.is_alive() for t in th), "a rank did not finish"
    if err:
        raise err[0]
    return out


def slabs_assemble(hz, ctxs, table, v, P, r):
    z0, nzl = parallel.slab_partition(NZ, P, r)
    vt = torch.from_numpy(np.ascontiguousarray(v[z0:z0 + nzl])).cuda()
    C = hz.hz_assemble_coeffs(ctxs[r], NX, NY, NZ, H, vt, F, table, npml=NPML, z0=z0, nz_local=nzl)
    return z0, nzl, C


@pytest.mark.parametrize("P", [2, 3, 5, 16])
def test_loopback_apply_is_bitwise_single_domain(hz, table, model, P):
    u = synth.random_field((3, NZ, NY, NX), seed=41)
    ctx1 = hz.hz_ctx_create(0)
    C1 = hz.hz_assemble_coeffs(ctx1, NX, NY, NZ, H, torch.from_numpy(model).cuda(), F, table, npml=NPML)
    ud, ad = C1.alloc_field(3), C1.alloc_field(3)
    ud[:, 1:-1] = torch.from_numpy(u).cuda()
    hz.hz_apply_impedance(C1, ud, ad)
    torch.cuda.synchronize()
    full = ad[:, 1:-1].cpu().numpy()
    ctxs = hz.hz_ctx_create_loopback(0, P)

    def rank(r):
        torch.cuda.set_device(0)
        z0, nzl, C = slabs_assemble(hz, ctxs, table, model, P, r)
        s = torch.cuda.Stream()
        us, as_ = C.alloc_field(3), C.alloc_field(3)
        us[:, 1:-1] = torch.from_numpy(u[:, z0:z0 + nzl]).cuda()
        torch.cuda.synchronize()
        hz.hz_apply_impedance(C, us, as_, stream=s)        # halo planes: the library's exchange
        s.synchronize()
        return z0, nzl, as_[:, 1:-1].cpu().numpy()
    out = np.zeros_like(full)
    for z0, nzl, a in run_ranks(P, rank):
        out[:, z0:z0 + nzl] = a
    assert np.array_equal(out, full), float(np.abs(out - full).max())


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_loopback_solve_decomposition_invariance(hz, table, model, P, ell):
    nodes = np.array([[22, 20, NPML + 2], [12, 30, 31]], dtype=np.int64)   # sources in different slabs
    ctx1 = hz.hz_ctx_create(0)
    C1 = hz.hz_assemble_coeffs(ctx1, NX, NY, NZ, H, torch.from_numpy(model).cuda(), F, table, npml=NPML)
    b1, x1 = C1.alloc_field(2), C1.alloc_field(2)
    hz.hz_point_sources(C1, nodes, b1)
    st1, rel1, its1, _ = hz.hz_solve(C1, b1, x1, rtol=1e-6, ell=ell)
    assert st1 == hz.HZ_OK
    ref = x1[:, 1:-1].cpu().numpy()
    ctxs = hz.hz_ctx_create_loopback(0, P)

    def rank(r):
        torch.cuda.set_device(0)
        z0, nzl, C = slabs_assemble(hz, ctxs, table, model, P, r)
        s = torch.cuda.Stream()
        b, x = C.alloc_field(2), C.alloc_field(2)
        hz.hz_point_sources(C, nodes, b, stream=s)
        st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-6, ell=ell, stream=s)
        s.synchronize()
        return z0, nzl, st, rel, its, x[:, 1:-1].cpu().numpy()
    res = run_ranks(P, rank)
    out = np.zeros_like(ref)
    for z0, nzl, st, rel, its, xs in res:
        assert st == hz.HZ_OK and np.all(rel <= 1e-6), (st, rel)
        out[:, z0:z0 + nzl] = xs
    # every rank reports the same global residuals and iteration counts (allreduced dots)
    assert all(np.array_equal(res[0][3], r[3]) and np.array_equal(res[0][4], r[4]) for r in res)
    its = res[0][4]
    assert np.all(np.abs(its - its1) <= np.maximum(0.1 * its1, 10)), (its, its1)
    for k in range(2):
        e = np.linalg.norm(out[k] - ref[k]) / np.linalg.norm(ref[k])
        assert e <= 1e-4, (k, e)
