"""GPU batched BiCGSTAB (through the C ABI) against the oracle's solves and the analytic field.

North-star bar: solved wavefields within 1e-4 (relative L2) of the oracle's at a fixed residual
tolerance of 1e-6.  Config 1 is solved by the oracle live; configs 2-3 compare against oracle
wavefields stored by tools/make_golden_solutions.py (oracle complex128 BiCGSTAB to 1e-10, sampled at
20000 seeded nodes), and every GPU wavefield is also checked by its residual with the ORACLE's
explicit matrix.
"""
import os

import numpy as np
import pytest

import synth
from conftest import GOLDEN
from oracle import analytic, metrics, operator as op, solvers

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


def setup(hz, ctx, table, cfg, dtype):
    v = synth.velocity_model(cfg)
    rd = np.float32 if dtype == "c64" else np.float64
    vt = torch.from_numpy(v.astype(rd)).cuda()
    C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, vt, cfg.freq, table, npml=cfg.npml,
                              dtype=hz.HZ_C64 if dtype == "c64" else hz.HZ_C128)
    return v.astype(rd).astype(np.float64), C


def gpu_solve(hz, C, nodes, rtol=1e-6, ell=1):
    b = C.alloc_field(len(nodes))
    hz.hz_point_sources(C, nodes, b)
    x = C.alloc_field(len(nodes))
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=rtol, max_iter=20000, ell=ell)
    torch.cuda.synchronize()
    return st, rel, its, x[:, 1:-1].cpu().numpy().astype(np.complex128)


def golden(name):
    """Stored oracle wavefields (tools/make_golden_solutions.py; oracle complex128 to a true residual of
    1e-10, sampled at 20000 seeded nodes).  A missing file is a failure, not a skip."""
    path = os.path.join(GOLDEN, f"solve_{name}.npz" if not isinstance(name, int) else f"solve_cfg{name}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing oracle golden {path}: run tools/make_golden_solutions.py")
    return np.load(path)


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_config1_solve_vs_oracle_and_analytic(hz, ctx, table, ga_table, dtype, ell):
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, dtype)
    nodes = synth.source_nodes(cfg)
    st, relres, its, x = gpu_solve(hz, C, nodes, ell=ell)
    assert st == hz.HZ_OK and relres[0] <= 1e-6, (st, relres)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    b = op.point_sources(P, nodes)[0].ravel()
    xo, rr, _ = solvers.bicgstab(A, b, rtol=1e-10)
    assert rel(x[0].ravel(), xo) <= 1e-4                      # north star: 1e-4
    assert np.linalg.norm(b - A @ x[0].ravel()) / np.linalg.norm(b) <= 1.5e-6
    # against the stored oracle wavefield as well (same model: v = 3000 is exact in float32)
    G = golden(1)
    assert rel(x[0].ravel()[G["idx"]], G["values"][0]) <= 1e-4
    # end to end against the analytic Green's function (north-star check 1)
    src = nodes[0]
    D = metrics.distance(v.shape, src, cfg.h)
    m = metrics.interior_mask(v.shape, cfg.npml, src)
    ref = analytic.homogeneous(np.where(D > 0, D, 1.0), 2 * np.pi * cfg.freq / 3000.0)
    assert metrics.eqerror(ref, x[0], D, m) <= 5e-3


@pytest.mark.parametrize("dtype,ell", [("c64", 1), ("c128", 1), ("c64", 2)])
def test_config2_batched_solve(hz, ctx, table, ga_table, dtype, ell):
    """4 RHS solved together: every wavefield against the stored oracle wavefield (1e-4) and by its
    residual with the oracle matrix (BiCGSTAB, and BiCGStab(2) for complex64)."""
    cfg = synth.get_config(2)
    v, C = setup(hz, ctx, table, cfg, dtype)
    nodes = synth.source_nodes(cfg)
    st, relres, its, x = gpu_solve(hz, C, nodes, ell=ell)
    assert st == hz.HZ_OK and np.all(relres <= 1e-6), (st, relres, its)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    B = op.point_sources(P, nodes)
    for r in range(len(nodes)):
        br = B[r].ravel()
        assert np.linalg.norm(br - A @ x[r].ravel()) / np.linalg.norm(br) <= 1.5e-6
    G = golden(2)
    for k, r in enumerate(G["rhs"]):
        assert rel(x[r].ravel()[G["idx"]], G["values"][k]) <= 1e-4, r


def test_config3_batched_solve(hz, ctx, table, ga_table):
    """Config 3 (16 RHS, c64, sharp contrasts): stored oracle wavefields for RHS 0 and 15 (1e-4), and the
    oracle-matrix residual of 4 RHS."""
    cfg = synth.get_config(3)
    v, C = setup(hz, ctx, table, cfg, "c64")
    nodes = synth.source_nodes(cfg)
    st, relres, its, x = gpu_solve(hz, C, nodes)
    assert st == hz.HZ_OK and np.all(relres <= 1e-6), (st, relres, its)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    B = op.point_sources(P, nodes[:4])
    for r in range(4):
        br = B[r].ravel()
        assert np.linalg.norm(br - A @ x[r].ravel()) / np.linalg.norm(br) <= 1.5e-6
    G = golden(3)
    for k, r in enumerate(G["rhs"]):
        assert rel(x[r].ravel()[G["idx"]], G["values"][k]) <= 1e-4, (r, rel(x[r].ravel()[G["idx"]], G["values"][k]))


@pytest.mark.parametrize("ell", [1, 2])
@pytest.mark.parametrize("key", ["crop4_5hz", "crop4_10hz", "crop5_10hz"])
def test_large_model_crops(hz, ctx, table, ga_table, key, ell):
    """Configs 4 and 5 (the overthrust and GO_3D_OBS stand-ins) on their seeded 201×201×101
    crops: own npml = 8 PML, the parent's h and f, one source; the GPU's complex64 solve
    at rtol 1e-6 against the oracle's complex128 wavefield (1e-10) within 1e-4 (north star), plus its
    residual with the oracle's explicit matrix."""
    ci, f = int(key[4]), float(key.split("_")[1][:-2])
    cfg = synth.crop_config(ci, f)
    v, C = setup(hz, ctx, table, cfg, "c64")
    nodes = synth.source_nodes(cfg)
    st, relres, its, x = gpu_solve(hz, C, nodes, ell=ell)
    assert st == hz.HZ_OK and relres[0] <= 1e-6, (st, relres, its)
    G = golden(key)
    e = rel(x[0].ravel()[G["idx"]], G["values"][0])
    assert e <= 1e-4, (e, its)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    b = op.point_sources(P, nodes)[0].ravel()
    assert np.linalg.norm(b - op.assemble(P) @ x[0].ravel()) / np.linalg.norm(b) <= 1.5e-6


def test_solver_edge_cases(hz, ctx, table):
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, "c64")
    b = C.alloc_field(3)
    hz.hz_point_sources(C, np.repeat(synth.source_nodes(cfg), 3, 0), b)
    b[1].zero_()                                    # b = 0 → x = 0, converged at iteration 0
    x = C.alloc_field(3)
    x[2].normal_()                                  # non-zero initial guess
    st, relres, its, stats = hz.hz_solve(C, b, x, rtol=1e-6)
    assert st == hz.HZ_OK and its[1] == 0 and float(x[1].abs().max()) == 0.0
    assert np.all(relres <= 1e-6)
    x2 = C.alloc_field(3)
    st, relres, its, stats = hz.hz_solve(C, b, x2, rtol=1e-12, max_iter=7)
    assert st == hz.HZ_NOT_CONVERGED and its[0] == 7
    assert stats["apply_launches"] > 0 and stats["kernel_launches"] >= stats["apply_launches"]
    # host (numpy) buffers through the same ABI: staged by the library, same answer
    bh = C.alloc_field(3, device="cpu")
    bh.copy_(b.cpu())
    xh = C.alloc_field(3, device="cpu")
    st2, rel2, its2, _ = hz.hz_solve(C, bh, xh, rtol=1e-6)
    x3 = C.alloc_field(3)
    st3, rel3, its3, _ = hz.hz_solve(C, b, x3, rtol=1e-6)
    assert st2 == hz.HZ_OK and np.array_equal(its2, its3)
    assert np.array_equal(xh.numpy(), x3.cpu().numpy())


@pytest.mark.parametrize("seed,ell", [(0, 1), (1, 1), (2, 1), (3, 1), (0, 2), (1, 2), (2, 2)])
def test_solve_random_small(hz, ctx, table, ga_table, seed, ell):
    """Batched solve on random small models (RHS converging at different iterations, RHS pairs with a
    retired member, odd RHS counts): every returned x meets rtol on the ORACLE matrix's residual."""
    rng = np.random.default_rng(3000 + seed)
    nz, ny, nx = (int(t) for t in rng.integers(14, 22, 3))
    npml = 3
    nrhs = int(rng.integers(2, 6))
    v = rng.uniform(1500.0, 3500.0, (nz, ny, nx)).astype(np.float32)
    C = hz.hz_assemble_coeffs(ctx, nx, ny, nz, 25.0, torch.from_numpy(v).cuda(), 5.0, table, npml=npml)
    nodes = np.stack([rng.integers(npml + 1, n - npml - 1, nrhs) for n in (nx, ny, nz)], axis=1)
    b = C.alloc_field(nrhs)
    hz.hz_point_sources(C, nodes, b)
    x = C.alloc_field(nrhs)
    st, relres, its, _ = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=20000, ell=ell)
    assert st == hz.HZ_OK and np.all(relres <= 1e-6), (st, relres, its)
    P = op.Problem(v.astype(np.float64), 25.0, 5.0, npml, ga_table)
    A = op.assemble(P)
    B = op.point_sources(P, nodes)
    X = x[:, 1:-1].cpu().numpy().astype(np.complex128)
    for r in range(nrhs):
        br = B[r].ravel()
        assert np.linalg.norm(br - A @ X[r].ravel()) / np.linalg.norm(br) <= 1.5e-6, r


def test_bicgstab2_edge_cases(hz, ctx, table):
    """BiCGStab(2): b = 0 retires at iteration 0, a non-zero initial guess, an iteration cap (counted in
    BiCGSTAB-equivalent steps of 2), host buffers equal to device buffers bit for bit, and a bad ell."""
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, "c64")
    b = C.alloc_field(3)
    hz.hz_point_sources(C, np.repeat(synth.source_nodes(cfg), 3, 0), b)
    b[1].zero_()
    x = C.alloc_field(3)
    x[2].normal_()
    st, relres, its, stats = hz.hz_solve(C, b, x, rtol=1e-6, ell=2)
    assert st == hz.HZ_OK and its[1] == 0 and float(x[1].abs().max()) == 0.0
    assert np.all(relres <= 1e-6) and its[0] % 2 == 0
    x2 = C.alloc_field(3)
    st, relres, its, stats = hz.hz_solve(C, b, x2, rtol=1e-12, max_iter=7, ell=2)
    assert st == hz.HZ_NOT_CONVERGED and its[0] == 8 and stats["iterations"] == 8
    # 4 applies per outer step (+ the initial and final residuals)
    assert stats["apply_launches"] >= 4 * 4
    bh = C.alloc_field(3, device="cpu")
    bh.copy_(b.cpu())
    xh = C.alloc_field(3, device="cpu")
    st2, rel2, its2, _ = hz.hz_solve(C, bh, xh, rtol=1e-6, ell=2)
    x3 = C.alloc_field(3)
    st3, rel3, its3, _ = hz.hz_solve(C, b, x3, rtol=1e-6, ell=2)
    assert st2 == hz.HZ_OK and np.array_equal(its2, its3)
    assert np.array_equal(xh.numpy(), x3.cpu().numpy())
    with pytest.raises(Exception):
        hz.hz_solve(C, b, x3, rtol=1e-6, ell=3)


@pytest.mark.parametrize("ell", [1, 2])
def test_stall_window(hz, ctx, table, ell):
    """stall_window < 0 never retires (the iteration cap ends the solve); a short window retires a
    RHS whose true residual has reached the complex64 floor (rtol 1e-14 is unreachable)."""
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, "c64")
    b = C.alloc_field(1)
    hz.hz_point_sources(C, synth.source_nodes(cfg), b)
    x = C.alloc_field(1)
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-14, max_iter=400, stall_window=-1, ell=ell)
    assert st == hz.HZ_NOT_CONVERGED and stats["stagnated"] == 0 and its[0] == 400, (st, its, stats)
    assert rel[0] <= 1e-6
    x = C.alloc_field(1)
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-14, max_iter=20000, stall_window=100, ell=ell)
    assert st == hz.HZ_NOT_CONVERGED and stats["stagnated"] == 1 and its[0] < 20000, (st, its, stats)
    assert rel[0] <= 1e-6


@pytest.mark.parametrize("key", [1, "crop4_5hz"])
def test_multigrid_preconditioned_solve(hz, ctx, table, ga_table, key):
    """NEXT-4 (opt-in, reading A27): right preconditioning by one complex shifted-Laplacian multigrid
    V-cycle.  Where it converges (config 1, the config-4 crop at 5 Hz) the wavefield equals the oracle's
    within the north star's 1e-4, with fewer iterations than the unpreconditioned BiCGSTAB."""
    cfg = synth.get_config(1) if key == 1 else synth.crop_config(4, 5.0)
    v, C = setup(hz, ctx, table, cfg, "c64")
    nodes = synth.source_nodes(cfg)[:1]
    b = C.alloc_field(1)
    hz.hz_point_sources(C, nodes, b)
    x = C.alloc_field(1)
    st, relres, its, _ = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=20000, precond=1)
    assert st == hz.HZ_OK and relres[0] <= 1e-6, (st, relres, its)
    x0 = C.alloc_field(1)
    st0, _, its0, _ = hz.hz_solve(C, b, x0, rtol=1e-6, max_iter=20000)
    assert its[0] < its0[0], (its, its0)
    G = golden(key)
    u = x[0, 1:-1, :, :cfg.nx].cpu().numpy().astype(np.complex128).ravel()
    assert rel(u[G["idx"]], G["values"][0]) <= 1e-4


def test_multigrid_preconditioner_rejects_unsupported(hz, ctx, table):
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, "c128")
    b = C.alloc_field(1)
    x = C.alloc_field(1)
    with pytest.raises(hz.HzError):
        hz.hz_solve(C, b, x, precond=1)      # complex128
    v, C = setup(hz, ctx, table, cfg, "c64")
    b = C.alloc_field(1)
    x = C.alloc_field(1)
    with pytest.raises(hz.HzError):
        hz.hz_solve(C, b, x, precond=1, ell=2)
