"""GPU batched BiCGSTAB (through the C ABI) against the oracle's solves and the analytic field."""
import numpy as np
import pytest

import synth
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


def gpu_solve(hz, C, nodes, rtol=1e-6):
    b = C.alloc_field(len(nodes))
    hz.hz_point_sources(C, nodes, b)
    x = C.alloc_field(len(nodes))
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=rtol, max_iter=20000)
    torch.cuda.synchronize()
    return st, rel, its, x[:, 1:-1].cpu().numpy().astype(np.complex128)


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_config1_solve_vs_oracle_and_analytic(hz, ctx, table, ga_table, dtype):
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, dtype)
    nodes = synth.source_nodes(cfg)
    st, rel, its, x = gpu_solve(hz, C, nodes)
    assert st == hz.HZ_OK and rel[0] <= 1e-6, (st, rel)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    b = op.point_sources(P, nodes)[0].ravel()
    xo, rr, _ = solvers.bicgstab(A, b, rtol=1e-10)
    assert np.linalg.norm(x[0].ravel() - xo) / np.linalg.norm(xo) <= 1e-4       # north star: 1e-4
    assert np.linalg.norm(b - A @ x[0].ravel()) / np.linalg.norm(b) <= 2e-6
    # end to end against the analytic Green's function (check 1)
    src = nodes[0]
    D = metrics.distance(v.shape, src, cfg.h)
    m = metrics.interior_mask(v.shape, cfg.npml, src)
    ref = analytic.homogeneous(np.where(D > 0, D, 1.0), 2 * np.pi * cfg.freq / 3000.0)
    assert metrics.eqerror(ref, x[0], D, m) <= 5e-3


@pytest.mark.parametrize("dtype", ["c64", "c128"])
def test_config2_batched_solve(hz, ctx, table, ga_table, dtype):
    """4 RHS solved together; RHS 0 against the oracle's own solve at 1e-10, all RHS by the
    oracle matrix residual of the GPU solution."""
    cfg = synth.get_config(2)
    v, C = setup(hz, ctx, table, cfg, dtype)
    nodes = synth.source_nodes(cfg)
    st, rel, its, x = gpu_solve(hz, C, nodes)
    assert st == hz.HZ_OK and np.all(rel <= 1e-6), (st, rel, its)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    B = op.point_sources(P, nodes)
    for r in range(len(nodes)):
        br = B[r].ravel()
        assert np.linalg.norm(br - A @ x[r].ravel()) / np.linalg.norm(br) <= 2e-6
    xo, rr, _ = solvers.bicgstab(A, B[0].ravel(), rtol=1e-10)
    assert np.linalg.norm(x[0].ravel() - xo) / np.linalg.norm(xo) <= 1e-4


def test_config3_residual_property(hz, ctx, table, ga_table):
    """Config 3 (16 RHS, c64): each GPU wavefield solves the oracle's matrix to the tolerance."""
    cfg = synth.get_config(3)
    v, C = setup(hz, ctx, table, cfg, "c64")
    nodes = synth.source_nodes(cfg)
    st, rel, its, x = gpu_solve(hz, C, nodes)
    assert st == hz.HZ_OK and np.all(rel <= 1e-6), (st, rel, its)
    P = op.Problem(v, cfg.h, cfg.freq, cfg.npml, ga_table)
    A = op.assemble(P)
    B = op.point_sources(P, nodes[:4])
    for r in range(4):
        br = B[r].ravel()
        assert np.linalg.norm(br - A @ x[r].ravel()) / np.linalg.norm(br) <= 3e-6


def test_solver_edge_cases(hz, ctx, table):
    cfg = synth.get_config(1)
    v, C = setup(hz, ctx, table, cfg, "c64")
    b = C.alloc_field(3)
    hz.hz_point_sources(C, np.repeat(synth.source_nodes(cfg), 3, 0), b)
    b[1].zero_()                                    # b = 0 → x = 0, converged at iteration 0
    x = C.alloc_field(3)
    x[2].normal_()                                  # non-zero initial guess
    st, rel, its, stats = hz.hz_solve(C, b, x, rtol=1e-6)
    assert st == hz.HZ_OK and its[1] == 0 and float(x[1].abs().max()) == 0.0
    assert np.all(rel <= 1e-6)
    x2 = C.alloc_field(3)
    st, rel, its, stats = hz.hz_solve(C, b, x2, rtol=1e-12, max_iter=7)
    assert st == hz.HZ_NOT_CONVERGED and its[0] == 7
    assert stats["apply_launches"] > 0 and stats["kernel_launches"] >= stats["apply_launches"]
