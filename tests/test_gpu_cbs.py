"""NEXT-3 on the GPU: the convergent Born series reference (hz_cbs_solve, reading A26)
against the CPU oracle (oracle/cbs.py), the free-space Green's function, the paper's 1e-12 backward
error on config 3, and the paper's Table-2 comparison structure: the adaptive stencil's
wavefield is closer to the CBS reference than the non-adaptive ones."""
import numpy as np
import pytest

import synth
from oracle import cbs, metrics

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


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("placement", ["device", "host"])
def test_cbs_matches_oracle(hz, ctx, placement):
    rng = np.random.default_rng(21)
    v = rng.uniform(1500.0, 4000.0, (12, 14, 16))
    h, f, pad, src = 30.0, 6.0, 8, [(5, 6, 4), (11, 2, 9)]
    amps = [1.0, 0.5 - 0.25j]
    box = cbs.box_k2(v, f, h, pad=pad, absorb=1.0)
    s = cbs.point_source_box(box, src, amps)
    uo, beo, ito, _ = cbs.cbs_solve(box, s, tol=1e-12, check_every=20)
    ref = cbs.model_region(box, uo)
    if placement == "device":
        vd = torch.from_numpy(v).cuda()
        ud = torch.zeros(v.shape, dtype=torch.complex128, device="cuda")
    else:
        vd = np.ascontiguousarray(v)
        ud = np.zeros(v.shape, dtype=np.complex128)
    st, stats = hz.hz_cbs_solve(ctx, vd, h, f, src, ud, amps=amps, pad=pad, absorb=1.0, tol=1e-12, check_every=20)
    got = ud.cpu().numpy() if placement == "device" else ud
    assert st == hz.HZ_OK and stats["backward_error"] <= 1e-12, stats
    assert abs(stats["k0sq"] - box.k0sq) <= 1e-12 * box.k0sq and abs(stats["eps"] - box.eps) <= 1e-12 * box.eps
    assert stats["box"] == (16 + 2 * pad, 14 + 2 * pad, 12 + 2 * pad)
    assert abs(stats["iterations"] - ito) <= 20, (stats["iterations"], ito)
    assert rel(got, ref) <= 1e-10, rel(got, ref)


def test_cbs_homogeneous_green(hz, ctx):
    n, h, f = 40, 50.0, 5.0   # G = 12
    v = torch.full((n, n, n), 3000.0, dtype=torch.float64, device="cuda")
    u = torch.zeros((n, n, n), dtype=torch.complex128, device="cuda")
    src = (n // 2, n // 2, n // 2)
    st, stats = hz.hz_cbs_solve(ctx, v, h, f, [src], u, pad=24, tol=1e-10)
    assert st == hz.HZ_OK, stats
    um = u.cpu().numpy()
    K, J, I = np.meshgrid(*[np.arange(n)] * 3, indexing="ij")
    r = h * np.sqrt((I - src[0]) ** 2 + (J - src[1]) ** 2 + (K - src[2]) ** 2)
    m = (r >= 4 * h) & (r <= 12 * h)
    k = 2 * np.pi * f / 3000.0
    ana = -np.exp(1j * k * r[m]) / (4 * np.pi * r[m])
    assert rel(um[m], ana) <= 1.5e-2, rel(um[m], ana)


def test_cbs_rejects_bad_input(hz, ctx):
    v = np.full((6, 6, 6), 2000.0)
    u = np.zeros((6, 6, 6), dtype=np.complex128)
    with pytest.raises(hz.HzError):
        hz.hz_cbs_solve(ctx, v, 25.0, 5.0, [(9, 0, 0)], u)          # source outside the model
    v[2, 2, 2] = -1.0
    with pytest.raises(hz.HzError):
        hz.hz_cbs_solve(ctx, v, 25.0, 5.0, [(1, 1, 1)], u)          # v <= 0


def test_table2_ordering_config3(hz, ctx, ga_table):
    """Config 3 (the salt stand-in): CBS reference to the paper's backward error 1e-12,
    then the GA (adaptive), Gm and G4 (non-adaptive) wavefields of one source compared with
    it through the paper's err (reading A20): the Table 2 ordering err(GA) < err(Gm) <
    err(G4).  The G4 stencil, tuned for G = 4, is far off at this model's G = 8.6-25.7 and
    BiCGStab(2) does not converge on it (the paper factorises it directly): its err is reported, not
    asserted."""
    from oracle import weights
    cfg = synth.get_config(3)
    v = synth.velocity_model(cfg).astype(np.float32).astype(np.float64)
    # one of the config's source columns at mid depth: the configured 25 m depth puts the source one
    # cell below the 10-cell top PML, whose reflections (0.6 λ thick at 3.5 Hz) then dominate the
    # FD-vs-CBS difference (err 0.64 at 7 Hz, 0.70 at 3.5 Hz, amplitude ratio 0.77-0.83; 0.18 and
    # ratio 1.00 at mid depth: profiles/r02_cbs.md)
    node = tuple(int(t) for t in synth.source_nodes(cfg)[5])
    node = (node[0], node[1], cfg.nz // 2)
    vd = torch.from_numpy(v).cuda()
    uc = torch.zeros(v.shape, dtype=torch.complex128, device="cuda")
    st, stats = hz.hz_cbs_solve(ctx, vd, cfg.h, cfg.freq, [node], uc, tol=1e-12)
    print(f"\nCBS config 3: {stats}")
    assert st == hz.HZ_OK and stats["backward_error"] <= 1e-12, stats
    ref = uc.cpu().numpy()
    vf = torch.from_numpy(v.astype(np.float32)).cuda()
    tables = {
        "GA": hz.hz_table_import(ga_table.g_min, ga_table.dg, ga_table.u5),
        "Gm": hz.hz_table_import(4.0, 0.1, weights.gm_weights()[None]),
        "G4": hz.hz_table_import(4.0, 0.1, weights.g4_weights()[None]),
    }
    W = metrics.distance(v.shape, node, cfg.h)
    mask = metrics.interior_mask(v.shape, cfg.npml, node, cfg.h, 2.0)
    err = {}
    for name, T in tables.items():
        C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, vf, cfg.freq, T, npml=cfg.npml)
        b = C.alloc_field(1)
        hz.hz_point_sources(C, [node], b, consistent=False)     # delta at the node
        x = C.alloc_field(1)
        st2, relres, its, _ = hz.hz_solve(C, b, x, rtol=1e-6, max_iter=20000, ell=2)
        if name == "G4" and st2 != hz.HZ_OK:
            print(f"G4: not converged ({st2}, relres {relres[0]:.2e})")
            continue
        assert st2 == hz.HZ_OK, (name, st2, relres)
        u = x[0, 1:-1, :, :cfg.nx].cpu().numpy().astype(np.complex128)
        err[name] = metrics.eqerror(ref, u, W, mask)
    print(f"err vs CBS: {err}")
    assert err["GA"] < err["Gm"], err
    if "G4" in err:
        assert err["Gm"] < err["G4"], err
