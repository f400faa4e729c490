"""World-size-2 tests of the z-slab (N>1) host path on CPU with the gloo backend.

The data path of N>1 runs inside libhz over NCCL (halo planes, dot allreduces) and needs GPUs; these
tests cover what runs on the host around it: the slab partition, source ownership, the unique-id
broadcast, the max/sum reductions bench.py reports, gathering slabs, rank-local model generation, and
— with the ORACLE operator — that one halo plane on each side is exactly what a slab's rows need.
"""
import importlib.util
import os
import socket

import numpy as np
import pytest

from conftest import ROOT

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def load_parallel():
    # by path: the package __init__ loads libhz (GPU product); parallel.py itself is host-only
    spec = importlib.util.spec_from_file_location(
        "hz_parallel", os.path.join(ROOT, "paper_2108_08730_b200", "parallel.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, ws, port, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        res = globals()[fn_name](rank, ws)
        q.put((rank, "ok", res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run2(fn_name, ws=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, fn_name, q)) for r in range(ws)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(ws):
        r, status, res = q.get(timeout=300)
        assert status == "ok", res
        out[r] = res
    for p in procs:
        p.join(timeout=60)
    return out


# ------------------------------------------------------------------------------------------------
def test_slab_partition_covers_every_plane_once():
    par = load_parallel()
    for nz in (3, 41, 101, 187, 401):
        for P in (1, 2, 3, 4, 8):
            if nz < P:
                continue
            slabs = par.all_slabs(nz, P)
            owned = np.concatenate([np.arange(z0, z0 + n) for z0, n in slabs])
            assert np.array_equal(owned, np.arange(nz))
            sizes = [n for _, n in slabs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        par.slab_partition(3, 4, 0)


def test_sources_on_rank():
    par = load_parallel()
    nodes = np.array([[5, 5, 0], [5, 5, 9], [5, 5, 10], [5, 5, 20]])
    # slab [10, 20): the consistent source at z = 9 (±1 plane) reaches plane 10; z = 20 reaches 19
    assert list(par.sources_on_rank(nodes, 10, 10)) == [1, 2, 3]
    assert list(par.sources_on_rank(nodes, 0, 10)) == [0, 1, 2]


def _reductions(rank, ws):
    par = load_parallel()
    mx = par.rank_max([float(rank + 1), -float(rank)])
    sm = par.rank_sum([float(rank + 1)])
    uid = par.broadcast_bytes(bytes(range(128)) if rank == 0 else None)
    return mx, sm, uid


def test_rank_reductions_and_uid_broadcast():
    out = run2("_reductions")
    for r in (0, 1):
        mx, sm, uid = out[r]
        assert mx == [2.0, 0.0] and sm == [3.0]
        assert uid == bytes(range(128))


def _gather(rank, ws):
    par = load_parallel()
    nz, ny, nx = 13, 4, 5
    z0, nzl = par.slab_partition(nz, ws, rank)
    glob = np.arange(2 * nz * ny * nx, dtype=np.float64).reshape(2, nz, ny, nx)
    out = par.gather_slabs(glob[:, z0:z0 + nzl].copy(), nz)
    return None if out is None else bool(np.array_equal(out, glob))


def test_gather_slabs():
    out = run2("_gather")
    assert out[0] is True and out[1] is None


def _model_slabs(rank, ws):
    import synth
    par = load_parallel()
    res = []
    for ci in (2, 3):
        cfg = synth.get_config(ci)
        z0, nzl = par.slab_partition(cfg.nz, ws, rank)
        res.append((ci, z0, synth.velocity_slab(cfg, z0, nzl)))
    return res


def test_rank_local_models_match_the_global_model():
    """Every rank generates its slab independently (generators are functions of global position)."""
    import synth
    out = run2("_model_slabs")
    for ci in (2, 3):
        full = synth.velocity_model(synth.get_config(ci))
        for r in (0, 1):
            for c, z0, v in out[r]:
                if c == ci:
                    assert np.array_equal(v, full[z0:z0 + v.shape[0]])


def _oracle_halo(rank, ws):
    """Rows of the owned planes from slab-local data: u and v outside [z0-1, z0+nzl] are poisoned with
    NaN, so any access beyond one halo plane would show up in the result."""
    import synth
    from oracle import operator as op
    from oracle import weights
    par = load_parallel()
    tab = weights.build_adaptive_table(4.0, 40.0, 0.5, 1e-2)
    rng = np.random.default_rng(7)
    nz, ny, nx, h, f, npml = 9, 7, 8, 25.0, 7.0, 2
    v = rng.uniform(1500.0, 4500.0, (nz, ny, nx))
    u = synth.random_field((nz, ny, nx), seed=11).astype(np.complex128)
    z0, nzl = par.slab_partition(nz, ws, rank)
    lo, hi = max(z0 - 1, 0), min(z0 + nzl + 1, nz)
    vp, up = np.full_like(v, np.nan), np.full_like(u, np.nan)
    vp[lo:hi], up[lo:hi] = v[lo:hi], u[lo:hi]
    prob = op.Problem(vp, h, f, npml, tab, v_pml=float(v.max()))
    nodes = np.array([[x, y, z] for z in range(z0, z0 + nzl) for y in range(ny) for x in range(nx)])
    local = op.apply_rows(prob, up, nodes).reshape(nzl, ny, nx)
    full = par.gather_slabs(local, nz)
    if rank != 0:
        return None
    ref = op.apply(op.assemble(op.Problem(v, h, f, npml, tab, v_pml=float(v.max()))), u)
    return float(np.max(np.abs(full - ref)) / np.max(np.abs(ref)))


def test_one_halo_plane_suffices_oracle():
    out = run2("_oracle_halo")
    assert out[0] is not None and out[0] <= 1e-13
