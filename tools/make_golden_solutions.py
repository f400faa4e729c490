"""Write tests/golden/solve_cfg{1,2,3}.npz: ORACLE wavefields (complex128 BiCGSTAB to a true relative
residual of 1e-10 on the oracle's explicit CSR matrix) of BASELINE configs 1-3, sampled at seeded
node sets, so the GPU solve-parity tests can compare wavefields without re-running a many-minute CPU
solve.  Calls only oracle/ and synth/ (task rule: a stored expected value is written by a committed
script that calls only the oracle).

Usage: python tools/make_golden_solutions.py [cfg ...]     (each RHS solve runs in its own process)
"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("MKL_NUM_THREADS", "1")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

RHS = {1: [0], 2: [0, 1, 2, 3], 3: [0, 15]}
NSAMPLE = 20000
RTOL = 1e-10


def problem(ci):
    from oracle import operator as op
    from oracle import weights
    cfg = synth.get_config(ci)
    tab = weights.build_adaptive_table(4.0, 40.0, 0.1, 1e-2)
    # the c64 GPU path receives float32 velocities: the oracle solves that exact model
    v = synth.velocity_model(cfg).astype(np.float32).astype(np.float64)
    return cfg, op.Problem(v, cfg.h, cfg.freq, cfg.npml, tab)


def solve_one(args):
    ci, r = args
    from oracle import operator as op
    from oracle import solvers
    cfg, P = problem(ci)
    A = op.assemble(P)
    nodes = synth.source_nodes(cfg)
    b = op.point_sources(P, nodes[r:r + 1])[0].ravel()
    x, rel, it = solvers.bicgstab(A, b, rtol=RTOL)
    print(f"cfg {ci} rhs {r}: {it} iterations, true relres {rel:.2e}", flush=True)
    return ci, r, x, rel, it


def write(ci, d):
    cfg = synth.get_config(ci)
    rng = np.random.Generator(np.random.Philox(synth.BASE_SEED + 7000 + ci))
    idx = np.sort(rng.choice(cfg.npoints, size=min(NSAMPLE, cfg.npoints), replace=False))
    rhs = sorted(d)
    np.savez_compressed(
        os.path.join(ROOT, "tests", "golden", f"solve_cfg{ci}.npz"),
        rhs=np.array(rhs), idx=idx,
        values=np.stack([d[r][0][idx] for r in rhs]),
        full_norm=np.array([np.linalg.norm(d[r][0]) for r in rhs]),
        relres=np.array([d[r][1] for r in rhs]), iters=np.array([d[r][2] for r in rhs]),
        note=np.array("oracle complex128 BiCGSTAB, true relres <= 1e-10, float32-rounded velocity; "
                      "written by tools/make_golden_solutions.py"))
    print(f"wrote solve_cfg{ci}.npz", flush=True)


def main():
    cfgs = [int(a) for a in sys.argv[1:]] or [1, 2, 3]
    jobs = [(ci, r) for ci in cfgs for r in RHS[ci]]
    out = {}
    with ProcessPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
        futs = [ex.submit(solve_one, j) for j in jobs]
        from concurrent.futures import as_completed
        for f in as_completed(futs):
            ci, r, x, rel, it = f.result()
            out.setdefault(ci, {})[r] = (x, rel, it)
            if len(out[ci]) == len(RHS[ci]):   # every RHS of this config done: write it now
                write(ci, out[ci])


if __name__ == "__main__":
    main()
