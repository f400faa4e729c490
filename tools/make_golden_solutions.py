"""Write tests/golden/solve_cfg{1,2,3}.npz and solve_crop{4,5}_{f}hz.npz: ORACLE wavefields (complex128 BiCGSTAB to a true relative
residual of 1e-10 on the oracle's explicit CSR matrix) of BASELINE configs 1-3, sampled at seeded
node sets, so the GPU solve-parity tests can compare wavefields without re-running a many-minute CPU
solve.  Calls only oracle/ and synth/ (task rule: a stored expected value is written by a committed
script that calls only the oracle).

Configs 4-5 are solved on their seeded 201x201x101 crops (synth.crop_config): keys
"4c5", "4c10" (config 4 at 5 / 10 Hz) and "5c10".  Config 3 and the crops are solved with the oracle's
BiCGStab(2): complex128 BiCGSTAB stagnates above 1e-10 on these sharp-contrast models (DESIGN.md
reading A23; a config-3 BiCGSTAB run did not finish in 3.7 h).

Usage: python tools/make_golden_solutions.py [key ...]     (each RHS solve runs in its own process)
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

RHS = {1: [0], 2: [0, 1, 2, 3], 3: [0, 15], "4c5": [0], "4c10": [0], "5c10": [0]}
NSAMPLE = 20000
RTOL = 1e-10


def config_of(key):
    if isinstance(key, str) and "c" in key:
        ci, f = key.split("c")
        return synth.crop_config(int(ci), float(f))
    return synth.get_config(int(key))


def out_name(key):
    if isinstance(key, str) and "c" in key:
        ci, f = key.split("c")
        return f"solve_crop{ci}_{f}hz.npz"
    return f"solve_cfg{key}.npz"


def problem(ci):
    from oracle import operator as op
    from oracle import weights
    cfg = config_of(ci)
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
    if isinstance(ci, str) or ci == 3:   # blocky config 3, crops of 4-5: BiCGStab(2) (BiCGSTAB stagnates, A23)
        x, rel, it = solvers.bicgstab_l(A, b, ell=2, rtol=RTOL, max_iter=16000)
    else:
        x, rel, it = solvers.bicgstab(A, b, rtol=RTOL)
    print(f"cfg {ci} rhs {r}: {it} iterations, true relres {rel:.2e}", flush=True)
    return ci, r, x, rel, it


def write(ci, d):
    cfg = config_of(ci)
    seed = ci if isinstance(ci, int) else 100 * int(ci.split("c")[0]) + int(ci.split("c")[1])
    rng = np.random.Generator(np.random.Philox(synth.BASE_SEED + 7000 + seed))
    idx = np.sort(rng.choice(cfg.npoints, size=min(NSAMPLE, cfg.npoints), replace=False))
    rhs = sorted(d)
    np.savez_compressed(
        os.path.join(ROOT, "tests", "golden", out_name(ci)),
        rhs=np.array(rhs), idx=idx,
        values=np.stack([d[r][0][idx] for r in rhs]),
        full_norm=np.array([np.linalg.norm(d[r][0]) for r in rhs]),
        relres=np.array([d[r][1] for r in rhs]), iters=np.array([d[r][2] for r in rhs]),
        note=np.array("oracle complex128 BiCGSTAB, true relres <= 1e-10, float32-rounded velocity; "
                      "written by tools/make_golden_solutions.py"))
    print(f"wrote {out_name(ci)}", flush=True)


def main():
    cfgs = [a if "c" in a else int(a) for a in sys.argv[1:]] or [1, 2, 3]
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
