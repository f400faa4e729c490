"""Sweep the complex64 apply's work-plan knobs (HZ_CP_XYF: x/y-PML chunk factor; HZ_CP_ZC: planes
per z-chunk) on BASELINE configs: mean in-solve apply time per launch (CUDA events inside libhz).
Each setting runs in a fresh process (the plan is built once per coefficients object).
Usage: python tools/cp_sweep.py CFG NRHS"""
import itertools
import os
import subprocess
import sys

if len(sys.argv) > 3:   # worker
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import synth
    from paper_2108_08730_b200 import hz
    ci, nrhs = int(sys.argv[1]), int(sys.argv[2])
    cfg = synth.get_config(ci)
    v = torch.from_numpy(synth.velocity_slab(cfg, 0, cfg.nz, device="cuda" if ci == 5 else None).astype(np.float32)).cuda()
    ctx = hz.hz_ctx_create(0)
    T = hz.hz_build_weight_table(4.0, 40.0, 0.1, 1e-2)
    C = hz.hz_assemble_coeffs(ctx, cfg.nx, cfg.ny, cfg.nz, cfg.h, v, cfg.freqs[-1], T, npml=cfg.npml)
    nodes = np.resize(synth.source_nodes(cfg), (nrhs, 3))
    b = C.alloc_field(nrhs)
    hz.hz_point_sources(C, nodes, b)
    best = 1e9
    for rep in range(3):
        x = C.alloc_field(nrhs)
        st, rel, its, stt = hz.hz_solve(C, b, x, rtol=1e-14, max_iter=40, timing=True, replace_every=1000)
        # the 2 fp64 residual applies are in the totals too: subtract nothing, compare like with like
        best = min(best, stt["apply_ms_total"] / stt["apply_launches"])
    print(f"{best:.4f}")
    sys.exit(0)

ci, nrhs = sys.argv[1], sys.argv[2]
for xyf, zc in itertools.product(["1.0", "1.5", "2.0", "3.0"], ["", "8", "16", "32"]):
    env = dict(os.environ)
    env.pop("HZ_CP_ZC", None)
    env["HZ_CP_XYF"] = xyf
    if zc:
        env["HZ_CP_ZC"] = zc
    out = subprocess.run([sys.executable, __file__, ci, nrhs, "w"], env=env, capture_output=True, text=True)
    print(f"cfg {ci} nrhs {nrhs} XYF {xyf} ZC {zc or 'auto'}: {out.stdout.strip() or out.stderr[-300:]} ms/apply", flush=True)
