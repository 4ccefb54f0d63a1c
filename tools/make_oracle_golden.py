"""Write oracle results for the full-size BASELINE configs into tests/golden/ (test fixtures).

Calls ONLY oracle/ (and the seeded input recipe in synthetic/); nothing here touches the CUDA
library.  The full-size oracle solves take minutes to an hour on a CPU, far too long for the GPU
test run, so the GPU parity tests at full size compare against these stored oracle values:
the WHOLE solution vector (free DOFs in the exported order; gated per block at relative L2
<= 1e-8), iterations, Lanczos kappa, primal counts, norms and a seeded sample of 20000 rhs
entries (SURVEY §8(c) gates).

  python tools/make_oracle_golden.py c2 c3 c4 c5
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

N_SAMPLE = 20000


def make(name, outdir=None):
    from synthetic import make_problem
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    t0 = time.time()
    prob = make_problem(name)
    gs = GlobalSystem(prob)
    print(name, "system assembled %.0f s" % (time.time() - t0), flush=True)
    bd = BDDC(gs)
    print(name, "BDDC set up %.0f s" % (time.time() - t0), flush=True)
    u, p, rep = bd.solve(rtol=1e-10)
    x = np.concatenate([u, p])
    rng = np.random.default_rng(12345)
    idx = np.sort(rng.choice(x.size, min(N_SAMPLE, x.size), replace=False)).astype(np.int64)
    out = os.path.join(outdir or os.path.join(ROOT, "tests", "golden"), "oracle_%s_full.npz" % name)
    meta = dict(config=name, iterations=int(rep["iterations"]), kappa=float(rep["kappa"]),
                lambda_min=float(rep["lambda_min"]), n_primal=int(bd.NPi), n_coarse=int(bd.NPi + bd.N),
                n_adaptive=int(getattr(bd, "adaptive_count", 0)),
                adaptive_margin=float(getattr(bd, "adaptive_margin", np.inf)),
                n_free_vel=int(gs.dofs.n_free_vel), n_pres=int(gs.dofs.npres),
                n_dofs_paper=int(gs.dofs.n_dofs_paper()), norm_u=float(np.linalg.norm(u)),
                norm_p=float(np.linalg.norm(p)), norm_rhs=float(np.linalg.norm(np.concatenate([gs.rhs_u, gs.rhs_p]))),
                seconds=time.time() - t0,
                source="tools/make_oracle_golden.py (oracle/ only), rtol 1e-10, seed 20230419")
    rhs = np.concatenate([gs.rhs_u, gs.rhs_p])
    np.savez_compressed(out, idx=idx, x_full=x, rhs=rhs[idx], meta=json.dumps(meta))
    print(name, json.dumps(meta), flush=True)


if __name__ == "__main__":
    args = sys.argv[1:]
    outdir = None
    if "--out" in args:
        i = args.index("--out")
        outdir = args[i + 1]
        del args[i:i + 2]
        os.makedirs(outdir, exist_ok=True)
    for name in args or ["c2", "c3", "c4"]:
        make(name, outdir)
