"""Debug aid: 1-rank vs R-rank (loopback) solves on small configs; prints iterations/kappa/status."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from test_gpu_multirank import _run_ranks
    cases = [("c1", {}, (2, 2, 2)), ("c1", {}, (2, 1, 1)), ("c1", {}, (2, 2, 1)), ("c1", dict(n=8), (2, 2, 2))]
    if len(sys.argv) > 1:
        cases = cases[1:3]
    for name, kw, grid in cases:
        prob = make_problem(name, **kw)
        ctx = vb.context_for(prob)
        ctx.factor()
        rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
        ctx.build_rhs(vb.problem_args(prob), rhs)
        x = torch.zeros_like(rhs)
        rep = ctx.pcg_solve(rhs, x, rtol=1e-10, raise_on_error=False)
        print(name, kw, grid, "1-rank:", rep["status"], rep["iterations"], "%.6g" % rep["kappa"], rep["n_primal"], flush=True)
        try:
            outs = _run_ranks(prob, grid, check_operator=False)
            for r, o in enumerate(outs):
                print("   rank", r, o["rep"]["status"], o["rep"]["iterations"], "%.6g" % o["rep"]["kappa"], o["rep"]["n_primal"], flush=True)
        except Exception as e:
            print("   R-rank failed:", e, flush=True)


if __name__ == "__main__":
    main()
