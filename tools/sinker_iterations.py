import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2304_09770_b200 as vb
from synthetic import make_problem
from oracle.assemble import GlobalSystem
from oracle.bddc import BDDC
if __name__ == "__main__":
    prob = make_problem("c4", n=8, sub=(4, 4, 4), constraints=dict(adaptive_tau=0.0))
    gs = GlobalSystem(prob, processes=1)
    bd = BDDC(gs)
    x_o, rep_o = bd.pcg(rtol=1e-10)
    ctx = vb.context_for(prob); ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda"); ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs); rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    print("oracle it", rep_o["iterations"], "kappa", rep_o["kappa"], "gpu it", rep["iterations"], "kappa", rep["kappa"])
    res = rep_o["residuals"]; r0 = res[0]
    print("oracle rel residual tail", [float("%.3e" % (v / r0)) for v in res[-6:]])
