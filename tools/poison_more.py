import sys, concurrent.futures as cf, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import paper_2304_09770_b200 as vb
from synthetic import make_problem
def solve(prob, constraints=None, **kw):
    ctx = vb.context_for(prob, constraints=constraints, **kw); ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda"); x = torch.zeros_like(rhs)
    torch.cuda.synchronize(); ctx.build_rhs(vb.problem_args(prob), rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10); ids = ctx.dof_layout(); xh = x.cpu().numpy()
    y = torch.zeros_like(rhs); ctx.apply_operator(x, y); torch.cuda.synchronize()
    res = float(torch.linalg.norm(rhs - y) / torch.linalg.norm(rhs)); ctx.close()
    return rep, ids, xh, res
for name, kw, cons in (("c3", dict(n=8), None), ("c1", dict(n=8), dict(scaling=vb.VB_MULTIPLICITY)), ("c4", dict(n=16), None), ("c1", dict(n=18, sub=(9, 9, 9)), None)):
    rep, ids, x, res = solve(make_problem(name, **kw), cons)
    print(name, kw, rep["status"], rep["iterations"], "res %.2e" % res, np.all(np.isfinite(x)), flush=True)
prob = make_problem("c4", n=16)
rep1, ids1, x1, _ = solve(prob)
world = vb.LoopbackWorld(4); srank = vb.box_ranks(prob.sub_grid, (2, 2, 1))
streams = [torch.cuda.Stream() for _ in range(4)]
with cf.ThreadPoolExecutor(4) as ex:
    outs = list(ex.map(lambda r: solve(prob, stream=streams[r], rank=r, nranks=4, subdomain_rank=srank, world=world), range(4)))
world.close()
print("c4 n=16 4 ranks", [(o[0]["status"], o[0]["iterations"], o[0]["n_adaptive"]) for o in outs], rep1["iterations"], rep1["n_adaptive"])
