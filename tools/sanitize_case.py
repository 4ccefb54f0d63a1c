"""Small solves for compute-sanitizer (one tool per run): config 1 (single rank, CUDA-graph
iteration), config 4 at n = 8 with the adaptive coarse space, and config 1 on 2 loopback ranks.

  compute-sanitizer --tool memcheck python tools/sanitize_case.py
"""
import concurrent.futures as cf
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def solve(prob, **kw):
    import torch
    import paper_2304_09770_b200 as vb
    ctx = vb.context_for(prob, **kw)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(rhs)
    torch.cuda.synchronize()
    ctx.build_rhs(vb.problem_args(prob), rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    y = torch.zeros_like(rhs)
    ctx.apply_operator(x, y)
    torch.cuda.synchronize()
    ctx.close()
    return rep


def main():
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    r = solve(make_problem("c1"))
    print("c1", r["status"], r["iterations"])
    r = solve(make_problem("c4", n=8))
    print("c4 n=8 adaptive", r["status"], r["iterations"], r["n_adaptive"])
    prob = make_problem("c1")
    world = vb.LoopbackWorld(2)
    srank = vb.box_ranks(prob.sub_grid, (1, 1, 2))
    streams = [torch.cuda.Stream() for _ in range(2)]
    with cf.ThreadPoolExecutor(2) as ex:
        reps = list(ex.map(lambda q: solve(prob, stream=streams[q], rank=q, nranks=2, subdomain_rank=srank,
                                           world=world), range(2)))
    world.close()
    print("c1 2 ranks", [(rp["status"], rp["iterations"]) for rp in reps])


if __name__ == "__main__":
    main()
