"""Debug aid: R-rank loopback solve with an arbitrary subdomain -> rank map; prints every rank's
outcome (or its exception) separately."""
import concurrent.futures as cf
import os
import sys
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    prob = make_problem("c1", n=8)
    sub = np.arange(int(np.prod(prob.sub_grid)))
    gx, gy, _ = prob.sub_grid
    i = sub % gx
    srank, R = (i % 3).astype(np.int32), 3
    if len(sys.argv) > 1 and sys.argv[1] == "halves":
        srank, R = (i // 2).astype(np.int32), 2
    world = vb.LoopbackWorld(R)
    streams = [torch.cuda.Stream() for _ in range(R)]

    def rank_main(r):
        try:
            ctx = vb.context_for(prob, stream=streams[r], rank=r, nranks=R, subdomain_rank=srank, world=world)
            print("rank", r, "setup ok", flush=True)
            ctx.factor()
            print("rank", r, "factor ok", flush=True)
            rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
            x = torch.zeros_like(rhs)
            torch.cuda.synchronize()
            ctx.build_rhs(vb.problem_args(prob), rhs)
            rep = ctx.pcg_solve(rhs, x, rtol=1e-10, raise_on_error=False)
            print("rank", r, rep["status"], rep["iterations"], vb._vb_last_error(ctx._h).decode() if rep["status"] != "OK" else "", flush=True)
        except Exception:
            print("rank", r, "FAILED:\n" + traceback.format_exc(), flush=True)

    with cf.ThreadPoolExecutor(R) as ex:
        list(ex.map(rank_main, range(R)))
    world.close()


if __name__ == "__main__":
    main()
