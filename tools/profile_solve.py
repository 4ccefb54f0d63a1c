"""Run setup+factor of a config, then ONE profiled vb_pcg_solve between cudaProfilerStart/Stop
(use with `ncu --profile-from-start off`).  Not a benchmark."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--factor", action="store_true", help="profile the factorisation instead")
    ap.add_argument("--with-k7", action="store_true", help="also one vb_apply_operator (K7) in the profiled range")
    args = ap.parse_args()
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS
    prob = make_problem(args.config, dims=C5_DIMS[1] if args.config == "c5" else None)
    ctx = vb.context_for(prob)
    if args.factor:
        torch.cuda.profiler.start()
    ctx.factor()
    if args.factor:
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        return
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    ctx.pcg_solve(rhs, x)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    rep = ctx.pcg_solve(rhs, x)
    if args.with_k7:
        y = torch.empty_like(x)
        ctx.apply_operator(x, y)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("iterations", rep["iterations"])


if __name__ == "__main__":
    main()
