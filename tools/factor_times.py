"""Stage wall times of vb_factor on config 5 (VB_FACTOR_TIMES=1 prints them on stderr), factored
twice on the same context (the second run shows the steady state).  Not a benchmark."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("VB_FACTOR_TIMES", "1")


def main():
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS
    prob = make_problem(sys.argv[1] if len(sys.argv) > 1 else "c5", dims=C5_DIMS[1])
    t = time.time()
    ctx = vb.context_for(prob)
    print("setup %.3f s" % (time.time() - t), flush=True)
    for _ in range(2):
        t = time.time()
        ctx.factor()
        torch.cuda.synchronize()
        print("factor %.3f s, GEMM flops %.3e" % (time.time() - t, ctx.stats()["factor_gemm_flops"]), flush=True)


if __name__ == "__main__":
    main()
