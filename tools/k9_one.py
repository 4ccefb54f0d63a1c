"""One vb_setup of config 5 (K9 element kernel runs once): for ncu captures of vem_element_kernel."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if __name__ == "__main__":
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS
    ctx = vb.context_for(make_problem(sys.argv[1] if len(sys.argv) > 1 else "c5", dims=C5_DIMS[1]))
    torch.cuda.synchronize()
    print("ok", ctx.stats()["nv_max"])
