"""K7 (vb_apply_operator) device time on config 5 with the per-launch CUDA events of the library
(VB_KERNEL_TIMING=1): median ms of elem_apply, algorithmic bytes 8 sum_K (nv(nv+1)/2 + np nv)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    from synthetic.configs import C5_DIMS
    prob = make_problem("c5", dims=C5_DIMS[1])
    ctx = vb.context_for(prob)
    st = ctx.stats()
    x = torch.randn(ctx.n_free, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    os.environ["VB_KERNEL_TIMING"] = "1"
    ctx.apply_operator(x, y)
    ts = []
    for _ in range(10):
        ctx.apply_operator(x, y)
        ts.append(ctx.kernel_times()["elem_apply K7 (packed element matrices)"])
    ms = float(np.median(ts))
    b = 8.0 * st["n_cells"] * (st["nv_max"] * (st["nv_max"] + 1) / 2 + 4 * st["nv_max"])
    print("K7 elem_apply: %.4f ms, %.3f GB algorithmic, %.0f GB/s" % (ms, b / 1e9, b / ms / 1e6))


if __name__ == "__main__":
    main()
