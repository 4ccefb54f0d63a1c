"""Trend check in the spirit of the paper's Table T2 and T3 on the
BASELINE-style CUBE meshes (homogeneous Dirichlet, box partitions): PCG iterations and Lanczos
kappa of the GPU solver for the minimal coarse space (vertex + face flux, nu_tol = inf in the
paper's terms), the BASELINE space (vertex + edge + face averages + flux) and the adaptive space
(tau = 2, the paper's nu_tol = 2), as H/h grows at a fixed subdomain count, and as k grows.
Context only: the paper's meshes and partitions differ.  With --neumann the faces
x = 1 and y = 1 carry the natural condition, as in the paper's runs (DESIGN A35).

  python tools/trend_table.py > profiles/r01_trends.txt
  python tools/trend_table.py --neumann > profiles/r02y_trends_neumann.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def run(prob, cons):
    import torch
    import paper_2304_09770_b200 as vb
    ctx = vb.context_for(prob, constraints=cons)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-8)          # the paper's stopping rule
    ctx.close()
    return rep


def main():
    from synthetic import make_problem
    neu = ("x1", "y1") if "--neumann" in sys.argv else None
    ks = (2, 3, 4) if neu else (2, 3)
    if neu:
        print("Neumann faces x = 1, y = 1 (homogeneous traction), Dirichlet elsewhere")
    spaces = {
        "minimal (vertex+flux)": dict(vertex=1, edge_avg=0, face_avg=0, face_flux=1, adaptive_tau=0.0),
        "BASELINE (vertex+edge+face)": dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0),
        "adaptive tau=2": dict(vertex=1, edge_avg=1, face_avg=0, face_flux=1, adaptive_tau=2.0),
    }
    print("H/h sweep: 4^3 subdomains, k = 2, nu = 1, rtol 1e-8")
    print("%-30s %6s %10s %8s %10s %8s" % ("space", "H/h", "nDofs", "N_Pi", "iterations", "kappa"))
    for name, cons in spaces.items():
        for hh in (2, 3, 4, 6):
            prob = make_problem("c2", n=4 * hh, sub=(hh, hh, hh), neumann=neu)
            rep = run(prob, cons)
            print("%-30s %6d %10d %8d %10d %8.2f" % (name, hh, rep["n_dofs_paper"], rep["n_primal"],
                                                     rep["iterations"], rep["kappa"]), flush=True)
    print("\nk sweep: CUBE 8^3, 2^3 subdomains, nu = 1, rtol 1e-8")
    for name, cons in spaces.items():
        for k in ks:
            prob = make_problem("c1", n=8, sub=(4, 4, 4), k=k, neumann=neu)
            try:
                rep = run(prob, cons)
            except Exception as e:   # e.g. adaptive k = 4 faces beyond the Jacobi GEVP kernel (EINVAL)
                print("%-30s k=%d  not run: %s" % (name, k, e), flush=True)
                continue
            print("%-30s k=%d %10d %8d %10d %8.2f" % (name, k, rep["n_dofs_paper"], rep["n_primal"],
                                                      rep["iterations"], rep["kappa"]), flush=True)


if __name__ == "__main__":
    main()
