"""The paper's Neumann setting on the GPU (Neumann conditions on two faces of the cube,
homogeneous Dirichlet on the others; DESIGN A35): face_on_dirichlet = 2 on x = 1 and y = 1.

Parity with the oracle (tests/test_oracle_neumann.py pins the oracle against the sparse direct solve
and the exact limit): solution blocks to relative L2 1e-8, iterations +-1, kappa within 1 %; the
dense coarse inverse, the coarse dissection over subdomain blocks, and two loopback ranks."""
import numpy as np
import pytest

from synthetic import make_problem

pytestmark = pytest.mark.gpu

NEU = ("x1", "y1")


def _gpu_solve(prob, rtol=1e-10, options=None):
    import torch
    import paper_2304_09770_b200 as vb
    ctx = vb.context_for(prob)
    for k, v in (options or {}).items():
        ctx.set_option(k, v)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=rtol)
    return ctx, rhs, x, rep


def _check(ctx, x, rep, prob, rtol=1e-10):
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    gs = GlobalSystem(prob)
    u, p, rep_o = BDDC(gs).solve(rtol=rtol)
    xh = x.cpu().numpy() if hasattr(x, "cpu") else x
    du = np.linalg.norm(xh[:ctx.n_vel] - u) / np.linalg.norm(u)
    dp = np.linalg.norm(xh[ctx.n_vel:] - p) / np.linalg.norm(p)
    assert du <= 1e-8 and dp <= 1e-8, (du, dp)
    assert abs(rep["iterations"] - rep_o["iterations"]) <= 1, (rep["iterations"], rep_o["iterations"])
    assert abs(rep["kappa"] - rep_o["kappa"]) <= 0.01 * rep_o["kappa"], (rep["kappa"], rep_o["kappa"])
    return du, dp, rep_o


@pytest.mark.parametrize("name,kw", [
    ("c1", dict()),                       # 4^3 cells, 8 subdomains, k = 2
    ("c1", dict(k=3)),
    ("c1", dict(n=6, sub=(3, 3, 3))),     # 3^3-cell subdomains
    ("c1", dict(n=8)),                    # 64 subdomains: interior subdomains without a patch
    ("c3", dict(n=4, sub=(2, 2, 2))),     # jittered, triangulated faces, k = 3
])
def test_neumann_parity(name, kw):
    prob = make_problem(name, neumann=NEU, **kw)
    ctx, rhs, x, rep = _gpu_solve(prob)
    assert rep["status"] == "OK"
    _check(ctx, x, rep, prob)


def test_neumann_one_face_and_true_residual():
    import torch
    prob = make_problem("c1", n=8, neumann=("x1",))
    ctx, rhs, x, rep = _gpu_solve(prob, options=dict(true_residual=1))
    _check(ctx, x, rep, prob)
    assert 0 <= rep["true_rel_residual"] <= 1e-8


def test_neumann_coarse_dissection():
    """Coarse dissection over subdomain blocks without the p_0 gauge: same solution."""
    prob = make_problem("c1", n=8, neumann=NEU)
    ctx, rhs, x, rep = _gpu_solve(prob, options=dict(coarse_dissection=1, coarse_blocks=4))
    _check(ctx, x, rep, prob)


def test_neumann_two_loopback_ranks():
    from test_gpu_multirank import _run_ranks, _assemble, _global_free_ids
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem("c1", n=8, neumann=NEU)
    outs = _run_ranks(prob, (2, 1, 1))
    gs = GlobalSystem(prob)
    gid = _global_free_ids(gs)                  # dof_layout ids are global (velocity, then pressure)
    pos = {int(g): i for i, g in enumerate(gid)}
    x, b = _assemble([dict(o, ids=np.array([pos[int(g)] for g in o["ids"]])) for o in outs], gid.size)
    u, p, rep_o = BDDC(gs).solve(rtol=1e-10)
    nv = gs.dofs.n_free_vel
    assert np.linalg.norm(x[:nv] - u) <= 1e-8 * np.linalg.norm(u)
    assert np.linalg.norm(x[nv:] - p) <= 1e-8 * np.linalg.norm(p)
    for o in outs:
        assert abs(o["rep"]["iterations"] - rep_o["iterations"]) <= 1
        assert np.allclose(o["x_host"], o["x"], rtol=0, atol=1e-12 * np.abs(o["x"]).max())


def test_bad_boundary_code_rejected():
    import paper_2304_09770_b200 as vb
    prob = make_problem("c1")
    fb = np.array(prob.mesh.face_on_boundary).copy()
    fb[np.nonzero(fb)[0][0]] = 3
    import dataclasses
    bad = dataclasses.replace(prob, mesh=dataclasses.replace(prob.mesh, face_on_boundary=fb))
    with pytest.raises(Exception, match="face_on_dirichlet"):
        vb.context_for(bad)


def test_neumann_cvt():
    """Voronoi cells (the paper's CVT family) with the two Neumann faces."""
    from synthetic.configs import poly_problem
    from synthetic.mesh import cvt_mesh, mark_neumann
    prob = poly_problem(mark_neumann(cvt_mesh(5, seed=20230419), NEU), (2, 2, 2), 2)
    ctx, rhs, x, rep = _gpu_solve(prob)
    _check(ctx, x, rep, prob)
