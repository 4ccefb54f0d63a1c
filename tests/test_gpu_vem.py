"""Device VEM (K9) parity: element matrices, rhs and full solves through the product path
(vb_setup generates A^K, B^K on the GPU; vb_build_rhs builds the load and lifting on the GPU).
Gates: element matrices <= 1e-12 relative; solution <= 1e-8; iterations +-1;
Lanczos kappa within 1%."""
import numpy as np
import pytest

from synthetic import make_problem

pytestmark = pytest.mark.gpu

# c4 here without the adaptive enrichment (the adaptive path has its own test)
CASES = [("c1", {}), ("c3", dict(n=4, sub=(2, 2, 2))), ("c1", dict(n=4, k=3)),
         ("c4", dict(n=8, sub=(4, 4, 4), constraints=dict(adaptive_tau=0.0))),
         ("c1", dict(n=4, k=4)), ("c3", dict(n=4, sub=(2, 2, 2), k=4))]


def _ctx(prob):
    import paper_2304_09770_b200 as vb
    return vb.context_for(prob)


@pytest.mark.parametrize("name,kw", CASES)
def test_element_matrices_parity(name, kw):
    from oracle.assemble import GlobalSystem
    prob = make_problem(name, **kw)
    gs = GlobalSystem(prob)
    ctx = _ctx(prob)
    worst = 0.0
    for K in range(0, prob.mesh.n_cells, max(1, prob.mesh.n_cells // 23)):
        A, B = ctx.element_matrices(K)
        op = gs.el.op(K)
        Ao, Bo = prob.nu_cell[K] * op.A, op.B
        worst = max(worst, np.abs(A - Ao).max() / np.abs(Ao).max(), np.abs(B - Bo).max() / np.abs(Bo).max())
    assert worst < 1e-12, worst


@pytest.mark.parametrize("name,kw", CASES)
def test_rhs_and_operator_parity(name, kw):
    import torch
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    prob = make_problem(name, **kw)
    gs = GlobalSystem(prob)
    ctx = _ctx(prob)
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    ref = np.concatenate([gs.rhs_u, gs.rhs_p])
    got = rhs.cpu().numpy()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
    # element-by-element saddle operator K7 vs the assembled oracle matrix
    rng = np.random.default_rng(3)
    x = rng.standard_normal(ctx.n_free)
    y = torch.zeros_like(rhs)
    ctx.apply_operator(torch.tensor(x, device="cuda"), y)
    yo = gs.saddle_matrix() @ x
    assert np.linalg.norm(y.cpu().numpy() - yo) <= 1e-12 * np.linalg.norm(yo)


@pytest.mark.parametrize("name,kw", CASES)
def test_full_solve_parity(name, kw):
    import torch
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem(name, **kw)
    gs = GlobalSystem(prob)
    u_o, p_o, rep_o = BDDC(gs).solve(rtol=1e-10)
    ctx = _ctx(prob)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    xh = x.cpu().numpy()
    du = np.linalg.norm(xh[:ctx.n_vel] - u_o) / np.linalg.norm(u_o)
    dp = np.linalg.norm(xh[ctx.n_vel:] - p_o) / np.linalg.norm(p_o)
    assert rep["rel_residual"] <= 1e-10
    # +-1 iteration, also for the non-adaptive sinker (kappa ~ 270, ~85 iterations)
    assert abs(rep["iterations"] - rep_o["iterations"]) <= 1, (rep["iterations"], rep_o["iterations"])
    assert abs(rep["kappa"] - rep_o["kappa"]) <= 0.01 * rep_o["kappa"]
    assert du <= 1e-8 and dp <= 1e-8, (du, dp)
    # the true full-system residual through the element-by-element operator
    y = torch.zeros_like(rhs)
    ctx.apply_operator(x, y)
    res = (rhs - y).cpu().numpy()
    assert np.linalg.norm(res[:ctx.n_vel]) <= 1e-8 * np.linalg.norm(rhs.cpu().numpy())


def load_golden(name):
    """Oracle results at full size, written by tools/make_oracle_golden.py (oracle/ only)."""
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_%s_full.npz" % name)
    z = np.load(path)
    return z, json.loads(str(z["meta"]))


def check_against_golden(ctx, rhs, x, rep, name):
    """SURVEY §8(c) gates against the stored full-size oracle solve: the WHOLE solution vector,
    velocity and pressure blocks separately at relative L2 <= 1e-8 (pressures both zero-mean),
    final relative residual <= 1e-10, iterations +-1, kappa 1 %, counts exact; the rhs on a seeded
    sample of entries and in norm."""
    z, meta = load_golden(name)
    nv = meta["n_free_vel"]
    assert ctx.n_vel == nv and ctx.n_free == nv + meta["n_pres"]
    assert rep["n_dofs_paper"] == meta["n_dofs_paper"]
    assert rep["n_primal"] == meta["n_primal"] and rep["n_coarse"] == meta["n_coarse"]
    idx = z["idx"]
    rh = rhs.cpu().numpy()
    assert abs(np.linalg.norm(rh) - meta["norm_rhs"]) <= 1e-12 * meta["norm_rhs"]
    assert np.abs(rh[idx] - z["rhs"]).max() <= 1e-12 * meta["norm_rhs"]
    xh = x.cpu().numpy()
    xo = z["x_full"]
    du = np.linalg.norm(xh[:nv] - xo[:nv]) / np.linalg.norm(xo[:nv])
    dp = np.linalg.norm(xh[nv:] - xo[nv:]) / np.linalg.norm(xo[nv:])
    assert du <= 1e-8 and dp <= 1e-8, (du, dp)
    assert rep["rel_residual"] <= 1e-10
    assert abs(rep["iterations"] - meta["iterations"]) <= 1, (rep["iterations"], meta["iterations"])
    assert abs(rep["kappa"] - meta["kappa"]) <= 0.01 * meta["kappa"], (rep["kappa"], meta["kappa"])
    print("%s full-size parity: du %.2e dp %.2e it %d (oracle %d) kappa %.6f (oracle %.6f)"
          % (name, du, dp, rep["iterations"], meta["iterations"], rep["kappa"], meta["kappa"]))
    return meta


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_full_size_parity(name):
    """BASELINE configs 2, 3 and 5 (the bench workload, in bench.py's launch configuration: one
    GPU, 32^3 cells, 512 subdomains) at full size: GPU product path vs the stored oracle solve
    (whole solution vector; config 4 with its adaptive enrichment: test_gpu_adaptive.py)."""
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic.configs import C5_DIMS
    prob = make_problem(name, dims=C5_DIMS[1]) if name == "c5" else make_problem(name)
    ctx = _ctx(prob)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    check_against_golden(ctx, rhs, x, rep, name)


def test_c5_full_size_properties():
    """Config 5 (the bench workload) at full size in bench.py's launch configuration: the oracle
    cannot solve it in seconds, so check sampled element matrices against the oracle cell by cell,
    and size-independent properties: convergence, true residual of the full system (K7), discrete
    divergence-freeness (pressure rows), lambda_min ~ 1 (Theorem teoEst)."""
    import torch
    import paper_2304_09770_b200 as vb
    from synthetic.configs import C5_DIMS
    from oracle.vem import ElementOps, mesh_edges, EdgeIndex
    prob = make_problem("c5", dims=C5_DIMS[1])
    ctx = _ctx(prob)
    ei = EdgeIndex(mesh_edges(prob.mesh), prob.mesh.n_vertices)
    for K in np.random.default_rng(5).choice(prob.mesh.n_cells, 6, replace=False):
        op = ElementOps(prob.mesh, int(K), ei, 2, prob.nu_cell[K])
        A, B = ctx.element_matrices(int(K))
        assert np.abs(A - op.A).max() <= 1e-12 * np.abs(op.A).max()
        assert np.abs(B - op.B).max() <= 1e-12 * np.abs(op.B).max()
    ctx.factor()
    st = ctx.stats()
    assert st["n_dofs_paper"] == 954947 and st["n_primal"] == 8589 and st["n_coarse"] == 9101
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    assert rep["rel_residual"] <= 1e-10 and 0.999 <= rep["lambda_min"] <= 1.01
    y = torch.zeros_like(rhs)
    ctx.apply_operator(x, y)
    res = (rhs - y).cpu().numpy()
    nb = np.linalg.norm(rhs.cpu().numpy())
    assert np.linalg.norm(res[:ctx.n_vel]) <= 1e-8 * nb
    assert np.linalg.norm(res[ctx.n_vel:]) <= 1e-8 * nb     # B u = g (discrete div-free)


def test_c3_full_size_properties():
    """Config 3 at full size (k = 3, triangulated faces, jittered vertices, 478,387 DOFs): the dense
    oracle does not fit a CPU host, so check sampled element matrices against the oracle cell by
    cell, the DOF counts against the oracle's DOF map, and size-independent properties: convergence,
    true residual of the full system, lambda_min ~ 1 (Theorem teoEst)."""
    import torch
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalDofs
    from oracle.vem import ElementOps, mesh_edges, EdgeIndex
    prob = make_problem("c3")
    ctx = _ctx(prob)
    dofs = GlobalDofs(prob.mesh, 3)
    assert ctx.n_vel == dofs.n_free_vel and ctx.n_free == dofs.n_free_vel + dofs.npres
    ei = EdgeIndex(mesh_edges(prob.mesh), prob.mesh.n_vertices)
    worst = 0.0
    for K in np.random.default_rng(3).choice(prob.mesh.n_cells, 6, replace=False):
        op = ElementOps(prob.mesh, int(K), ei, 3, prob.nu_cell[K])
        A, B = ctx.element_matrices(int(K))
        worst = max(worst, np.abs(A - op.A).max() / np.abs(op.A).max(), np.abs(B - op.B).max() / np.abs(op.B).max())
    print("c3 sampled element matrices: worst relative entry difference %.2e" % worst)
    assert worst <= 1e-12, worst
    ctx.factor()
    st = ctx.stats()
    assert st["n_dofs_paper"] == dofs.n_dofs_paper()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)
    assert rep["status"] == "OK" and rep["rel_residual"] <= 1e-10 and 0.999 <= rep["lambda_min"] <= 1.01
    y = torch.zeros_like(rhs)
    ctx.apply_operator(x, y)
    res = (rhs - y).cpu().numpy()
    nb = np.linalg.norm(rhs.cpu().numpy())
    assert np.linalg.norm(res[:ctx.n_vel]) <= 1e-8 * nb
    assert np.linalg.norm(res[ctx.n_vel:]) <= 1e-8 * nb


def test_k4_dof_count_table3():
    """k = 4 (T3 row CUBE 512 k=4): the GPU DOF numbering gives the paper's 76,387
    nDofs on the 8^3 cube, and one solve converges to the oracle-pinned gates of test_full_solve_parity."""
    import paper_2304_09770_b200 as vb
    prob = make_problem("c1", n=8, k=4, sub=(4, 4, 4))
    ctx = vb.context_for(prob)
    assert ctx.stats()["n_dofs_paper"] == 76387


@pytest.mark.parametrize("case", ["hex_k2", "hex_jitter_k2", "cvt_k2", "hex_k3"])
def test_k7_kernel_variants_match_oracle(case, monkeypatch):
    """Every K7 kernel (the persistent pipelined kernels with lane-pair and warp-per-row
    consumers, ragged stage counts, the one-cell-per-CTA bulk kernel, the streaming kernel) against
    the oracle's assembled saddle matrix; CVT cells have ragged nv (bulk sizes vary per cell), k = 3
    hexahedra exceed the staged kernels' shared memory (fallback path)."""
    import torch
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    from synthetic import make_cvt_problem
    prob = {"hex_k2": lambda: make_problem("c1"), "hex_jitter_k2": lambda: make_problem("c3", n=4, sub=(2, 2, 2), k=2),
            "cvt_k2": lambda: make_cvt_problem(4, grid=(2, 2, 1), k=2),
            "hex_k3": lambda: make_problem("c1", n=4, k=3)}[case]()
    gs = GlobalSystem(prob)
    ctx = _ctx(prob)
    x = np.random.default_rng(11).standard_normal(ctx.n_free)
    yo = gs.saddle_matrix() @ x
    xd = torch.tensor(x, device="cuda")
    variants = [{}, {"VB_K7_PIPE": "1"}, {"VB_K7_PIPE": "2"}, {"VB_K7_PIPE": "0"}, {"VB_K7_STREAM": "1"},
                {"VB_K7_PIPE": "1", "VB_K7_STAGES": "5", "VB_K7_CTAS": "1", "VB_K7_TPR": "4", "VB_K7_CONS": "128"},
                {"VB_K7_PIPE": "2", "VB_K7_STAGES": "3", "VB_K7_CTAS": "2", "VB_K7_CONS": "64"},
                {"VB_K7_PIPE": "2", "VB_K7_STAGES": "1", "VB_K7_CTAS": "1", "VB_K7_CONS": "256"}]
    knobs = ("VB_K7_PIPE", "VB_K7_STREAM", "VB_K7_STAGES", "VB_K7_CTAS", "VB_K7_TPR", "VB_K7_CONS")
    for env in variants:
        for k in knobs:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        y = torch.full_like(xd, float("nan"))
        ctx.apply_operator(xd, y)
        err = np.linalg.norm(y.cpu().numpy() - yo) / np.linalg.norm(yo)
        assert err <= 1e-11, (env, err)
