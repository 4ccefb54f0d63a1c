"""Edge and degenerate cases of the GPU path: a single subdomain (no interface),
every interface DOF primal (M^-1 = S^-1, one iteration), multiplicity scaling
(Eq.(pseudoinv)) against the oracle, the exact viscosity invariance nu -> c nu (F9),
maxit reached (VB_ENOTCONV, "NC" P:1233) and out-of-order calls."""
import numpy as np
import pytest

from synthetic import make_problem

pytestmark = pytest.mark.gpu


def _gpu_solve(prob, rtol=1e-10, maxit=2000, raise_on_error=True, **kw):
    import torch
    import paper_2304_09770_b200 as vb
    ctx = vb.context_for(prob, **kw)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=rtol, maxit=maxit, raise_on_error=raise_on_error)
    return ctx, rhs, x, rep


def test_single_subdomain_direct():
    """One subdomain: no interface, the coarse problem is the single p0 (gauge-fixed to 0); the
    solve is the back-substitution alone and must equal the dense direct solve of Eq.(MatrixForm)."""
    import torch
    from oracle.assemble import GlobalSystem
    prob = make_problem("c1", sub=(4, 4, 4))
    assert int(prob.cell_subdomain.max()) == 0
    ctx, rhs, x, rep = _gpu_solve(prob)
    assert rep["iterations"] == 0 and rep["status"] == "OK"
    gs = GlobalSystem(prob)
    u, p = gs.direct_solve()
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh[:ctx.n_vel] - u) <= 1e-10 * np.linalg.norm(u)
    assert np.linalg.norm(xh[ctx.n_vel:] - p) <= 1e-10 * np.linalg.norm(p)


def test_all_primal_exact_limit():
    """Every interface DOF primal: S~ = S^, so M^-1 S^ = I on the benign space and CG stops after
    one step; the oracle does the same."""
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem("c1")
    ctx, rhs, x, rep = _gpu_solve(prob, constraints=dict(all_primal=1))
    assert rep["iterations"] == 1
    u_o, p_o, rep_o = BDDC(GlobalSystem(prob), constraints=dict(all_primal=1)).solve()
    assert rep_o["iterations"] == 1
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh[:ctx.n_vel] - u_o) <= 1e-8 * np.linalg.norm(u_o)


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c1", dict(n=8))])
def test_multiplicity_scaling_parity(name, kw):
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    prob = make_problem(name, **kw)
    ctx, rhs, x, rep = _gpu_solve(prob, constraints=dict(scaling=vb.VB_MULTIPLICITY))
    u_o, p_o, rep_o = BDDC(GlobalSystem(prob), scaling="multiplicity").solve()
    assert abs(rep["iterations"] - rep_o["iterations"]) <= 1
    assert abs(rep["kappa"] - rep_o["kappa"]) <= 0.01 * rep_o["kappa"]
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh[:ctx.n_vel] - u_o) <= 1e-8 * np.linalg.norm(u_o)
    assert np.linalg.norm(xh[ctx.n_vel:] - p_o) <= 1e-8 * np.linalg.norm(p_o)


@pytest.mark.parametrize("name,kw", [("c1", dict(n=8)), ("c1", dict(n=8, k=3)),
                                     ("c3", dict(n=8, sub=(2, 2, 2)))])
def test_minimal_coarse_space_parity(name, kw):
    """The paper's minimal primal space: vertices + face fluxes only (nu_tol = infinity, P:1197-1199;
    SURVEY f3), against the oracle with the same constraints (SURVEY §8(c) gates)."""
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    cons = dict(vertex=1, edge_avg=0, face_avg=0, face_flux=1)
    prob = make_problem(name, constraints=cons, **kw)
    ctx, rhs, x, rep = _gpu_solve(prob)
    u_o, p_o, rep_o = BDDC(GlobalSystem(prob)).solve()
    assert rep["n_primal"] == rep_o["n_primal"]
    assert abs(rep["iterations"] - rep_o["iterations"]) <= 1, (rep["iterations"], rep_o["iterations"])
    assert abs(rep["kappa"] - rep_o["kappa"]) <= 0.01 * rep_o["kappa"]
    xh = x.cpu().numpy()
    assert np.linalg.norm(xh[:ctx.n_vel] - u_o) <= 1e-8 * np.linalg.norm(u_o)
    assert np.linalg.norm(xh[ctx.n_vel:] - p_o) <= 1e-8 * np.linalg.norm(p_o)


def test_viscosity_scaling_invariance():
    """F9: nu -> 1000 nu with the same rhs: identical iterations and kappa, u / 1000, p unchanged."""
    import torch
    import paper_2304_09770_b200 as vb
    p1 = make_problem("c1", n=8)
    p2 = make_problem("c1", n=8, nu=1000.0)
    c1, rhs, x1, r1 = _gpu_solve(p1)
    c2 = vb.context_for(p2)
    c2.factor()
    x2 = torch.zeros_like(rhs)
    r2 = c2.pcg_solve(rhs, x2, rtol=1e-10)
    assert r1["iterations"] == r2["iterations"]
    assert abs(r1["kappa"] - r2["kappa"]) <= 1e-8 * r1["kappa"]
    a, b = x1.cpu().numpy(), x2.cpu().numpy()
    nv = c1.n_vel
    assert np.linalg.norm(a[:nv] - 1000.0 * b[:nv]) <= 1e-9 * np.linalg.norm(a[:nv])
    assert np.linalg.norm(a[nv:] - b[nv:]) <= 1e-9 * np.linalg.norm(a[nv:])


def test_maxit_and_state_errors():
    import torch
    import paper_2304_09770_b200 as vb
    prob = make_problem("c1", n=8)
    ctx = vb.context_for(prob)
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(rhs)
    with pytest.raises(vb.VBError) as e:     # solve before factor
        ctx.pcg_solve(rhs, x)
    assert e.value.status == vb.VB_ESTATE
    ctx.factor()
    ctx.build_rhs(vb.problem_args(prob), rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-14, maxit=3, raise_on_error=False)
    assert rep["status"] == "ENOTCONV" and rep["iterations"] == 3
    assert rep["rel_residual"] > 1e-14
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10)          # the context is still usable
    assert rep["status"] == "OK"


def test_two_contexts_interleaved():
    """Two live contexts of different subdomain sizes in one process, solved alternately: kernel
    launch limits are process-wide, so preparing the small one must not break the large one, and
    each keeps its own results (bitwise repeatable solves)."""
    import torch
    import paper_2304_09770_b200 as vb
    big = make_problem("c1", n=8, sub=(4, 4, 4))
    small = make_problem("c1")
    cb, rb, xb, repb = _gpu_solve(big)
    cs, rs, xs, reps = _gpu_solve(small)
    xb2 = torch.zeros_like(xb)
    rep2 = cb.pcg_solve(rb, xb2, rtol=1e-10)
    assert rep2["iterations"] == repb["iterations"] and torch.equal(xb2, xb)
    xs2 = torch.zeros_like(xs)
    rep3 = cs.pcg_solve(rs, xs2, rtol=1e-10)
    assert rep3["iterations"] == reps["iterations"] and torch.equal(xs2, xs)
    cb.close()
    cs.close()


def test_large_subdomains_big_gemv():
    """Subdomains of 9^3 cells (n_D ~ 17.6k): the packed-GEMV vectors exceed shared memory, so the
    subdomain GEMVs run the L2-vector (BIG) variant.  The discrete solution is unique, so it must equal
    the solve of the same mesh with 3^3-cell subdomains (shared-memory GEMVs); both reach the true
    residual of the element-by-element operator, and lambda_min ~ 1 (Theorem teoEst)."""
    import torch
    import paper_2304_09770_b200 as vb
    pb = make_problem("c1", n=18, sub=(9, 9, 9))
    ps = make_problem("c1", n=18, sub=(3, 3, 3))
    cb, rb, xb, repb = _gpu_solve(pb)
    assert max(cb.stats()["max_n"], 1) > 17000
    cs, rs, xs, reps = _gpu_solve(ps)
    assert torch.equal(rb, rs)
    for c, r, x, rep in ((cb, rb, xb, repb), (cs, rs, xs, reps)):
        assert rep["status"] == "OK" and 0.999 <= rep["lambda_min"] <= 1.01
        y = torch.zeros_like(r)
        c.apply_operator(x, y)
        assert torch.linalg.norm(r - y) <= 1e-8 * torch.linalg.norm(r)
    nv = cb.n_vel
    assert torch.linalg.norm(xb[:nv] - xs[:nv]) <= 1e-8 * torch.linalg.norm(xs[:nv])
    assert torch.linalg.norm(xb[nv:] - xs[nv:]) <= 1e-8 * torch.linalg.norm(xs[nv:])
    cb.close()
    cs.close()


def test_refactor_then_solve():
    """vb_factor twice on one context (e.g. new viscosity data would do the same): the solve state
    is rebuilt against the new factors; the solve is bitwise that of a single factorisation."""
    import torch
    prob = make_problem("c1", n=8)
    c1, rhs, x1, r1 = _gpu_solve(prob)
    c1.factor()
    x2 = torch.zeros_like(rhs)
    r2 = c1.pcg_solve(rhs, x2, rtol=1e-10)
    assert r2["iterations"] == r1["iterations"] and torch.equal(x1, x2)
    c1.close()


def test_no_uninitialised_reads_poisoned_memory():
    """Every device allocation filled with NaN bits (VB_POISON=1, in a fresh process): a 1-rank solve,
    an adaptive solve, a 2-rank loopback solve and the coarse dissection (4 blocks on one rank; two
    levels on 2 ranks x 2 blocks) must still converge to the same answers -- no kernel
    may read memory it has not written (regression: the first CG direction once read p)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = r'''
import sys, concurrent.futures as cf, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
import paper_2304_09770_b200 as vb
from synthetic import make_problem
def solve(prob, opts=(), **kw):
    ctx = vb.context_for(prob, **kw)
    for k, v in opts: ctx.set_option(k, v)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda"); x = torch.zeros_like(rhs)
    torch.cuda.synchronize(); ctx.build_rhs(vb.problem_args(prob), rhs)
    rep = ctx.pcg_solve(rhs, x, rtol=1e-10); ids = ctx.dof_layout(); xh = x.cpu().numpy(); ctx.close()
    return rep, ids, xh
for name, kw in (("c1", dict(n=8)), ("c4", dict(n=8))):
    rep, ids, x = solve(make_problem(name, **kw))
    assert rep["status"] == "OK" and np.all(np.isfinite(x)), (name, rep)
prob = make_problem("c1", n=8)
rep1, ids1, x1 = solve(prob)
world = vb.LoopbackWorld(2); srank = vb.box_ranks(prob.sub_grid, (1, 1, 2))
streams = [torch.cuda.Stream() for _ in range(2)]
with cf.ThreadPoolExecutor(2) as ex:
    outs = list(ex.map(lambda r: solve(prob, stream=streams[r], rank=r, nranks=2, subdomain_rank=srank, world=world), range(2)))
world.close()
pos = {int(g): i for i, g in enumerate(ids1)}
xr = np.full(x1.size, np.nan)
for rep, ids, x in outs:
    assert rep["status"] == "OK"
    xr[[pos[int(g)] for g in ids]] = x
assert np.linalg.norm(xr - x1) <= 1e-10 * np.linalg.norm(x1)
# the coarse dissection over 4 blocks on one rank, and two levels (2 ranks x 2 blocks)
cd = (("coarse_dissection", 1), ("coarse_blocks", 4))
rep, ids, x = solve(prob, opts=cd)
assert rep["status"] == "OK" and np.linalg.norm(x - x1) <= 1e-10 * np.linalg.norm(x1)
world = vb.LoopbackWorld(2)
with cf.ThreadPoolExecutor(2) as ex:
    outs = list(ex.map(lambda r: solve(prob, opts=(("coarse_blocks", 2),), stream=streams[r], rank=r, nranks=2,
                                        subdomain_rank=srank, world=world), range(2)))
world.close()
xr = np.full(x1.size, np.nan)
for rep, ids, x in outs:
    assert rep["status"] == "OK"
    xr[[pos[int(g)] for g in ids]] = x
assert np.linalg.norm(xr - x1) <= 1e-10 * np.linalg.norm(x1)
print("POISON_OK")
''' % (root, os.path.join(root, "tests"))
    env = dict(os.environ, VB_POISON="1")
    r = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert "POISON_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
