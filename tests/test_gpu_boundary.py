"""C-ABI boundary conformance on the GPU:
* a flux-incompatible rhs (pressure rows not integrating to zero against constants)
  returns VB_EINVAL instead of being silently projected;
* vb_set_option("true_residual") fills vb_report.true_rel_residual with ||b - K x|| / ||b|| of the
  full saddle system through the element-by-element operator K7;
* vb_report.flux_violation_max = max_i |b_0^(i) x_Gamma| of the final iterate (benign space,
  Assumption ass1 P:526-528) is at rounding level;
* a wrong-signed velocity pivot (an element matrix with negative energy) is VB_ESINGULAR naming
  the subdomain (relative, signed pivot test: velocity > 0, pressure < 0, reading A5);
* the NCCL transport runs eagerly and captured inside a conditional WHILE graph body on one GPU.
"""
import numpy as np
import pytest

from synthetic import make_problem

pytestmark = pytest.mark.gpu


def _ctx_rhs(prob, **kw):
    import torch
    import paper_2304_09770_b200 as vb
    ctx = vb.context_for(prob, **kw)
    ctx.factor()
    rhs = torch.zeros(ctx.n_free, dtype=torch.float64, device="cuda")
    ctx.build_rhs(vb.problem_args(prob), rhs)
    return ctx, rhs


def test_flux_incompatible_rhs_is_einval():
    import torch
    import paper_2304_09770_b200 as vb
    prob = make_problem("c1")
    ctx, rhs = _ctx_rhs(prob)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x)                                  # compatible: converges
    assert rep["status"] == "OK"
    bad = rhs.clone()
    bad[ctx.n_vel] += 1.0                                        # constant-mode DOF of cell 0
    with pytest.raises(vb.VBError) as ei:
        ctx.pcg_solve(bad, x)
    assert ei.value.status == vb.VB_EINVAL and "flux-incompatible" in str(ei.value)
    # the context stays usable
    rep = ctx.pcg_solve(rhs, x)
    assert rep["status"] == "OK"


@pytest.mark.parametrize("name,kw", [("c1", {}), ("c3", dict(n=4, sub=(2, 2, 2)))])
def test_true_residual_and_flux_violation(name, kw):
    import torch
    prob = make_problem(name, **kw)
    ctx, rhs = _ctx_rhs(prob)
    x = torch.zeros_like(rhs)
    rep = ctx.pcg_solve(rhs, x)
    assert rep["true_rel_residual"] == -1.0                      # off by default (no extra pass)
    ctx.set_option("true_residual", 1)
    rep = ctx.pcg_solve(rhs, x)
    y = torch.zeros_like(rhs)
    ctx.apply_operator(x, y)
    ref = float(torch.linalg.norm(rhs - y) / torch.linalg.norm(rhs))
    assert 0 <= rep["true_rel_residual"] <= 1e-8
    assert abs(rep["true_rel_residual"] - ref) <= 1e-3 * ref + 1e-15
    assert rep["flux_violation_max"] <= 1e-12 * float(torch.linalg.norm(x))


def test_wrong_sign_pivot_names_subdomain():
    import paper_2304_09770_b200 as vb
    from oracle.assemble import GlobalSystem
    prob = make_problem("c1")
    gs = GlobalSystem(prob)
    pa, A, pb, B = [0], [], [0], []
    bad_sub = 3
    for K in range(prob.mesh.n_cells):
        op = gs.el.op(K)
        sgn = -1.0 if prob.cell_subdomain[K] == bad_sub else 1.0
        A.append((sgn * prob.nu_cell[K] * op.A).ravel()); B.append(op.B.ravel())
        pa.append(pa[-1] + op.A.size); pb.append(pb[-1] + op.B.size)
    ctx = vb.context_for(prob, elements=(np.array(pa), np.concatenate(A), np.array(pb), np.concatenate(B)))
    with pytest.raises(vb.VBError) as ei:
        ctx.factor()
    assert ei.value.status == vb.VB_ESINGULAR
    assert "subdomain %d" % bad_sub in str(ei.value) and "Dirichlet" in str(ei.value)


def test_nccl_transport_selftest():
    import torch  # noqa: F401  (loads torch's libnccl into the process)
    import paper_2304_09770_b200 as vb
    r = vb.nccl_selftest(0)
    assert r["eager_ok"], r
    print("NCCL graph capture:", r)
    assert r["graph_ok"] and r["graph_iterations"] == 3, r


def test_binding_rejects_bad_buffers():
    import torch
    prob = make_problem("c1")
    ctx, rhs = _ctx_rhs(prob)
    x = torch.zeros_like(rhs)
    for bad in (rhs.float(), rhs.cpu(), rhs[:-1], torch.zeros(2 * ctx.n_free, dtype=torch.float64,
                                                               device="cuda")[::2]):
        with pytest.raises(ValueError):
            ctx.pcg_solve(bad, x)
    with pytest.raises(ValueError):
        ctx.pcg_solve_host(rhs.cpu().numpy().astype(np.float32), np.zeros(ctx.n_free))


def test_coarse_options_state_machine():
    """vb_set_option("coarse_dissection" / "coarse_blocks") are read by vb_factor: VB_ESTATE after
    it; unknown option names are VB_EINVAL; the auto rule picks the dense inverse for a small coarse
    problem (c1: N_c = 65) and the blocked dissection for N_c >= 4096 (include/vbddc.h)."""
    import paper_2304_09770_b200 as vb
    from synthetic import make_problem
    ctx = vb.context_for(make_problem("c1"))
    with pytest.raises(vb.VBError) as e:
        ctx.set_option("coarse_nonsense", 1)
    assert e.value.status == vb.VB_EINVAL
    ctx.factor()
    assert ctx.stats()["n_coarse_root"] == 0          # auto: dense inverse for N_c = 65
    for name in ("coarse_dissection", "coarse_blocks"):
        with pytest.raises(vb.VBError) as e:
            ctx.set_option(name, 1)
        assert e.value.status == vb.VB_ESTATE
    ctx.close()
