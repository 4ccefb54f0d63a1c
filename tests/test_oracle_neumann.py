"""Oracle pins for the paper's Neumann setting ("Neumann boundary conditions on two faces of
the cube and homogeneous Dirichlet boundary conditions on the other ones"; DESIGN A35): homogeneous
traction on the faces x = 1 and y = 1, the DOFs of those faces free and on the subdomain interface.

Pinned against things other than the oracle's own BDDC arithmetic:
  * the global saddle matrix: with Dirichlet data everywhere the constant pressure is in the kernel
    of B^T (int div v = 0 for v in H^1_0), with Neumann faces it is not (the pressure is unique) --
    so a Neumann marking that is silently ignored fails;
  * the BDDC-PCG solution equals a sparse direct solve of the global system (library LU, no gauge);
  * every interface DOF primal: S~ = S^, one CG step (the exact limit);
  * lambda_min of the preconditioned operator >= 1 (BDDC lower bound);
  * the entity structure of a 2x2x2 box partition: one single-sharer face entity (a Neumann patch
    with its flux row) per subdomain touching the Neumann faces, the lines where two subdomains
    meet on the Neumann faces as edges, the point where four meet as a vertex.
"""
import numpy as np
import pytest

from synthetic import make_problem
from synthetic.mesh import mark_neumann, hex_mesh

NEU = ("x1", "y1")


def test_mark_neumann_counts():
    m = mark_neumann(hex_mesh(4), NEU)
    fb = m.face_on_boundary
    assert int(np.sum(fb == 2)) == 2 * 16 and int(np.sum(fb == 1)) == 4 * 16
    assert int(np.sum(hex_mesh(4).face_on_boundary == 1)) == 6 * 16


def test_constant_pressure_leaves_kernel():
    from oracle.assemble import GlobalSystem
    for neu, zero in ((None, True), (NEU, False)):
        gs = GlobalSystem(make_problem("c1", neumann=neu))
        # the DOF vector of q = 1 (D_Q of the constant, per subdomain c_i)
        from oracle.bddc import BDDC
        b = BDDC(gs)
        cg = np.zeros(gs.dofs.npres)
        for S in b.sub:
            cg[S.P] = S.c
        v = gs.Bf.T @ cg
        scale = np.abs(gs.Bf).sum()
        if zero:
            assert np.linalg.norm(v) <= 1e-12 * scale
        else:
            assert np.linalg.norm(v) >= 1e-3 * np.linalg.norm(gs.Bf.data)


@pytest.mark.parametrize("kw", [dict(), dict(k=3), dict(n=6, sub=(3, 3, 3))])
def test_bddc_equals_direct_solve(kw):
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    gs = GlobalSystem(make_problem("c1", neumann=NEU, **kw))
    ud, pd = gs.direct_solve()
    # the direct solve itself: residual of the unreduced saddle system
    K = gs.saddle_matrix()
    rhs = np.concatenate([gs.rhs_u, gs.rhs_p])
    assert np.linalg.norm(K @ np.concatenate([ud, pd]) - rhs) <= 1e-10 * np.linalg.norm(rhs)
    u, p, rep = BDDC(gs).solve(rtol=1e-12)
    assert rep["status"] == "ok"
    assert np.linalg.norm(u - ud) <= 1e-9 * np.linalg.norm(ud)
    assert np.linalg.norm(p - pd) <= 1e-9 * np.linalg.norm(pd)
    assert rep["lambda_min"] >= 1.0 - 1e-8


def test_exact_limit_all_primal():
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    gs = GlobalSystem(make_problem("c1", neumann=NEU))
    u, p, rep = BDDC(gs, constraints=dict(all_primal=1)).solve(rtol=1e-10)
    assert rep["iterations"] == 1
    ud, pd = gs.direct_solve()
    assert np.linalg.norm(u - ud) <= 1e-9 * np.linalg.norm(ud)


def test_entity_structure():
    from oracle.assemble import GlobalSystem
    from oracle.bddc import BDDC
    gs = GlobalSystem(make_problem("c1", neumann=NEU))     # 4^3 cells, 2x2x2 subdomains
    b = BDDC(gs)
    dofs = gs.dofs
    onN = dofs.free_on_neumann
    neu_ents = [E for E in b.ents if np.all(onN[E.dofs])]
    assert all(not np.any(onN[E.dofs]) for E in b.ents if E not in neu_ents)
    single = [E for E in neu_ents if len(E.sharers) == 1]
    # subdomains touching x = 1 or y = 1: 6 of 8, each with one Neumann patch (face: average + flux;
    # on a planar patch the flux row is the normal average, so 3 primal DOFs survive the SVD filter,
    # 4 on the two patches folded over the edge x = y = 1)
    assert len(single) == 6 and all(E.kind == "face" for E in single)
    assert sorted(E.r for E in single) == [3, 3, 3, 3, 4, 4]
    # lines where two subdomains meet on the Neumann faces: edges (vertex/edge DOFs, no face
    # moments), 3 on x = 1, 3 on y = 1, and the L-shaped one at z = 1/2 over the fold shared by the
    # two subdomains in the corner x, y > 1/2 (counted once): 7
    two = [E for E in neu_ents if len(E.sharers) == 2]
    assert len(two) == 7 and all(E.kind == "edge" and E.r == 3 for E in two)
    four = [E for E in neu_ents if len(E.sharers) == 4]
    assert len(four) == 2 and all(E.kind == "vertex" for E in four)
    # Dirichlet run of the same mesh has no Neumann entity and no single-sharer entity
    b0 = BDDC(GlobalSystem(make_problem("c1")))
    assert all(len(E.sharers) >= 2 for E in b0.ents)
