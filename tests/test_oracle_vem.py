"""Pins of the oracle's VEM discretisation against what the paper and mathematics fix.

* DOF closed forms reproduce the nDofs printed in T2-T4.
* The spaces contain [P_k]^3 x P_{k-1} (P:175-177 Remark): projectors reproduce polynomials.
* a_h^K is consistent on [P_k]^3: compared with closed-form box integrals.
* ker a_h^K = rigid modes; b exact: compared with closed-form fluxes.
* Quadrature rules vs closed-form simplex moments.
* Patch test and convergence orders (Eq.(teoConv)).
"""
import math
import numpy as np
import pytest

from synthetic import hex_mesh, make_problem
from oracle.poly import dim3, exps3, triangle_rule, tet_rule, gauss_lobatto01
from oracle.vem import ElementOps, mesh_edges, EdgeIndex
from oracle.assemble import GlobalDofs, GlobalSystem


def _ops(n, K, k, jitter=0.0, tri=False, seed=3):
    m = hex_mesh(n, jitter=jitter, seed=seed, triangulate=tri)
    ei = EdgeIndex(mesh_edges(m), m.n_vertices)
    return ElementOps(m, K, ei, k, 1.0)


# ------------------------------------------------------------------ DOF counts (F1)
def _closed_form(n, k):
    dP = lambda m: 0 if m < 0 else (m + 1) * (m + 2) * (m + 3) // 6
    nv, ne, nf, nc = (n + 1) ** 3, 3 * n * (n + 1) ** 2, 3 * n * n * (n + 1), n ** 3
    cell = 3 * dP(k - 3) - dP(k - 4) + dP(k - 1) - 1
    return 3 * nv + 3 * (k - 1) * ne + 3 * k * (k - 1) // 2 * nf + cell * nc + dP(k - 1) * nc


@pytest.mark.parametrize("n,k,printed,line", [
    (16, 2, 124195, "P:1043 T2 CUBE 4096"), (24, 2, 408243, "P:1047 T2 CUBE 13824"),
    (28, 2, 643387, "P:1049 T2 CUBE 21952"), (32, 2, 954947, "P:1051 T2 CUBE 32768"),
    (8, 2, 16787, "P:1093 T3 CUBE 512 k=2"), (8, 3, 40667, "P:1095 T3 CUBE 512 k=3"),
    (8, 4, 76387, "P:1097 T3 CUBE 512 k=4"), (24, 3, 1009803, "P:1134 T4 CUBE 13824 k=3"),
    (20, 4, 1119523, "P:1136 T4 CUBE 8000 k=4")])
def test_dof_closed_form_matches_paper(n, k, printed, line):
    assert _closed_form(n, k) == printed, line


def test_dof_typo_T2_8000():
    # P:1045 prints 239,763 for CUBE 8000 k=2; the closed form gives 238,763
    assert _closed_form(20, 2) == 238763


@pytest.mark.parametrize("n,k", [(4, 2), (8, 2), (4, 3)])
def test_global_dof_numbering_counts(n, k):
    d = GlobalDofs(hex_mesh(n), k)
    assert d.n_dofs_paper() == _closed_form(n, k)


def test_single_cube_dofs():
    op = _ops(1, 0, 2)
    assert op.L.nv == 81 and op.L.np == 4


def test_triangulated_counts():
    # 16^3 jittered+triangulated: 24,576 faces, 25,392 edges, nDofs 478,387
    m = hex_mesh(16, jitter=0.2, seed=20230419, triangulate=True)
    E = mesh_edges(m)
    assert m.n_faces == 24576 and len(E) == 25392
    d = GlobalDofs(m, 3)
    assert d.n_dofs_paper() == 478387


# ------------------------------------------------------------------ quadrature
@pytest.mark.parametrize("n", [3, 4, 5])
def test_triangle_rule_exact(n):
    a, b, c = np.zeros(3), np.array([1.0, 0, 0]), np.array([0, 1.0, 0])
    p, w = triangle_rule(a, b, c, n)
    for i in range(2 * n - 1):
        for j in range(2 * n - 1 - i):
            exact = math.factorial(i) * math.factorial(j) / math.factorial(i + j + 2)
            assert abs(np.sum(w * p[:, 0] ** i * p[:, 1] ** j) - exact) < 1e-14


@pytest.mark.parametrize("n", [4, 5, 6])
def test_tet_rule_exact(n):
    e = np.eye(3)
    p, w = tet_rule(np.zeros(3), e[0], e[1], e[2], n)
    for i in range(2 * n - 2):
        for j in range(2 * n - 2 - i):
            for l in range(2 * n - 2 - i - j):
                exact = (math.factorial(i) * math.factorial(j) * math.factorial(l)
                         / math.factorial(i + j + l + 3))
                assert abs(np.sum(w * p[:, 0] ** i * p[:, 1] ** j * p[:, 2] ** l) - exact) < 1e-14


def test_gauss_lobatto():
    x, w = gauss_lobatto01(4)
    assert np.allclose(x, [0, (1 - 1 / np.sqrt(5)) / 2, (1 + 1 / np.sqrt(5)) / 2, 1])
    assert np.allclose(w, [1 / 12, 5 / 12, 5 / 12, 1 / 12])


# ------------------------------------------------------------------ projector reproduction
CELLS = [(2, 0.0, False), (3, 0.0, False), (2, 0.2, True), (3, 0.2, True), (4, 0.0, False), (4, 0.2, True)]


@pytest.mark.parametrize("k,jit,tri", CELLS)
def test_projectors_reproduce_polynomials(k, jit, tri):
    op = _ops(3, 13, k, jit, tri)
    Dk = dim3(k)
    rng = np.random.default_rng(1)
    a = rng.standard_normal(3 * Dk)
    dofs = op.DOFpoly @ a
    for c in range(3):
        assert np.allclose(op.PiN[c] @ dofs, a[c * Dk:(c + 1) * Dk], atol=1e-10)
        assert np.allclose(op.P0[c] @ dofs, a[c * Dk:(c + 1) * Dk], atol=1e-9 if k < 4 else 1e-8)
    # Pi^0_{k-1} grad reproduces grad p exactly (degree k-1)
    E = exps3(k); idx = {e: i for i, e in enumerate(exps3(k - 1))}
    for c in range(3):
        for d in range(3):
            g = np.zeros(dim3(k - 1))
            for j, e in enumerate(E):
                if e[d] > 0:
                    ee = tuple(e[q] - (1 if q == d else 0) for q in range(3))
                    g[idx[ee]] += e[d] / op.g.h * a[c * Dk + j]
            assert np.allclose(op.Grad[c][d] @ dofs, g, atol=1e-9)


# ------------------------------------------------------------------ exact integrals on a box
def _box_int(e, lo, hi, xc, h):
    """Exact int over the box of prod ((x_i - xc_i)/h)^e_i."""
    out = 1.0
    for i in range(3):
        a, b = (lo[i] - xc[i]) / h, (hi[i] - xc[i]) / h
        out *= h * (b ** (e[i] + 1) - a ** (e[i] + 1)) / (e[i] + 1)
    return out


def _grad_coeffs(a, k, h):
    """d p_c/d x_d coefficient vectors in the degree-(k-1) basis."""
    Dk = dim3(k); E = exps3(k); idx = {e: i for i, e in enumerate(exps3(k - 1))}
    G = np.zeros((3, 3, dim3(k - 1)))
    for c in range(3):
        for j, e in enumerate(E):
            for d in range(3):
                if e[d] > 0:
                    ee = tuple(e[q] - (1 if q == d else 0) for q in range(3))
                    G[c, d, idx[ee]] += e[d] / h * a[c * Dk + j]
    return G


@pytest.mark.parametrize("k", [2, 3])
def test_consistency_on_polynomials_closed_form(k):
    """a_h^K(p,q) = int nu eps(p):eps(q) for p,q in [P_k]^3 on a box (closed-form integrals)."""
    op = _ops(2, 0, k)
    g = op.g
    lo, hi = g.X.min(0), g.X.max(0)
    E1 = exps3(k - 1)
    M = np.array([[_box_int(tuple(x + y for x, y in zip(e1, e2)), lo, hi, g.xc, g.h) for e2 in E1]
                  for e1 in E1])
    rng = np.random.default_rng(2)
    for _ in range(3):
        a, b = rng.standard_normal(3 * dim3(k)), rng.standard_normal(3 * dim3(k))
        Ga, Gb = _grad_coeffs(a, k, g.h), _grad_coeffs(b, k, g.h)
        ex = 0.0
        for c in range(3):
            for d in range(3):
                ea = 0.5 * (Ga[c, d] + Ga[d, c]); eb = 0.5 * (Gb[c, d] + Gb[d, c])
                ex += ea @ M @ eb
        got = (op.DOFpoly @ a) @ op.A @ (op.DOFpoly @ b)
        assert abs(got - ex) < 1e-10 * max(1.0, abs(ex))


@pytest.mark.parametrize("k,jit,tri", CELLS)
def test_rigid_kernel_and_psd(k, jit, tri):
    op = _ops(3, 13, k, jit, tri)
    ev = np.linalg.eigvalsh(op.A)
    scale = ev[-1]
    assert np.sum(np.abs(ev) < 1e-11 * scale) == 6          # exactly the rigid modes
    assert ev[0] > -1e-11 * scale
    rng = np.random.default_rng(5)
    for _ in range(3):
        w, t = rng.standard_normal(3), rng.standard_normal(3)
        r = op.dofs_of_field(lambda x: np.cross(w, x) + t)
        assert np.linalg.norm(op.A @ r) < 1e-11 * scale * np.linalg.norm(r)


@pytest.mark.parametrize("k", [2, 3])
def test_divergence_exact_on_box(k):
    """B row for the constant pressure = flux = int div p; full B dofs(p) = |K| * coeffs(div p)."""
    op = _ops(2, 0, k)
    g = op.g
    lo, hi = g.X.min(0), g.X.max(0)
    rng = np.random.default_rng(4)
    a = rng.standard_normal(3 * dim3(k))
    G = _grad_coeffs(a, k, g.h)
    div = G[0, 0] + G[1, 1] + G[2, 2]
    E1 = exps3(k - 1)
    exact_int = sum(div[j] * _box_int(e, lo, hi, g.xc, g.h) for j, e in enumerate(E1))
    c1 = np.array([_box_int(e, lo, hi, g.xc, g.h) for e in E1]) / g.vol     # D_Q of q = 1
    dofs = op.DOFpoly @ a
    assert abs(c1 @ (op.B @ dofs) - exact_int) < 1e-11
    assert np.allclose(op.B @ dofs, g.vol * div, atol=1e-10)


# ------------------------------------------------------------------ global patch test & orders
def _patch_fields(k):
    # divergence-free u in [P_k]^3 and p in P_{k-1}
    if k == 2:
        u = lambda x: np.stack([x[:, 1] ** 2 + x[:, 2], x[:, 2] ** 2 - x[:, 0], x[:, 0] * x[:, 1]], 1)
        lap = np.array([2.0, 2.0, 0.0])
        p = lambda x: x[:, 0] - 2 * x[:, 1] + 0.5 * x[:, 2]
        gp = np.array([1.0, -2.0, 0.5])
    else:
        u = lambda x: np.stack([x[:, 1] ** 3, x[:, 2] ** 3 + x[:, 0] ** 2, x[:, 0] * x[:, 1] ** 2], 1)
        lap = None
        p = lambda x: x[:, 0] ** 2 - x[:, 1] * x[:, 2]
        gp = None
    return u, p, lap, gp


@pytest.mark.parametrize("jit,tri", [(0.0, False), (0.2, True)])
def test_patch_test_k2(jit, tri):
    """u in [P_2]^3 div-free, p in P_1 are reproduced exactly."""
    u, p, lap, gp = _patch_fields(2)
    nu = 1.3
    f = lambda nuK: (lambda x: np.tile(-0.5 * nuK * lap - gp, (x.shape[0], 1)))
    pr = make_problem("c1", n=3, sub=(1, 1, 1))
    if tri:
        pr.mesh = hex_mesh(3, jitter=jit, seed=7, triangulate=True)
    pr.nu_cell[:] = nu
    gs = GlobalSystem(pr, u_bc=u, f_of_nu=f)
    uh, ph = gs.direct_solve()
    ui = np.zeros(gs.dofs.nvel)
    for K in range(pr.mesh.n_cells):
        op = gs.el.op(K)
        iv, _ = gs.el.l2g[K]
        sh = gs.el.shift[K]
        ui[iv] = op.dofs_of_field(lambda x: u(x + sh))
    assert np.max(np.abs(uh - ui[gs.dofs.free_vel])) < 1e-10
    # pressure: compare against the DOFs (moments) of p - mean(p)
    eh1, ep = gs.errors(uh, ph)
    mean_p = 0.5 - 1.0 + 0.25
    err = 0.0
    for K in range(pr.mesh.n_cells):
        op = gs.el.op(K); _, ip = gs.el.l2g[K]
        err += op.l2_pressure_error_sq(ph[ip], p, gs.el.shift[K], pmean=mean_p)
    assert np.sqrt(err) < 1e-10
    assert np.max(np.abs(gs.Bf @ uh + gs.B[:, gs.dofs.bnd_vel] @ gs.uD[gs.dofs.bnd_vel])) < 1e-12


@pytest.mark.slow
def test_convergence_order_k2():
    """Eq.(teoConv): |u-u_h|_1 and ||p-p_h|| decay like h^k (k=2) for the smooth solution."""
    eu, ep = [], []
    for n in (2, 4, 8):
        gs = GlobalSystem(make_problem("c1", n=n, sub=(1, 1, 1)))
        u, p = gs.direct_solve()
        a, b = gs.errors(u, p)
        eu.append(a); ep.append(b)
        assert np.max(np.abs(gs.Bf @ u + gs.B[:, gs.dofs.bnd_vel] @ gs.uD[gs.dofs.bnd_vel])) < 1e-12
    ru = np.log2(eu[1] / eu[2]); rp = np.log2(ep[1] / ep[2])
    assert 1.8 < ru < 2.3 and 1.8 < rp < 2.4, (eu, ep)


# ------------------------------------------------------------------ CVT (Voronoi) polyhedra, SURVEY f4
@pytest.fixture(scope="module")
def cvt5():
    from synthetic import cvt_mesh
    return cvt_mesh(5, seed=20230419)


def test_cvt_mesh_is_a_valid_polyhedral_partition(cvt5):
    """Planar convex faces, closed cells (sum_f s_f |f| n_f = 0), positive volumes summing to |[0,1]^3|,
    every interior face in exactly two cells with opposite signs (S:28-33 checks)."""
    m = cvt5
    from oracle.vem import face_geometry
    count = np.zeros(m.n_faces, dtype=int)
    total = 0.0
    for K in range(m.n_cells):
        fs, ss = m.cell_faces(K)
        acc = np.zeros(3)
        for f, s in zip(fs, ss):
            F = face_geometry(m, f, 2)
            X = m.xyz[m.face(f)]
            assert np.abs((X - X.mean(0)) @ F.n).max() < 1e-12          # planar
            acc += s * F.area * F.n
            count[f] += 1
        assert np.linalg.norm(acc) < 1e-13
        ei = EdgeIndex(mesh_edges(m), m.n_vertices)
        total += ElementOps(m, K, ei, 2, 1.0).g.vol
    assert abs(total - 1.0) < 1e-12
    assert np.all(count[m.face_on_boundary == 1] == 1) and np.all(count[m.face_on_boundary == 0] == 2)
    assert np.diff(m.face_ptr).max() > 4 and np.diff(m.cell_ptr).max() > 12   # genuinely polyhedral


@pytest.mark.parametrize("k", [2, 3])
def test_cvt_projectors_and_kernel(cvt5, k):
    """On Voronoi cells (up to 17 faces, 8-gon faces): projectors reproduce [P_k]^3, ker a_h^K = the
    six rigid modes, a_h^K symmetric PSD."""
    m = cvt5
    ei = EdgeIndex(mesh_edges(m), m.n_vertices)
    K = int(np.argmax(np.diff(m.cell_ptr)))          # the cell with the most faces
    op = ElementOps(m, K, ei, k, 1.0)
    Dk = dim3(k)
    a = np.random.default_rng(2).standard_normal(3 * Dk)
    dofs = op.DOFpoly @ a
    for c in range(3):
        assert np.allclose(op.PiN[c] @ dofs, a[c * Dk:(c + 1) * Dk], atol=1e-9)
        assert np.allclose(op.P0[c] @ dofs, a[c * Dk:(c + 1) * Dk], atol=1e-8)
    ev = np.linalg.eigvalsh(op.A)
    assert np.sum(np.abs(ev) < 1e-11 * ev[-1]) == 6 and ev[0] > -1e-11 * ev[-1]


def test_cvt_patch_test_k2():
    """Global patch test on the CVT mesh: div-free u in [P_2]^3 and p in P_1 reproduced exactly."""
    from synthetic import make_cvt_problem
    u, p, lap, gp = _patch_fields(2)
    f = lambda nuK: (lambda x: np.tile(-0.5 * nuK * lap - gp, (x.shape[0], 1)))
    pr = make_cvt_problem(4, grid=(1, 1, 1))
    gs = GlobalSystem(pr, u_bc=u, f_of_nu=f)
    uh, ph = gs.direct_solve()
    ui = np.zeros(gs.dofs.nvel)
    for K in range(pr.mesh.n_cells):
        op = gs.el.op(K)
        iv, _ = gs.el.l2g[K]
        ui[iv] = op.dofs_of_field(lambda x: u(x + gs.el.shift[K]))
    assert np.max(np.abs(uh - ui[gs.dofs.free_vel])) < 1e-9
    err = 0.0
    for K in range(pr.mesh.n_cells):
        op = gs.el.op(K); _, ip = gs.el.l2g[K]
        err += op.l2_pressure_error_sq(ph[ip], p, gs.el.shift[K], pmean=0.5 - 1.0 + 0.25)
    assert np.sqrt(err) < 1e-9
