"""Pins of the oracle's BDDC / PCG against what the paper and mathematics fix.

* PCG + back-substitution reproduces the sparse direct solution of Eq.(DiscProblem).
* Interface reduction: dense S^, g^ -> solve -> expand equals the direct solve.
* M^-1 symmetric; its output is benign (B_0G z = 0, Assumption ass1 P:526-528).
* lambda_min(M^-1 S^) = 1 on the benign space and Lanczos kappa ~ dense kappa (Theorem teoEst,
  P:557-564).
* All interface DOFs primal => M^-1 = S^-1 => one CG step (exact limit).
* Deluxe partition of unity sum_m D^(m) = I.
* nu -> c nu invariance.
* Adaptive eigenvalues in [0,1] and monotone selection.
* Independent brute-force constructions (bordered dense elimination of the assembled subdomain
  saddle matrix, independent null-space bases, KKT minimum-energy extension, general
  eigensolver) of S_Gamma^(i), the deluxe D_G^(m) and the adaptive face pencils; the stiffer
  side of a 1e6 viscosity jump takes the whole deluxe weight.
"""
import numpy as np
import pytest
import scipy.linalg as sla

from synthetic import make_problem
from oracle.assemble import GlobalSystem
from oracle.bddc import BDDC, lanczos_extremes


@pytest.fixture(scope="module")
def c1():
    gs = GlobalSystem(make_problem("c1"))
    return gs, BDDC(gs)


def _dense(op, n):
    return np.column_stack([op(e) for e in np.eye(n)])


def test_pcg_matches_direct(c1):
    gs, bd = c1
    ud, pd = gs.direct_solve()
    u, p, rep = bd.solve(rtol=1e-12)
    assert rep["status"] == "ok"
    assert np.linalg.norm(u - ud) / np.linalg.norm(ud) < 1e-10
    assert np.linalg.norm(p - pd) / np.linalg.norm(pd) < 1e-8
    assert bd.NPi == 57 and bd.NPi + bd.N == 65


def test_interface_reduction_bruteforce(c1):
    gs, bd = c1
    n = bd.nG + bd.N
    S = _dense(bd.apply_S, n)
    assert np.abs(S - S.T).max() < 1e-12 * np.abs(S).max()
    g = bd.condensed_rhs()
    # gauge on p0: sum vol_i p0_i = 0 (A5)
    M = np.zeros((n + 1, n + 1)); M[:n, :n] = S
    M[n, bd.nG:n] = bd.vols; M[bd.nG:n, n] = bd.vols
    x = np.linalg.solve(M, np.concatenate([g, [0.0]]))[:n]
    u, p = bd.back_substitute(x)
    ud, pd = gs.direct_solve()
    assert np.linalg.norm(u - ud) / np.linalg.norm(ud) < 1e-10
    assert np.linalg.norm(p - pd) / np.linalg.norm(pd) < 1e-9


def test_preconditioner_symmetric_and_benign(c1):
    gs, bd = c1
    n = bd.nG + bd.N
    Minv = _dense(bd.apply_M, n)
    assert np.abs(Minv - Minv.T).max() < 1e-10 * np.abs(Minv).max()
    rng = np.random.default_rng(0)
    r = rng.standard_normal(n)
    r[bd.nG:] = 0.0                          # benign residual (zero p0 block)
    z = bd.apply_M(r)
    for i, S in enumerate(bd.sub):
        assert abs(S.b0 @ z[:bd.nG][S.Gpos]) < 1e-12 * np.linalg.norm(z)
    # with a flux-compatible p0 block the coarse problem reproduces it: B_0 z = r_0
    r0 = rng.standard_normal(bd.N); r0 -= r0.mean()
    r[bd.nG:] = r0
    z = bd.apply_M(r)
    for i, S in enumerate(bd.sub):
        assert abs(S.b0 @ z[:bd.nG][S.Gpos] - r0[i]) < 1e-10 * np.linalg.norm(z)


def test_spectrum_lambda_min_one(c1):
    gs, bd = c1
    n = bd.nG + bd.N
    S = _dense(bd.apply_S, n)
    Minv = _dense(bd.apply_M, n)
    # benign subspace: B_0 u = 0 for every subdomain, p0 free; eigenvalues of M^-1 S there
    B0 = np.zeros((bd.N, n))
    for i, Sd in enumerate(bd.sub):
        B0[i, Sd.Gpos] = Sd.b0
    Q = sla.null_space(B0)
    ev = np.linalg.eigvals(np.linalg.pinv(Q) @ Minv @ S @ Q)
    ev = np.sort(ev.real[np.abs(ev) > 1e-8])
    assert abs(ev[0] - 1.0) < 1e-8
    _, rep = bd.pcg(rtol=1e-13)
    assert 0.999 <= rep["lambda_min"] <= 1.01
    assert abs(rep["kappa"] - ev[-1] / ev[0]) / (ev[-1] / ev[0]) < 0.05


def test_all_primal_one_iteration():
    gs = GlobalSystem(make_problem("c1"))
    bd = BDDC(gs, constraints=dict(all_primal=1))
    _, rep = bd.pcg(rtol=1e-10)
    assert rep["iterations"] == 1


def test_deluxe_partition_of_unity(c1):
    _, bd = c1
    for E in bd.ents:
        if E.nd:
            Ssum = sum(E.D[m] for m in E.sharers)
            assert np.allclose(Ssum, np.eye(E.nd), atol=1e-12)


def test_viscosity_scaling_invariance():
    """F9: A -> cA with the same rhs: same iterations and kappa, u/c, p unchanged."""
    p1 = make_problem("c1")
    gs1 = GlobalSystem(p1)
    p2 = make_problem("c1", nu=1000.0)
    gs2 = GlobalSystem(p2)
    gs2.rhs_u, gs2.rhs_p = gs1.rhs_u.copy(), gs1.rhs_p.copy()
    u1, q1, r1 = BDDC(gs1).solve()
    u2, q2, r2 = BDDC(gs2).solve()
    assert r1["iterations"] == r2["iterations"]
    assert abs(r1["kappa"] - r2["kappa"]) < 1e-6 * r1["kappa"]
    assert np.linalg.norm(1000 * u2 - u1) < 1e-8 * np.linalg.norm(u1)
    assert np.linalg.norm(q2 - q1) < 1e-8 * np.linalg.norm(q1)


def test_multiplicity_scaling_same_solution(c1):
    gs, bd = c1
    u, p, rep = bd.solve()
    bm = BDDC(gs, scaling="multiplicity")
    um, pm, repm = bm.solve()
    assert repm["status"] == "ok"
    assert np.linalg.norm(u - um) / np.linalg.norm(u) < 1e-8
    assert repm["iterations"] >= rep["iterations"]


def test_lanczos_tridiagonal_textbook():
    """Lanczos extremes from CG coefficients equal the extreme eigenvalues of a Jacobi-PCG problem."""
    rng = np.random.default_rng(3)
    n = 40
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = Q @ np.diag(np.linspace(1, 50, n)) @ Q.T
    Dm = np.diag(1 / np.diag(A))
    b = rng.standard_normal(n)
    x = np.zeros(n); r = b.copy(); z = Dm @ r; p = z.copy(); rz = r @ z
    al, be = [], []
    for _ in range(n):
        q = A @ p; a = rz / (p @ q); x += a * p; r -= a * q
        al.append(a); z = Dm @ r; rzn = r @ z; be.append(rzn / rz); rz = rzn; p = z + be[-1] * p
        if np.linalg.norm(r) < 1e-14:
            break
    lmin, lmax = lanczos_extremes(al, be)
    ev = np.linalg.eigvals(Dm @ A).real
    assert abs(lmin - ev.min()) < 1e-6 * ev.max() and abs(lmax - ev.max()) < 1e-6 * ev.max()


def test_adaptive_eigenvalues_and_monotone():
    pr = make_problem("c4", n=8, sub=(2, 2, 2))
    gs = GlobalSystem(pr)
    counts = []
    for tau in (2.0, 10.0, 100.0):
        bd = BDDC(gs, adaptive_tau=tau)
        counts.append(bd.adaptive_count)
        u, p, rep = bd.solve()
        assert rep["status"] == "ok" and rep["lambda_min"] > 0.999
    assert counts[0] >= counts[1] >= counts[2]


# ---------------------------------------------------------------------------------------------
# Independent brute-force constructions (the deluxe and adaptive steps were pinned
# only by invariants a plausible mistake also satisfies).

def _bf_subdomain_schur(gs, m):
    """S_Gamma^(m) by dense elimination of the BORDERED subdomain saddle matrix
    [[A, B^T, 0], [B, 0, mv], [0, mv^T, 0]] on (u, p over all cell pressure DOFs, lambda), the
    multiplier lambda imposing int p = 0 (p in Q_I; a different route from the oracle's
    Z-basis of Q_I and sparse LU).  Assembled from the element matrices of the subdomain's cells
    (Eq.(MatrixForm)).  Returns (Gamma DOF ids of m in increasing order, S)."""
    prob, dofs, el = gs.prob, gs.dofs, gs.el
    csub = prob.cell_subdomain
    owner = {}
    for K in range(prob.mesh.n_cells):
        fr = dofs.vel2free[el.l2g[K][0]]
        for d in fr[fr >= 0]:
            owner.setdefault(int(d), set()).add(int(csub[K]))
    cells = np.nonzero(csub == m)[0]
    vel = sorted({int(d) for K in cells for d in dofs.vel2free[el.l2g[K][0]] if d >= 0})
    gam = [d for d in vel if len(owner[d]) > 1]
    intr = [d for d in vel if len(owner[d]) == 1]
    pres = sorted({int(q) for K in cells for q in el.l2g[K][1]})
    lv = {d: j for j, d in enumerate(intr + gam)}
    lp = {q: j for j, q in enumerate(pres)}
    nv, npr = len(vel), len(pres)
    A = np.zeros((nv, nv)); B = np.zeros((npr, nv))
    for K in cells:
        iv, ip = el.l2g[K]
        fr = dofs.vel2free[iv]
        kp = fr >= 0
        li = [lv[int(d)] for d in fr[kp]]
        pi = [lp[int(q)] for q in ip]
        A[np.ix_(li, li)] += prob.nu_cell[K] * el.op(K).A[np.ix_(kp, kp)]
        B[np.ix_(pi, li)] += el.op(K).B[:, kp]
    mv = gs.pmass[pres]
    nI, nGm = len(intr), len(gam)
    n = nv + npr + 1
    Kb = np.zeros((n, n))
    Kb[:nv, :nv] = A; Kb[:nv, nv:nv + npr] = B.T; Kb[nv:nv + npr, :nv] = B
    Kb[nv:nv + npr, -1] = mv; Kb[-1, nv:nv + npr] = mv
    g = np.arange(nI, nI + nGm)
    o = np.concatenate([np.arange(nI), np.arange(nv, n)])
    S = Kb[np.ix_(g, g)] - Kb[np.ix_(g, o)] @ np.linalg.solve(Kb[np.ix_(o, o)], Kb[np.ix_(o, g)])
    return np.array(gam), 0.5 * (S + S.T)


def _minor(gam, S, ids):
    pos = {int(d): j for j, d in enumerate(gam)}
    j = [pos[int(d)] for d in ids]
    return S[np.ix_(j, j)]


def test_subdomain_schur_bruteforce(c1):
    """Setup-stage gate: the oracle's S_Gamma^(i) (sparse LU on the Z-basis) equals the
    bordered dense elimination, per subdomain, to 1e-11 relative (Frobenius)."""
    gs, bd = c1
    for m, S in enumerate(bd.sub):
        gam, Sbf = _bf_subdomain_schur(gs, m)
        assert sorted(S.G.tolist()) == gam.tolist()
        Sor = _minor(gam, Sbf, S.G)
        assert np.linalg.norm(S.SG - Sor) <= 1e-11 * np.linalg.norm(Sor)


def test_deluxe_bruteforce(c1):
    """D_G^(m) = (sum_m' N^T S_GG^(m') N)^-1 N^T S_GG^(m) N (SURVEY O-11) rebuilt from the
    bordered brute-force S_Gamma^(m) and an independent null-space basis N' of C_G
    (scipy null_space): the basis-invariant operators N D N^T agree for every entity and sharer.
    A swapped side, a wrong principal minor or a transposed solve fails this."""
    gs, bd = c1
    bf = {m: _bf_subdomain_schur(gs, m) for m in range(bd.N)}
    checked = 0
    for E in bd.ents:
        if E.nd == 0:
            continue
        Nn = sla.null_space(E.C) if E.r else np.eye(len(E.dofs))
        blk = {m: Nn.T @ _minor(*bf[m], E.dofs) @ Nn for m in E.sharers}
        tot = sum(blk.values())
        for m in E.sharers:
            Dn = np.linalg.solve(tot, blk[m])
            ref = Nn @ Dn @ Nn.T
            got = E.N @ E.D[m] @ E.N.T
            assert np.linalg.norm(got - ref) <= 1e-9 * max(1.0, np.linalg.norm(ref))
            checked += 1
    assert checked > 0


def test_deluxe_stiff_side_dominates():
    """Viscosity jump 1e6 : 1 across the faces and edges of subdomain 0 (c1 layout): deluxe gives the
    stiffer side the whole weight, D^(stiff) -> I and D^(soft) -> 0 (the point of deluxe
    scaling for coefficient jumps).  Multiplicity scaling would give 1/2, 1/4."""
    pr = make_problem("c1")
    pr.nu_cell[pr.cell_subdomain == 0] = 1e6
    gs = GlobalSystem(pr)
    bd = BDDC(gs)
    n = 0
    for E in bd.ents:
        if E.nd == 0 or 0 not in E.sharers:
            continue
        I = np.eye(E.nd)
        assert np.linalg.norm(E.D[0] - I, 2) < 1e-4
        for m in E.sharers:
            if m != 0:
                assert np.linalg.norm(E.D[m], 2) < 1e-4
        n += 1
    assert n >= 3 + 3       # 3 faces and 3 edges of subdomain 0 carry dual DOFs


@pytest.fixture(scope="module")
def sinker_small():
    pr = make_problem("c4", n=8, sub=(2, 2, 2))
    gs = GlobalSystem(pr)
    return pr, gs, BDDC(gs, adaptive_tau=10.0, keep_pencils=True)


def test_adaptive_spectrum_bounds_and_selection(sinker_small):
    """The parallel sum is monotone and S~ <= S, so every GEVP eigenvalue lies in [0, 1] (
    0 on faces between floating subdomains, reading A28); a swapped pencil gives 1/lambda >= 1.
    With the sinker's 10^4 viscosity contrast, tau = 10 selects eigenvectors (lambda < 1/tau) on
    faces with a viscosity jump across them, and on every face lambda_max is close to 1."""
    pr, gs, bd = sinker_small
    lam = np.concatenate(list(bd.adaptive_spectra.values()))
    assert lam.min() >= -1e-9 and lam.max() <= 1.0 + 1e-9
    jump_sel = 0
    for e, l in bd.adaptive_spectra.items():
        E = bd.ents[e]
        a, b = (pr.nu_cell[bd.sub_cells[m]].max() for m in E.sharers)
        if max(a, b) / min(a, b) > 100:
            jump_sel += int((l < 0.1).sum())
    assert jump_sel > 0 and bd.adaptive_count > 0


def test_adaptive_pencil_bruteforce(sinker_small):
    """S~_FD^(m) (Schur complement onto F's dual coordinates eliminating Gamma_m minus F_D)
    recomputed as the minimum-energy extension: S~ w = -mu from the KKT system
    [[S_Gamma, E^T], [E, 0]] [u; mu] = [0; w] with E = N_F^T on F's DOFs (least squares: rigid modes
    of floating subdomains), S_Gamma from the bordered brute force; then the parallel sums
    X:Y = X (X+Y)^+ Y (reading A28) and the spectrum by the general (non-symmetric) eigensolver.
    Checked on the faces with the largest viscosity contrast."""
    pr, gs, bd = sinker_small
    faces = sorted(bd.adaptive_pencils, key=lambda e: -np.ptp(np.log(np.concatenate(
        [pr.nu_cell[bd.sub_cells[m]] for m in bd.ents[e].sharers]))))[:3]
    cache = {}
    for e in faces:
        E, pc = bd.ents[e], bd.adaptive_pencils[e]
        Nf = pc["N"]
        St = []
        for m in E.sharers:
            if m not in cache:
                cache[m] = _bf_subdomain_schur(gs, m)
            gam, S = cache[m]
            pos = {int(d): j for j, d in enumerate(gam)}
            Em = np.zeros((Nf.shape[1], len(gam)))
            Em[:, [pos[int(d)] for d in E.dofs]] = Nf.T
            nd = Nf.shape[1]
            KKT = np.block([[S, Em.T], [Em, np.zeros((nd, nd))]])
            rhs = np.vstack([np.zeros((len(gam), nd)), np.eye(nd)])
            sol = np.linalg.lstsq(KKT, rhs, rcond=1e-13)[0]
            Stm = -sol[len(gam):]
            St.append(0.5 * (Stm + Stm.T))
            Sff = Nf.T @ _minor(gam, S, E.dofs) @ Nf
            assert np.linalg.norm(pc["Sf"][len(St) - 1] - Sff) <= 1e-10 * np.linalg.norm(Sff)
            assert np.linalg.norm(pc["St"][len(St) - 1] - St[-1]) <= 1e-8 * np.linalg.norm(Sff)
        par = lambda X, Y: X @ np.linalg.pinv(X + Y, rcond=1e-12) @ Y
        A = par(St[0], St[1])
        Bm = par(*[Nf.T @ _minor(*cache[m], E.dofs) @ Nf for m in E.sharers])
        lam = np.sort(sla.eigvals(A, Bm).real)
        assert np.abs(lam - bd.adaptive_spectra[e]).max() <= 1e-8


def test_adaptive_spectrum_viscosity_scale_invariant():
    """nu -> 1000 nu (all cells) scales every S^(m) and S~^(m) alike: the face spectra are unchanged
    (SURVEY F9 applied to the pencil)."""
    spectra = []
    for scale in (1.0, 1000.0):
        pr = make_problem("c4", n=4, sub=(2, 2, 2))
        pr.nu_cell *= scale
        bd = BDDC(GlobalSystem(pr), adaptive_tau=10.0)
        spectra.append(np.concatenate([bd.adaptive_spectra[e] for e in sorted(bd.adaptive_spectra)]))
    assert np.abs(spectra[0] - spectra[1]).max() <= 1e-9
