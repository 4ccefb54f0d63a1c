"""Pins of the oracle's BDDC / PCG against what the paper and mathematics fix.

* PCG + back-substitution reproduces the sparse direct solution of Eq.(DiscProblem).
* Interface reduction: dense S^, g^ -> solve -> expand equals the direct solve.
* M^-1 symmetric; its output is benign (B_0G z = 0, Assumption ass1 P:526-528).
* lambda_min(M^-1 S^) = 1 on the benign space and Lanczos kappa ~ dense kappa (Theorem teoEst,
  P:557-564).
* All interface DOFs primal => M^-1 = S^-1 => one CG step (exact limit).
* Deluxe partition of unity sum_m D^(m) = I.
* nu -> c nu invariance.
* Adaptive eigenvalues in (0,1] and monotone selection.
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
