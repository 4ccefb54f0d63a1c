"""Divergence-free VEM of degree k on a polyhedron (oracle; test infrastructure only).

Follows PAPER.md §3:
  * pressure Q_h^K = P_{k-1}(K), DOFs D_Q = moments;
  * face space B^_k(f) with enhancement (iii), which makes
    Pi^0_{k+1,f} computable from Pi^nabla_{k,f};
  * element space V_h^K with the super-enhancement;
  * DOFs D1..D5;
  * a_h^K = consistency (Pi^0_{k-1} eps : Pi^0_{k-1} eps) + D-recipe stabilisation on
    (I - Pi^nabla_k) (P:216-226 Eq.(discreteA)); b exact (with SURVEY F2);
  * load (f_h, v)_K = int Pi^0_k f . v (P:228-230 Eq.(discreteF)).
Conventions pinned in SURVEY §8(c) O-2..O-5 (frames, normalisations, GL edge points).
The origin of x in x^[P]^3 is the element centroid, scaled by h_K.
"""
import numpy as np
from .poly import (dim2, dim3, exps2, exps3, mono2, mono3, gauss_lobatto01,
                   triangle_rule, tet_rule)


# ----------------------------------------------------------------------------- topology
def mesh_edges(mesh):
    """Global edges = unique (min,max) vertex pairs of face loops, sorted lexicographically."""
    pairs = []
    for f in range(mesh.n_faces):
        lp = mesh.face(f)
        a = lp; b = np.roll(lp, -1)
        pairs.append(np.stack([np.minimum(a, b), np.maximum(a, b)], 1))
    P = np.concatenate(pairs, 0)
    E = np.unique(P, axis=0)
    return E


class EdgeIndex:
    def __init__(self, edges, n_vertices):
        self.edges = edges
        self.nv = n_vertices
        self.key = edges[:, 0].astype(np.int64) * n_vertices + edges[:, 1]

    def __call__(self, a, b):
        a, b = (a, b) if a < b else (b, a)
        i = np.searchsorted(self.key, a * self.nv + b)
        assert self.key[i] == a * self.nv + b
        return int(i)


# ----------------------------------------------------------------------------- geometry
class FaceGeom:
    pass


def face_geometry(mesh, f, k):
    """Area, unit loop normal n_f, area centroid, diameter, frame (t1 = first loop edge,
    t2 = n x t1; SURVEY O-2) and a collapsed quadrature exact to degree 2k+2."""
    F = FaceGeom()
    lp = mesh.face(f)
    P = mesh.xyz[lp]
    F.gid, F.loop = int(f), lp
    av = 0.5 * sum(np.cross(P[i], P[(i + 1) % len(P)]) for i in range(len(P)))
    F.area = np.linalg.norm(av)
    F.n = av / F.area
    cen = np.zeros(3); asum = 0.0
    for i in range(1, len(P) - 1):
        ai = 0.5 * np.dot(np.cross(P[i] - P[0], P[i + 1] - P[0]), F.n)
        cen += ai * (P[0] + P[i] + P[i + 1]) / 3.0; asum += ai
    F.xc = cen / asum
    F.h = float(np.max(np.linalg.norm(P[:, None, :] - P[None, :, :], axis=2)))
    F.t1 = (P[1] - P[0]) / np.linalg.norm(P[1] - P[0])
    F.t2 = np.cross(F.n, F.t1)
    assert np.max(np.abs((P - F.xc) @ F.n)) < 1e-10 * F.h, "non-planar face %d" % f
    qp, qw = [], []
    for i in range(1, len(P) - 1):
        p_, w_ = triangle_rule(P[0], P[i], P[i + 1], k + 2)
        qp.append(p_); qw.append(w_)
    F.qp = np.concatenate(qp); F.qw = np.concatenate(qw)
    return F


class CellGeom:
    """Geometry of cell K: vertices/edges/faces in increasing global id (local DOF order)."""

    def __init__(self, mesh, K, eidx, k):
        self.k = k
        fids, sgn = mesh.cell_faces(K)
        order = np.argsort(fids)
        fids, sgn = fids[order], sgn[order]
        loops = [mesh.face(f) for f in fids]
        self.verts = np.unique(np.concatenate(loops))
        self.X = mesh.xyz[self.verts]
        ed = set()
        for lp in loops:
            for i in range(len(lp)):
                ed.add(eidx(lp[i], lp[(i + 1) % len(lp)]))
        self.edges = np.array(sorted(ed), dtype=np.int64)
        self.edge_vtx = eidx.edges[self.edges]
        self.faces = fids
        self.signs = sgn.astype(np.float64)
        vloc = {int(v): i for i, v in enumerate(self.verts)}
        eloc = {int(e): i for i, e in enumerate(self.edges)}
        xv0 = self.X.mean(0)  # star centre for the sub-tetrahedra (SURVEY O-1)
        self.F = []
        vol = 0.0; mom1 = np.zeros(3)
        tets = []
        for lf, (f, s, lp) in enumerate(zip(fids, sgn, loops)):
            F = face_geometry(mesh, f, k)
            F.sign = float(s)
            P = mesh.xyz[lp]
            # loop edges with GL node DOF maps (filled later by the element)
            F.loop_edges = []
            for i in range(len(lp)):
                a, b = int(lp[i]), int(lp[(i + 1) % len(lp)])
                e = eloc[eidx(a, b)]
                F.loop_edges.append((vloc[a], vloc[b], e, a < b, P[i], P[(i + 1) % len(P)]))
            self.F.append(F)
            # outward-oriented fan triangles -> sub-tetrahedra with apex xv0
            for i in range(1, len(P) - 1):
                a, b, c = (P[0], P[i], P[i + 1]) if s > 0 else (P[0], P[i + 1], P[i])
                v6 = np.dot(a - xv0, np.cross(b - xv0, c - xv0))
                assert v6 > 0, "non-positive sub-tetrahedron in cell %d" % K
                vol += v6 / 6.0; mom1 += v6 / 6.0 * (xv0 + a + b + c) / 4.0
                tets.append((xv0, a, b, c))
        self.vol = vol
        self.xc = mom1 / vol
        self.h = float(np.max(np.linalg.norm(self.X[:, None, :] - self.X[None, :, :], axis=2)))
        nqv = k + 3  # collapsed tet rule exact to 2(k+3)-3 = 2k+3
        qp, qw = [], []
        for t in tets:
            p_, w_ = tet_rule(*t, nqv)
            qp.append(p_); qw.append(w_)
        self.qp = np.concatenate(qp); self.qw = np.concatenate(qw)


# ----------------------------------------------------------------------------- DOF layout
class Layout:
    """Local DOF layout D1..D5 of P:178-198 for a cell (velocity), and D_Q (pressure)."""

    def __init__(self, g, k):
        self.k = k
        self.nV, self.nE, self.nF = len(g.verts), len(g.edges), len(g.faces)
        self.nm = dim2(k - 2)                              # face moments per (face, direction)
        self.n4 = 3 * dim3(k - 3) - dim3(k - 4)            # dim x^[P_{k-3}]^3
        self.n5 = dim3(k - 1) - 1                          # dim P^_{k-1\0}
        self.oE = 3 * self.nV
        self.oF = self.oE + 3 * (k - 1) * self.nE
        self.o4 = self.oF + 3 * self.nm * self.nF
        self.o5 = self.o4 + self.n4
        self.nv = self.o5 + self.n5
        self.np = dim3(k - 1)

    def vdof(self, lv, c):
        return 3 * lv + c

    def edof(self, le, j, c):
        return self.oE + 3 * (self.k - 1) * le + 3 * j + c

    def fdof(self, lf, t, a):
        return self.oF + lf * 3 * self.nm + t * self.nm + a


def cross_basis(n):
    """Spanning set of x^[H_d]^3 for d = 0..n as triples (d, m-exponent, component c).

    x^(m e_c) with x = scaled coordinates; the set is linearly dependent (x^(x q) = 0),
    which the oracle handles by least squares (SURVEY O-4 'drop the rank deficiency')."""
    out = []
    for d in range(n + 1):
        for e in exps3(n):
            if sum(e) == d:
                for c in range(3):
                    out.append((e, c))
    return out


def cross_coeffs(e, c, n_out):
    """Coefficients of x^(m_e e_c) in the standard basis {m_a e_comp} (comp-major) of degree n_out."""
    E = exps3(n_out); idx = {ee: i for i, ee in enumerate(E)}
    D = len(E)
    v = np.zeros(3 * D)
    up = lambda e, i: tuple(e[j] + (1 if j == i else 0) for j in range(3))
    # x cross e_c: e1 -> (0, x3, -x2); e2 -> (-x3, 0, x1); e3 -> (x2, -x1, 0)
    table = {0: [(1, 2, +1), (2, 1, -1)], 1: [(0, 2, -1), (2, 0, +1)], 2: [(0, 1, +1), (1, 0, -1)]}
    for comp, xi, sgn in table[c]:
        v[comp * D + idx[up(e, xi)]] += sgn
    return v


def d4_basis(k):
    """Basis of x^[P_{k-3}]^3 used by the D4 moments (SURVEY O-4 reading A24): the fields
    x^(m e_c) for monomials m of degree 0..k-3 (exps3 order), components c = 1, 2, 3, omitting
    c = 1 when x_1 divides m (x^(x_1 q e_1) = x_1 x^(q e_1) ... the relation x^(x q) = 0 removes
    exactly one field per monomial of degree >= 1: dim = 3 dim P_{k-3} - dim P_{k-4}).
    k = 2: none; k = 3: x^e_1, x^e_2, x^e_3; k = 4: 11 fields."""
    out = []
    for d in range(k - 2):
        for e in exps3(d):
            if sum(e) != d:
                continue
            for c in range(3):
                if c == 0 and e[0] > 0:
                    continue
                out.append((e, c))
    assert len(out) == 3 * dim3(k - 3) - dim3(k - 4)
    return out


# ----------------------------------------------------------------------------- element operators
class ElementOps:
    """All VEM operators of one cell as dense matrices acting on the local velocity DOF vector."""

    def Gram(self, n1, n2):
        """(int_K m_a m_b) for |a| <= n1, |b| <= n2 by the cell quadrature (a method, not a closure,
        so element operators can be returned from worker processes)."""
        return (self.Mq[:, :dim3(n1)] * self.wq[:, None]).T @ self.Mq[:, :dim3(n2)]

    def __init__(self, mesh, K, eidx, k, nu):
        self.k, self.nu = k, nu
        g = self.g = CellGeom(mesh, K, eidx, k)
        L = self.L = Layout(g, k)
        nv = L.nv
        for F in g.F:
            F.m3v, F.m3g = mono3(F.qp, g.xc, g.h, k + 1)
        self._face_ops()
        xq, wq = g.qp, g.qw
        Mk1, Gk1 = mono3(xq, g.xc, g.h, k + 1)
        self.Mq, self.Gq, self.wq = Mk1, Gk1, wq
        d = lambda n: dim3(n)
        Gram = self.Gram
        # ---- (1) divergence: div v in P_{k-1} (Ṽ_h^K (iii)); moments via flux + D5
        Rdiv = np.zeros((d(k - 1), nv))
        for lf, F in enumerate(g.F):
            Rdiv[0, L.fdof(lf, 0, 0)] += F.sign * F.area
        for a in range(1, d(k - 1)):
            Rdiv[a, L.o5 + a - 1] = g.vol / g.h
        self.Rdiv = Rdiv
        self.DIVc = np.linalg.solve(Gram(k - 1, k - 1), Rdiv)
        # ---- (2) moments against [P_{k-2}]^3 via grad P_{k-1} (+) x^[P_{k-3}]^3
        self.Mom2 = self._moments(k - 2, use_piN=False)
        # ---- (3) Pi^nabla_{k,K} per component
        Dk = d(k)
        Gn = np.zeros((Dk, Dk))
        Gn[1:, :] = np.einsum("q,qai,qbi->ab", wq, Gk1[:, 1:Dk, :], Gk1[:, :Dk, :])
        for F in g.F:
            Gn[0, :] += F.qw @ F.m3v[:, :Dk]
        E2 = exps3(k - 2); i2 = {e: i for i, e in enumerate(E2)}
        Ek = exps3(k)
        self.PiN = []
        for c in range(3):
            R = np.zeros((Dk, nv))
            for b in range(1, Dk):
                e = Ek[b]
                for cc in range(3):      # -int Lap(m_b) v_c
                    if e[cc] >= 2:
                        ee = tuple(e[j] - (2 if j == cc else 0) for j in range(3))
                        R[b] -= e[cc] * (e[cc] - 1) / g.h ** 2 * self.Mom2[c][i2[ee]]
            for lf, F in enumerate(g.F):
                dn = (F.m3g[:, :Dk] @ F.n) * F.sign          # grad m_b . n_K^f
                R[1:] += (dn[:, 1:] * F.qw[:, None]).T @ F.V[c]
                R[0] += F.qw @ F.V[c]
            self.PiN.append(np.linalg.solve(Gn, R))
        # ---- (4) moments against [P_k]^3 with the super-enhancement -> Pi^0_{k,K}
        self.MomK = self._moments(k, use_piN=True)
        Gkk = Gram(k, k)
        self.P0 = [np.linalg.solve(Gkk, self.MomK[c]) for c in range(3)]
        # ---- (5) Pi^0_{k-1} grad v
        Ek1 = exps3(k - 1); ik = {e: i for i, e in enumerate(Ek)}
        G1 = Gram(k - 1, k - 1)
        self.Grad = [[None] * 3 for _ in range(3)]
        for c in range(3):
            for dd in range(3):
                R = np.zeros((d(k - 1), nv))
                for a, e in enumerate(Ek1):
                    if e[dd] > 0:
                        ee = tuple(e[j] - (1 if j == dd else 0) for j in range(3))
                        R[a] -= e[dd] / g.h * self.MomK[c][ik[ee]]
                for F in g.F:
                    mv = F.m3v[:, :d(k - 1)]
                    R += F.sign * F.n[dd] * ((mv * F.qw[:, None]).T @ F.V[c])
                self.Grad[c][dd] = np.linalg.solve(G1, R)
        # ---- (6) consistency + D-recipe stabilisation (Eq.(discreteA))
        Acons = np.zeros((nv, nv))
        for c in range(3):
            for dd in range(3):
                Ecd = 0.5 * (self.Grad[c][dd] + self.Grad[dd][c])
                Acons += Ecd.T @ G1 @ Ecd
        Acons *= nu
        self.DOFpoly = self.dofs_of_basis()
        Pihat = sum(self.DOFpoly[:, c * Dk:(c + 1) * Dk] @ self.PiN[c] for c in range(3))
        dstab = np.maximum(np.diag(Acons), nu * g.h)
        IP = np.eye(nv) - Pihat
        self.Acons = Acons
        self.Pihat = Pihat
        self.A = Acons + IP.T @ (dstab[:, None] * IP)
        self.A = 0.5 * (self.A + self.A.T)
        # ---- (7) B^K_{j,i} = int div phi_i psi_j, psi dual to D_Q (SURVEY O-5)
        self.B = g.vol * self.DIVc

    # -------------------------------------------------------------------------
    def _face_ops(self):
        """Per face f and component c: V[c] = values of Pi^0_{k+1,f} v_c at the face quadrature
        points as a matrix on the element DOFs (P:146-151 enhancement, P:118-124 Pi^nabla)."""
        g, L, k = self.g, self.L, self.k
        nv = L.nv
        xg, wg = gauss_lobatto01(k + 1)
        E2k = exps2(k); i2 = {e: i for i, e in enumerate(exps2(k + 1))}
        for lf, F in enumerate(g.F):
            tfr = np.stack([F.t1, F.t2])                      # 2x3
            xi = lambda x: (np.atleast_2d(x) - F.xc) @ tfr.T
            # interior moments of v_c: int_f v_c m_a = |f| (n_c D3n + t1_c D3t1 + t2_c D3t2)
            mom = np.zeros((3, L.nm, nv))
            for c in range(3):
                for a in range(L.nm):
                    for t, tau in enumerate((F.n, F.t1, F.t2)):
                        mom[c, a, L.fdof(lf, t, a)] += F.area * tau[c]
            # boundary nodal values on each loop edge: GL nodes (SURVEY O-3: exact edge traces)
            Dk = dim2(k)
            Gn = np.zeros((Dk, Dk))
            mqv, mqg = mono2(xi(F.qp), k + 1, F.h)
            Gn[1:, :] = np.einsum("q,qai,qbi->ab", F.qw, mqg[:, 1:Dk, :], mqg[:, :Dk, :])
            Rb = np.zeros((3, Dk, nv))
            for (la, lb, le, fwd, Pa, Pb) in F.loop_edges:
                el = np.linalg.norm(Pb - Pa)
                ne = np.cross((Pb - Pa) / el, F.n)            # outward in-plane normal
                ne2 = tfr @ ne
                for j, (tj, wj) in enumerate(zip(xg, wg)):
                    xj = Pa + tj * (Pb - Pa)
                    mv, mg = mono2(xi(xj), k, F.h)
                    for c in range(3):
                        if j == 0:
                            col = L.vdof(la, c)
                        elif j == k:
                            col = L.vdof(lb, c)
                        else:
                            jj = j - 1 if fwd else k - 2 - (j - 1)
                            col = L.edof(le, jj, c)
                        Rb[c, 1:, col] += el * wj * (mg[0, 1:, :] @ ne2)
                        Rb[c, 0, col] += el * wj
                        Gn[0, :] += 0 if c else el * wj * mv[0, :Dk]
            # Laplacian of 2D monomials in P_{k-2}
            F.V = []
            D1 = dim2(k + 1)
            G0 = (mqv * F.qw[:, None]).T @ mqv
            for c in range(3):
                R = Rb[c].copy()
                for b in range(1, Dk):
                    p, q = E2k[b]
                    if p >= 2:
                        R[b] -= p * (p - 1) / F.h ** 2 * mom[c, i2[(p - 2, q)]]
                    if q >= 2:
                        R[b] -= q * (q - 1) / F.h ** 2 * mom[c, i2[(p, q - 2)]]
                piN = np.linalg.solve(Gn, R)                  # Pi^nabla_{k,f} v_c
                R0 = np.zeros((D1, nv))
                R0[:L.nm] = mom[c]
                R0[L.nm:] = G0[L.nm:, :Dk] @ piN              # enhancement (iii)
                P0f = np.linalg.solve(G0, R0)
                F.V.append(mqv @ P0f)

    def _moments(self, n, use_piN):
        """int_K v . (m_a e_c) for |a| <= n, via [P_n]^3 = grad P_{n+1} (+) x^[P_{n-1}]^3
        (SURVEY O-4).  x^ part: D4 for degree <= k-3, super-enhancement for k-2..k-1."""
        g, L, k = self.g, self.L, self.k
        nv = L.nv
        Dn = dim3(n)
        En1 = exps3(n + 1); In = {e: i for i, e in enumerate(exps3(n))}
        rows, vals = [], []
        # grad m_b, 1 <= |b| <= n+1:  -int div v m_b + sum_f s_f int_f (v.n_f) m_b
        Gdiv = self.Gram(n + 1, k - 1) @ self.DIVc
        for b in range(1, dim3(n + 1)):
            e = En1[b]
            coef = np.zeros(3 * Dn)
            for c in range(3):
                if e[c] > 0:
                    ee = tuple(e[j] - (1 if j == c else 0) for j in range(3))
                    coef[c * Dn + In[ee]] = e[c] / g.h
            val = -Gdiv[b].copy()
            for F in g.F:
                wm = F.qw * F.m3v[:, b] * F.sign
                for c in range(3):
                    val += F.n[c] * (wm @ F.V[c])
            rows.append(coef); vals.append(val)
        # x^ part
        d4 = d4_basis(k)
        for i, (e, c) in enumerate(d4):
            if sum(e) <= n - 1:
                rows.append(cross_coeffs(e, c, n)); vals.append(g.vol * np.eye(nv)[L.o4 + i])
        if use_piN:
            Dk = dim3(k)
            for (e, c) in cross_basis(n - 1):
                if sum(e) < k - 2:
                    continue
                w = cross_coeffs(e, c, n)                        # vector field coefficients
                val = np.zeros(nv)
                for comp in range(3):
                    # int (Pi^nabla v)_comp * w_comp
                    wv = self.Mq[:, :Dn] @ w[comp * Dn:(comp + 1) * Dn]
                    val += ((wv * self.wq) @ self.Mq[:, :Dk]) @ self.PiN[comp]
                rows.append(w); vals.append(val)
        T = np.array(rows); V = np.array(vals)
        assert np.linalg.matrix_rank(T) == 3 * Dn
        Qt, Rt = np.linalg.qr(T)                     # consistent full-column-rank system (least squares)
        mS = np.linalg.solve(Rt, Qt.T @ V)
        return [mS[c * Dn:(c + 1) * Dn] for c in range(3)]

    # -------------------------------------------------------------------------
    def dofs_of_field(self, u, divu=None):
        """D1..D5 of a vector field u(x)->[n,3] (DOF interpolant; SURVEY O-5/O-6)."""
        g, L, k = self.g, self.L, self.k
        out = np.zeros(L.nv)
        out[:L.oE] = u(g.X).ravel()
        xg, _ = gauss_lobatto01(k + 1)
        for le, (a, b) in enumerate(g.edge_vtx):
            Pa, Pb = self._vx(a), self._vx(b)
            for j in range(k - 1):
                out[L.edof(le, j, 0):L.edof(le, j, 0) + 3] = u((Pa + xg[j + 1] * (Pb - Pa))[None])[0]
        for lf, F in enumerate(g.F):
            mv, _ = mono2((F.qp - F.xc) @ np.stack([F.t1, F.t2]).T, k - 2, F.h)
            uq = u(F.qp)
            for t, tau in enumerate((F.n, F.t1, F.t2)):
                out[L.fdof(lf, t, 0):L.fdof(lf, t, 0) + L.nm] = ((F.qw * (uq @ tau)) @ mv) / F.area
        uq = u(g.qp)
        for i, (e, c) in enumerate(d4_basis(k)):
            D1 = dim3(k - 2)
            w = cross_coeffs(e, c, k - 2)
            wq = np.stack([self.Mq[:, :D1] @ w[cc * D1:(cc + 1) * D1] for cc in range(3)], 1)
            out[L.o4 + i] = (g.qw * np.sum(uq * wq, 1)).sum() / g.vol
        if L.n5:
            dq = divu(g.qp) if divu is not None else np.zeros(len(g.qw))
            out[L.o5:] = g.h / g.vol * ((g.qw * dq) @ self.Mq[:, 1:dim3(k - 1)])
        return out

    def _vx(self, gv):
        return self.X_of[int(gv)]

    @property
    def X_of(self):
        return {int(v): x for v, x in zip(self.g.verts, self.g.X)}

    def dofs_of_basis(self):
        """DOFs of the polynomial basis {m_a e_c} of [P_k]^3 (columns comp-major)."""
        g, L, k = self.g, self.L, self.k
        Dk = dim3(k)
        out = np.zeros((L.nv, 3 * Dk))
        # vectorised: evaluate all monomials at the DOF sample points
        mv, _ = mono3(g.X, g.xc, g.h, k)
        for c in range(3):
            out[c:L.oE:3, c * Dk:(c + 1) * Dk] = mv
        xg, _ = gauss_lobatto01(k + 1)
        Xo = self.X_of
        for le, (a, b) in enumerate(g.edge_vtx):
            for j in range(k - 1):
                x = Xo[int(a)] + xg[j + 1] * (Xo[int(b)] - Xo[int(a)])
                mv, _ = mono3(x[None], g.xc, g.h, k)
                for c in range(3):
                    out[L.edof(le, j, c), c * Dk:(c + 1) * Dk] = mv[0]
        for lf, F in enumerate(g.F):
            m2, _ = mono2((F.qp - F.xc) @ np.stack([F.t1, F.t2]).T, k - 2, F.h)
            m3 = F.m3v[:, :Dk]
            I = (m2 * F.qw[:, None]).T @ m3 / F.area           # [nm, Dk]
            for t, tau in enumerate((F.n, F.t1, F.t2)):
                for c in range(3):
                    out[L.fdof(lf, t, 0):L.fdof(lf, t, 0) + L.nm, c * Dk:(c + 1) * Dk] += tau[c] * I
        D1 = dim3(k - 2)
        for i, (e, c0) in enumerate(d4_basis(k)):
            w = cross_coeffs(e, c0, k - 2)
            for c in range(3):
                wq = self.Mq[:, :D1] @ w[c * D1:(c + 1) * D1]
                out[L.o4 + i, c * Dk:(c + 1) * Dk] = ((g.qw * wq) @ self.Mq[:, :Dk]) / g.vol
        if L.n5:
            for c in range(3):
                # (h/|K|) int d_c m_g m_a, a >= 1
                out[L.o5:, c * Dk:(c + 1) * Dk] = g.h / g.vol * (
                    (self.Mq[:, 1:dim3(k - 1)] * g.qw[:, None]).T @ self.Gq[:, :Dk, c])
        return out

    def load(self, f, shift=0.0):
        """(f_h, phi_i)_K = int Pi^0_k f . phi_i (Eq.(discreteF)), f(x)->[n,3].
        `shift` translates the cell (operators of congruent translated cells are identical)."""
        g = self.g
        Dk = dim3(self.k)
        fq = f(g.qp + shift)
        Fm = [(g.qw * fq[:, c]) @ self.Mq[:, :Dk] for c in range(3)]   # int f_c m_a
        return sum(Fm[c] @ self.P0[c] for c in range(3))

    def h1_error_sq(self, ul, grad_u, shift=0.0):
        """int_K |grad u - Pi^0_{k-1} grad u_h|^2 (SURVEY O-16 velocity error)."""
        g = self.g
        Gq = grad_u(g.qp + shift)
        D = dim3(self.k - 1)
        err = 0.0
        for c in range(3):
            for d in range(3):
                v = self.Mq[:, :D] @ (self.Grad[c][d] @ ul)
                err += np.sum(g.qw * (Gq[:, c, d] - v) ** 2)
        return err

    def l2_pressure_error_sq(self, pl, p, shift=0.0, pmean=0.0):
        """int_K |p - p_h|^2 with p_h = sum_j pl_j psi_j, psi dual to D_Q."""
        g = self.g
        D = dim3(self.k - 1)
        Gp = self.Gram(self.k - 1, self.k - 1) / g.vol
        coef = np.linalg.solve(Gp, pl)
        ph = self.Mq[:, :D] @ coef
        return np.sum(g.qw * (p(g.qp + shift) - pmean - ph) ** 2)
