"""BDDC-preconditioned CG for the interface saddle problem (oracle; test infrastructure only).

Follows PAPER.md §4 and §6:
  * splitting V = V_I (+) V_Gamma, Q = Q_I (+) Q_0 (P:313-325 Eq.(discVQ));
  * static condensation by subdomain Dirichlet saddle problems (P:359-392 Eq.(uipi));
  * interface saddle problem S^ [u_G; p_0] = g^ (P:393-445 Eq.(globInt)),
    S_G^(i) from Eq.(firstSchur), assembled by Eq.(ScapGdef);
  * partially assembled space with an explicit change of basis to primal DOFs;
  * scaled restriction R~_D and average E_D with deluxe scaling (
    edges by the same formula) or multiplicity scaling Eq.(pseudoinv);
  * M^-1 = R~_D^T S~^-1 R~_D = local + coarse (P:510-514 Eq.(BDDCprec));
  * primal constraints: vertices, edge averages, face averages + face flux,
    SVD-filtered;
  * CG with stopping rule ||r||_2 <= rtol ||r_0||_2 and Lanczos k_2
    (SURVEY A12);
  * adaptive coarse space: per-face generalized eigenproblems on deluxe Schur complements
    (SURVEY O-12).
Everything is in ORIGINAL interface coordinates with T_G = [N_G, C_G^T (C_G C_G^T)^-1]
(SURVEY A9).  Q_I is handled with an explicit (sparse) basis Z of {q : int q = 0}
("Z-basis").  Per subdomain only S_G (dense), the sparse LU of K_DD and the factored
dual block are kept, so the full-size configs 3 and 5 fit a CPU host (SURVEY O-8).
"""
import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla


def _sym(M):
    return 0.5 * (M + M.T)


class Entity:
    pass


class BDDC:
    def __init__(self, gs, scaling="deluxe", constraints=None, adaptive_tau=None, svd_tol=1e-10,
                 keep_pencils=False):
        self.gs = gs
        self.keep_pencils = keep_pencils      # tests: keep each face's (N_F, S~^(m), S_FD^(m), A, B)
        prob = gs.prob
        self.prob = prob
        mesh, dofs, k = prob.mesh, gs.dofs, prob.k
        self.k = k
        cons = dict(prob.constraints)
        if constraints:
            cons.update(constraints)
        self.cons = cons
        tau = cons.get("adaptive_tau", 0.0) if adaptive_tau is None else adaptive_tau
        self.scaling = scaling
        self.svd_tol = svd_tol
        csub = prob.cell_subdomain
        N = self.N = int(csub.max()) + 1
        el = gs.el
        nvf = dofs.n_free_vel
        # ---------------- subdomain DOF sets (free velocity indices), sharer sets
        sub_vel = [set() for _ in range(N)]
        self.sub_cells = [np.nonzero(csub == i)[0] for i in range(N)]
        for K in range(mesh.n_cells):
            iv, _ = el.l2g[K]
            fr = dofs.vel2free[iv]
            sub_vel[csub[K]].update(int(x) for x in fr[fr >= 0])
        sharers = {}
        for i in range(N):
            for d in sub_vel[i]:
                sharers.setdefault(d, []).append(i)
        # Gamma_i = the free DOFs on the subdomain boundary: shared DOFs, and with Neumann faces
        # also the DOFs on the subdomain's part of the Neumann boundary (one sharer), so
        # the flux row b_0^(i) keeps acting on Gamma only (DESIGN A35)
        self.neumann = bool(dofs.neumann)
        onN = dofs.free_on_neumann
        gam = sorted(d for d, s in sharers.items() if len(s) > 1 or onN[d])
        self.gamma = np.array(gam, dtype=np.int64)        # interface DOFs (free-velocity ids)
        self.nG = len(gam)
        gpos = {d: j for j, d in enumerate(gam)}
        # ---------------- entities = classes of interface DOFs with equal sharer sets
        # (with Neumann faces the class key also says whether the DOF lies on the Neumann boundary,
        # so the lines and points where subdomains meet on it are entities of their own; DESIGN A35)
        classes = {}
        for d in gam:
            classes.setdefault(tuple(sharers[d]) + ((-1,) if onN[d] else ()), []).append(d)
        ents = sorted(classes.items(), key=lambda kv: min(kv[1]))
        self.ents = []
        for key, dl in ents:
            E = Entity()
            E.sharers = [x for x in key if x >= 0]
            E.dofs = np.array(sorted(dl), dtype=np.int64)          # free-velocity ids
            E.gpos = np.array([gpos[d] for d in E.dofs])           # interface positions
            gv = dofs.free_vel[E.dofs]                             # global velocity ids
            if np.all(gv < dofs.oE) and len(np.unique(gv // 3)) == 1:
                E.kind = "vertex"
            elif key[-1] == -1:          # on the Neumann boundary: face iff it holds face moments
                E.kind = "face" if np.any((gv >= dofs.oF) & (gv < dofs.oC)) else "edge"
            elif len(key) == 2:
                E.kind = "face"
            else:
                E.kind = "edge"
            self.ents.append(E)
        # ---------------- subdomain local orderings
        self.sub = []
        for i in range(N):
            S = Entity()
            S.vel = np.array(sorted(sub_vel[i]), dtype=np.int64)
            S.ents = [e for e, E in enumerate(self.ents) if i in E.sharers]
            S.G = np.concatenate([self.ents[e].dofs for e in S.ents])   # local Gamma order
            S.Gpos = np.concatenate([self.ents[e].gpos for e in S.ents])
            isG = set(S.G.tolist())
            S.I = np.array([d for d in S.vel if d not in isG], dtype=np.int64)
            S.P = np.concatenate([el.l2g[K][1] for K in self.sub_cells[i]])
            S.P.sort()
            self.sub.append(S)
        self._subdomain_matrices()
        self._constraints()
        self._factor(tau)

    # ------------------------------------------------------------------ subdomain operators
    def _subdomain_matrices(self):
        """K^(i) = sum of element saddle matrices (O-8), stored sparse; K_DD^(i) on (u_I, Q_I) is
        factored by a sparse LU (library solve); S_G^(i) = K_GG - K_GD K_DD^-1 K_DG
        (Eq.(firstSchur)) is the only dense per-subdomain matrix kept (memory-lean:
        configs 3 and 5 at full size fit a CPU host, SURVEY O-8)."""
        gs, dofs, el = self.gs, self.gs.dofs, self.gs.el
        nu = self.prob.nu_cell
        for i, S in enumerate(self.sub):
            lv = {int(d): j for j, d in enumerate(np.concatenate([S.I, S.G]))}
            lp = {int(d): j for j, d in enumerate(S.P)}
            nI, nGl, nP = len(S.I), len(S.G), len(S.P)
            ar, ac, av, br, bc, bv = [], [], [], [], [], []
            c = np.zeros(nP); m = np.zeros(nP)
            for K in self.sub_cells[i]:
                op = el.op(K)
                iv, ip = el.l2g[K]
                fr = dofs.vel2free[iv]
                keep = fr >= 0
                li = np.array([lv[int(x)] for x in fr[keep]])
                pi = np.array([lp[int(x)] for x in ip])
                ar.append(np.repeat(li, li.size)); ac.append(np.tile(li, li.size))
                av.append((nu[K] * op.A[np.ix_(keep, keep)]).ravel())
                br.append(np.repeat(pi, li.size)); bc.append(np.tile(li, pi.size))
                bv.append(op.B[:, keep].ravel())
                # DOFs of the constant 1 (D_Q of q=1) and m = int psi_j
                c[pi] = op.Gram(self.k - 1, 0)[:, 0] / op.g.vol
                m[pi[0]] = op.g.vol
            n = nI + nGl
            A = sp.csr_matrix((np.concatenate(av), (np.concatenate(ar), np.concatenate(ac))), shape=(n, n))
            B = sp.csr_matrix((np.concatenate(bv), (np.concatenate(br), np.concatenate(bc))), shape=(nP, n))
            S.c, S.m = c, m
            S.vol = float(m.sum())
            S.nI, S.nGl = nI, nGl
            # Q_I basis: columns e_j - (m_j / m_j0) e_j0, j != j0 (m^T z = 0; sparse)
            j0 = int(np.flatnonzero(m)[0])
            oth = np.delete(np.arange(nP), j0)
            S.Z = sp.csr_matrix((np.concatenate([np.ones(nP - 1), -m[oth] / m[j0]]),
                                 (np.concatenate([oth, np.full(nP - 1, j0)]),
                                  np.concatenate([np.arange(nP - 1)] * 2))), shape=(nP, nP - 1))
            AII, AIG, AGG = A[:nI, :nI], A[:nI, nI:], A[nI:, nI:]
            BI, BG = B[:, :nI], B[:, nI:]
            ZB = (S.Z.T @ BI).tocsr()
            KDD = sp.bmat([[AII, ZB.T], [ZB, None]]).tocsc()
            KDG = sp.vstack([AIG, S.Z.T @ BG]).tocsc()
            S.KDG = KDG
            S.KDD_lu = spla.splu(KDD)
            X = S.KDD_lu.solve(KDG.toarray())
            S.SG = _sym(AGG.toarray() - KDG.T @ X)               # Eq.(firstSchur)
            del X
            S.b0 = BG.T @ S.c                                    # flux row B_0G^(i)
            S.b0_int = BI.T @ S.c                                # must vanish (interior DOFs)

    # ------------------------------------------------------------------ primal constraints
    def _entity_constraints(self, E):
        gs, dofs, mesh, k = self.gs, self.gs.dofs, self.prob.mesh, self.k
        gv = dofs.free_vel[E.dofs]
        pos = {int(g): j for j, g in enumerate(gv)}
        n = len(gv)
        rows = []
        if self.cons.get("all_primal", 0):
            return np.eye(n)            # exact-limit check: every interface DOF primal
        if E.kind == "vertex":
            return np.eye(3) if self.cons.get("vertex", 1) else np.zeros((0, 3))
        if E.kind == "edge":
            if not self.cons.get("edge_avg", 1):
                return np.zeros((0, n))
            from .poly import gauss_lobatto01
            _, wg = gauss_lobatto01(k + 1)
            C = np.zeros((3, n))
            # fine edges whose DOFs belong to the macro edge (SURVEY O-9)
            eids = np.unique((gv[gv >= dofs.oE] - dofs.oE) // (3 * (k - 1)))
            for e in eids:
                a, b = dofs.edges[e]
                L = np.linalg.norm(mesh.xyz[b] - mesh.xyz[a])
                for d in range(3):
                    for j in range(k - 1):
                        C[d, pos[dofs.oE + 3 * (k - 1) * e + 3 * j + d]] += L * wg[j + 1]
                    for (v, w) in ((a, wg[0]), (b, wg[k])):
                        if 3 * v + d in pos:
                            C[d, pos[3 * v + d]] += L * w
            return C
        # face
        from .vem import face_geometry
        fids = np.unique((gv[(gv >= dofs.oF) & (gv < dofs.oC)] - dofs.oF) // (3 * dofs.nm))
        s_owner = E.sharers[0]
        avg = np.zeros((3, n)); flux = np.zeros((1, n))
        for f in fids:
            F = face_geometry(mesh, f, k)
            # orientation of n_f w.r.t. the outward normal of the first sharer
            sgn = self._face_sign_in_subdomain(f, s_owner)
            for t, tau in enumerate((F.n, F.t1, F.t2)):
                col = pos[dofs.oF + 3 * dofs.nm * f + t * dofs.nm]
                avg[:, col] += F.area * tau
            flux[0, pos[dofs.oF + 3 * dofs.nm * f]] += sgn * F.area
        if self.cons.get("face_avg", 1):
            rows.append(avg)
        if self.cons.get("face_flux", 1):
            rows.append(flux)
        return np.vstack(rows) if rows else np.zeros((0, n))

    def _face_sign_in_subdomain(self, f, i):
        mesh = self.prob.mesh
        if not hasattr(self, "_face_cell_sign"):
            self._face_cell_sign = {}
            csub = self.prob.cell_subdomain
            for K in range(mesh.n_cells):
                fs, ss = mesh.cell_faces(K)
                for ff, s in zip(fs, ss):
                    self._face_cell_sign[(int(ff), int(csub[K]))] = int(s)
        return self._face_cell_sign[(int(f), int(i))]

    def _constraints(self, extra=None):
        """C_G, SVD filter, T_G = [N_G, P_G] with P_G = C^T (C C^T)^-1 (SURVEY O-9)."""
        for e, E in enumerate(self.ents):
            C = self._entity_constraints(E)
            if extra is not None and e in extra:
                C = np.vstack([C, extra[e]])
            n = len(E.dofs)
            if C.shape[0]:
                U, s, Vt = np.linalg.svd(C, full_matrices=True)
                r = int(np.sum(s > self.svd_tol * s[0]))
                C = (s[:r, None] * Vt[:r])                  # span-preserving filtered rows
                N = Vt[r:].T
                P = C.T @ np.linalg.inv(C @ C.T)
            else:
                r = 0
                C = np.zeros((0, n)); N = np.eye(n); P = np.zeros((n, 0))
            E.C, E.N, E.P, E.r = C, N, P, r
            E.nd = n - r
        # global primal numbering (entity order) and local transformed layouts
        off = 0
        for E in self.ents:
            E.pi = np.arange(off, off + E.r); off += E.r
        self.NPi = off

    def _factor(self, tau):
        adaptive = bool(tau and tau > 0)
        self._keep_ST = adaptive            # the face pencils need S_T (memory-lean otherwise)
        self._local_transform()
        self._deluxe()
        if adaptive:
            self._adaptive(tau)
            self._keep_ST = False
            self._local_transform()
            self._deluxe()
        self._coarse()

    def _local_transform(self):
        """S_T = T^T S_G T, S_DD, Phi_D = -S_DD^-1 S_DP, S_c = S_PP + S_PD Phi (O-10)."""
        for i, S in enumerate(self.sub):
            nG = S.nGl
            blocksN, blocksP = [], []
            offs = 0
            S.ent_off = []
            for e in S.ents:
                E = self.ents[e]
                S.ent_off.append(offs); offs += len(E.dofs)
            nd = sum(self.ents[e].nd for e in S.ents)
            npi = sum(self.ents[e].r for e in S.ents)
            T = np.zeros((nG, nd + npi))
            S.d_off, S.p_off = [], []
            dd = 0; pp = nd
            S.pi_glob = []
            for e, o in zip(S.ents, S.ent_off):
                E = self.ents[e]
                n = len(E.dofs)
                T[o:o + n, dd:dd + E.nd] = E.N
                T[o:o + n, pp:pp + E.r] = E.P
                S.d_off.append(dd); S.p_off.append(pp)
                S.pi_glob.append(E.pi)
                dd += E.nd; pp += E.r
            S.pi_glob = np.concatenate(S.pi_glob).astype(np.int64)
            S.T, S.nd, S.npi = T, nd, npi
            ST = _sym(T.T @ S.SG @ T)
            S.ST = ST
            S.SDD = ST[:nd, :nd]; S.SDP = ST[:nd, nd:]; S.SPP = ST[nd:, nd:]
            S.b0T = S.b0 @ T
            S.SDD_chol = sla.cho_factor(S.SDD)
            S.Phi = -sla.cho_solve(S.SDD_chol, S.SDP)
            S.Sc = _sym(S.SPP + S.SDP.T @ S.Phi)
            S.T = S.SDD = S.SDP = S.SPP = None          # factor-time only (memory-lean)
            if not self._keep_ST:
                S.ST = None

    def _deluxe(self):
        """D_G^(m) = (sum_m' S_GD^(m'))^-1 S_GD^(m) or 1/card(I_x) (Eq.(pseudoinv))."""
        for e, E in enumerate(self.ents):
            E.D = {}
            if E.nd == 0:
                continue
            blocks = {}
            for m in E.sharers:
                S = self.sub[m]
                j = S.ents.index(e)
                o = S.ent_off[j]; n = len(E.dofs)
                SGG = S.SG[o:o + n, o:o + n]
                blocks[m] = _sym(E.N.T @ SGG @ E.N)
            if self.scaling == "deluxe":
                Ssum = sum(blocks.values())
                ch = sla.cho_factor(Ssum)
                for m in E.sharers:
                    E.D[m] = sla.cho_solve(ch, blocks[m])
            else:
                for m in E.sharers:
                    E.D[m] = np.eye(E.nd) / len(E.sharers)
            E.Sblocks = blocks

    def _coarse(self):
        """Coarse saddle problem on (u_Pi, p_0) (SURVEY O-13) with gauge sum vol_i p0_i = 0
        (no gauge with Neumann faces: the Neumann patches' flux constraints make it nonsingular)."""
        N, NPi = self.N, self.NPi
        nc = NPi + N
        Kc = np.zeros((nc, nc))
        for i, S in enumerate(self.sub):
            g = S.pi_glob
            Kc[np.ix_(g, g)] += S.Sc
            b = S.b0T[S.nd:]
            Kc[NPi + i, g] += b
            Kc[g, NPi + i] += b
        self.Kc = Kc
        vol = np.array([S.vol for S in self.sub])
        self.vols = vol
        if self.neumann:
            self.Kc_lu = sla.lu_factor(Kc)
            return
        Mb = np.zeros((nc + 1, nc + 1))
        Mb[:nc, :nc] = Kc
        Mb[nc, NPi:nc] = vol; Mb[NPi:nc, nc] = vol
        self.Kc_lu = sla.lu_factor(Mb)
        self.vols = vol

    def coarse_solve(self, rc):
        if self.neumann:
            return sla.lu_solve(self.Kc_lu, rc)
        x = sla.lu_solve(self.Kc_lu, np.concatenate([rc, [0.0]]))
        return x[:-1]

    # ------------------------------------------------------------------ interface operator
    def apply_S(self, x):
        """S^ [u; p0] = [sum R^T (S_G u^(i) + b0^T p0_i); (b0 u^(i))_i] (Eq.(globInt))."""
        u, p0 = x[:self.nG], x[self.nG:]
        q = np.zeros(self.nG); q0 = np.zeros(self.N)
        for i, S in enumerate(self.sub):
            ui = u[S.Gpos]
            qi = S.SG @ ui + S.b0 * p0[i]
            np.add.at(q, S.Gpos, qi)
            q0[i] = S.b0 @ ui
        return np.concatenate([q, q0])

    def apply_M(self, r):
        """z = M^-1 r = R~_D^T S~^-1 R~_D r (Eq.(BDDCprec))."""
        rG, r0 = r[:self.nG], r[self.nG:]
        NPi, N = self.NPi, self.N
        rc = np.zeros(NPi + N)
        rc[NPi:] = r0
        for E in self.ents:                                    # primal part, unscaled
            if E.r:
                rc[E.pi] += E.P.T @ rG[E.gpos]
        rD = []
        for i, S in enumerate(self.sub):
            v = np.zeros(S.nd)
            for e, dd in zip(S.ents, S.d_off):
                E = self.ents[e]
                if E.nd:
                    v[dd:dd + E.nd] = E.D[i].T @ (E.N.T @ rG[E.gpos])   # scaled dual restriction
            rD.append(v)
            rc[S.pi_glob] += S.Phi.T @ v
        uc = self.coarse_solve(rc)
        uPi, p0 = uc[:NPi], uc[NPi:]
        z = np.zeros(self.nG)
        for E in self.ents:
            if E.r:
                z[E.gpos] += E.P @ uPi[E.pi]
        for i, S in enumerate(self.sub):
            w = sla.cho_solve(S.SDD_chol, rD[i]) + S.Phi @ uPi[S.pi_glob]
            for e, dd in zip(S.ents, S.d_off):
                E = self.ents[e]
                if E.nd:
                    z[E.gpos] += E.N @ (E.D[i] @ w[dd:dd + E.nd])
        return np.concatenate([z, p0])

    # ------------------------------------------------------------------ rhs and back-substitution
    def condensed_rhs(self):
        """g^: g_G = b_G - sum R^T K_GD K_DD^-1 b_D; g_0^(i) = c_i^T g_p^(i)."""
        gs = self.gs
        g = gs.rhs_u[self.gamma].copy()
        g0 = np.zeros(self.N)
        self._bD = []
        for i, S in enumerate(self.sub):
            bI = gs.rhs_u[S.I]
            gp = gs.rhs_p[S.P]
            bD = np.concatenate([bI, S.Z.T @ gp])
            self._bD.append(bD)
            g[S.Gpos] -= S.KDG.T @ S.KDD_lu.solve(bD)
            g0[i] = S.c @ gp
        return np.concatenate([g, g0])

    def back_substitute(self, x):
        """u_I, p_I from Dirichlet solves; p = p_I + p_0 c_i; zero global mean (O-16)."""
        gs, dofs = self.gs, self.gs.dofs
        u = np.zeros(dofs.n_free_vel); p = np.zeros(dofs.npres)
        uG, p0 = x[:self.nG], x[self.nG:]
        u[self.gamma] = uG
        for i, S in enumerate(self.sub):
            y = S.KDD_lu.solve(self._bD[i] - S.KDG @ uG[S.Gpos])
            u[S.I] = y[:S.nI]
            p[S.P] = S.Z @ y[S.nI:] + p0[i] * S.c
        if self.neumann:
            return u, p
        mean = (gs.pmass @ p) / gs.pmass[::dofs.np_].sum()
        cglob = np.zeros(dofs.npres)
        for i, S in enumerate(self.sub):
            cglob[S.P] = S.c
        p -= mean * cglob
        return u, p

    # ------------------------------------------------------------------ adaptive coarse space
    def _adaptive(self, tau):
        """Per face F shared by i,j: S~_FD^(m) (eliminate F' = Gamma_m minus F_D), parallel sums
        A = S~i:S~j, B = Si:Sj, GEVP A psi = lam B psi, keep lam < 1/tau, add rows (B Psi)^T N_F^T
        to C_F (SURVEY O-12)."""
        extra = {}
        self.adaptive_spectra = {}
        self.adaptive_margin = np.inf
        self.adaptive_count = 0
        self.adaptive_pencils = {}
        for e, E in enumerate(self.ents):
            if E.kind != "face" or E.nd == 0 or len(E.sharers) != 2:
                continue
            St, Sf = [], []
            for m in E.sharers:
                S = self.sub[m]
                j = S.ents.index(e)
                dd = S.d_off[j]
                idx = np.arange(dd, dd + E.nd)
                rest = np.setdiff1d(np.arange(S.nd + S.npi), idx)
                ST = S.ST
                SFF = ST[np.ix_(idx, idx)]
                SFr = ST[np.ix_(idx, rest)]
                Srr = ST[np.ix_(rest, rest)]
                St.append(_sym(SFF - SFr @ np.linalg.solve(Srr, SFr.T)))
                Sf.append(SFF)
            par = lambda X, Y: _sym(X @ np.linalg.solve(X + Y, Y))
            Aop = par(St[0], St[1]); Bop = par(Sf[0], Sf[1])
            lam, Psi = sla.eigh(Aop, Bop)
            self.adaptive_spectra[e] = lam
            if self.keep_pencils:
                self.adaptive_pencils[e] = dict(N=E.N.copy(), St=St, Sf=Sf, A=Aop, B=Bop)
            sel = lam < 1.0 / tau
            self.adaptive_margin = min(self.adaptive_margin, float(np.min(np.abs(lam - 1.0 / tau))))
            if np.any(sel):
                rows = (Bop @ Psi[:, sel]).T @ E.N.T
                extra[e] = rows
                self.adaptive_count += int(sel.sum())
        self._constraints(extra)

    # ------------------------------------------------------------------ PCG
    def pcg(self, rtol=1e-10, maxit=2000, record=False):
        """Preconditioned CG on Eq.(globInt) from x0 = 0 (SURVEY O-15)."""
        b = self.condensed_rhs()
        x = np.zeros_like(b)
        r = b.copy()
        r0n = np.linalg.norm(r)
        z = self.apply_M(r)
        p = z.copy()
        rz = r @ z
        alphas, betas, res = [], [], [r0n]
        it = 0
        status = "ok"
        while True:
            if np.linalg.norm(r) <= rtol * r0n:
                break
            if it >= maxit:
                status = "notconv"; break
            q = self.apply_S(p)
            pq = p @ q
            if pq <= 0 or rz <= 0:
                status = "breakdown"; break
            a = rz / pq
            x += a * p
            r -= a * q
            it += 1
            res.append(np.linalg.norm(r))
            alphas.append(a)
            z = self.apply_M(r)
            rz_new = r @ z
            bta = rz_new / rz
            betas.append(bta)
            rz = rz_new
            p = z + bta * p
        lmin, lmax = lanczos_extremes(alphas, betas)
        rep = dict(iterations=it, status=status, r0=r0n, rfinal=res[-1], rel=res[-1] / r0n,
                   lambda_min=lmin, lambda_max=lmax, kappa=lmax / lmin if lmin > 0 else np.inf,
                   residuals=np.array(res), alphas=np.array(alphas), betas=np.array(betas[:len(alphas)]),
                   n_primal=self.NPi, n_coarse=self.NPi + self.N)
        return x, rep

    def solve(self, rtol=1e-10, maxit=2000):
        x, rep = self.pcg(rtol, maxit)
        u, p = self.back_substitute(x)
        return u, p, rep


def lanczos_extremes(alphas, betas):
    """Extreme Ritz values of the CG Lanczos tridiagonal (SURVEY O-15 index convention):
    T_00 = 1/a_0, T_jj = 1/a_j + b_{j-1}/a_{j-1}, T_{j,j-1} = sqrt(b_{j-1})/a_{j-1}."""
    m = len(alphas)
    if m == 0:
        return 1.0, 1.0
    T = np.zeros((m, m))
    for j in range(m):
        T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j > 0 else 0.0)
        if j > 0:
            T[j, j - 1] = T[j - 1, j] = np.sqrt(betas[j - 1]) / alphas[j - 1]
    ev = np.linalg.eigvalsh(T)
    return float(ev[0]), float(ev[-1])
