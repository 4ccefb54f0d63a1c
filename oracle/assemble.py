"""Global VEM Stokes system (oracle; test infrastructure only).

Global DOF numbering (SURVEY O-6 "entity-type-major, entity-id-minor"):
  velocity: vertex v -> 3v+c; edge e (global (min,max) order, GL point j along min->max)
            -> oE + 3(k-1)e + 3j + c; face f -> oF + 3 nm f + t nm + a (t: n, t1, t2);
            cell K -> oC + K (n4+n5) + i (D4 then D5);
  pressure: cell K -> K np + a.
Boundary DOFs (all D1-D3 of entities on the boundary) are removed; the exact trace is lifted by
its DOF interpolant.  The discrete problem is Eq.(DiscProblem) in the
matrix form Eq.(MatrixForm).
"""
import os
import numpy as np
import scipy.sparse as sp
from .vem import ElementOps, mesh_edges, EdgeIndex, face_geometry, Layout
from .poly import dim2, dim3, mono2, gauss_lobatto01
from . import problems


class GlobalDofs:
    def __init__(self, mesh, k):
        self.k = k
        self.edges = mesh_edges(mesh)
        self.eidx = EdgeIndex(self.edges, mesh.n_vertices)
        nV, nE, nF, nK = mesh.n_vertices, len(self.edges), mesh.n_faces, mesh.n_cells
        self.nm = dim2(k - 2)
        self.n4 = 3 * dim3(k - 3) - dim3(k - 4)
        self.n5 = dim3(k - 1) - 1
        self.np_ = dim3(k - 1)
        self.oE = 3 * nV
        self.oF = self.oE + 3 * (k - 1) * nE
        self.oC = self.oF + 3 * self.nm * nF
        self.nvel = self.oC + nK * (self.n4 + self.n5)
        self.npres = nK * self.np_
        # boundary entities: face_on_boundary 1 = Dirichlet, 2 = Neumann (natural condition, the
        # DOFs of the face closure stay free unless they also lie on a Dirichlet face; DESIGN A35)
        bf = np.nonzero(mesh.face_on_boundary == 1)[0]
        bverts = set(); bedges = set()
        for f in bf:
            lp = mesh.face(f)
            for i in range(len(lp)):
                bverts.add(int(lp[i]))
                bedges.add(self.eidx(lp[i], lp[(i + 1) % len(lp)]))
        nf = np.nonzero(mesh.face_on_boundary == 2)[0]
        self.neumann = nf.size > 0
        on_neu = np.zeros(self.nvel, dtype=bool)
        for f in nf:
            lp = mesh.face(f)
            for i in range(len(lp)):
                on_neu[3 * int(lp[i]) + np.arange(3)] = True
                e = self.eidx(lp[i], lp[(i + 1) % len(lp)])
                on_neu[self.oE + 3 * (k - 1) * e + np.arange(3 * (k - 1))] = True
            on_neu[self.oF + 3 * self.nm * f + np.arange(3 * self.nm)] = True
        self.bverts = np.array(sorted(bverts), dtype=np.int64)
        self.bedges = np.array(sorted(bedges), dtype=np.int64)
        self.bfaces = bf
        isb = np.zeros(self.nvel, dtype=bool)
        for c in range(3):
            isb[3 * self.bverts + c] = True
        for j in range(3 * (k - 1)):
            isb[self.oE + 3 * (k - 1) * self.bedges + j] = True
        for j in range(3 * self.nm):
            isb[self.oF + 3 * self.nm * bf + j] = True
        self.is_bnd = isb
        self.free_vel = np.nonzero(~isb)[0]
        self.bnd_vel = np.nonzero(isb)[0]
        self.n_free_vel = self.free_vel.size
        self.vel2free = -np.ones(self.nvel, dtype=np.int64)
        self.vel2free[self.free_vel] = np.arange(self.free_vel.size)
        self.free_on_neumann = on_neu[self.free_vel]      # per free velocity DOF

    def n_dofs_paper(self):
        """nDofs as counted in T2-T4: all velocity DOFs incl. boundary + all pressure."""
        return self.nvel + self.npres

    def local_to_global(self, op, K):
        g, L, k = op.g, op.L, self.k
        idx = np.empty(L.nv, dtype=np.int64)
        for lv, v in enumerate(g.verts):
            idx[3 * lv:3 * lv + 3] = 3 * v + np.arange(3)
        for le, e in enumerate(g.edges):
            s = L.edof(le, 0, 0)
            idx[s:s + 3 * (k - 1)] = self.oE + 3 * (k - 1) * e + np.arange(3 * (k - 1))
        for lf, f in enumerate(g.faces):
            s = L.fdof(lf, 0, 0)
            idx[s:s + 3 * self.nm] = self.oF + 3 * self.nm * f + np.arange(3 * self.nm)
        nc = self.n4 + self.n5
        idx[L.o4:L.o4 + nc] = self.oC + K * nc + np.arange(nc)
        pidx = K * self.np_ + np.arange(self.np_)
        return idx, pidx


def _topology_key(mesh, K, dofs):
    fids, sgn = mesh.cell_faces(K)
    order = np.argsort(fids)
    loops = [mesh.face(f) for f in fids[order]]
    verts = np.unique(np.concatenate(loops))
    loc = {int(v): i for i, v in enumerate(verts)}
    X = mesh.xyz[verts]
    topo = tuple(tuple(loc[int(v)] for v in lp) for lp in loops) + (tuple(sgn[order]),)
    return (X - X[0]).tobytes() + repr(topo).encode(), X[0]


def _build_op(args):
    mesh, K, k, eidx = args
    return ElementOps(mesh, K, eidx, k, 1.0)


class ElementSet:
    """Element operators for every cell.  Cells that are exact translates of each other (same
    relative coordinates and local topology) share one ElementOps evaluated at nu=1; a_h^K is
    linear in nu_K (consistency and D-recipe both scale with nu), so A_K = nu_K A(1)."""

    def __init__(self, prob, dofs, processes=None):
        mesh, k = prob.mesh, prob.k
        self.keys, self.shift, uniq = [], [], {}
        for K in range(mesh.n_cells):
            key, x0 = _topology_key(mesh, K, dofs)
            if key not in uniq:
                uniq[key] = (K, x0)
            self.keys.append(key)
            self.shift.append(x0 - uniq[key][1])
        todo = [(mesh, K, k, dofs.eidx) for (K, _) in uniq.values()]
        nproc = processes or min(os.cpu_count() or 1, 16)
        if len(todo) > 64 and nproc > 1:
            import multiprocessing as mp
            # spawn, not fork: forking a process whose BLAS threads are running can deadlock;
            # one BLAS thread per worker (the children inherit the environment at spawn)
            keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
            saved = {key: os.environ.get(key) for key in keys}
            for key in keys:
                os.environ[key] = "1"
            try:
                with mp.get_context("spawn").Pool(nproc) as pool:
                    ops = pool.map(_build_op, todo, chunksize=16)
            finally:
                for key, v in saved.items():
                    if v is None:
                        os.environ.pop(key, None)
                    else:
                        os.environ[key] = v
        else:
            ops = [_build_op(t) for t in todo]
        self.ops = dict(zip(uniq.keys(), ops))
        self.ref_cell = {key: K for key, (K, _) in uniq.items()}
        self.prob, self.dofs = prob, dofs
        self.l2g = []
        for K in range(mesh.n_cells):
            op = self.ops[self.keys[K]]
            # the local->global map must be built from this cell's own topology
            self.l2g.append(self._l2g(K))

    def _l2g(self, K):
        mesh, dofs, k = self.prob.mesh, self.dofs, self.prob.k
        fids, _ = mesh.cell_faces(K)
        fids = np.sort(fids)
        loops = [mesh.face(f) for f in fids]
        verts = np.unique(np.concatenate(loops))
        ed = sorted({dofs.eidx(lp[i], lp[(i + 1) % len(lp)]) for lp in loops for i in range(len(lp))})

        class G:
            pass
        g = G(); g.verts, g.edges, g.faces = verts, np.array(ed), fids
        op = self.ops[self.keys[K]]

        class O:
            pass
        o = O(); o.g, o.L = g, op.L
        return dofs.local_to_global(o, K)

    def op(self, K):
        return self.ops[self.keys[K]]


class GlobalSystem:
    """Assembled A, B, load, lifted rhs on the free DOFs (SURVEY O-6)."""

    def __init__(self, prob, processes=None, u_bc=None, f_of_nu=None):
        self.prob = prob
        mesh, k = prob.mesh, prob.k
        self.dofs = dofs = GlobalDofs(mesh, k)
        self.el = el = ElementSet(prob, dofs, processes)
        nu = prob.nu_cell
        rows, cols, vals = [], [], []
        brow, bcol, bval = [], [], []
        fvel = np.zeros(dofs.nvel)
        if f_of_nu is not None:
            self.f = f_of_nu
        elif prob.kind == "manufactured":
            self.f = problems.f_manufactured
        else:
            fs = problems.f_sinker(prob.params)
            self.f = lambda nuK: fs
        for K in range(mesh.n_cells):
            op = el.op(K)
            iv, ip = el.l2g[K]
            A = nu[K] * op.A
            rows.append(np.repeat(iv, iv.size)); cols.append(np.tile(iv, iv.size)); vals.append(A.ravel())
            brow.append(np.repeat(ip, iv.size)); bcol.append(np.tile(iv, ip.size)); bval.append(op.B.ravel())
            fvel[iv] += op.load(self.f(nu[K]), el.shift[K])
        self.A = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                               shape=(dofs.nvel, dofs.nvel))
        self.B = sp.csr_matrix((np.concatenate(bval), (np.concatenate(brow), np.concatenate(bcol))),
                               shape=(dofs.npres, dofs.nvel))
        self.fvel = fvel
        # lifting of the exact trace; sinker: homogeneous
        uD = np.zeros(dofs.nvel)
        if u_bc is not None:
            uD = self.boundary_interpolant(u_bc)
        elif prob.kind == "manufactured":
            uD = self.boundary_interpolant(problems.u_exact)
        self.uD = uD
        fr, bd = dofs.free_vel, dofs.bnd_vel
        self.Aff = self.A[fr][:, fr].tocsr()
        self.Bf = self.B[:, fr].tocsr()
        self.rhs_u = fvel[fr] - self.A[fr][:, bd] @ uD[bd]
        self.rhs_p = -(self.B[:, bd] @ uD[bd])
        # m_j = int psi_j (pressure dual basis): vol_K for the constant moment
        self.pmass = np.zeros(dofs.npres)
        for K in range(mesh.n_cells):
            self.pmass[K * dofs.np_] = el.op(K).g.vol
        self.n_free = dofs.n_free_vel + dofs.npres

    def boundary_interpolant(self, u):
        """D1-D3 of u on the boundary entities (vertex values, GL edge points, face moments)."""
        mesh, dofs, k = self.prob.mesh, self.dofs, self.prob.k
        out = np.zeros(dofs.nvel)
        X = mesh.xyz
        out[3 * dofs.bverts[:, None] + np.arange(3)] = u(X[dofs.bverts])
        xg, _ = gauss_lobatto01(k + 1)
        for e in dofs.bedges:
            a, b = dofs.edges[e]
            for j in range(k - 1):
                s = dofs.oE + 3 * (k - 1) * e + 3 * j
                out[s:s + 3] = u((X[a] + xg[j + 1] * (X[b] - X[a]))[None])[0]
        for f in dofs.bfaces:
            F = face_geometry(mesh, f, k)
            m2, _ = mono2((F.qp - F.xc) @ np.stack([F.t1, F.t2]).T, k - 2, F.h)
            uq = u(F.qp)
            for t, tau in enumerate((F.n, F.t1, F.t2)):
                s = dofs.oF + 3 * dofs.nm * f + t * dofs.nm
                out[s:s + dofs.nm] = ((F.qw * (uq @ tau)) @ m2) / F.area
        return out

    def saddle_matrix(self):
        """Free-DOF saddle matrix [[A, B^T], [B, 0]] (sparse)."""
        return sp.bmat([[self.Aff, self.Bf.T], [self.Bf, None]]).tocsr()

    def direct_solve(self):
        """Sparse direct solve of Eq.(DiscProblem) with the zero-mean pressure gauge
        (Q_{h,0}) imposed by a Lagrange multiplier; with Neumann faces the
        pressure is unique and the saddle matrix is solved as it stands."""
        import scipy.sparse.linalg as spla
        nvf, npr = self.dofs.n_free_vel, self.dofs.npres
        if self.dofs.neumann:
            x = spla.spsolve(self.saddle_matrix().tocsc(), np.concatenate([self.rhs_u, self.rhs_p]))
            return x[:nvf], x[nvf:]
        m = sp.csr_matrix(self.pmass[None, :])
        M = sp.bmat([[self.Aff, self.Bf.T, None], [self.Bf, None, m.T], [None, m, None]]).tocsc()
        rhs = np.concatenate([self.rhs_u, self.rhs_p, [0.0]])
        x = spla.spsolve(M, rhs)
        return x[:nvf], x[nvf:nvf + npr]

    def full_velocity(self, u_free):
        u = self.uD.copy()
        u[self.dofs.free_vel] = u_free
        return u

    def errors(self, u_free, p):
        """H1-seminorm velocity error and L2 pressure error (SURVEY O-16)."""
        mesh = self.prob.mesh
        u = self.full_velocity(u_free)
        eh1 = ep = 0.0
        for K in range(mesh.n_cells):
            op = self.el.op(K)
            iv, ip = self.el.l2g[K]
            eh1 += op.h1_error_sq(u[iv], problems.grad_u_exact, self.el.shift[K])
            ep += op.l2_pressure_error_sq(p[ip], problems.p_exact, self.el.shift[K])
        return np.sqrt(eh1), np.sqrt(ep)
