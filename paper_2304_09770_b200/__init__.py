"""B200-native BDDC-preconditioned CG for the 3D divergence-free VEM Stokes system (arXiv 2304.09770).

Thin ctypes binding of the C ABI in include/vbddc.h: argument marshalling only -- every step of
setup/factor/solve runs in libvbddc.so's sm_100a kernels.  torch is used for device memory and the
CUDA stream.  There is no CPU fallback: importing fails loudly if the library is missing.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libvbddc.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libvbddc.so not built: run `python -c 'import __graft_entry__ as g; g.build()'` "
                      "(the CUDA library is required; there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

VB_OK, VB_EINVAL, VB_ESTATE, VB_ENOMEM, VB_ECUDA, VB_ENCCL, VB_ESINGULAR, VB_EBREAKDOWN, VB_ENOTCONV = range(9)
STATUS = {0: "OK", 1: "EINVAL", 2: "ESTATE", 3: "ENOMEM", 4: "ECUDA", 5: "ENCCL", 6: "ESINGULAR",
          7: "EBREAKDOWN", 8: "ENOTCONV"}
VB_DELUXE, VB_MULTIPLICITY = 0, 1

_p = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_dp = ctypes.POINTER(ctypes.c_double)


class VBMesh(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int32), ("n_vertices", ctypes.c_int64), ("xyz", _dp),
                ("n_faces", ctypes.c_int64), ("face_ptr", _i64p), ("face_vtx", _i64p),
                ("n_cells", ctypes.c_int64), ("cell_ptr", _i64p), ("cell_face", _i64p),
                ("cell_face_sign", ctypes.POINTER(ctypes.c_int8)),
                ("face_on_dirichlet", ctypes.POINTER(ctypes.c_uint8))]


class VBConstraints(ctypes.Structure):
    _fields_ = [("vertex", ctypes.c_int32), ("edge_avg", ctypes.c_int32), ("face_avg", ctypes.c_int32),
                ("face_flux", ctypes.c_int32), ("adaptive_tau", ctypes.c_double),
                ("scaling", ctypes.c_int32), ("svd_rel_tol", ctypes.c_double)]


class VBDist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("nranks", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_unique_id", _p), ("stream", _p), ("loopback_world", _p)]


class VBProblem(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n_sinkers", ctypes.c_int32), ("centres", _dp),
                ("delta", ctypes.c_double), ("omega", ctypes.c_double), ("beta", ctypes.c_double)]


class VBReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("r0_norm", ctypes.c_double), ("r_final_norm", ctypes.c_double), ("rel_residual", ctypes.c_double),
                ("lambda_min", ctypes.c_double), ("lambda_max", ctypes.c_double), ("kappa", ctypes.c_double),
                ("true_rel_residual", ctypes.c_double),
                ("t_setup_s", ctypes.c_double), ("t_factor_s", ctypes.c_double), ("t_solve_s", ctypes.c_double),
                ("bytes_per_iter_model", ctypes.c_double), ("flux_violation_max", ctypes.c_double),
                ("n_primal", ctypes.c_int32), ("n_coarse", ctypes.c_int32), ("n_dofs_paper", ctypes.c_int64),
                ("n_adaptive", ctypes.c_int32), ("adaptive_margin", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


def _sig(name, res, args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = args
    return f


_vb_setup = _sig("vb_setup", ctypes.c_int, [ctypes.POINTER(VBMesh), _i32p, ctypes.c_int32, _i32p,
                                           ctypes.POINTER(VBConstraints), _dp, ctypes.POINTER(VBDist), ctypes.POINTER(_p)])
_vb_setup_el = _sig("vb_setup_from_elements", ctypes.c_int,
                    [ctypes.POINTER(VBMesh), _i32p, ctypes.c_int32, _i32p, ctypes.POINTER(VBConstraints), _dp,
                     ctypes.POINTER(VBDist), _i64p, _dp, _i64p, _dp, ctypes.POINTER(_p)])
_vb_factor = _sig("vb_factor", ctypes.c_int, [_p])
_vb_build_rhs = _sig("vb_build_rhs", ctypes.c_int, [_p, ctypes.POINTER(VBProblem), _p])
_vb_pcg_solve = _sig("vb_pcg_solve", ctypes.c_int, [_p, _p, _p, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(VBReport)])
_vb_pcg_solve_host = _sig("vb_pcg_solve_host", ctypes.c_int,
                          [_p, _dp, _dp, ctypes.c_double, ctypes.c_int32, ctypes.POINTER(VBReport)])
_vb_apply_operator = _sig("vb_apply_operator", ctypes.c_int, [_p, _p, _p])
_vb_num_free_dofs = _sig("vb_num_free_dofs", ctypes.c_int, [_p, _i64p, _i64p])
_vb_dof_layout = _sig("vb_dof_layout", ctypes.c_int, [_p, _i64p])
_vb_cell_local_dofs = _sig("vb_cell_local_dofs", ctypes.c_int, [_p, ctypes.c_int64, _i64p, _i32p, _i64p, _i32p])
_vb_get_element_matrices = _sig("vb_get_element_matrices", ctypes.c_int, [_p, ctypes.c_int64, _dp, _dp])
_vb_stats = _sig("vb_stats", ctypes.c_int, [_p, _i64p])
_vb_last_error = _sig("vb_last_error", ctypes.c_char_p, [_p])
_vb_kernel_times = _sig("vb_kernel_times", ctypes.c_int, [_p, _dp, ctypes.c_int32, _i32p])
_vb_kernel_time_name = _sig("vb_kernel_time_name", ctypes.c_char_p, [ctypes.c_int32])
_vb_destroy = _sig("vb_destroy", ctypes.c_int, [_p])
_vb_nccl_unique_id = _sig("vb_nccl_unique_id", ctypes.c_int, [_p])
_vb_debug_iop = _sig("vb_debug_interface_op", ctypes.c_int, [_p, ctypes.c_int32, _dp, _dp])
_vb_interface_dofs = _sig("vb_interface_dofs", ctypes.c_int, [_p, _i64p, _i64p])
_vb_set_option = _sig("vb_set_option", ctypes.c_int, [_p, ctypes.c_char_p, ctypes.c_double])
_vb_debug_subop = _sig("vb_debug_subdomain_op", ctypes.c_int, [_p, ctypes.c_int32, ctypes.c_int32, _i64p, _dp, _i64p])
_vb_nccl_selftest = _sig("vb_debug_nccl_selftest", ctypes.c_int, [ctypes.c_int32, _dp])
_vb_debug_gemm = _sig("vb_debug_gemm", ctypes.c_int,
                     [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_double, _p, ctypes.c_int32,
                      ctypes.c_int32, _p, ctypes.c_int32, ctypes.c_int32, _p, ctypes.c_double, _p,
                      ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _p,
                      ctypes.c_int32, ctypes.c_int32, ctypes.c_int32])

EXPORTED = ["vb_plan_exchange", "vb_plan_coarse_dissection", "vb_nccl_unique_id", "vb_loopback_world_create", "vb_loopback_world_destroy", "vb_setup", "vb_setup_from_elements", "vb_factor", "vb_build_rhs",
            "vb_pcg_solve", "vb_pcg_solve_host", "vb_apply_operator", "vb_debug_interface_op", "vb_debug_gemm",
            "vb_interface_dofs", "vb_num_free_dofs", "vb_dof_layout",
            "vb_cell_local_dofs", "vb_get_element_matrices", "vb_stats", "vb_kernel_times",
            "vb_kernel_time_name", "vb_last_error", "vb_destroy", "vb_set_option", "vb_debug_nccl_selftest",
            "vb_debug_subdomain_op"]


class VBError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a, ctype):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


def _cons(constraints):
    c = dict(vertex=1, edge_avg=1, face_avg=1, face_flux=1, adaptive_tau=0.0, scaling=VB_DELUXE, svd_rel_tol=1e-10)
    if constraints:
        c.update({k: v for k, v in constraints.items() if k in c})
        if constraints.get("all_primal"):
            c["svd_rel_tol"] = -1.0
    return VBConstraints(int(c["vertex"]), int(c["edge_avg"]), int(c["face_avg"]), int(c["face_flux"]),
                         float(c["adaptive_tau"]), int(c["scaling"]), float(c["svd_rel_tol"]))


class Context:
    """One vb_ctx (one GPU).  Call factor(), then build_rhs()/pcg_solve() any number of times."""

    def __init__(self, mesh, k, cell_subdomain, n_subdomains, viscosity, constraints=None, stream=None,
                 device=0, elements=None, rank=0, nranks=1, subdomain_rank=None, nccl_id=None, world=None):
        """Multi-rank (one rank per GPU): pass rank, nranks, subdomain_rank and either
        nccl_id (128 bytes from nccl_unique_id() on rank 0, broadcast by the caller) or world (a
        LoopbackWorld: ranks as threads of one process on one GPU, test transport)."""
        import torch
        self._keep = []
        xyz = _arr(mesh.xyz, np.float64)
        fp, fv = _arr(mesh.face_ptr, np.int64), _arr(mesh.face_vtx, np.int64)
        cp, cf = _arr(mesh.cell_ptr, np.int64), _arr(mesh.cell_face, np.int64)
        cs = _arr(mesh.cell_face_sign, np.int8)
        fb = _arr(mesh.face_on_boundary, np.uint8)
        self._keep += [xyz, fp, fv, cp, cf, cs, fb]
        m = VBMesh(int(k), xyz.shape[0], _ptr(xyz, ctypes.c_double), fp.size - 1, _ptr(fp, ctypes.c_int64),
                   _ptr(fv, ctypes.c_int64), cp.size - 1, _ptr(cp, ctypes.c_int64), _ptr(cf, ctypes.c_int64),
                   _ptr(cs, ctypes.c_int8), _ptr(fb, ctypes.c_uint8))
        sub = _arr(cell_subdomain, np.int32)
        nu = _arr(viscosity, np.float64)
        if stream is None:
            stream = torch.cuda.current_stream(device)
        self.stream = stream
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(idbuf)
        dist = VBDist(int(rank), int(nranks), int(device), ctypes.cast(idbuf, _p) if idbuf is not None else None,
                      ctypes.c_void_p(stream.cuda_stream), world.handle if world is not None else None)
        srank = None
        if subdomain_rank is not None:
            sr = _arr(subdomain_rank, np.int32)
            self._keep.append(sr)
            srank = _ptr(sr, ctypes.c_int32)
        cons = _cons(constraints)
        h = _p()
        if elements is None:
            st = _vb_setup(ctypes.byref(m), _ptr(sub, ctypes.c_int32), int(n_subdomains), srank, ctypes.byref(cons),
                           _ptr(nu, ctypes.c_double), ctypes.byref(dist), ctypes.byref(h))
        else:
            pa, A, pb, B = [_arr(x, t) for x, t in zip(elements, (np.int64, np.float64, np.int64, np.float64))]
            st = _vb_setup_el(ctypes.byref(m), _ptr(sub, ctypes.c_int32), int(n_subdomains), srank, ctypes.byref(cons),
                              _ptr(nu, ctypes.c_double), ctypes.byref(dist), _ptr(pa, ctypes.c_int64),
                              _ptr(A, ctypes.c_double), _ptr(pb, ctypes.c_int64), _ptr(B, ctypes.c_double),
                              ctypes.byref(h))
        if st != VB_OK:
            raise VBError(st, _vb_last_error(None).decode())
        self._h = h
        nv, npr = ctypes.c_int64(), ctypes.c_int64()
        _vb_num_free_dofs(self._h, ctypes.byref(nv), ctypes.byref(npr))
        self.n_vel, self.n_p = nv.value, npr.value
        self.n_free = self.n_vel + self.n_p

    def _dev(self, t, name):
        """Device vector argument: CUDA, float64, contiguous, exactly this rank's n_free entries."""
        import torch
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()
                and t.numel() == self.n_free):
            raise ValueError("%s must be a contiguous float64 CUDA tensor of %d entries" % (name, self.n_free))
        return ctypes.c_void_p(t.data_ptr())

    def _host(self, a, name):
        """Host vector argument: float64 numpy array, C-contiguous, exactly n_free entries."""
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
                and a.size == self.n_free):
            raise ValueError("%s must be a C-contiguous float64 numpy array of %d entries" % (name, self.n_free))
        return _ptr(a, ctypes.c_double)

    def _check(self, st):
        if st != VB_OK:
            raise VBError(st, _vb_last_error(self._h).decode())

    def factor(self):
        self._check(_vb_factor(self._h))

    def set_option(self, name, value):
        """vb_set_option: "true_residual" (0/1) -> vb_report.true_rel_residual through K7;
        "p2p" (0/1, before factor) -> peer-store interface exchanges in the PCG step;
        "coarse_dissection" (1/0/-1 auto, before factor) -> rank-level dissection of the coarse problem."""
        self._check(_vb_set_option(self._h, name.encode(), float(value)))

    def build_rhs(self, problem, out):
        """problem: dict(kind='manufactured'|'sinker', centres, delta, omega, beta); out: cuda float64 tensor."""
        if problem.get("kind", "manufactured") == "sinker":
            cen = _arr(problem["centres"], np.float64)
            self._keep.append(cen)
            p = VBProblem(1, cen.shape[0], _ptr(cen, ctypes.c_double), problem["delta"], problem["omega"], problem["beta"])
        else:
            p = VBProblem(0, 0, None, 0.0, 0.0, 0.0)
        self._check(_vb_build_rhs(self._h, ctypes.byref(p), self._dev(out, "out")))
        return out

    def pcg_solve(self, rhs, x, rtol=1e-10, maxit=2000, raise_on_error=True):
        rep = VBReport()
        st = _vb_pcg_solve(self._h, self._dev(rhs, "rhs"), self._dev(x, "x"), float(rtol),
                           int(maxit), ctypes.byref(rep))
        d = rep.as_dict()
        d["status"] = STATUS[st]
        if raise_on_error and st != VB_OK:
            self._check(st)
        return d

    def pcg_solve_host(self, rhs_host, x_host, rtol=1e-10, maxit=2000):
        rep = VBReport()
        self._check(_vb_pcg_solve_host(self._h, self._host(rhs_host, "rhs_host"), self._host(x_host, "x_host"),
                                       float(rtol), int(maxit), ctypes.byref(rep)))
        return rep.as_dict()

    def apply_operator(self, x, y):
        self._check(_vb_apply_operator(self._h, self._dev(x, "x"), self._dev(y, "y")))
        return y

    def interface_dofs(self):
        n = ctypes.c_int64()
        self._check(_vb_interface_dofs(self._h, None, ctypes.byref(n)))
        ids = np.zeros(n.value, np.int64)
        self._check(_vb_interface_dofs(self._h, _ptr(ids, ctypes.c_int64), ctypes.byref(n)))
        return ids

    def interface_op(self, which, vec):
        """which: 'S' (interface saddle operator) or 'M' (BDDC preconditioner); original coordinates."""
        v = _arr(vec, np.float64)
        out = np.zeros_like(v)
        self._check(_vb_debug_iop(self._h, 0 if which == "S" else 1, _ptr(v, ctypes.c_double),
                                  _ptr(out, ctypes.c_double)))
        return out

    def subdomain_op(self, sub, which):
        """(free velocity ids, dense operator) of local subdomain `sub`: which 'S' = S_Gamma^(i),
        'M' = N (D S_DD^-1 D^T) N^T (vb_debug_subdomain_op)."""
        n = ctypes.c_int64()
        w = 0 if which == "S" else 1
        self._check(_vb_debug_subop(self._h, int(sub), w, None, None, ctypes.byref(n)))
        ids = np.zeros(n.value, np.int64)
        out = np.zeros((n.value, n.value))
        self._check(_vb_debug_subop(self._h, int(sub), w, _ptr(ids, ctypes.c_int64), _ptr(out, ctypes.c_double),
                                    ctypes.byref(n)))
        return ids, out.T.copy()     # column-major -> row-major

    def dof_layout(self):
        ids = np.zeros(self.n_free, np.int64)
        self._check(_vb_dof_layout(self._h, _ptr(ids, ctypes.c_int64)))
        return ids

    def cell_local_dofs(self, cell):
        if not hasattr(self, "_nv_max"):
            self._nv_max = int(self.stats()["nv_max"])
        v = np.zeros(self._nv_max, np.int64); p = np.zeros(64, np.int64)
        nv, npr = ctypes.c_int32(), ctypes.c_int32()
        self._check(_vb_cell_local_dofs(self._h, int(cell), _ptr(v, ctypes.c_int64), ctypes.byref(nv),
                                        _ptr(p, ctypes.c_int64), ctypes.byref(npr)))
        return v[:nv.value].copy(), p[:npr.value].copy()

    def element_matrices(self, cell):
        v, p = self.cell_local_dofs(cell)
        A = np.zeros((v.size, v.size)); B = np.zeros((p.size, v.size))
        self._check(_vb_get_element_matrices(self._h, int(cell), _ptr(A, ctypes.c_double), _ptr(B, ctypes.c_double)))
        return A, B

    def stats(self):
        o = np.zeros(28, np.int64)
        self._check(_vb_stats(self._h, _ptr(o, ctypes.c_int64)))
        keys = ["n_dofs_paper", "n_free_vel", "n_pres", "n_sub", "n_ent", "n_gamma", "n_primal", "n_coarse",
                "n_delta", "max_n", "max_nG", "max_nd", "n_edges", "bytes_per_iter", "nv_max", "n_colors",
                "sum_pk_G", "sum_pk_D", "sum_dlx_sq", "sum_phi", "pk_coarse", "last_iterations", "n_cells",
                "factor_gemm_flops", "factor_alloc_us", "factor_gemm_us", "n_coarse_root", "n_coarse_local"]
        return dict(zip(keys, o.tolist()))

    def kernel_times(self):
        """{category name: average ms per launch} of the last solve (needs VB_KERNEL_TIMING=1)."""
        ms = np.zeros(16)
        n = ctypes.c_int32()
        self._check(_vb_kernel_times(self._h, _ptr(ms, ctypes.c_double), 16, ctypes.byref(n)))
        return {_vb_kernel_time_name(i).decode(): float(ms[i]) for i in range(n.value)}

    def close(self):
        if getattr(self, "_h", None):
            _vb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_vb_nccl_uid = _sig("vb_nccl_unique_id", ctypes.c_int, [_p])
_vb_lw_create = _sig("vb_loopback_world_create", ctypes.c_int, [ctypes.c_int32, ctypes.POINTER(_p)])
_vb_lw_destroy = _sig("vb_loopback_world_destroy", ctypes.c_int, [_p])


def nccl_unique_id():
    """128-byte NCCL unique id (rank 0), to broadcast with torch.distributed before Context()."""
    buf = ctypes.create_string_buffer(128)
    st = _vb_nccl_uid(ctypes.cast(buf, _p))
    if st != VB_OK:
        raise VBError(st, _vb_last_error(None).decode())
    return bytes(buf.raw)


def nccl_selftest(device=0):
    """vb_debug_nccl_selftest on one GPU: dict(eager_ok, graph_ok, graph_iterations, max_err, message)."""
    out = np.zeros(4)
    st = _vb_nccl_selftest(int(device), _ptr(out, ctypes.c_double))
    if st != VB_OK:
        raise VBError(st, _vb_last_error(None).decode())
    return dict(eager_ok=bool(out[0]), graph_ok=bool(out[1]), graph_iterations=int(out[2]), max_err=float(out[3]),
                message=_vb_last_error(None).decode() if not out[1] else "")


def debug_gemm(A, B, C, alpha=1.0, beta=0.0, d=None, transA=False, transB=False, kz=None):
    """C_b = alpha op(A_b) diag(d) op(B_b) + beta C_b with the factorisation's DMMA GEMM
    (vb_debug_gemm).  A, B, C: CUDA float64 tensors of shape (batch, cols, rows) holding each matrix
    COLUMN-major (i.e. the transposes of the logical matrices, contiguous); C is updated in place.
    kz = (kzA, kzB): triangular operands, op(A)(i, k) = 0 for k < i + kzA, op(B)(k, j) = 0 for
    k < j + kzB (the kernel skips those K slabs)."""
    import torch
    for t in (A, B, C):
        assert t.is_cuda and t.dtype == torch.float64 and t.is_contiguous() and t.dim() == 3
    batch = C.shape[0]
    M, N = C.shape[2], C.shape[1]
    K = A.shape[2] if transA else A.shape[1]
    st = _vb_debug_gemm(M, N, K, alpha, ctypes.c_void_p(A.data_ptr()), A.shape[2], int(transA),
                        ctypes.c_void_p(B.data_ptr()), B.shape[2], int(transB),
                        ctypes.c_void_p(d.data_ptr()) if d is not None else None, beta,
                        ctypes.c_void_p(C.data_ptr()), C.shape[2], batch,
                        A.shape[1] * A.shape[2] if A.shape[0] > 1 else 0,
                        B.shape[1] * B.shape[2] if B.shape[0] > 1 else 0, C.shape[1] * C.shape[2],
                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), 1 if kz else 0,
                        kz[0] if kz else 0, kz[1] if kz else 0)
    if st != VB_OK:
        raise VBError(st, _vb_last_error(None).decode())
    return C


class LoopbackWorld:
    """Test transport: nranks library ranks as threads of this process sharing one GPU."""

    def __init__(self, nranks):
        self.handle = _p()
        st = _vb_lw_create(int(nranks), ctypes.byref(self.handle))
        if st != VB_OK:
            raise VBError(st, "loopback world")
        self.nranks = nranks

    def close(self):
        if self.handle:
            _vb_lw_destroy(self.handle)
            self.handle = None


def box_ranks(sub_grid, rank_grid):
    """Subdomain -> rank for a box partition: sub_grid (sx, sy, sz) subdomains (x fastest),
    rank_grid (rx, ry, rz) ranks, each owning a contiguous box of subdomains."""
    sx, sy, sz = sub_grid
    rx, ry, rz = rank_grid
    assert sx % rx == 0 and sy % ry == 0 and sz % rz == 0
    out = np.zeros(sx * sy * sz, np.int32)
    for k in range(sz):
        for j in range(sy):
            for i in range(sx):
                out[i + sx * (j + sy * k)] = (i // (sx // rx)) + rx * ((j // (sy // ry)) + ry * (k // (sz // rz)))
    return out


_vb_plan = _sig("vb_plan_exchange", ctypes.c_int, [ctypes.POINTER(VBMesh), _i32p, ctypes.c_int32, _i32p,
                                                    ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, _i64p, _i64p,
                                                    _i64p])


def plan_exchange(mesh, k, cell_subdomain, subdomain_rank, rank, nranks, mode=0):
    """Host-only (no GPU): (send_counts[nranks], recv_counts[nranks], n_owned_free) of this rank's
    interface exchange plan (vb_plan_exchange)."""
    keep = []
    m = _mesh_struct(mesh, k, keep)
    sub = _arr(cell_subdomain, np.int32)
    sr = _arr(subdomain_rank, np.int32)
    snd = np.zeros(nranks, np.int64); rcv = np.zeros(nranks, np.int64)
    own = ctypes.c_int64()
    st = _vb_plan(ctypes.byref(m), _ptr(sub, ctypes.c_int32), int(sub.max()) + 1, _ptr(sr, ctypes.c_int32), int(rank),
                  int(nranks), int(mode), _ptr(snd, ctypes.c_int64), _ptr(rcv, ctypes.c_int64), ctypes.byref(own))
    if st != VB_OK:
        raise VBError(st, _vb_last_error(None).decode())
    return snd, rcv, own.value


_vb_plan_cd = _sig("vb_plan_coarse_dissection", ctypes.c_int, [ctypes.POINTER(VBMesh), _i32p, ctypes.c_int32, _i32p,
                                                              ctypes.c_int32, ctypes.c_int32, _i32p, _i64p])


def plan_coarse_dissection(mesh, k, cell_subdomain, subdomain_rank, rank, nranks, primal_per_kind=(3, 3, 3)):
    """Host-only (no GPU): sizes of this rank's coarse dissection (vb_plan_coarse_dissection):
    dict(n_interior, n_S, n_sep, n_root, n_local, n_primal)."""
    keep = []
    m = _mesh_struct(mesh, k, keep)
    sub = _arr(cell_subdomain, np.int32)
    sr = _arr(subdomain_rank if subdomain_rank is not None else np.zeros(int(sub.max()) + 1), np.int32)
    ppk = np.asarray(primal_per_kind, np.int32)
    out = np.zeros(6, np.int64)
    st = _vb_plan_cd(ctypes.byref(m), _ptr(sub, ctypes.c_int32), int(sub.max()) + 1, _ptr(sr, ctypes.c_int32),
                     int(rank), int(nranks), _ptr(ppk, ctypes.c_int32), _ptr(out, ctypes.c_int64))
    if st != VB_OK:
        raise VBError(st, _vb_last_error(None).decode())
    return dict(zip(["n_interior", "n_S", "n_sep", "n_root", "n_local", "n_primal"], out.tolist()))


def _mesh_struct(mesh, k, keep):
    xyz = _arr(mesh.xyz, np.float64)
    fp, fv = _arr(mesh.face_ptr, np.int64), _arr(mesh.face_vtx, np.int64)
    cp, cf = _arr(mesh.cell_ptr, np.int64), _arr(mesh.cell_face, np.int64)
    cs = _arr(mesh.cell_face_sign, np.int8)
    fb = _arr(mesh.face_on_boundary, np.uint8)
    keep += [xyz, fp, fv, cp, cf, cs, fb]
    return VBMesh(int(k), xyz.shape[0], _ptr(xyz, ctypes.c_double), fp.size - 1, _ptr(fp, ctypes.c_int64),
                  _ptr(fv, ctypes.c_int64), cp.size - 1, _ptr(cp, ctypes.c_int64), _ptr(cf, ctypes.c_int64),
                  _ptr(cs, ctypes.c_int8), _ptr(fb, ctypes.c_uint8))


def problem_args(prob):
    """Library problem descriptor for a synthetic.Problem."""
    if prob.kind == "sinker":
        return dict(kind="sinker", centres=prob.params["centres"], delta=prob.params["delta"],
                    omega=prob.params["omega"], beta=prob.params["beta"])
    return dict(kind="manufactured")


def context_for(prob, elements=None, constraints=None, stream=None, **dist):
    cons = dict(prob.constraints)
    if constraints:
        cons.update(constraints)
    return Context(prob.mesh, prob.k, prob.cell_subdomain, int(prob.cell_subdomain.max()) + 1, prob.nu_cell,
                   constraints=cons, stream=stream, elements=elements, **dist)
