/*
 * vbddc.h -- C ABI of the B200-native BDDC-preconditioned CG for the 3D divergence-free
 * VEM discretisation of Stokes (arXiv 2304.09770).  `P:n` = PAPER.md line n.
 *
 * Call sequence:  vb_setup -> vb_factor -> vb_pcg_solve (repeatable)
 *                                   -> vb_destroy.
 * All functions return vb_status; no C++ exception or longjmp crosses the ABI.  On failure
 * vb_last_error(ctx) (or vb_last_error(NULL) for failures before a context exists) returns a
 * NUL-terminated message naming the failing subdomain/entity where applicable.
 * A context is single-threaded (one driving call at a time) and bound to one CUDA device.
 * All arithmetic of the method runs in the library's sm_100a kernels; nothing here falls back
 * to the CPU.
 */
#ifndef VBDDC_H
#define VBDDC_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vb_ctx vb_ctx; /* opaque; one per rank / GPU */

typedef enum {
  VB_OK = 0,
  VB_EINVAL = 1,      /* bad argument (message says which)                                  */
  VB_ESTATE = 2,      /* call out of order (setup -> factor -> solve)                       */
  VB_ENOMEM = 3,      /* device allocation failed                                           */
  VB_ECUDA = 4,       /* CUDA runtime error                                                 */
  VB_ENCCL = 5,       /* NCCL error                                                         */
  VB_ESINGULAR = 6,   /* zero/wrong-sign pivot in a local, deluxe or coarse factorisation   */
  VB_EBREAKDOWN = 7,  /* p^T S p <= 0 or r^T z <= 0: iterate left the benign space */
  VB_ENOTCONV = 8     /* maxit reached ("NC"); x holds the last iterate            */
} vb_status;

/* General polyhedral mesh.  Host arrays, copied by vb_setup (borrowed only for the
 * duration of the call).  Face loops must be planar; cell_face_sign[j] = +1 iff the right-hand
 * normal of the loop of cell_face[j] points out of the cell.  face_on_dirichlet = 1 marks
 * boundary faces (homogeneous Dirichlet after lifting, Eq.(ContinuousProblem)); = 2 marks
 * a Neumann face (homogeneous traction, the paper's two Neumann faces of P:1197, DESIGN A35): its
 * velocity DOFs stay free, belong to the subdomain interface, and the pressure has no gauge (no
 * zero-mean projection, no flux-compatibility check of the rhs).  Other values: VB_EINVAL. */
typedef struct {
  int32_t k;                       /* VEM degree: 2 or 3                         */
  int64_t n_vertices; const double *xyz;              /* [n_vertices][3]                      */
  int64_t n_faces; const int64_t *face_ptr; const int64_t *face_vtx;   /* CSR vertex loops    */
  int64_t n_cells; const int64_t *cell_ptr; const int64_t *cell_face;  /* CSR face lists      */
  const int8_t *cell_face_sign;
  const uint8_t *face_on_dirichlet;
} vb_mesh;

/* Primal constraints per interface entity and scaling. */
enum { VB_DELUXE = 0, VB_MULTIPLICITY = 1 };
typedef struct {
  int32_t vertex, edge_avg, face_avg, face_flux;   /* booleans                              */
  double adaptive_tau;   /* 0 = off; else add face GEVP eigenvectors with lambda < 1/tau */
  int32_t scaling;       /* VB_DELUXE | VB_MULTIPLICITY                                       */
  double svd_rel_tol;    /* constraint filter; <= 0 means 1e-10                       */
} vb_constraints;

/* Distribution: one rank per GPU; each rank owns the subdomains with
 * subdomain_rank == rank and exchanges interface sums, coarse pieces and dot partials with the
 * others over NCCL (NVLink).  nranks = 1 needs no NCCL id.  `stream` is a cudaStream_t owned by
 * the caller (torch); the library works on it.  loopback_world (test infrastructure): when set,
 * the ranks are threads of one process sharing one GPU (vb_loopback_world_create) and exchange by
 * host-synchronised device copies instead of NCCL. */
typedef struct {
  int32_t rank, nranks, device;
  const void *nccl_unique_id;      /* 128 bytes from vb_nccl_unique_id on rank 0, or NULL     */
  void *stream;
  void *loopback_world;            /* NULL = NCCL                                              */
} vb_dist;

/* Analytic problem data evaluated by the library's kernels (BASELINE.json configs).
 *  kind 0 = manufactured: u = curl(sin(pi x)sin(pi y)sin(pi z)(1,1,1)), p = sin(2 pi x)cos(pi y)z,
 *           f = (3 pi^2 nu_K / 2) u - grad p, boundary data lifted;
 *  kind 1 = multi-sinker force f = (0,0,beta(chi-1)) with sinker centres c_i, homogeneous BC. */
typedef struct {
  int32_t kind;
  int32_t n_sinkers; const double *centres;        /* [n_sinkers][3]                         */
  double delta, omega, beta;
} vb_problem;

typedef struct {
  int32_t iterations, converged;
  double r0_norm, r_final_norm, rel_residual;   /* interface residual ||r||_2        */
  double lambda_min, lambda_max, kappa;         /* Lanczos from the CG coefficients  */
  double true_rel_residual;                     /* ||b - K x||_2 / ||b||_2 of the full saddle
                                                   system through the element-by-element K7
                                                    when vb_set_option(ctx,
                                                   "true_residual", 1); else -1 (one extra pass) */
  double t_setup_s, t_factor_s, t_solve_s;
  double bytes_per_iter_model;
  double flux_violation_max;                    /* max_i |b_0^(i) x_Gamma^(i)| of the final
                                                   interface iterate (benign space, Assumption
                                                   ass1 P:526-528); meaningful on
                                                   VB_EBREAKDOWN                               */
  int32_t n_primal, n_coarse;
  int64_t n_dofs_paper;                         /* nDofs as counted in T2-T4                   */
  int32_t n_adaptive;                           /* primal rows added by the face GEVPs */
  double adaptive_margin;                       /* min |lambda - 1/tau| over all face pencils  */
} vb_report;

/* rank 0: fills 128 bytes to broadcast with torch.distributed before vb_setup. */
vb_status vb_nccl_unique_id(void *out128);
/* Test transport: a world of nranks in-process ranks (threads) on one GPU; destroy after every
 * context using it is destroyed. */
vb_status vb_loopback_world_create(int32_t nranks, void **world);
vb_status vb_loopback_world_destroy(void *world);

/* Host-only planning, no GPU needed (tests of the multi-rank bookkeeping): for one double per
 * interface DOF per sending sharer, the doubles this rank would send to (send_counts[p]) and
 * receive from (recv_counts[p]) every rank p under exchange `mode` (0: every sharer sends,
 * 1: only the entity's lowest sharer, 2: the lowest sharer on each rank), and the number of free
 * DOFs this rank owns in the vb_dof_layout sense.  Arrays have nranks entries. */
vb_status vb_plan_exchange(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                           const int32_t *subdomain_rank, int32_t rank, int32_t nranks, int32_t mode,
                           int64_t *send_counts, int64_t *recv_counts, int64_t *n_owned_free);

/* Host-only planning, no GPU needed: the sizes of the single-level coarse
 * dissection this rank would build if every interface entity of kind q (0 vertex, 1 edge, 2 face)
 * carried min(n_e, primal_per_kind[q]) primal DOFs (the factor computes the true counts by the
 * pivoted QR of the constraint rows; for the BASELINE constraints on hexahedral meshes they are
 * 3 / 3 / 3).  out6 = {interior DOFs n_I of this rank, its root list n_S (touched separator DOFs +
 * its p_0's), separator DOFs n_sep, root order n_root = n_sep + n_subdomains, local packed order
 * ceil32(n_I) + n_S, N_Pi}. */
vb_status vb_plan_coarse_dissection(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                                    const int32_t *subdomain_rank, int32_t rank, int32_t nranks,
                                    const int32_t *primal_per_kind, int64_t *out6);

/* Build the context: topology, DOF numbering, box-free general subdomain
 * classification, interface entities, and the VEM element matrices A^K, B^K computed
 * on the device from the geometry and the per-cell viscosity.
 *   cell_subdomain[n_cells]  subdomain id per cell (0..n_subdomains-1)
 *   subdomain_rank[n_subdomains] owning rank (NULL = all rank 0); every rank must own at
 *                            least one subdomain (VB_EINVAL naming the rank otherwise)
 *   cell_viscosity[n_cells]  nu_K > 0                                               */
vb_status vb_setup(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                   const int32_t *subdomain_rank, const vb_constraints *cons,
                   const double *cell_viscosity, const vb_dist *dist, vb_ctx **out);

/* Bring-up/testing variant: identical, but the element matrices are supplied (host, row-major,
 * per cell in the library's local DOF order -- see vb_cell_local_dofs) instead of generated. */
vb_status vb_setup_from_elements(const vb_mesh *mesh, const int32_t *cell_subdomain,
                                 int32_t n_subdomains, const int32_t *subdomain_rank,
                                 const vb_constraints *cons, const double *cell_viscosity,
                                 const vb_dist *dist, const int64_t *elem_ptr_A,
                                 const double *elem_A, const int64_t *elem_ptr_B,
                                 const double *elem_B, vb_ctx **out);

/* Factorisations feeding the hot path: subdomain Dirichlet LDL^T and
 * interface Schur S_G (Eq.(firstSchur)), change of basis, dual Schur inverse, coarse
 * basis, deluxe operators, adaptive enrichment, coarse saddle inverse. */
vb_status vb_factor(vb_ctx *ctx);

/* Right-hand side of Eq.(DiscProblem) on the free DOFs (velocity free DOFs in global order, then
 * pressure): load (f_h, v) = int Pi^0_k f . v (Eq.(discreteF)) minus the lifted
 * boundary data.  rhs_dev: device buffer of vb_num_free_dofs doubles (caller-owned).          */
vb_status vb_build_rhs(vb_ctx *ctx, const vb_problem *prob, double *rhs_dev);

/* PCG on the interface saddle problem Eq.(globInt) preconditioned by
 * M^-1 = R~_D^T S~^-1 R~_D (Eq.(BDDCprec)), x0 = 0, stop at ||r|| <= rtol ||r0||.
 * rhs_dev, x_dev: caller-owned device buffers in the rank's free-DOF layout (vb_dof_layout: the
 * velocity DOFs whose lowest sharing subdomain is on this rank, then the pressure DOFs of its
 * cells; for one rank, all free DOFs in global order); x gets the full solution (interior
 * back-substitution, pressure with zero global mean).  maxit <= 0 means 2000.
 * The pressure rows of rhs must be flux-compatible, sum_i g0_i = 0 (integral of the pressure rhs
 * against constants): |sum_i g0_i| > 1e-8 (sum_j |c_j g_pj| + ||r0||_2) returns VB_EINVAL
 * (c = DOFs of the constant pressure, g_p = the pressure rows, r0 = the condensed rhs); within that
 * bound the rounding is removed (reading A30).  VB_EBREAKDOWN (p^T S p <= 0 or
 * r^T z <= 0) and VB_ENOTCONV (maxit) leave the last iterate in x and fill the report.
 * Collective: every rank calls it with the same rtol/maxit. */
vb_status vb_pcg_solve(vb_ctx *ctx, const double *rhs_dev, double *x_dev, double rtol,
                       int32_t maxit, vb_report *rep);

/* Context options (host, any time after vb_setup):
 *   "true_residual" (0/1, default 0): vb_pcg_solve also fills vb_report.true_rel_residual
 *                   (one element-by-element K7 pass and two norms after the solve).
 *   "p2p" (0/1, default 0; also VB_P2P=1; multi-rank only): the two interface exchanges of every
 *                   PCG step (copies of p for S^ p, scaled extension products of z = M^-1 r;
 *                   SURVEY §8(e) C1) become direct stores from the producing kernels into the
 *                   peers' receive areas (NVLink peer memory mapped by CUDA IPC under NCCL, plain
 *                   pointers under the loopback transport), followed by a stream barrier -- no
 *                   pack kernel and no send/recv.  Read by vb_factor (collective: every rank the
 *                   same value); VB_ESTATE after vb_factor, VB_EINVAL (from vb_factor) together
 *                   with the VB_POOL allocator.  Results are bit-identical to the default path.
 *   "coarse_dissection" (1 on, 0 off, -1 auto = the default: on for nranks > 1; SURVEY f1,
 *                   DESIGN.md §9): the coarse saddle problem by block elimination over
 *                   parts -- the ranks, or on one rank blocks of its subdomains -- each part's
 *                   primal DOFs of entities all of whose sharers lie in it are eliminated by that
 *                   part alone (explicit local inverse and coupling kept packed), and only the
 *                   separator primal DOFs between parts plus every p_0 form the root problem that
 *                   all ranks assemble (the parts' Schur contributions, allgathered, part order),
 *                   factor and invert (sliced over ranks).  Off: the whole N_c x N_c coarse matrix
 *                   is assembled, factored and inverted on every rank.  Same solution up to
 *                   rounding.  Read by vb_factor (collective: every rank the same value); VB_ESTATE
 *                   after it.
 *   "coarse_blocks" (>= 1, or -1 auto = the default: the largest power of two <= 8 with at least
 *                   16 of the rank's subdomains per block, e.g. 8 for 512): blocks of this
 *                   rank's subdomains by recursive coordinate bisection of their centroids.  One
 *                   rank: the blocks are the parts.  Several ranks, > 1: two levels -- the rank
 *                   first eliminates its blocks' interiors, then the separator between its blocks
 *                   from the sum of their Schur contributions; the root is unchanged.  Read by
 *                   vb_factor.
 * VB_EINVAL on an unknown name. */
vb_status vb_set_option(vb_ctx *ctx, const char *name, double value);

/* Self-test of the NCCL transport on ONE GPU (1-rank communicator): a grouped send/recv to self
 * and an all-gather, eagerly and captured inside a CUDA-graph conditional WHILE body (the way
 * the PCG iteration graph captures them).  result[4] = {eager ok, graph ok, graph iterations,
 * max abs error}; VB_ENCCL if NCCL is not loaded; capture failures are reported in result[1] = 0
 * with the message in vb_last_error(NULL), not as an error status. */
vb_status vb_debug_nccl_selftest(int32_t device, double *result);

/* Same, with HOST rhs/x buffers: the host<->device copies are part of the call (e2e timing). */
vb_status vb_pcg_solve_host(vb_ctx *ctx, const double *rhs_host, double *x_host, double rtol,
                            int32_t maxit, vb_report *rep);

/* y = K x with the element-by-element saddle operator on the free DOFs (device). */
vb_status vb_apply_operator(vb_ctx *ctx, const double *x_dev, double *y_dev);

/* Parity/debug: y = S^ x (which = 0, Eq.(globInt)) or y = M^-1 x (which = 1, Eq.(BDDCprec)) on a
 * HOST vector in original interface coordinates: the vb_interface_dofs order (entity-major),
 * then one p_0 per subdomain.  Requires vb_factor.                                            */
vb_status vb_debug_interface_op(vb_ctx *ctx, int32_t which, const double *in_host, double *out_host);

/* Parity/debug (setup-stage gates): a dense operator of the rank-local subdomain
 * `sub` (0-based, local order) in ORIGINAL local interface coordinates -- its interface entities in
 * the library's order, each entity's free velocity DOFs increasing; ids (may be NULL) receives those
 * free velocity ids:
 *   which 0: S_Gamma^(i) (Eq.(firstSchur)), assembled back as T S_T T^T;
 *   which 1: the deluxe-scaled local dual operator N_G (D S_DD^-1 D^T) N_G^T.
 * out: host, nG x nG column-major, or NULL to query *n.  Requires vb_factor.                  */
vb_status vb_debug_subdomain_op(vb_ctx *ctx, int32_t sub, int32_t which, int64_t *ids, double *out,
                                int64_t *n);

/* Parity/debug and microbenchmark: the factorisation's grouped DMMA GEMM on DEVICE buffers,
 *   C_b = alpha * op(A_b) * diag(d) * op(B_b) + beta * C_b,   b = 0 .. batch-1,
 * column-major, op(X) = X or X^T (trans* = 0/1), X_b = X + b * strideX (elements); d (length K,
 * unit stride) may be NULL.  kz_on = 1 declares triangular operands, op(A)(i, k) = 0 for
 * k < i + kzA and op(B)(k, j) = 0 for k < j + kzB, whose zero K slabs are skipped (the caller
 * guarantees the zeros).  Runs on `stream` (a cudaStream_t, NULL = legacy default) and
 * synchronises it before returning.  VB_EINVAL on non-positive sizes or leading dimensions.      */
vb_status vb_debug_gemm(int32_t M, int32_t N, int32_t K, double alpha, const double *A, int32_t lda,
                        int32_t transA, const double *B, int32_t ldb, int32_t transB, const double *d,
                        double beta, double *C, int32_t ldc, int32_t batch, int64_t strideA,
                        int64_t strideB, int64_t strideC, void *stream, int32_t kz_on, int32_t kzA,
                        int32_t kzB);
/* Interface DOFs (free velocity ids) in the library's entity-major order; *n = count.
 * ids may be NULL to query the count only.                                                     */
vb_status vb_interface_dofs(const vb_ctx *ctx, int64_t *ids, int64_t *n);

/* Queries. */
vb_status vb_num_free_dofs(const vb_ctx *ctx, int64_t *n_vel, int64_t *n_p);
vb_status vb_dof_layout(const vb_ctx *ctx, int64_t *global_ids);   /* free -> global DOF id    */
vb_status vb_cell_local_dofs(const vb_ctx *ctx, int64_t cell, int64_t *vel_ids, int32_t *n_vel,
                             int64_t *p_ids, int32_t *n_p);       /* local order -> global id  */
vb_status vb_get_element_matrices(const vb_ctx *ctx, int64_t cell, double *A, double *B);
/* 28 counters (host-owned out28): sizes of the decomposition and operators, bytes per iteration,
 * factor GEMM flops, factor allocation time (us) and, after a vb_factor run with
 * VB_KERNEL_TIMING=1 in the environment, the GEMM kernel time of that factorisation (us; else 0).
 * Order: the keys of paper_2304_09770_b200.Context.stats. */
vb_status vb_stats(const vb_ctx *ctx, int64_t *out28);
/* Average per-launch device time (ms) of each timed launch category of the last vb_pcg_solve,
 * recorded with CUDA events on the library stream when VB_KERNEL_TIMING=1 in the environment. */
vb_status vb_kernel_times(const vb_ctx *ctx, double *ms_out, int32_t n_max, int32_t *n_out);
const char *vb_kernel_time_name(int32_t i);
const char *vb_last_error(const vb_ctx *ctx);
vb_status vb_destroy(vb_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* VBDDC_H */
