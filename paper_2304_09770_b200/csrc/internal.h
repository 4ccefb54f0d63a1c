// Internal state of a vb_ctx (not part of the ABI).
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/vbddc.h"
#include "comm.h"

#ifdef __CUDACC__
#define HD_INLINE __host__ __device__ __forceinline__
#else
#define HD_INLINE inline
#endif

namespace vb {

struct Error {
  vb_status st;
  std::string msg;
};

#define VB_CUDA(x)                                                                              \
  do {                                                                                          \
    cudaError_t _e = (x);                                                                       \
    if (_e != cudaSuccess)                                                                      \
      throw ::vb::Error{VB_ECUDA, std::string(#x) + ": " + cudaGetErrorString(_e) + " at " +    \
                                      __FILE__ + ":" + std::to_string(__LINE__)};               \
  } while (0)
#define VB_CHECK_LAUNCH() VB_CUDA(cudaGetLastError())
#define VB_REQUIRE(cond, code, m)                                                               \
  do {                                                                                          \
    if (!(cond)) throw ::vb::Error{code, std::string(m)};                                       \
  } while (0)

// ------------------------------------------------------------------ device buffer
// cumulative wall time (s) spent in allocation / release by DBuf (diagnostics, VB_FACTOR_TIMES)
extern thread_local double g_malloc_s, g_free_s;
double wall_now();

// Device memory: cudaMalloc / cudaFree by default; with VB_POOL=1 the device's stream-ordered pool
// (cudaMallocAsync / cudaFreeAsync on the stream of the context being served, release threshold
// raised so freed blocks are reused).  Measured on config 5 the pool removed the synchronous cudaFree
// cost but raised the factor's first-touch mapping (its footprint grows), 1.25 s against 0.8 s
// typical.  Every ABI entry point sets g_alloc_stream (AllocStreamScope).
extern thread_local cudaStream_t g_alloc_stream;
extern bool g_use_pool;   // VB_POOL=1: stream-ordered pool; default plain cudaMalloc / cudaFree
extern bool g_poison;     // VB_POISON=1: fill every new device allocation with NaN bits (tests)
void pool_init();
void pool_trim(cudaStream_t s);
struct vb_ctx_fwd;   // sync s, then return unused pool memory to the device
struct AllocStreamScope {
  cudaStream_t prev;
  explicit AllocStreamScope(cudaStream_t s) : prev(g_alloc_stream) { g_alloc_stream = s; }
  ~AllocStreamScope() { g_alloc_stream = prev; }
};

template <class T>
struct DBuf {
  T *p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf &) = delete;
  DBuf &operator=(const DBuf &) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) {
      const double t0 = wall_now();
      if (g_use_pool) cudaFreeAsync(p, g_alloc_stream); else cudaFree(p);
      g_free_s += wall_now() - t0;
    }
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count) {
    release();
    if (count == 0) return;
    pool_init();
    const double t0 = wall_now();
    cudaError_t e = g_use_pool ? cudaMallocAsync((void **)&p, count * sizeof(T), g_alloc_stream)
                               : cudaMalloc((void **)&p, count * sizeof(T));
    g_malloc_s += wall_now() - t0;
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      p = nullptr;
      throw Error{VB_ENOMEM, "cudaMallocAsync of " + std::to_string(count * sizeof(T)) + " bytes failed"};
    }
    n = count;
    if (g_poison) cudaMemsetAsync(p, 0xFF, count * sizeof(T), g_alloc_stream);   // all-ones = NaN
  }
  void zero(cudaStream_t s) {
    if (n) VB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  void upload(const std::vector<T> &h, cudaStream_t s) {
    alloc(h.size());
    if (n) VB_CUDA(cudaMemcpyAsync(p, h.data(), n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void download(std::vector<T> &h, cudaStream_t s) const {
    h.resize(n);
    if (n) VB_CUDA(cudaMemcpyAsync(h.data(), p, n * sizeof(T), cudaMemcpyDeviceToHost, s));
  }
};

// ------------------------------------------------------------------ grouped GEMM descriptor
// C(MxN) = beta*C + alpha * op(A) * diag(d) * op(B), column-major, op = transpose if flag.
struct GemmProb {
  const double *A;
  const double *B;
  double *C;
  const double *d;   // optional diagonal scaling (length K), stride dstride
  int lda, ldb, ldc, dstride;
  int M, N, K;
  double alpha, beta;
  int transA, transB;
  int lower;         // only compute tiles intersecting the lower triangle (i >= j)
  // triangular operands: op(A)(i, k) = 0 for k < i + kzA and op(B)(k, j) = 0 for k < j + kzB, so
  // tile (m0, n0) starts its K loop at max(m0 + kzA, n0 + kzB) (kz_on = 1 enables it)
  int kz_on, kzA, kzB;
};

// ------------------------------------------------------------------ packed symmetric tiles
// Lower triangle of a symmetric n x n matrix as 32x32 tiles (I >= J) in row-of-tiles order, each
// tile row-major (diagonal tiles hold the full symmetric block); the tiles of the last tile row
// store only its rv = n - 32 (nt - 1) valid rows, so no padding rows are streamed.
HD_INLINE int64_t ptile_row_start(int64_t I) { return 1024 * (I * (I + 1) / 2); }
HD_INLINE int ld4(int n) { return (n + 3) & ~3; }   // leading dimensions with 32-byte aligned columns
HD_INLINE int64_t ptile_off(int n, int I, int J) {   // offset of tile (I, J), J <= I
  const int nt = (n + 31) / 32;
  const int64_t rows = (I == nt - 1) ? n - 32 * (nt - 1) : 32;
  return ptile_row_start(I) + (int64_t)J * rows * 32;
}
HD_INLINE int64_t packed_size(int n) {               // doubles
  if (n <= 0) return 0;
  const int nt = (n + 31) / 32;
  const int64_t rv = n - 32 * (nt - 1);
  return ptile_row_start(nt - 1) + (int64_t)nt * rv * 32;
}

struct GEnt {                  // global interface entity (every rank holds the whole list)
  std::vector<int> sharers;     // global subdomain ids (sorted)
  int n = 0, kind = 0, r = -1;  // DOFs, kind, primal rank (after the constraint filter)
  int64_t off_pi = 0;           // offset of its primal coordinates in the global u_Pi
};

struct Entity {                 // interface entity touched by a local subdomain
  int gid = -1;                 // global entity id
  int kind = 0;                 // 0 vertex, 1 edge, 2 face
  std::vector<int> sharers;     // GLOBAL subdomain ids (sorted), local or not
  std::vector<int64_t> dofs;    // free velocity ids (sorted)
  int n = 0, r = 0, nd = 0;
  int64_t off_d = 0;            // offset of its dual coords in the (rank-local) PCG vector
  int64_t off_p = 0;            // offset of its primal coords within the GLOBAL u_Pi
  int64_t off_pl = 0;           // offset of its primal coords within the rank-local primal block
  int64_t off_T = 0;            // offset of T_G (n x n, column-major) in the T buffer
  int64_t off_C = 0;            // offset of constraint rows C_G (rows x n, row-major)
  int nrows_C = 0;
  int64_t off_D = 0;            // offset of deluxe blocks (one nd x nd per sharer, row-major)
};

struct Sub {
  std::vector<int> cells;
  std::vector<int64_t> I;       // interior free velocity ids
  std::vector<int64_t> P;       // pressure global ids
  std::vector<int> ents;        // entity ids (sorted by entity id)
  std::vector<int> ent_offG, ent_offD, ent_offP;
  int nI = 0, nP = 0, nG = 0, nD = 0, n = 0, nd = 0, npi = 0;
  int64_t off_K = 0;            // dense (n x n) subdomain matrix, column-major, ld = n
  int64_t off_ST = 0;           // dense transformed Schur S_T (nG x nG), column-major
  int64_t off_STp = 0;          // packed tiles of S_T
  int64_t off_SDi = 0;          // packed tiles of S_DD^-1
  int64_t off_Phi = 0;          // Phi (nd x npi), row-major
  int64_t off_Sc = 0;           // S_c (npi x npi) column-major
  int64_t off_vecG = 0;         // offset into per-subdomain vectors of length nG
  int64_t off_vecD = 0;         // offset into per-subdomain vectors of length nd
  int64_t off_vecPi = 0;        // offset into per-subdomain vectors of length npi
  int64_t off_vecDfull = 0;     // offset into per-subdomain vectors of length nD
  int color = 0;
  double vol = 0, gamma = 0;
};

// Device-side descriptors (plain data, uploaded once).
struct SubDev {
  int nI, nP, nG, nD, n, nd, npi;
  int cell_begin, cell_end;   // into sub_cells
  int slot_begin, slot_end;   // into the subdomain-major slot index list
  int ldk;                    // leading dimension of the dense subdomain matrix: n rounded up to 4
  int64_t off_K;              // dense n x n (column-major, ld = ldk; 32-byte aligned columns)
  int64_t off_ST;             // dense nG x nG: S_T, then its partial LDL^T
  int64_t off_STp;            // packed tiles of S_T
  int64_t off_SDi;            // packed tiles of S_DD^-1
  int64_t off_Phi;            // Phi, nd x npi column-major
  int64_t off_G;              // offset into length-nG per-subdomain vectors
  int64_t off_Dv;             // offset into length-nd vectors
  int64_t off_Pi;             // offset into length-npi vectors
  int64_t off_P;              // offset into length-nP vectors
  int64_t off_I;              // offset into length-nI vectors
  int64_t off_Dn;             // offset into length-nD vectors
  int64_t off_X;              // scratch square (nG x nG) offset
  int64_t off_KDi;            // packed tiles of K_DD^-1 (Q_I-augmented, A5)
  double vol, gamma;
};

struct SlotDev {              // one (entity, sharer) pair; slots are entity-major
  int sub, ent, n, nd, r;
  int offG;                   // local original-Gamma offset in the subdomain
  int offD;                   // local dual offset (0..nd_sub)
  int offPi;                  // local primal offset (0..npi_sub)
  int64_t off_T;              // T_G of the entity
  int64_t off_Dlx;            // deluxe block D_G^(sub) (nd x nd, column-major)
  int64_t off_side;           // scratch for S_GD^(sub)
};

struct EntDev {
  int n, nd, r, nsides, side_begin, kind, nrowsC, nsh;   // nsides: local sharers; nsh: all sharers
  int64_t off_T, off_C, off_xd, off_pi, off_gam, off_sum, off_W;
  int64_t off_pl;             // rank-local primal offset (x = [dual | local primal | p0])
};

// one part of the coarse dissection eliminated by this rank (factor.cu; the solve fields are set
// by prepare_solve)
struct CdPart {
  int part = 0;                 // part id (rank, or block of one rank's subdomains)
  int P1 = 0, P2 = 0;           // GEMV chunks of pass 1 (all tile rows) / pass 2 (the S tile rows)
  int64_t nI = 0, nIp = 0, nS = 0, nloc = 0;   // interior, interior padded to 32, root list, nIp + nS
  int64_t koff = 0;             // packed matrix offset in d_Kloc
  int64_t p1off = 0, p2off = 0; // chunk partials of pass 1 / 2 (chunk q at + q nloc)
  int64_t yoff = 0;             // y_I = E g_I in the Y buffer
  int64_t moff = 0;             // gather maps (nloc each)
  int64_t ioff = 0;             // interior global indices
};

struct KTimer {
  std::string name;
  cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace vb

struct vb_ctx {
  // ---------------- configuration
  int k = 2;
  vb_constraints cons{};
  int rank = 0, nranks = 1, device = 0;
  vb::Comm *comm = nullptr;          // null for nranks = 1
  cudaStream_t stream = nullptr;
  std::string err;
  int state = 0;  // 1 = setup, 2 = factored
  // ---------------- mesh (host copy)
  int64_t nV = 0, nF = 0, nK = 0, nE = 0;
  std::vector<double> xyz;
  std::vector<int64_t> face_ptr, face_vtx, cell_ptr, cell_face;
  std::vector<int8_t> cell_sign;
  std::vector<uint8_t> face_bnd;                   // 0 interior, 1 Dirichlet, 2 Neumann
  std::vector<char> vel_on_neu;                    // per velocity DOF: on a Neumann face's closure
  bool neumann = false;                            // any Neumann face: no pressure gauge (DESIGN A35)
  std::vector<int64_t> edges;        // [nE][2] (a<b), lexicographic
  std::vector<double> nu;
  // ---------------- DOF numbering
  int nm = 0, n4 = 0, n5 = 0, np = 0, nv_max = 0;
  int64_t oE = 0, oF = 0, oC = 0, nvel = 0, npres = 0;
  std::vector<int64_t> vel2free;     // -1 for Dirichlet DOFs
  std::vector<int64_t> free2vel;
  int64_t n_free_vel = 0;
  // per cell local topology
  std::vector<int> cell_nv;              // local velocity dof count
  std::vector<int64_t> cell_l2g_ptr;     // CSR into cell_l2g (velocity global ids)
  std::vector<int64_t> cell_l2g;
  std::vector<int> cell_topo;            // packed local topology for the element kernel
  int topo_stride = 0;
  // ---------------- subdomains / entities (global view + the local part of this rank)
  int Ng = 0;                        // global subdomain count
  std::vector<int> sub_rank, sub_gid, sub_lid;     // rank of each global sub; local<->global ids
  std::vector<int64_t> cell_gid, cell_lid;         // local<->global cell ids
  int64_t nKl = 0;                   // local cells
  std::vector<int> gsub_ncell;
  std::vector<int> dof_owner_sub, dof_nsh;         // per free velocity DOF: lowest sharer, #sharers
  std::vector<vb::GEnt> gents;
  std::vector<std::vector<int>> gsub_ents;         // global sub -> global entities (sorted)
  std::vector<int> gent_lid;                       // global entity -> local entity (-1)
  std::vector<double> gsub_vol;                    // volumes of all subdomains
  int64_t NPi_g = 0;                 // global primal count (coarse = NPi_g + Ng)
  int N = 0;                         // local subdomains
  std::vector<int> cell_sub;
  std::vector<vb::Sub> subs;
  std::vector<vb::Entity> ents;
  int64_t nGamma = 0;                // number of interface (original) DOFs
  int64_t n_delta_glob = 0;          // dual coordinates of the local entities
  int64_t NPi = 0;                   // primal coordinates of the local entities
  int64_t nx = 0;                    // rank-local PCG vector length = n_delta_glob + NPi + N
  int ncolors = 0;
  // ---------------- device data
  vb::DBuf<double> d_xyz, d_nu;
  vb::DBuf<int> d_topo;
  vb::DBuf<double> d_elA, d_elB;     // element matrices: A [nK][nv_max^2], B [nK][np*nv_max]
  vb::DBuf<double> d_elAp;           // K7: lower triangles of A^K, packed rows [nK][nv_max (nv_max+1)/2]
  vb::DBuf<int64_t> d_cell_l2g;      // [nK][nv_max] global velocity ids (-1 pad)
  vb::DBuf<int> d_cell_loc;          // [nK][nv_max + np] position in subdomain matrix (-1 = drop)
  std::vector<int> h_cell_loc;       // host copy (B0/B8 coupling plans)
  vb::DBuf<int> d_cell_nv;
  vb::DBuf<int64_t> d_vel2free;
  double flux_violation = 0;
  vb::DBuf<double> d_P0;             // per cell Pi^0_{k,K} coefficients (3 dim P_k x nv), for the load
  void *solve_state = nullptr;
  int debug = 0;
  vb::DBuf<double> w_hostio;
  vb::DBuf<double> w_k9;             // K9 scratch while the element kernel overlaps the host layout (vb_setup)
  int max_npi = 0, geo_stride = 0;
  std::vector<double> cellgeo;       // host copy of d_cellgeo
  vb::DBuf<double> d_K;              // subdomain dense matrices
  vb::DBuf<double> d_ST, d_STp, d_SDi /* D S_DD^-1 D^T */, d_Phi /* D Phi */, d_Sc, d_KDi;
  int64_t len_KDi = 0;
  vb::DBuf<double> d_T, d_C, d_Dlx;  // per-entity T_G, constraint rows, deluxe blocks
  vb::DBuf<double> d_Kc, d_Kcp;      // coarse dense & packed inverse
  int64_t Nc = 0;
  // descriptors
  std::vector<vb::SubDev> h_sub;
  std::vector<vb::SlotDev> h_slot;
  std::vector<vb::EntDev> h_ent;
  std::vector<int> h_sub_slots;      // subdomain-major list of slot ids
  vb::DBuf<vb::SubDev> d_sub;
  vb::DBuf<vb::SlotDev> d_slot;
  vb::DBuf<vb::EntDev> d_ent;
  vb::DBuf<int> d_sub_slots, d_sub_cells;
  int64_t len_G = 0, len_Dv = 0, len_Pi = 0, len_P = 0, len_I = 0, len_Dn = 0;
  int64_t len_K = 0, len_ST = 0, len_STp = 0, len_SDi = 0, len_Phi = 0, len_X = 0;
  int64_t len_T = 0, len_Dlx = 0, len_side = 0, len_sum = 0, len_W = 0;
  // per-subdomain vectors
  vb::DBuf<double> d_b0;             // original flux row on local Gamma (len_G)
  vb::DBuf<double> d_b0T;            // transformed flux row on local Pi (len_Pi)
  vb::DBuf<double> d_cvec, d_mvec;   // D_Q of q = 1 and int psi_j (len_P)
  vb::DBuf<int64_t> d_loc2x;         // local transformed coord -> x index (len_G)
  vb::DBuf<int64_t> d_subG_free;     // local original Gamma -> free vel id (len_G)
  vb::DBuf<int64_t> d_subI_free;     // interior -> free vel id (len_I)
  vb::DBuf<int64_t> d_subP_glob;     // pressure -> pressure global id (len_P)
  vb::DBuf<int64_t> d_pi_glob;       // local primal -> global primal index (len_Pi)
  // x coordinate -> local copies (sub-local transformed positions, global offsets into len_G)
  vb::DBuf<int64_t> d_xcopy_ptr, d_xcopy;
  vb::DBuf<int64_t> d_gam_free;      // interface DOFs (free ids), entity-major order
  vb::DBuf<double> d_cellgeo;        // per cell: vol, centroid(3), h, c-vector(np)
  vb::DBuf<int> d_info;
  // solve workspaces
  vb::DBuf<double> w_x, w_r, w_z, w_p, w_q, w_part, w_locD, w_locY, w_locC, w_uc, w_rc, w_ucp,
      w_scal, w_gam, w_bD, w_zG, w_dots, w_elt, w_elx, w_yDp, w_xD;   // w_elx: K7 per-cell inputs
  int P_kd = 4;
  vb::DBuf<int> d_op_work, d_loc_work, d_c_work;   // packed-GEMV chunk work lists
  int n_op_work = 0, n_loc_work = 0, n_c_work = 0, P_op = 4, P_loc = 4, P_c = 148;
  vb::DBuf<int64_t> d_op_part_off, d_loc_part_off;
  vb::DBuf<int64_t> d_el_ptr, d_el_ent;   // K7: free dof -> (cell, local) contributions
  double bytes_per_iter = 0;
  // timing
  bool timing = false;
  int opt_p2p = 0;                   // vb_set_option("p2p"): peer stores for the C1 exchanges of the PCG step
  int opt_true_residual = 0;         // vb_set_option("true_residual"): ||b - K x|| / ||b|| via K7
  std::vector<double> ktime_ms;
  std::vector<int> ktime_count;
  int last_iterations = 0;
  std::vector<std::string> ktime_name;
  double t_setup = 0, t_factor = 0;
  // adaptive coarse space (A6): extra constraint rows per entity (rows x n, row-major)
  std::vector<std::vector<double>> extra_rows;
  int n_adaptive = 0;
  double adaptive_margin = 0;
  // multi-rank
  vb::DBuf<double> w_red;            // C3 scratch (nranks x k)
  vb::DBuf<int64_t> d_cell_gid;      // local cell -> global cell (pressure indexing)
  std::vector<int> gsub_color;       // colouring of the global subdomain adjacency (coarse assembly)
  std::vector<int64_t> owned_free;   // ABI layout: owned free DOF ids (global free numbering)
  vb::DBuf<int64_t> d_owned_free;
  vb::DBuf<double> w_rhsg, w_xg;     // global-layout free vectors (nranks > 1)
  vb::DBuf<double> d_Kcs;            // distributed coarse: this rank's tile rows of the packed inverse
  int64_t coarse_tlo = 0, coarse_thi = 0;   // ... tile rows [tlo, thi) (balanced by tile count)
  // dissection of the coarse saddle problem (factor.cu coarse_dissection).
  // Parts = ranks (R > 1) or blocks of one rank's subdomains (R = 1); interior = primal DOFs of
  // entities whose sharers all lie in one part (eliminated by that part alone); root = the other
  // primal DOFs and every p_0 (replicated, sliced over ranks).
  int opt_coarse_dis = -1;           // vb_set_option("coarse_dissection"): -1 auto = on for nranks > 1
  int opt_coarse_blocks = -1;        // vb_set_option("coarse_blocks"): parts on one rank (-1 auto)
  bool cdis = false;                 // the last vb_factor used it
  int cd_nparts = 0;
  int64_t Nroot = 0, cd_nsep = 0, cd_maxS = 0;   // root size (= cd_nsep separator DOFs + Ng p_0)
  std::vector<vb::CdPart> cd_parts;  // the parts this rank eliminates
  std::vector<std::vector<int64_t>> cd_I, cd_S;   // per owned part: interior / root list -> global coarse index
  std::vector<int64_t> cd_root_glob;
  std::vector<int64_t> cd_rptr, cd_ridx;   // root entry <- t entries p * maxS + q, part order
  // two levels (R > 1 with coarse_blocks > 1): level 0 = this rank's blocks (t stride cd_maxS0),
  // level 1 = the rank's separator between its blocks (cd2_RS) against its root list (cd2_S)
  bool cd_two = false;
  int64_t cd_maxS0 = 0;
  vb::CdPart cd2_part;
  std::vector<int64_t> cd2_RS, cd2_S;
  std::vector<int64_t> cd2_ptr, cd2_idx;   // level-1 position <- block t entries b * maxS0 + q
  vb::DBuf<double> d_Kloc2;
  vb::DBuf<double> d_Kloc;           // per owned part, packed [[A_II^-1, sym], [A_SI A_II^-1, 0]] (n_loc = nIp + nS)
  double factor_flops = 0;     // DMMA GEMM flops of the last vb_factor
  double factor_gemm_s = 0;    // their kernel time (CUDA events; VB_KERNEL_TIMING=1 only, else 0)
  double factor_alloc_s = 0;   // wall time of device allocation / release inside the last vb_factor
};
