#pragma once
#include <algorithm>
#include <exception>
#include <thread>
#include "internal.h"

namespace vb {
// Local cell topology packing (one int block of TOPO_STRIDE per cell).
// General polyhedra: hexahedra, triangulated jittered hexahedra and centroidal Voronoi
// cells (up to ~17 faces, 30 vertices, 45 edges and 8-gon faces on the CVT family).
constexpr int MAXV = 40;     // vertices per cell
constexpr int MAXE = 64;     // edges per cell
constexpr int MAXF = 24;     // faces per cell
constexpr int MAXL = 10;     // vertices per face loop
constexpr int MAXT = 96;     // fan triangles per cell (sum over faces of loop length - 2)
constexpr int FACE_STRIDE = 2 + 3 * MAXL;    // sign, len, loop vertices, loop edges, forward flags
constexpr int TOPO_V = 3;
constexpr int TOPO_E = TOPO_V + MAXV;
constexpr int TOPO_F = TOPO_E + 2 * MAXE;
constexpr int TOPO_STRIDE = TOPO_F + MAXF * FACE_STRIDE;

// VB_DEBUG=1: synchronise and check after every stage, naming it in the error.
inline void dbg(vb_ctx *c, const char *what) {
  if (!c->debug) return;
  cudaError_t e = cudaStreamSynchronize(c->stream);
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e != cudaSuccess) throw Error{VB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e)};
}

#define VB_STR_(x) #x
#define VB_XSTR(x) VB_STR_(x)
#define VB_STAGE()                                                                              \
  do {                                                                                          \
    VB_CHECK_LAUNCH();                                                                          \
    dbg(c, __FILE__ ":" VB_XSTR(__LINE__));                                                     \
  } while (0)

// host thread pool for the per-cell / per-subdomain setup passes: f(begin, end) on contiguous
// chunks of [0, n); an exception thrown in any chunk is rethrown on the caller's thread
template <class F>
void parallel_for(int64_t n, F f, int64_t min_chunk = 2048) {
  static const int env_threads = getenv("VB_HOST_THREADS") ? atoi(getenv("VB_HOST_THREADS")) : 0;
  int T = (int)std::min<int64_t>(env_threads > 0 ? env_threads : std::max(1u, std::thread::hardware_concurrency()), 32);
  T = (int)std::min<int64_t>(T, (n + min_chunk - 1) / min_chunk);
  if (T <= 1) { if (n > 0) f((int64_t)0, n); return; }
  std::vector<std::thread> th;
  std::vector<std::exception_ptr> err(T);
  for (int t = 0; t < T; ++t)
    th.emplace_back([&, t] {
      try { f(n * t / T, n * (t + 1) / T); } catch (...) { err[t] = std::current_exception(); }
    });
  for (auto &x : th) x.join();
  for (auto &e : err) if (e) std::rethrow_exception(e);
}

void gauss_legendre01(int n, double *x, double *w);
void gauss_lobatto01(int npts, double *x, double *w);
void build_topology(vb_ctx *c, const vb_mesh *m);
void build_subdomains(vb_ctx *c, const int32_t *cell_sub, int Ng, const int32_t *sub_rank);
void face_frame(const vb_ctx *c, int64_t f, double *area, double n[3], double t1[3], double t2[3]);
void build_constraint_rows(vb_ctx *c, std::vector<double> &rows_out);

// SURVEY f1 (factor.cu): the host plan of the coarse dissection from the global entity list
// (gents[].r, off_pi, sharers), gsub_ents, NPi_g, Ng and a part per global subdomain (ranks, or
// blocks of one rank's subdomains)
struct CoarsePlan {
  int nparts = 1;
  std::vector<int> part;                     // global subdomain -> part
  std::vector<int> owned;                    // parts this rank eliminates (R > 1: its rank; R = 1: all)
  std::vector<int64_t> root;                 // global coarse indices (separator, then every p_0)
  std::vector<std::vector<int64_t>> I, S;    // per part: interior DOFs; touched separator DOFs, then its p_0's
  std::vector<int64_t> rptr, ridx;           // root entry <- t entries p * maxS + q, part order
  int64_t nsep = 0, maxS = 1;
};
CoarsePlan plan_coarse_dissection(const vb_ctx *c, const std::vector<int> &part, int nparts);

// device-side stages (defined in the .cu files)
void cell_geometry_device(vb_ctx *c);                    // vem.cu
void layout_phase_a(vb_ctx *c, cudaStream_t s_upload = nullptr);   // abi.cu (uploads on s_upload if given)
void build_transformed_maps(vb_ctx *c);                  // abi.cu (after the entity ranks)
void prepare_solve(vb_ctx *c);                           // solve.cu
void destroy_solve_state(vb_ctx *c);                     // solve.cu
void element_matrices_device(vb_ctx *c, bool wait = true);   // vem.cu (K9; wait = false: c->w_k9 keeps the scratch)
void build_rhs_device(vb_ctx *c, const vb_problem *p, double *rhs);   // vem.cu
void factor_device(vb_ctx *c);                           // factor.cu
void adaptive_enrich(vb_ctx *c, double tau, const DBuf<double> &sidebuf);   // adaptive.cu (A6)
void pcg_device(vb_ctx *c, const double *rhs, double *x, double rtol, int maxit, vb_report *rep);
void apply_operator_device(vb_ctx *c, const double *x, double *y);    // solve.cu (K7)
void debug_interface_op(vb_ctx *c, int which, const double *in, double *out);   // solve.cu
void debug_subdomain_op(vb_ctx *c, int sub, int which, int64_t *ids, double *out, int64_t *n);   // solve.cu
void element_gather(vb_ctx *c, const double *yel, double *out);      // solve.cu: per-DOF sums
const char *kernel_time_name(int i);                                  // solve.cu
}  // namespace vb
