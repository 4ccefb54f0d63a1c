// Factor stage: subdomain assembly, partial LDL^T giving the interface
// Stokes Schur complement S_G (Eq.(firstSchur)), orthogonal change of basis to explicit
// primal coordinates, dual Schur inverse, coarse basis Phi, deluxe operators,
// coarse saddle matrix on (u_Pi, p_0) and its inverse.
//
// Q_I (zero-mean interior pressure) is imposed by augmenting the pressure block with
// -gamma m m^T and projecting the pressure-velocity coupling with Pi^T = I - m c^T / vol
// (reading A5); this gives exactly the Q_I Schur complement.
#include <algorithm>
#include <array>
#include <functional>
#include <cmath>
#include <map>
#include <set>
#include <cstring>
#include <chrono>
#include "dense.cuh"
#include "setup.h"
#include "exchange.h"

namespace vb {

thread_local double g_malloc_s = 0.0, g_free_s = 0.0;
thread_local cudaStream_t g_alloc_stream = nullptr;
bool g_use_pool = getenv("VB_POOL") && atoi(getenv("VB_POOL"));   // opt-in
bool g_poison = getenv("VB_POISON") && atoi(getenv("VB_POISON"));

void pool_init() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_dev = dev;
}

void pool_trim(cudaStream_t s) {
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaStreamSynchronize(s) == cudaSuccess && cudaGetDevice(&dev) == cudaSuccess &&
      cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess)
    cudaMemPoolTrimTo(pool, 0);
}
double wall_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}


static void stage_time(vb_ctx *c, const char *name) {
  static const bool on = getenv("VB_FACTOR_TIMES") && atoi(getenv("VB_FACTOR_TIMES"));
  if (!on) return;
  static double last = 0;
  VB_CUDA(cudaStreamSynchronize(c->stream));
  const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  if (name)
    fprintf(stderr, "[vb factor rank %d] %-22s %8.3f s  (cumulative cudaMalloc %.3f s, cudaFree %.3f s)\n", c->rank,
            name, now - last, g_malloc_s, g_free_s);
  last = now;
}

#define STAGE_T(name) stage_time(c, name)


// ------------------------------------------------------------------ assembly (one CTA / subdomain)
__global__ void assemble_kernel(const SubDev *__restrict__ subs, const int *__restrict__ sub_cells,
                                const int *__restrict__ cell_loc, const int *__restrict__ cell_nv,
                                const double *__restrict__ elA, const double *__restrict__ elB,
                                int nvmax, int np, const double *__restrict__ cvec,
                                const double *__restrict__ mvec, double *Kall, double *b0all) {
  const SubDev S = subs[blockIdx.x];
  double *K = Kall + S.off_K;
  const double *c = cvec + S.off_P;
  const double *m = mvec + S.off_P;
  double *b0 = b0all + S.off_G;
  const int64_t ld = S.ldk;
  const int nI = S.nI, nP = S.nP, nG = S.nG;
  const int stride = nvmax + np;
  for (int q = S.cell_begin; q < S.cell_end; ++q) {
    const int cell = sub_cells[q];
    const int nv = cell_nv[cell];
    const int *loc = cell_loc + (int64_t)cell * stride;
    const double *A = elA + (int64_t)cell * nvmax * nvmax;
    const double *B = elB + (int64_t)cell * np * nvmax;
    for (int idx = threadIdx.x; idx < nv * nv; idx += blockDim.x) {
      int a = idx / nv, b = idx % nv;
      int pa = loc[a], pb = loc[b];
      if (pa >= 0 && pb >= 0) K[pa + pb * ld] += A[(int64_t)a * nv + b];
    }
    for (int idx = threadIdx.x; idx < np * nv; idx += blockDim.x) {
      int p = idx / nv, b = idx % nv;
      int pp = loc[nvmax + p], pb = loc[b];
      if (pb >= 0) {
        double v = B[(int64_t)p * nv + b];
        K[pp + pb * ld] += v;
        K[pb + pp * ld] += v;
      }
    }
    __syncthreads();
  }
  // augmentation of the pressure block: -gamma m m^T
  for (int idx = threadIdx.x; idx < nP * nP; idx += blockDim.x) {
    int a = idx / nP, b = idx % nP;
    if (m[a] != 0.0 && m[b] != 0.0) K[(nI + a) + (int64_t)(nI + b) * ld] -= S.gamma * m[a] * m[b];
  }
  __syncthreads();
  // projection Pi^T of the pressure rows on every velocity column: K[P,v] -= m (c^T K[P,v]) / vol
  for (int v = threadIdx.x; v < nI + nG; v += blockDim.x) {
    const int col = v < nI ? v : v + nP;
    double s = 0.0;
    for (int a = 0; a < nP; ++a) s += c[a] * K[(nI + a) + (int64_t)col * ld];
    if (v >= nI) b0[v - nI] = s;      // flux row B_0G^(i) on the local interface
    for (int a = 0; a < nP; ++a) {
      if (m[a] != 0.0) K[(nI + a) + (int64_t)col * ld] -= m[a] * s / S.vol;
      K[col + (int64_t)(nI + a) * ld] = K[(nI + a) + (int64_t)col * ld];
    }
  }
}

// ------------------------------------------------------------------ change of basis per entity
// Householder QR with column pivoting of C_G^T; T_G = [N_G | Q_1] (dual coordinates first),
// rank by |R_jj| > tol |R_00|.  One CTA per entity; T (n x n col-major) in global memory.
__device__ double block_sum(double v, double *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
  return s;
}

__global__ void entity_basis_kernel(const EntDev *__restrict__ ents, const double *__restrict__ Crows,
                                    double *Tall, double *work, int *rank_out, double tol) {
  const EntDev E = ents[blockIdx.x];
  const int n = E.n, nr = E.nrowsC;
  double *T = Tall + E.off_T;
  const double *C = Crows + E.off_C;     // nr x n row-major
  double *W = work + E.off_C;            // n x nr column-major (same size as C)
  __shared__ double red[32];
  for (int idx = threadIdx.x; idx < n * nr; idx += blockDim.x) {
    int row = idx % n, col = idx / n;
    W[row + (int64_t)col * n] = C[(int64_t)col * n + row];
  }
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) T[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  __syncthreads();
  double r00 = 0.0;
  int r = 0;
  for (int j = 0; j < nr && j < n; ++j) {
    int pc = j;
    double best = -1.0;
    for (int col = j; col < nr; ++col) {
      double s = 0.0;
      for (int row = j + threadIdx.x; row < n; row += blockDim.x) s += W[row + (int64_t)col * n] * W[row + (int64_t)col * n];
      s = block_sum(s, red);
      if (s > best) { best = s; pc = col; }
    }
    if (pc != j) {
      for (int row = threadIdx.x; row < n; row += blockDim.x) {
        double t = W[row + (int64_t)j * n];
        W[row + (int64_t)j * n] = W[row + (int64_t)pc * n];
        W[row + (int64_t)pc * n] = t;
      }
    }
    __syncthreads();
    double nrm = sqrt(best);
    if (j == 0) r00 = nrm;
    if (!(nrm > tol * r00)) break;
    r = j + 1;
    double x0 = W[j + (int64_t)j * n];
    double alpha = x0 >= 0 ? -nrm : nrm;
    __syncthreads();
    if (threadIdx.x == 0) W[j + (int64_t)j * n] = x0 - alpha;
    __syncthreads();
    double vv = 0.0;
    for (int row = j + threadIdx.x; row < n; row += blockDim.x) vv += W[row + (int64_t)j * n] * W[row + (int64_t)j * n];
    vv = block_sum(vv, red);
    const double beta = 2.0 / vv;
    for (int col = j + 1; col < nr; ++col) {
      double s = 0.0;
      for (int row = j + threadIdx.x; row < n; row += blockDim.x) s += W[row + (int64_t)j * n] * W[row + (int64_t)col * n];
      s = block_sum(s, red) * beta;
      for (int row = j + threadIdx.x; row < n; row += blockDim.x) W[row + (int64_t)col * n] -= s * W[row + (int64_t)j * n];
      __syncthreads();
    }
    for (int row = 0; row < n; ++row) {     // Q <- Q H_j
      double s = 0.0;
      for (int q = j + threadIdx.x; q < n; q += blockDim.x) s += T[row + (int64_t)q * n] * W[q + (int64_t)j * n];
      s = block_sum(s, red) * beta;
      for (int q = j + threadIdx.x; q < n; q += blockDim.x) T[row + (int64_t)q * n] -= s * W[q + (int64_t)j * n];
      __syncthreads();
    }
  }
  __syncthreads();
  // Q = [Q1 (r) | Q2 (n-r)] -> T = [Q2 | Q1]; W (n*nr >= n*r) is free scratch now
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) W[idx] = T[idx];
  __syncthreads();
  for (int col = 0; col < n - r; ++col) {
    for (int row = threadIdx.x; row < n; row += blockDim.x) T[row + (int64_t)col * n] = T[row + (int64_t)(col + r) * n];
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < n * r; idx += blockDim.x) T[(int64_t)(n - r) * n + idx] = W[idx];
  if (threadIdx.x == 0) rank_out[blockIdx.x] = r;
}

// b~0 = b0 T on the primal coordinates; max |b0 T_Delta| / |b0| is the benign check (Eq.(ass1)).
__global__ void b0_transform_kernel(const SlotDev *__restrict__ slots, int nslot, const SubDev *__restrict__ subs,
                                    const double *__restrict__ T, const double *__restrict__ b0all,
                                    double *b0T, unsigned long long *viol) {
  int w = blockIdx.x;
  if (w >= nslot) return;
  const SlotDev s = slots[w];
  const SubDev S = subs[s.sub];
  const double *Te = T + s.off_T;
  const double *b0 = b0all + S.off_G + s.offG;
  const int n = s.n;
  double nb = 0.0;
  for (int j = threadIdx.x; j < n; j += 32) nb += b0[j] * b0[j];
  for (int o = 16; o; o >>= 1) nb += __shfl_xor_sync(0xffffffffu, nb, o);
  for (int col = 0; col < n; ++col) {
    double sum = 0.0;
    for (int j = threadIdx.x; j < n; j += 32) sum += b0[j] * Te[j + (int64_t)col * n];
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (threadIdx.x == 0) {
      if (col >= s.nd) b0T[S.off_Pi + s.offPi + (col - s.nd)] = sum;
      else if (nb > 0) atomicMax(viol, (unsigned long long)__double_as_longlong(fabs(sum) / sqrt(nb)));
    }
  }
}

// ------------------------------------------------------------------ deluxe helpers
__global__ void deluxe_gather_kernel(const SlotDev *__restrict__ slots, const SubDev *__restrict__ subs,
                                     const double *__restrict__ Kall, double *sidebuf) {
  const SlotDev s = slots[blockIdx.y];
  const SubDev S = subs[s.sub];
  const double *ST = Kall + S.off_K + (int64_t)S.nD * (S.ldk + 1);
  const int64_t ld = S.ldk;
  const int nd = s.nd;
  double *out = sidebuf + s.off_side;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < nd * nd; idx += gridDim.x * blockDim.x) {
    int a = idx % nd, b = idx / nd;
    int ra = s.offD + a, rb = s.offD + b;
    out[idx] = ra >= rb ? ST[ra + rb * ld] : ST[rb + ra * ld];
  }
}

__global__ void multiplicity_kernel(const SlotDev *__restrict__ slots, const EntDev *__restrict__ ents, double *Dlx) {
  const SlotDev s = slots[blockIdx.y];
  const double v = 1.0 / ents[s.ent].nsh;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < s.nd * s.nd; idx += gridDim.x * blockDim.x)
    Dlx[s.off_Dlx + idx] = (idx % s.nd == idx / s.nd) ? v : 0.0;
}

// batched: out[o_b + i] = 1 / A_b(i, i) for the matrices described by MatDesc (A, n = order, ld)
struct DiagDesc {
  const double *A;
  int64_t ld, out_off;
  int n, pad;
};
__global__ void recip_diag_batched_kernel(const DiagDesc *__restrict__ d, double *out) {
  const DiagDesc D = d[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < D.n; i += gridDim.x * blockDim.x)
    out[D.out_off + i] = 1.0 / D.A[i + i * D.ld];
}

static void recip_diag_batched(const std::vector<DiagDesc> &v, double *out, cudaStream_t s) {
  if (v.empty()) return;
  DBuf<DiagDesc> d;
  std::vector<DiagDesc> h(v);
  d.upload(h, s);
  recip_diag_batched_kernel<<<dim3(8, v.size()), 256, 0, s>>>(d.p, out);
  VB_CHECK_LAUNCH();
  VB_CUDA(cudaStreamSynchronize(s));
}

__global__ void recip_diag_kernel(const double *A, int64_t ld, int n, double *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = 1.0 / A[i + i * ld];
}

// ------------------------------------------------------------------ coarse assembly (colored)
// tile rows [tlo, tlo + gridDim.y) of the packed symmetric layout (internal.h) from a row block
// Kr = A[lo:hi, :] (column-major, leading dimension ld) of a symmetric n x n matrix A; tile (I, J)
// goes to ptile_off(n, I, J) - ptile_row_start(tlo)
__global__ void pack_rows_kernel(const double *__restrict__ Kr, int64_t ld, int64_t lo, int64_t n, int64_t tlo,
                                 double *out) {
  const int64_t I = tlo + blockIdx.y, J = blockIdx.x;
  if (J > I) return;
  const int64_t nt = (n + 31) / 32;
  const int rows = (I == nt - 1) ? (int)(n - 32 * (nt - 1)) : 32;
  double *o = out + ptile_off(n, I, J) - ptile_row_start(tlo);
  for (int e = threadIdx.x; e < rows * 32; e += blockDim.x) {
    const int r = e >> 5, cc = e & 31;
    const int64_t gj = 32 * J + cc;
    o[e] = gj < n ? Kr[(32 * I + r - lo) + gj * ld] : 0.0;
  }
}

__global__ void coarse_augment_kernel(const double *__restrict__ vol, int N, double gam, double *Kc, int64_t ldc, int64_t NPi) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)N * N; idx += (int64_t)gridDim.x * blockDim.x) {
    int a = idx % N, b = idx / N;
    Kc[(NPi + a) + (NPi + b) * ldc] -= gam * vol[a] * vol[b];
  }
}

// C4 pieces: [S_c (npi x npi, full) | b~0 on Pi (npi)] per local subdomain, concatenated
__global__ void coarse_piece_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Kall,
                                    const double *__restrict__ b0T, const int64_t *__restrict__ poff, double *buf) {
  const SubDev S = subs[blockIdx.y];
  const int npi = S.npi;
  const double *Sc = Kall + S.off_K + (int64_t)(S.nD + S.nd) * (S.ldk + 1);
  double *o = buf + poff[blockIdx.y];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < npi * npi + npi; idx += gridDim.x * blockDim.x) {
    if (idx < npi * npi) {
      const int a = idx % npi, b = idx / npi;
      o[idx] = a >= b ? Sc[a + (int64_t)b * S.ldk] : Sc[b + (int64_t)a * S.ldk];
    } else {
      o[idx] = b0T[S.off_Pi + (idx - npi * npi)];
    }
  }
}

// coarse assembly from the gathered pieces of one colour class of GLOBAL subdomains
__global__ void coarse_assemble_kernel2(const int *__restrict__ color_subs, const int64_t *__restrict__ poff,
                                        const int *__restrict__ pnpi, const int64_t *__restrict__ pimoff,
                                        const int64_t *__restrict__ pimap, const double *__restrict__ buf,
                                        double *Kc, int64_t ldc, int64_t NPi) {
  const int i = color_subs[blockIdx.y];
  const int npi = pnpi[i];
  const double *Sc = buf + poff[i];
  const double *b0 = Sc + (int64_t)npi * npi;
  const int64_t *g = pimap + pimoff[i];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < npi * npi; idx += gridDim.x * blockDim.x) {
    const int a = idx % npi, b = idx / npi;
    Kc[g[a] + g[b] * ldc] += Sc[idx];
  }
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < npi; a += gridDim.x * blockDim.x) {
    Kc[(NPi + i) + g[a] * ldc] += b0[a];
    Kc[g[a] + (NPi + i) * ldc] += b0[a];
  }
}

// f1 (coarse dissection): each owned part's coarse matrix on [interior | pad | separator + p_0]
// from the pieces of one colour class of the LOCAL subdomains (lmap: piece row -> position in its
// part's matrix at kbase, leading dimension kld)
__global__ void coarse_assemble_local_kernel(const int *__restrict__ lsubs, const int64_t *__restrict__ lpoff,
                                             const int *__restrict__ lnpi, const int64_t *__restrict__ mapoff,
                                             const int64_t *__restrict__ lmap, const int64_t *__restrict__ p0pos,
                                             const double *__restrict__ buf, double *Kall,
                                             const int64_t *__restrict__ kbase, const int *__restrict__ kld) {
  const int i = lsubs[blockIdx.y];
  double *K = Kall + kbase[i];
  const int64_t ld = kld[i];
  const int npi = lnpi[i];
  const double *Sc = buf + lpoff[i];
  const double *b0 = Sc + (int64_t)npi * npi;
  const int64_t *g = lmap + mapoff[i];
  const int64_t p = p0pos[i];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < npi * npi; idx += gridDim.x * blockDim.x) {
    const int a = idx % npi, b = idx / npi;
    K[g[a] + g[b] * ld] += Sc[idx];
  }
  for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < npi; a += gridDim.x * blockDim.x) {
    K[p + g[a] * ld] += b0[a];
    K[g[a] + p * ld] += b0[a];
  }
}

__global__ void unit_diag_kernel(double *K, int64_t ld, int64_t lo, int64_t hi) {
  for (int64_t j = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < hi; j += (int64_t)gridDim.x * blockDim.x)
    K[j + j * ld] = 1.0;
}

// dst (n x n, ld dst_ld) = the symmetric matrix whose lower triangle is src's
__global__ void copy_sym_lower_kernel(const double *__restrict__ src, int64_t lds, int64_t n, double *dst, int64_t ldd) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx % n, b = idx / n;
    dst[a + b * ldd] = a >= b ? src[a + b * lds] : src[b + a * lds];
  }
}

// root += one rank's Schur contribution (n x n, ld ldp) at root positions rp (one launch per rank,
// ranks in order: the summation order is fixed and the same on every rank)
__global__ void root_scatter_add_kernel(const double *__restrict__ piece, int64_t ldp, int64_t n,
                                        const int64_t *__restrict__ rp, double *Kr, int64_t ldr) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx % n, b = idx / n;
    Kr[rp[a] + rp[b] * ldr] += piece[a + b * ldp];
  }
}

// ------------------------------------------------------------------ host orchestration
static void sync(vb_ctx *c) { VB_CUDA(cudaStreamSynchronize(c->stream)); }

// pivot failures of a batched LDL^T (ldl_panel_kernel: zero, non-finite, or of the wrong sign /
// below kPivRel * max|diag| where MatDesc::npos asks for it), named by subdomain / entity id
static void check_info(vb_ctx *c, int nmat, const char *what, const std::vector<int> *names = nullptr,
                       const char *kind = "matrix") {
  std::vector<int> info(nmat);
  VB_CUDA(cudaMemcpyAsync(info.data(), c->d_info.p, nmat * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  sync(c);
  for (int b = 0; b < nmat; ++b)
    if (info[b])
      throw Error{VB_ESINGULAR, std::string(what) + ": pivot failure (zero, non-finite or wrong sign) at column " +
                                    std::to_string(info[b] - 1) + " of " + kind + " " +
                                    std::to_string(names ? (*names)[b] : b)};
}

// primal ranks of ALL entities (each provided by the entity's owner rank = rank of its lowest
// sharer) and the global primal numbering (entity order)
static void global_entity_ranks(vb_ctx *c, const std::vector<int> &rank) {
  const int nge = c->gents.size();
  std::vector<double> mine(nge, 0.0), all;
  for (size_t e = 0; e < c->ents.size(); ++e) {
    const Entity &E = c->ents[e];
    if (c->sub_rank[E.sharers[0]] == c->rank) mine[E.gid] = rank[e];
  }
  if (c->nranks == 1) {
    all = mine;
  } else {
    DBuf<double> dm, dg;
    dm.upload(mine, c->stream);
    dg.alloc((size_t)nge * c->nranks);
    c->comm->allgather(dm.p, dg.p, nge, c->stream);
    std::vector<double> g;
    dg.download(g, c->stream);
    sync(c);
    all.assign(nge, 0.0);
    for (int r = 0; r < c->nranks; ++r)
      for (int e = 0; e < nge; ++e) all[e] += g[(size_t)r * nge + e];
  }
  int64_t off = 0;
  for (int e = 0; e < nge; ++e) {
    c->gents[e].r = (int)all[e];
    c->gents[e].off_pi = off;
    off += c->gents[e].r;
  }
  c->NPi_g = off;
  for (size_t e = 0; e < c->ents.size(); ++e)
    VB_REQUIRE(c->gents[c->ents[e].gid].r == rank[e], VB_EINVAL,
               "primal rank of entity " + std::to_string(c->ents[e].gid) + " differs between ranks");
}

// layout after the ranks of the entity bases are known
static void layout_phase_b(vb_ctx *c, const std::vector<int> &rank) {
  global_entity_ranks(c, rank);
  int64_t xd = 0, pl = 0;
  for (size_t e = 0; e < c->ents.size(); ++e) {
    Entity &E = c->ents[e];
    EntDev &D = c->h_ent[e];
    E.r = rank[e]; E.nd = E.n - E.r;
    D.r = E.r; D.nd = E.nd;
    E.off_d = xd; D.off_xd = xd; xd += E.nd;
    E.off_p = c->gents[E.gid].off_pi; D.off_pi = E.off_p;
    E.off_pl = pl; D.off_pl = pl; pl += E.r;
  }
  c->n_delta_glob = xd;
  c->NPi = pl;
  c->nx = xd + pl + c->N;
  int64_t sum = 0, Dl = 0, side = 0;
  for (size_t e = 0; e < c->ents.size(); ++e) {
    EntDev &D = c->h_ent[e];
    D.off_sum = sum; D.off_W = sum; sum += (int64_t)D.nd * D.nd;
    for (int q = 0; q < D.nsides; ++q) {
      SlotDev &s = c->h_slot[D.side_begin + q];
      s.nd = D.nd; s.r = D.r;
      s.off_Dlx = Dl; Dl += (int64_t)D.nd * D.nd;
      s.off_side = side; side += (int64_t)D.nd * D.nd;
    }
  }
  c->len_sum = sum; c->len_Dlx = Dl; c->len_side = side;
  int64_t offDv = 0, offPi = 0, STp = 0, SDi = 0, Phi = 0;
  for (int i = 0; i < c->N; ++i) {
    SubDev &S = c->h_sub[i];
    int nd = 0, npi = 0;
    for (int q = S.slot_begin; q < S.slot_end; ++q) {
      SlotDev &s = c->h_slot[c->h_sub_slots[q]];
      s.offD = nd; nd += s.nd;
    }
    for (int q = S.slot_begin; q < S.slot_end; ++q) {
      SlotDev &s = c->h_slot[c->h_sub_slots[q]];
      s.offPi = npi; npi += s.r;
    }
    S.nd = nd; S.npi = npi;
    c->subs[i].nd = nd; c->subs[i].npi = npi;
    S.off_Dv = offDv; offDv += nd;
    S.off_Pi = offPi; offPi += npi;
    S.off_STp = STp; STp += packed_size(S.nG);
    S.off_SDi = SDi; SDi += packed_size(nd);
    S.off_Phi = Phi; Phi += (int64_t)nd * npi;
  }
  c->len_Dv = offDv; c->len_Pi = offPi; c->len_STp = STp; c->len_SDi = SDi; c->len_Phi = Phi;
}

// A1/A2: assembly, Dirichlet LDL^T, S_G in the trailing block of K, B0/B8 operators.
static void stage_dirichlet(vb_ctx *c) {
  cudaStream_t s = c->stream;
  const int N = c->N;
  // ---------------- A1: assemble subdomain matrices [I | P | Gamma]
  c->d_K.alloc(c->len_K);
  c->d_K.zero(s);
  c->d_b0.alloc(c->len_G);
  c->d_b0.zero(s);
  assemble_kernel<<<N, 256, 0, s>>>(c->d_sub.p, c->d_sub_cells.p, c->d_cell_loc.p, c->d_cell_nv.p,
                                    c->d_elA.p, c->d_elB.p, c->nv_max, c->np, c->d_cvec.p, c->d_mvec.p,
                                    c->d_K.p, c->d_b0.p);
  VB_STAGE();
  // ---------------- A1/A2: partial LDL^T eliminating (u_I, p) -> trailing block = S_G
  c->d_info.alloc(std::max<int64_t>(N, std::max<int64_t>(c->ents.size(), 1)) + 1);
  c->d_info.zero(s);
  std::vector<MatDesc> mats(N);
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    mats[i] = MatDesc{c->d_K.p + S.off_K, S.n, S.ldk, S.nD};
    mats[i].npos = S.nI;        // [u_I | p (Q_I, augmented) | Gamma]: velocity > 0, pressure < 0
  }
  STAGE_T("  assembly");
  ldl_partial_batched(mats, c->d_info.p, s);
  check_info(c, N, "subdomain Dirichlet LDL^T (A1)", &c->sub_gid, "subdomain");
  STAGE_T("  Dirichlet LDL^T");
  std::vector<MatDesc> sg(N);
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    sg[i] = MatDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.nG, S.ldk, 0};
  }
  symmetrize_lower_batched(sg, s);
  // ---------------- Dirichlet solve operator for B0/B8 as a packed GEMV operand:
  //   K_DD^-1 = L_DD^-T D^-1 L_DD^-1 (the couplings K_GD, K_DG are applied element by element)
  {
    int64_t lenWD = 0, lenKDi = 0;
    std::vector<int64_t> offWD(N), offKDi(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      offWD[i] = lenWD; lenWD += (int64_t)ld4(S.nD) * S.nD;
      offKDi[i] = lenKDi; lenKDi += packed_size(S.nD);
      c->h_sub[i].off_KDi = offKDi[i];
    }
    DBuf<double> WD, dD;
    WD.alloc(lenWD);
    WD.zero(s);
    std::vector<TriDesc> td(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      td[i] = TriDesc{c->d_K.p + S.off_K, S.ldk, WD.p + offWD[i], ld4(S.nD), S.nD};
    }
    tri_inverse_batched(td, s);
    STAGE_T("  L_DD^-1");
    dD.alloc(c->len_Dn);
    {
      std::vector<DiagDesc> dd;
      for (int i = 0; i < N; ++i) {
        const SubDev &S = c->h_sub[i];
        dd.push_back(DiagDesc{c->d_K.p + S.off_K, S.ldk, S.off_Dn, S.nD, 0});
      }
      recip_diag_batched(dd, dD.p, s);
    }
    VB_STAGE();
    // K_DD^-1 (lower) overwrites the consumed L_DD block of K (leading dimension n)
    GemmPlan plan;
    int l0 = plan.begin_launch();
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      GemmProb q{};
      q.A = WD.p + offWD[i]; q.lda = ld4(S.nD); q.transA = 1;
      q.d = dD.p + S.off_Dn; q.dstride = 1;
      q.B = WD.p + offWD[i]; q.ldb = ld4(S.nD);
      q.C = c->d_K.p + S.off_K; q.ldc = S.ldk;
      q.M = q.N = q.K = S.nD; q.alpha = 1.0; q.beta = 0.0; q.lower = 1;
      q.kz_on = 1;   // W lower triangular: only k >= max(i, j) contributes (site bit 1)
      plan.add(q);
    }
    plan.upload(s);
    plan.run(l0, s);
    sync(c);
    c->d_KDi.alloc(lenKDi);
    std::vector<PackDesc> pk(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      pk[i] = PackDesc{c->d_K.p + S.off_K, S.nD, S.ldk, c->d_KDi.p + offKDi[i]};
    }
    pack_tiles_batched(pk, s);
    c->len_KDi = lenKDi;
  }
}

// A3 (first half): entity bases, layout, S_T = T^T S_G T over the trailing block of K, packed S_T,
// deluxe side blocks S_GD^(m) (sidebuf) and their sums (sumbuf).
static void stage_interface(vb_ctx *c, DBuf<double> &sidebuf, DBuf<double> &sumbuf) {
  cudaStream_t s = c->stream;
  const int N = c->N;
  // ---------------- A3: entity bases T_G = [N_G | C'^T]
  std::vector<double> rows;
  build_constraint_rows(c, rows);
  int64_t lenT = 0;
  for (size_t e = 0; e < c->ents.size(); ++e) {
    EntDev &D = c->h_ent[e];
    D.off_C = c->ents[e].off_C; D.nrowsC = c->ents[e].nrows_C;
    D.off_T = lenT; lenT += (int64_t)D.n * D.n;
  }
  for (auto &sl : c->h_slot) sl.off_T = c->h_ent[sl.ent].off_T;
  c->len_T = lenT;
  c->d_C.upload(rows, s);
  c->d_T.alloc(lenT);
  DBuf<double> wq;
  wq.alloc(std::max<size_t>(rows.size(), 1));
  c->d_ent.upload(c->h_ent, s);
  DBuf<int> drank;
  drank.alloc(c->ents.size());
  double tol = c->cons.svd_rel_tol > 0 ? c->cons.svd_rel_tol : 1e-10;
  if (c->cons.svd_rel_tol < 0) tol = 1e-10;
  if (!c->ents.empty())
    entity_basis_kernel<<<c->ents.size(), 128, 0, s>>>(c->d_ent.p, c->d_C.p, c->d_T.p, wq.p, drank.p, tol);
  VB_STAGE();
  std::vector<int> rank;
  drank.download(rank, s);
  sync(c);
  layout_phase_b(c, rank);
  c->d_ent.upload(c->h_ent, s);
  c->d_slot.upload(c->h_slot, s);
  c->d_sub.upload(c->h_sub, s);
  build_transformed_maps(c);
  // ---------------- S_T = T^T S_G T (into the trailing block of K), via scratch X = S_G T
  DBuf<double> X;
  X.alloc(c->len_X);
  {
    GemmPlan plan;
    int l0 = plan.begin_launch();
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      double *SG = c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1);
      for (int q = S.slot_begin; q < S.slot_end; ++q) {
        const SlotDev &sl = c->h_slot[c->h_sub_slots[q]];
        const double *Te = c->d_T.p + sl.off_T;
        for (int part = 0; part < 2; ++part) {
          GemmProb p{};
          p.A = SG + (int64_t)sl.offG * S.ldk; p.lda = S.ldk;
          p.B = Te + (part ? (int64_t)sl.nd * sl.n : 0); p.ldb = sl.n;
          int oc = part ? S.nd + sl.offPi : sl.offD;
          p.C = X.p + S.off_X + (int64_t)oc * ld4(S.nG); p.ldc = ld4(S.nG);
          p.M = S.nG; p.N = part ? sl.r : sl.nd; p.K = sl.n; p.alpha = 1.0; p.beta = 0.0;
          plan.add(p);
        }
      }
    }
    int l1 = plan.begin_launch();
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      double *ST = c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1);
      for (int q = S.slot_begin; q < S.slot_end; ++q) {
        const SlotDev &sl = c->h_slot[c->h_sub_slots[q]];
        const double *Te = c->d_T.p + sl.off_T;
        for (int part = 0; part < 2; ++part) {
          GemmProb p{};
          p.A = Te + (part ? (int64_t)sl.nd * sl.n : 0); p.lda = sl.n; p.transA = 1;
          p.B = X.p + S.off_X + sl.offG; p.ldb = ld4(S.nG);
          int orow = part ? S.nd + sl.offPi : sl.offD;
          p.C = ST + orow; p.ldc = S.ldk;
          p.M = part ? sl.r : sl.nd; p.N = S.nG; p.K = sl.n; p.alpha = 1.0; p.beta = 0.0;
          plan.add(p);
        }
      }
    }
    plan.upload(s);
    plan.run(l0, s);
    plan.run(l1, s);
    sync(c);
  }
  // ---------------- operator matrix: packed tiles of S_T (per-iteration operator, B1)
  c->d_STp.alloc(c->len_STp);
  {
    std::vector<PackDesc> pk(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      pk[i] = PackDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.nG, S.ldk, c->d_STp.p + S.off_STp};
    }
    pack_tiles_batched(pk, s);
  }
  // ---------------- deluxe side blocks S_GD^(m) (before S_T is factored)
  const int nslot = c->h_slot.size();
  // sums over ALL sharers: blocks of sharers on other ranks arrive by a C1 exchange
  SlotExchange XD;
  auto L2 = [&](int e) { return (int64_t)c->h_ent[e].nd * c->h_ent[e].nd; };
  build_slot_exchange(c, XD, L2, [&](int sl, std::vector<int64_t> &out) {
    const int64_t b = c->h_slot[sl].off_side, n = L2(c->h_slot[sl].ent);
    for (int64_t q = 0; q < n; ++q) out.push_back(b + q);
  });
  sidebuf.alloc(std::max<int64_t>(c->len_side + XD.recv_len, 1));
  sumbuf.alloc(std::max<int64_t>(c->len_sum, 1));
  if (nslot) {
    deluxe_gather_kernel<<<dim3(16, nslot), 256, 0, s>>>(c->d_slot.p, c->d_sub.p, c->d_K.p, sidebuf.p);
    VB_STAGE();
  }
  run_slot_exchange(c, XD, sidebuf.p, sidebuf.p + c->len_side);
  EntitySum ES;
  build_entity_sum(c, ES, XD, L2, [&](int sl) { return c->h_slot[sl].off_side; }, c->len_side,
                   [&](int e) { return c->h_ent[e].off_sum; });
  run_entity_sum(c, ES, sidebuf.p, sumbuf.p);
  VB_STAGE();
  sync(c);
}

// VB_CD_DUMP=<dir>: debug dumps of the coarse matrices (dense Kc, the dissection root and lists)
static void cd_dump(vb_ctx *c, const char *name, const double *dev, int64_t rows, int64_t cols, int64_t ld) {
  const char *dir = getenv("VB_CD_DUMP");
  if (!dir) return;
  std::vector<double> h(rows * cols);
  VB_CUDA(cudaStreamSynchronize(c->stream));
  VB_CUDA(cudaMemcpy2D(h.data(), rows * 8, dev, ld * 8, rows * 8, cols, cudaMemcpyDeviceToHost));
  std::string f = std::string(dir) + "/" + name + "_r" + std::to_string(c->rank) + ".bin";
  FILE *fp = fopen(f.c_str(), "wb");
  if (!fp) return;
  int64_t hd[2] = {rows, cols};
  fwrite(hd, 8, 2, fp);
  fwrite(h.data(), 8, h.size(), fp);
  fclose(fp);
}
static void cd_dump_i(vb_ctx *c, const char *name, const std::vector<int64_t> &v) {
  const char *dir = getenv("VB_CD_DUMP");
  if (!dir) return;
  std::string f = std::string(dir) + "/" + name + "_r" + std::to_string(c->rank) + ".bin";
  FILE *fp = fopen(f.c_str(), "wb");
  if (!fp) return;
  int64_t hd[2] = {(int64_t)v.size(), 1};
  fwrite(hd, 8, 2, fp);
  fwrite(v.data(), 8, v.size(), fp);
  fclose(fp);
}

// Explicit inverse of an LDL^T-factored coarse (or dissection root) matrix of order n, packed
// (DESIGN.md §9): (K)^-1 = W^T D^-1 W with W = L^-1.  One rank keeps all of it; with R ranks,
// rank r computes and keeps only the tile rows [tlo, thi) of the packed symmetric inverse (a
// contiguous slice of the 1-rank layout, split by tile count), from the row block
// (W[:, lo:hi])^T D^-1 W[:, :hi] (W lower triangular: k >= lo suffices).  The solve streams the
// slice with the packed GEMV (row and transpose parts) and sums the ranks' partial vectors in rank
// order (C2): n^2 / (2R) doubles per rank per iteration.
static void coarse_inverse_pack(vb_ctx *c, DBuf<double> &Kc, int64_t ldC, int64_t Nc) {
  cudaStream_t s = c->stream;
  DBuf<double> Wc, dc;
  Wc.alloc(ldC * Nc);
  Wc.zero(s);
  tri_inverse_batched({TriDesc{Kc.p, (int)ldC, Wc.p, (int)ldC, (int)Nc}}, s);
  dc.alloc(Nc);
  recip_diag_kernel<<<(Nc + 255) / 256, 256, 0, s>>>(Kc.p, ldC, Nc, dc.p);
  VB_STAGE();
  if (c->nranks == 1) {
    GemmPlan plan;
    int l0 = plan.begin_launch();
    GemmProb p{};
    p.A = Wc.p; p.lda = ldC; p.transA = 1; p.d = dc.p; p.dstride = 1;
    p.B = Wc.p; p.ldb = ldC; p.C = Kc.p; p.ldc = ldC;
    p.M = p.N = p.K = Nc; p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
    p.kz_on = 8;   // W lower triangular (site bit 8)
    plan.add(p);
    plan.upload(s);
    plan.run(l0, s);
    sync(c);
    c->d_Kcp.alloc(packed_size(Nc));
    pack_tiles_batched({PackDesc{Kc.p, (int)Nc, (int)ldC, c->d_Kcp.p}}, s);
  } else {
    const int64_t nt = (Nc + 31) / 32, R = c->nranks;
    std::vector<int64_t> T(R + 1, nt);
    T[0] = 0;
    const double total = (double)nt * (nt + 1) / 2;
    for (int64_t r = 1, I = 0; r < R; ++r) {
      while (I < nt && (double)(I + 1) * (I + 2) / 2 < total * r / R) ++I;
      T[r] = std::max(T[r - 1], std::min<int64_t>(nt, I + 1));
    }
    c->coarse_tlo = T[c->rank];
    c->coarse_thi = T[c->rank + 1];
    const int64_t lo = 32 * c->coarse_tlo, hi = std::min<int64_t>(Nc, 32 * c->coarse_thi), mine = hi - lo;
    const int64_t slice = c->coarse_thi == nt ? packed_size(Nc) - ptile_row_start(c->coarse_tlo)
                                              : ptile_row_start(c->coarse_thi) - ptile_row_start(c->coarse_tlo);
    c->d_Kcs.alloc(std::max<int64_t>(slice, 1));
    if (mine > 0) {
      DBuf<double> Kr;
      Kr.alloc(mine * hi);
      GemmPlan plan;
      int l0 = plan.begin_launch();
      GemmProb p{};
      p.A = Wc.p + lo * ldC + lo; p.lda = ldC; p.transA = 1; p.d = dc.p + lo; p.dstride = 1;
      p.B = Wc.p + lo; p.ldb = ldC; p.C = Kr.p; p.ldc = mine;
      p.M = mine; p.N = hi; p.K = Nc - lo; p.alpha = 1.0; p.beta = 0.0;
      p.kz_on = 16; p.kzB = (int)-lo;   // (site bit 16)   // W(lo + k, lo + i) = 0 for k < i, W(lo + k, j) = 0 for k < j - lo
      plan.add(p);
      plan.upload(s);
      plan.run(l0, s);
      pack_rows_kernel<<<dim3(c->coarse_thi, c->coarse_thi - c->coarse_tlo), 256, 0, s>>>(
          Kr.p, mine, lo, Nc, c->coarse_tlo, c->d_Kcs.p);
      sync(c);
    }
    VB_STAGE();
  }
}

// Host part of the coarse dissection (also vb_plan_coarse_dissection, no device work).  Parts: the
// ranks (R > 1: part = subdomain_rank, this rank eliminates its own part) or, on one rank, blocks of
// its subdomains (coarse_blocks; this rank eliminates every part).  Interior DOFs of each part, the
// root (separator between parts, then every p_0), each part's root list S_p and the root-rhs
// sources p * maxS + q.
CoarsePlan plan_coarse_dissection(const vb_ctx *c, const std::vector<int> &part, int nparts) {
  CoarsePlan P;
  P.nparts = nparts;
  P.part = part;
  const int Ng = c->Ng;
  if (c->nranks > 1) P.owned = {c->rank};
  else for (int p = 0; p < nparts; ++p) P.owned.push_back(p);
  const int64_t NPi = c->NPi_g, Nc = NPi + Ng;
  const int ne = c->gents.size();
  std::vector<int> epart(ne, -1);   // the one part of all sharers, or -1 (separator)
  for (int e = 0; e < ne; ++e) {
    const GEnt &E = c->gents[e];
    if (E.r <= 0 || E.sharers.empty()) continue;
    int p0 = part[E.sharers[0]];
    for (int g : E.sharers)
      if (part[g] != p0) { p0 = -1; break; }
    epart[e] = p0;
  }
  std::vector<int64_t> &root = P.root;
  P.I.assign(nparts, {});
  for (int e = 0; e < ne; ++e) {
    const GEnt &E = c->gents[e];
    if (E.r <= 0) continue;
    for (int t = 0; t < E.r; ++t) {
      if (epart[e] < 0) root.push_back(E.off_pi + t);
      else P.I[epart[e]].push_back(E.off_pi + t);
    }
  }
  std::sort(root.begin(), root.end());
  for (auto &v : P.I) std::sort(v.begin(), v.end());
  const int64_t nsep = root.size();
  P.nsep = nsep;
  for (int g = 0; g < Ng; ++g) root.push_back(NPi + g);
  const int64_t nroot = root.size();
  std::vector<int64_t> rpos(Nc, -1);
  for (int64_t j = 0; j < nroot; ++j) rpos[root[j]] = j;
  // every part's root list: the separator DOFs its subdomains touch (sorted), then its p_0's
  std::vector<std::vector<int64_t>> &Sr = P.S;
  Sr.assign(nparts, {});
  for (int g = 0; g < Ng; ++g) {
    const int p = part[g];
    for (int e : c->gsub_ents[g])
      if (c->gents[e].r > 0 && epart[e] < 0)
        for (int t = 0; t < c->gents[e].r; ++t) Sr[p].push_back(c->gents[e].off_pi + t);
  }
  for (int p = 0; p < nparts; ++p) {   // an entity is seen once per sharing subdomain of the part
    std::sort(Sr[p].begin(), Sr[p].end());
    Sr[p].erase(std::unique(Sr[p].begin(), Sr[p].end()), Sr[p].end());
  }
  for (int g = 0; g < Ng; ++g) Sr[part[g]].push_back(NPi + g);
  int64_t &maxS = P.maxS;
  maxS = 1;
  for (int p = 0; p < nparts; ++p) maxS = std::max<int64_t>(maxS, Sr[p].size());
  // root rhs sources: root entry j <- t_p[q] (at p * maxS + q) for every S_p[q] = root[j]
  std::vector<int64_t> &rptr = P.rptr, &ridx = P.ridx;
  rptr.assign(nroot + 1, 0);
  for (int p = 0; p < nparts; ++p)
    for (int64_t v : Sr[p]) ++rptr[rpos[v] + 1];
  for (int64_t j = 0; j < nroot; ++j) rptr[j + 1] += rptr[j];
  ridx.resize(rptr[nroot]);
  {
    std::vector<int64_t> fill(rptr.begin(), rptr.end() - 1);
    for (int p = 0; p < nparts; ++p)
      for (size_t q = 0; q < Sr[p].size(); ++q) ridx[fill[rpos[Sr[p][q]]]++] = (int64_t)p * maxS + q;
  }
  return P;
}

// Blocks of one rank's subdomains for the coarse dissection on one GPU: recursive coordinate
// bisection of the subdomain centroids (volume-weighted cell centroids) into B parts (B a power of
// two): split the longest extent at the median, ties by subdomain id (deterministic).
static std::vector<int> coarse_blocks_rcb(const vb_ctx *c, int B) {
  const int N = c->N;
  std::vector<std::array<double, 3>> xc(N);
  for (int i = 0; i < N; ++i) {
    double v = 0, x[3] = {0, 0, 0};
    for (int l : c->subs[i].cells) {
      const double *g = &c->cellgeo[(int64_t)l * c->geo_stride];
      v += g[0];
      for (int d = 0; d < 3; ++d) x[d] += g[0] * g[1 + d];
    }
    for (int d = 0; d < 3; ++d) xc[i][d] = x[d] / v;
  }
  std::vector<int> part(c->Ng, 0);
  std::function<void(std::vector<int> &, int, int)> rec = [&](std::vector<int> &ids, int p0, int nb) {
    if (nb <= 1 || ids.size() <= 1) {
      for (int i : ids) part[c->sub_gid[i]] = p0;
      return;
    }
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
    for (int i : ids)
      for (int d = 0; d < 3; ++d) { lo[d] = std::min(lo[d], xc[i][d]); hi[d] = std::max(hi[d], xc[i][d]); }
    int ax = 0;
    for (int d = 1; d < 3; ++d) if (hi[d] - lo[d] > hi[ax] - lo[ax]) ax = d;
    std::sort(ids.begin(), ids.end(), [&](int a, int b) {
      return xc[a][ax] != xc[b][ax] ? xc[a][ax] < xc[b][ax] : a < b;
    });
    std::vector<int> L(ids.begin(), ids.begin() + ids.size() / 2), Rr(ids.begin() + ids.size() / 2, ids.end());
    rec(L, p0, nb / 2);
    rec(Rr, p0 + nb / 2, nb - nb / 2);
  };
  std::vector<int> all(N);
  for (int i = 0; i < N; ++i) all[i] = i;
  rec(all, 0, B);
  return part;
}

// One level of the coarse dissection: the parts j (index lists I_j, S_j of global coarse indices)
// each get a dense matrix on [I_j | pad | S_j] from `assemble` (K, Koff, D), a partial LDL^T
// eliminating I_j (A_II SPD), W = L_II^-1, E = W^T D^-1 W and F^T = L_SI W packed as
// [[E, .], [F^T, 0]] into Kpk, and their Schur contributions on S_j into pieces (part j at
// j maxS^2, full symmetric, leading dimension maxS).  All batched over the parts.
template <class Assemble>
static std::vector<CdPart> eliminate_level(vb_ctx *c, const std::vector<std::vector<int64_t>> &I,
                                           const std::vector<std::vector<int64_t>> &S, const std::vector<int> &ids,
                                           int64_t maxS, DBuf<double> &Kpk, DBuf<double> &pieces,
                                           const Assemble &assemble) {
  cudaStream_t s = c->stream;
  const int no = I.size();
  std::vector<CdPart> D(no);
  std::vector<int64_t> Koff(no + 1, 0), Woff(no + 1, 0);
  int64_t kpk = 0;
  for (int j = 0; j < no; ++j) {
    CdPart &d = D[j];
    d.part = ids[j];
    d.nI = I[j].size();
    d.nIp = (d.nI + 31) / 32 * 32;
    d.nS = S[j].size();
    d.nloc = d.nIp + d.nS;
    d.koff = kpk;
    kpk += packed_size((int)d.nloc);
    Koff[j + 1] = Koff[j] + (int64_t)ld4((int)d.nloc) * d.nloc;
    Woff[j + 1] = Woff[j] + (int64_t)ld4((int)std::max<int64_t>(d.nIp, 1)) * d.nIp;
  }
  DBuf<double> K;
  K.alloc(std::max<int64_t>(Koff[no], 1));
  K.zero(s);
  assemble(K.p, Koff, D);
  for (int j = 0; j < no; ++j)
    if (D[j].nIp > D[j].nI) {
      unit_diag_kernel<<<1, 64, 0, s>>>(K.p + Koff[j], ld4((int)D[j].nloc), D[j].nI, D[j].nIp);
      VB_STAGE();
    }
  Kpk.release();
  Kpk.alloc(std::max<int64_t>(kpk, 1));
  Kpk.zero(s);
  std::vector<MatDesc> lm;
  std::vector<int> who;
  for (int j = 0; j < no; ++j) {
    if (!D[j].nIp) continue;
    MatDesc m{K.p + Koff[j], (int)D[j].nloc, ld4((int)D[j].nloc), (int)D[j].nIp};
    m.npos = (int)D[j].nIp;   // A_II SPD
    lm.push_back(m);
    who.push_back(D[j].part);
  }
  if (!lm.empty()) {
    c->d_info.zero(s);
    ldl_partial_batched(lm, c->d_info.p, s);
    check_info(c, (int)lm.size(), "coarse interior LDL^T (f1)", &who, "part");
    DBuf<double> W, dI, M;
    W.alloc(std::max<int64_t>(Woff[no], 1));
    W.zero(s);
    std::vector<TriDesc> td;
    for (int j = 0; j < no; ++j)
      if (D[j].nIp)
        td.push_back(TriDesc{K.p + Koff[j], ld4((int)D[j].nloc), W.p + Woff[j], ld4((int)D[j].nIp), (int)D[j].nIp});
    tri_inverse_batched(td, s);
    std::vector<int64_t> doff(no + 1, 0);
    for (int j = 0; j < no; ++j) doff[j + 1] = doff[j] + D[j].nIp;
    dI.alloc(std::max<int64_t>(doff[no], 1));
    for (int j = 0; j < no; ++j)
      if (D[j].nIp) {
        recip_diag_kernel<<<(int)((D[j].nIp + 255) / 256), 256, 0, s>>>(K.p + Koff[j], ld4((int)D[j].nloc),
                                                                        (int)D[j].nIp, dI.p + doff[j]);
        VB_STAGE();
      }
    M.alloc(std::max<int64_t>(Koff[no], 1));
    M.zero(s);
    GemmPlan plan;
    int l0 = plan.begin_launch();
    for (int j = 0; j < no; ++j) {
      if (!D[j].nIp) continue;
      const int ldk = ld4((int)D[j].nloc), ldw = ld4((int)D[j].nIp);
      GemmProb p{};
      p.A = W.p + Woff[j]; p.lda = ldw; p.transA = 1; p.d = dI.p + doff[j]; p.dstride = 1;   // E = W^T D^-1 W
      p.B = W.p + Woff[j]; p.ldb = ldw; p.C = M.p + Koff[j]; p.ldc = ldk;
      p.M = p.N = p.K = (int)D[j].nIp; p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
      p.kz_on = 8;   // W lower triangular (site bit 8)
      plan.add(p);
      GemmProb q{};
      q.A = K.p + Koff[j] + D[j].nIp; q.lda = ldk;                                           // F^T = L_SI W
      q.B = W.p + Woff[j]; q.ldb = ldw; q.C = M.p + Koff[j] + D[j].nIp; q.ldc = ldk;
      q.M = (int)D[j].nS; q.N = (int)D[j].nIp; q.K = (int)D[j].nIp; q.alpha = 1.0; q.beta = 0.0;
      plan.add(q);
    }
    plan.upload(s);
    plan.run(l0, s);
    sync(c);
    std::vector<PackDesc> pk;
    for (int j = 0; j < no; ++j)
      if (D[j].nIp) pk.push_back(PackDesc{M.p + Koff[j], (int)D[j].nloc, ld4((int)D[j].nloc), Kpk.p + D[j].koff});
    pack_tiles_batched(pk, s);
  }
  pieces.alloc((size_t)maxS * maxS * std::max(no, 1));
  pieces.zero(s);
  for (int j = 0; j < no; ++j) {
    const int64_t n = D[j].nS, ldk = ld4((int)D[j].nloc);
    if (!n) continue;
    copy_sym_lower_kernel<<<(int)std::min<int64_t>((n * n + 255) / 256, 8192), 256, 0, s>>>(
        K.p + Koff[j] + D[j].nIp * (ldk + 1), ldk, n, pieces.p + (size_t)j * maxS * maxS, maxS);
    VB_STAGE();
  }
  sync(c);
  return D;
}

// dissection of the coarse saddle problem (solved by block elimination; DESIGN.md
// §9).  The primal DOFs of an entity whose sharers all lie in one part p are interior to p: only p's
// subdomains contribute to their rows and columns, so p is eliminated alone.  The other primal DOFs
// (the separator between parts) and every p_0 (coupled globally by the gauge augmentation -gamma m
// m^T, reading A5) form the root.  Each part keeps E = A_II^-1 and F^T = A_SI A_II^-1 = L_SI L_II^-1
// (its partial LDL^T gives A_SI = L_SI D L_II^T), packed as one symmetric matrix [[E, .], [F^T, 0]];
// the root Schur complement sum_p (A_SS^(p) - A_SI A_II^-1 A_IS) - gamma m m^T is assembled on every
// rank from the parts' contributions (allgathered across ranks, summed in part order) and inverted
// like the dense coarse matrix (coarse_inverse_pack, sliced over ranks).  Solve: y_I = E g_I,
// t = F^T g_I (one GEMV pass per part); x_S = S^-1 (g_S - sum_p t_p); x_I = y_I - F x_S.  Velocity
// DOFs first in the local and the root orderings (A_II SPD; the root's pressure Schur complement
// negative definite: the pivot test of ldl_panel).
// Parts: one GPU -- blocks of its subdomains (coarse_blocks); several ranks -- the ranks, and with
// blocks (two levels) each rank first eliminates its blocks' interiors, then the separator between
// its blocks (the rank-interior DOFs no block owns) from the sum of the blocks' Schur contributions;
// only the cut between rank boxes and the p_0's reach the replicated root.
static void coarse_dissection(vb_ctx *c, DBuf<double> &pieces, const std::vector<int64_t> &lpoff,
                              const std::vector<int> &gnpi, const std::vector<int64_t> &pimoff,
                              const std::vector<int64_t> &pimap, double gam_c, int blocks) {
  cudaStream_t s = c->stream;
  const int R = c->nranks, Ng = c->Ng, N = c->N;
  const int64_t NPi = c->NPi_g, Nc = c->Nc;
  const bool two = R > 1 && blocks > 1;
  // global plan (parts = ranks, or the one-GPU blocks): root, S lists, root-rhs sources
  const CoarsePlan G = plan_coarse_dissection(c, R > 1 ? c->sub_rank : coarse_blocks_rcb(c, blocks), R > 1 ? R : blocks);
  // level-0 parts: the owned parts of G, or (two levels) this rank's blocks, planned with every
  // other rank's subdomains in one extra part (entities they touch are never block-interior)
  CoarsePlan L;
  std::vector<std::vector<int64_t>> I0, S0;
  std::vector<int> ids0;
  int64_t maxS0 = G.maxS;
  if (two) {
    std::vector<int> part = coarse_blocks_rcb(c, blocks);
    for (int g = 0; g < Ng; ++g)
      if (c->sub_rank[g] != c->rank) part[g] = blocks;
    L = plan_coarse_dissection(c, part, blocks + 1);
    maxS0 = 1;
    for (int b = 0; b < blocks; ++b) {
      I0.push_back(L.I[b]); S0.push_back(L.S[b]); ids0.push_back(b);
      maxS0 = std::max<int64_t>(maxS0, L.S[b].size());
    }
  } else {
    for (int p : G.owned) { I0.push_back(G.I[p]); S0.push_back(G.S[p]); ids0.push_back(p); }
  }
  const int no = I0.size();
  // part of every level-0 interior DOF, its position; S positions by search in the sorted S lists
  std::vector<int> lpart(Nc, -1);
  std::vector<int64_t> lp(Nc, -1);
  for (int j = 0; j < no; ++j)
    for (size_t a = 0; a < I0[j].size(); ++a) { lp[I0[j][a]] = a; lpart[I0[j][a]] = j; }
  std::vector<int> sub_j(N, -1);
  {
    const std::vector<int> &part = two ? L.part : G.part;
    for (int i = 0; i < N; ++i) {
      const int pg = part[c->sub_gid[i]];
      for (int j = 0; j < no; ++j) if (ids0[j] == pg) sub_j[i] = j;
      VB_REQUIRE(sub_j[i] >= 0, VB_EINVAL, "internal: coarse dissection part");
    }
  }
  auto spos = [&](const std::vector<int64_t> &Sl, int64_t nIp, int64_t v) {
    const auto it = std::lower_bound(Sl.begin(), Sl.end(), v);   // separator DOFs, then p_0's: sorted
    VB_REQUIRE(it != Sl.end() && *it == v, VB_EINVAL, "internal: coarse dissection map");
    return nIp + (int64_t)(it - Sl.begin());
  };
  // ---- level 0: matrices from the local subdomains' (S_c, b~0) pieces (no communication)
  DBuf<double> P0;
  auto asm0 = [&](double *K, const std::vector<int64_t> &Koff, const std::vector<CdPart> &D) {
    std::vector<int64_t> lmap, mapoff(N + 1, 0), p0pos(N), kbase(N);
    std::vector<int> lnpi(N), kld(N);
    for (int i = 0; i < N; ++i) {
      const int g = c->sub_gid[i], j = sub_j[i];
      const CdPart &d = D[j];
      for (int64_t q = pimoff[g]; q < pimoff[g + 1]; ++q) {
        const int64_t v = pimap[q];
        lmap.push_back(lpart[v] == j ? lp[v] : spos(S0[j], d.nIp, v));
      }
      mapoff[i + 1] = lmap.size();
      p0pos[i] = spos(S0[j], d.nIp, NPi + g);
      lnpi[i] = gnpi[g];
      kbase[i] = Koff[j];
      kld[i] = ld4((int)d.nloc);
    }
    if (lmap.empty()) lmap.push_back(0);
    DBuf<int64_t> dlpoff, dmapoff, dlmap, dp0, dkb;
    DBuf<int> dlnpi, dkld;
    dlpoff.upload(lpoff, s); dmapoff.upload(mapoff, s); dlmap.upload(lmap, s); dp0.upload(p0pos, s);
    dlnpi.upload(lnpi, s); dkb.upload(kbase, s); dkld.upload(kld, s);
    std::vector<std::vector<int>> colors(c->ncolors);
    for (int i = 0; i < N; ++i) colors[c->gsub_color[c->sub_gid[i]]].push_back(i);
    for (auto &col : colors) {
      if (col.empty()) continue;
      DBuf<int> dcol;
      dcol.upload(col, s);
      coarse_assemble_local_kernel<<<dim3(8, col.size()), 256, 0, s>>>(dcol.p, dlpoff.p, dlnpi.p, dmapoff.p, dlmap.p,
                                                                       dp0.p, pieces.p, K, dkb.p, dkld.p);
      VB_STAGE();
      sync(c);
    }
  };
  std::vector<CdPart> D0 = eliminate_level(c, I0, S0, ids0, maxS0, c->d_Kloc, P0, asm0);
  STAGE_T("  coarse level-0 elimination (f1)");
  // ---- level 1 (two levels): this rank's matrix on [RS | pad | S_r], RS = the rank-interior DOFs
  // no block owns, from the sum of its blocks' Schur contributions (block order)
  DBuf<double> Ptop;
  std::vector<CdPart> D1;
  std::vector<int64_t> RS, l2ptr, l2idx;
  if (two) {
    {
      std::vector<char> inblk(Nc, 0);
      for (auto &v : I0) for (int64_t x : v) inblk[x] = 1;
      for (int64_t x : G.I[c->rank]) if (!inblk[x]) RS.push_back(x);
    }
    const std::vector<int64_t> &Sr = G.S[c->rank];
    const int64_t nRS = RS.size(), nRSp = (nRS + 31) / 32 * 32;
    auto pos1 = [&](int64_t v) {
      const auto it = std::lower_bound(RS.begin(), RS.end(), v);
      if (it != RS.end() && *it == v) return (int64_t)(it - RS.begin());
      return spos(Sr, nRSp, v);
    };
    // level-0 S entries -> level-1 positions (the scatter of the Schur pieces and, in the solve, of
    // the blocks' t vectors: CSR over level-1 positions, sources b * maxS0 + q in block order)
    std::vector<std::vector<int64_t>> pos0(no);
    for (int j = 0; j < no; ++j)
      for (int64_t v : S0[j]) pos0[j].push_back(pos1(v));
    const int64_t nl1 = nRSp + Sr.size();
    l2ptr.assign(nl1 + 1, 0);
    for (int j = 0; j < no; ++j) for (int64_t t : pos0[j]) ++l2ptr[t + 1];
    for (int64_t a = 0; a < nl1; ++a) l2ptr[a + 1] += l2ptr[a];
    l2idx.resize(l2ptr[nl1]);
    {
      std::vector<int64_t> fill(l2ptr.begin(), l2ptr.end() - 1);
      for (int j = 0; j < no; ++j)
        for (size_t q = 0; q < pos0[j].size(); ++q) l2idx[fill[pos0[j][q]]++] = (int64_t)j * maxS0 + q;
    }
    auto asm1 = [&](double *K, const std::vector<int64_t> &Koff, const std::vector<CdPart> &D) {
      const int64_t ld = ld4((int)D[0].nloc);
      for (int j = 0; j < no; ++j) {
        const int64_t n = S0[j].size();
        if (!n) continue;
        DBuf<int64_t> dp;
        dp.upload(pos0[j], s);
        root_scatter_add_kernel<<<(int)std::min<int64_t>((n * n + 255) / 256, 8192), 256, 0, s>>>(
            P0.p + (size_t)j * maxS0 * maxS0, maxS0, n, dp.p, K + Koff[0], ld);
        VB_STAGE();
        sync(c);
      }
    };
    D1 = eliminate_level(c, {RS}, {Sr}, {c->rank}, G.maxS, c->d_Kloc2, Ptop, asm1);
    P0.release();
    STAGE_T("  coarse level-1 elimination (f1)");
  }
  DBuf<double> &top = two ? Ptop : P0;
  // ---- root: the top level's Schur contributions (allgathered across ranks), summed in part
  // order, augmented, factored, inverted
  const std::vector<int64_t> &root = G.root;
  const int64_t nsep = G.nsep, nroot = root.size(), maxS = G.maxS;
  std::vector<int64_t> rpos(Nc, -1);
  for (int64_t j = 0; j < nroot; ++j) rpos[root[j]] = j;
  const int nparts = G.nparts;
  DBuf<double> gath;
  const double *all = top.p;   // part p at p * maxS^2 (one GPU: the owned parts are all parts, in order)
  if (R > 1) {
    gath.alloc((size_t)maxS * maxS * R);
    c->comm->allgather(top.p, gath.p, maxS * maxS, s);
    all = gath.p;
  }
  const int64_t ldR = ld4((int)nroot);
  DBuf<double> Kr, gvol;
  DBuf<int64_t> drp;
  Kr.alloc(ldR * nroot);
  Kr.zero(s);
  {
    std::vector<int64_t> rp((size_t)maxS * nparts, 0);
    for (int p = 0; p < nparts; ++p)
      for (size_t q = 0; q < G.S[p].size(); ++q) rp[(size_t)p * maxS + q] = rpos[G.S[p][q]];
    drp.upload(rp, s);
  }
  for (int p = 0; p < nparts; ++p) {
    const int64_t n = G.S[p].size();
    root_scatter_add_kernel<<<(int)std::min<int64_t>((n * n + 255) / 256, 8192), 256, 0, s>>>(
        all + (size_t)p * maxS * maxS, maxS, n, drp.p + (size_t)p * maxS, Kr.p, ldR);
    VB_STAGE();
  }
  gvol.upload(c->gsub_vol, s);
  coarse_augment_kernel<<<(int)std::min<int64_t>(((int64_t)Ng * Ng + 255) / 256, 4096), 256, 0, s>>>(
      gvol.p, Ng, gam_c, Kr.p, ldR, nsep);
  VB_STAGE();
  gath.release();
  top.release();
  STAGE_T("  coarse root assembly (f1)");
  cd_dump(c, "kroot", Kr.p, nroot, nroot, ldR);
  c->d_info.zero(s);
  std::vector<MatDesc> rm{MatDesc{Kr.p, (int)nroot, (int)ldR, (int)nroot}};
  rm[0].npos = (int)nsep;   // [separator u_Pi | p_0 (augmented)]
  ldl_partial_batched(rm, c->d_info.p, s);
  check_info(c, 1, "coarse root LDL^T (f1)");
  coarse_inverse_pack(c, Kr, ldR, nroot);
  STAGE_T("  coarse root inverse (f1)");
  c->Nroot = nroot; c->cd_nsep = nsep; c->cd_maxS = maxS; c->cd_maxS0 = maxS0; c->cd_nparts = nparts;
  c->cd_parts = D0;
  c->cd_I = I0; c->cd_S = S0;
  c->cd_two = two;
  if (two) {
    c->cd2_part = D1[0];
    c->cd2_RS = RS;
    c->cd2_S = G.S[c->rank];
    c->cd2_ptr = l2ptr; c->cd2_idx = l2idx;
  }
  c->cd_root_glob = root;
  c->cd_rptr = G.rptr; c->cd_ridx = G.ridx;
}

// A3 (second half) .. A5: dual Schur inverse, Phi, S_c, b~0, deluxe D_G^(m), coarse inverse.
static void stage_dual(vb_ctx *c, DBuf<double> &sidebuf, DBuf<double> &sumbuf) {
  cudaStream_t s = c->stream;
  const int N = c->N;
  const int nslot = c->h_slot.size();
  const int nent = c->h_ent.size();
  std::vector<MatDesc> mats(N), sg(N);
  // Y = S_DD^-1 (and later D S_DD^-1 D^T) lives in the dual block of the trailing matrix of K
  // (leading dimension n), whose L_DD is consumed by the triangular inverse into X
  DBuf<double> X, Wbuf, dinv;
  X.alloc(c->len_X);
  auto Yp = [&](const SubDev &S) { return c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1); };
  Wbuf.alloc(std::max<int64_t>(c->len_sum, 1));
  // ---------------- A3: partial LDL^T of S_T eliminating the dual block -> S_c trailing
  c->d_info.zero(s);
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    mats[i] = MatDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.nG, S.ldk, S.nd};
    mats[i].npos = S.nd;        // S_DD is SPD (the primal constraints remove the rigid modes)
  }
  ldl_partial_batched(mats, c->d_info.p, s);
  check_info(c, N, "dual Schur LDL^T (A3)", &c->sub_gid, "subdomain");
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    sg[i] = MatDesc{c->d_K.p + S.off_K + (int64_t)(S.nD + S.nd) * (S.ldk + 1), S.npi, S.ldk, 0};
  }
  symmetrize_lower_batched(sg, s);
  // W = L_DD^-1 (in X), Y = W^T D^-1 W = S_DD^-1, Phi = -W^T L_PiD^T
  X.zero(s);
  {
    std::vector<TriDesc> td(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      td[i] = TriDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.ldk, X.p + S.off_X, ld4(S.nd), S.nd};
    }
    tri_inverse_batched(td, s);
  }
  dinv.alloc(std::max<int64_t>(c->len_Dv, 1));
  {
    std::vector<DiagDesc> dd;
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      if (S.nd) dd.push_back(DiagDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.ldk, S.off_Dv, S.nd, 0});
    }
    recip_diag_batched(dd, dinv.p, s);
  }
  VB_STAGE();
  c->d_Phi.alloc(std::max<int64_t>(c->len_Phi, 1));
  {
    GemmPlan plan;
    int l0 = plan.begin_launch();
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      GemmProb p{};
      p.A = X.p + S.off_X; p.lda = ld4(S.nd); p.transA = 1;
      p.d = dinv.p + S.off_Dv; p.dstride = 1;
      p.B = X.p + S.off_X; p.ldb = ld4(S.nd);
      p.C = Yp(S); p.ldc = S.ldk;
      p.M = p.N = p.K = S.nd; p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
      p.kz_on = 2;   // W lower triangular (site bit 2)
      plan.add(p);
      GemmProb q{};
      q.A = X.p + S.off_X; q.lda = ld4(S.nd); q.transA = 1;
      q.B = c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1) + S.nd; q.ldb = S.ldk; q.transB = 1;
      q.C = c->d_Phi.p + S.off_Phi; q.ldc = S.nd;
      q.M = S.nd; q.N = S.npi; q.K = S.nd; q.alpha = -1.0; q.beta = 0.0;
      q.kz_on = 4; q.kzB = -(1 << 30);   // W^T: only k >= i contributes (site bit 4)
      plan.add(q);
    }
    plan.upload(s);
    plan.run(l0, s);
    sync(c);
  }
  STAGE_T("  L_DD^-1 / S_DD^-1 / Phi");
  // ---------------- b~0 and the benign check
  c->d_b0T.alloc(std::max<int64_t>(c->len_Pi, 1));
  c->d_b0T.zero(s);
  DBuf<unsigned long long> dviol;
  dviol.alloc(1);
  dviol.zero(s);
  if (nslot) b0_transform_kernel<<<nslot, 32, 0, s>>>(c->d_slot.p, nslot, c->d_sub.p, c->d_T.p, c->d_b0.p, c->d_b0T.p, dviol.p);
  VB_STAGE();
  unsigned long long vv = 0;
  VB_CUDA(cudaMemcpyAsync(&vv, dviol.p, 8, cudaMemcpyDeviceToHost, s));
  // ---------------- A4: deluxe D_G^(m) = (sum S)^-1 S^(m)
  c->d_Dlx.alloc(std::max<int64_t>(c->len_Dlx, 1));
  if (c->cons.scaling == VB_MULTIPLICITY) {
    if (nslot) multiplicity_kernel<<<dim3(16, nslot), 256, 0, s>>>(c->d_slot.p, c->d_ent.p, c->d_Dlx.p);
    VB_STAGE();
  } else {
    std::vector<MatDesc> em;
    std::vector<int> names;
    for (int e = 0; e < nent; ++e) {
      const EntDev &E = c->h_ent[e];
      if (E.nd) {
        em.push_back(MatDesc{sumbuf.p + E.off_sum, E.nd, E.nd, E.nd});
        em.back().npos = E.nd;  // sum of the sharers' S_GD (SPD)
        names.push_back(e);
      }
    }
    c->d_info.zero(s);
    ldl_partial_batched(em, c->d_info.p, s);
    check_info(c, em.size(), "deluxe sum LDL^T (A4)", &names, "entity");
    Wbuf.zero(s);
    std::vector<TriDesc> td;
    for (auto &M : em) td.push_back(TriDesc{M.A, M.n, Wbuf.p + (M.A - sumbuf.p), M.n, M.n});
    tri_inverse_batched(td, s);
    DBuf<double> edinv;
    edinv.alloc(std::max<int64_t>(c->len_sum, 1));
    {
      std::vector<DiagDesc> dd;
      for (auto &M : em) dd.push_back(DiagDesc{M.A, M.n, (int64_t)(M.A - sumbuf.p), M.n, 0});
      recip_diag_batched(dd, edinv.p, s);
    }
    VB_STAGE();
    {
      GemmPlan plan;
      int l0 = plan.begin_launch();
      for (auto &M : em) {
        int64_t off = M.A - sumbuf.p;
        GemmProb p{};
        p.A = Wbuf.p + off; p.lda = M.n; p.transA = 1;
        p.d = edinv.p + off; p.dstride = 1;
        p.B = Wbuf.p + off; p.ldb = M.n;
        p.C = sumbuf.p + off; p.ldc = M.n;
        p.M = p.N = p.K = M.n; p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
        plan.add(p);
      }
      plan.upload(s);
      plan.run(l0, s);
      sync(c);
    }
    for (auto &M : em) M.m = 0;
    symmetrize_lower_batched(em, s);
    {
      GemmPlan plan;
      int l0 = plan.begin_launch();
      for (int q = 0; q < nslot; ++q) {
        const SlotDev &sl = c->h_slot[q];
        if (!sl.nd) continue;
        const EntDev &E = c->h_ent[sl.ent];
        GemmProb p{};
        p.A = sumbuf.p + E.off_sum; p.lda = sl.nd;
        p.B = sidebuf.p + sl.off_side; p.ldb = sl.nd;
        p.C = c->d_Dlx.p + sl.off_Dlx; p.ldc = sl.nd;
        p.M = p.N = p.K = sl.nd; p.alpha = 1.0; p.beta = 0.0;
        plan.add(p);
      }
      plan.upload(s);
      plan.run(l0, s);
      sync(c);
    }
  }
  STAGE_T("  deluxe D_G (A4)");
  // ---------------- deluxe scaling folded into the per-iteration operators (DESIGN.md "scaled local
  // operators"): with D^(m) = blockdiag over the dual slots of D_G^(m), the local part of M^-1 is
  // D S_DD^-1 D^T and the coarse basis enters as D Phi, so the iteration never applies D itself:
  //   S^_DD = D (S_DD^-1) D^T  (packed into d_SDi),  Phi^ = D Phi  (replaces d_Phi).
  {
    std::vector<MatDesc> ym;
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      if (S.nd) ym.push_back(MatDesc{Yp(S), S.nd, S.ldk, 0});
    }
    symmetrize_lower_batched(ym, s);
    DBuf<double> PhiH;
    PhiH.alloc(std::max<int64_t>(c->len_Phi, 1));
    {
      GemmPlan plan;
      int l0 = plan.begin_launch();
      for (int q = 0; q < nslot; ++q) {        // Z = D Y (row blocks), Phi^ = D Phi (row blocks)
        const SlotDev &sl = c->h_slot[q];
        if (!sl.nd) continue;
        const SubDev &S = c->h_sub[sl.sub];
        GemmProb p{};
        p.A = c->d_Dlx.p + sl.off_Dlx; p.lda = sl.nd;
        p.B = Yp(S) + sl.offD; p.ldb = S.ldk;
        p.C = X.p + S.off_X + sl.offD; p.ldc = ld4(S.nd);
        p.M = sl.nd; p.N = S.nd; p.K = sl.nd; p.alpha = 1.0; p.beta = 0.0;
        plan.add(p);
        if (S.npi) {
          GemmProb f{};
          f.A = c->d_Dlx.p + sl.off_Dlx; f.lda = sl.nd;
          f.B = c->d_Phi.p + S.off_Phi + sl.offD; f.ldb = S.nd;
          f.C = PhiH.p + S.off_Phi + sl.offD; f.ldc = S.nd;
          f.M = sl.nd; f.N = S.npi; f.K = sl.nd; f.alpha = 1.0; f.beta = 0.0;
          plan.add(f);
        }
      }
      int l1 = plan.begin_launch();
      for (int q = 0; q < nslot; ++q) {        // S^ = Z D^T (column blocks)
        const SlotDev &sl = c->h_slot[q];
        if (!sl.nd) continue;
        const SubDev &S = c->h_sub[sl.sub];
        GemmProb p{};
        p.A = X.p + S.off_X + (int64_t)sl.offD * ld4(S.nd); p.lda = ld4(S.nd);
        p.B = c->d_Dlx.p + sl.off_Dlx; p.ldb = sl.nd; p.transB = 1;
        p.C = Yp(S) + (int64_t)sl.offD * S.ldk; p.ldc = S.ldk;
        p.M = S.nd; p.N = sl.nd; p.K = sl.nd; p.alpha = 1.0; p.beta = 0.0;
        plan.add(p);
      }
      plan.upload(s);
      plan.run(l0, s);
      plan.run(l1, s);
      sync(c);
    }
    if (c->len_Phi) VB_CUDA(cudaMemcpyAsync(c->d_Phi.p, PhiH.p, c->len_Phi * sizeof(double), cudaMemcpyDeviceToDevice, s));
    sync(c);
  }
  c->d_SDi.alloc(c->len_SDi);
  {
    std::vector<PackDesc> pk(N);
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      pk[i] = PackDesc{Yp(S), S.nd, S.ldk, c->d_SDi.p + S.off_SDi};
    }
    pack_tiles_batched(pk, s);
  }
  VB_STAGE();
  c->d_Dlx.release();
  STAGE_T("  fold D S_DD^-1 D^T, D Phi");
  // ---------------- A5: coarse saddle matrix on (u_Pi, p_0) of ALL subdomains
  const int Ng = c->Ng;
  const int64_t Nc = c->NPi_g + Ng;
  c->Nc = Nc;
  // blocks of this rank's subdomains (auto: the largest power of two <= 8 with at least 16
  // subdomains per block): the parts on one rank; the first level of two on several ranks
  int blocks = 1;
  if (c->opt_coarse_blocks > 0) blocks = c->opt_coarse_blocks;
  else while (blocks < 8 && 2 * blocks * 16 <= N) blocks *= 2;
  blocks = std::max(1, std::min(blocks, N));
  // auto: always for several ranks; on one rank for coarse problems of >= 4096 unknowns split into
  // >= 2 blocks (c5: 1,025 -> 1,055 M DOF*it/s; small coarse problems keep the dense inverse)
  c->cdis = c->opt_coarse_dis < 0 ? (c->nranks > 1 || (Nc >= 4096 && blocks >= 2)) : c->opt_coarse_dis != 0;
  {
    // global piece layout: rank-major, subdomains in order within a rank
    std::vector<int> gnpi(Ng, 0);
    std::vector<int64_t> pimoff(Ng + 1, 0), pimap;
    for (int g = 0; g < Ng; ++g) {
      for (int e : c->gsub_ents[g])
        for (int t = 0; t < c->gents[e].r; ++t) pimap.push_back(c->gents[e].off_pi + t);
      gnpi[g] = pimap.size() - pimoff[g];
      pimoff[g + 1] = pimap.size();
    }
    std::vector<int64_t> rlen(c->nranks, 0), poff(Ng, 0), lpoff(N, 0);
    for (int g = 0; g < Ng; ++g) {
      const int r = c->sub_rank[g];
      poff[g] = rlen[r];
      rlen[r] += (int64_t)gnpi[g] * gnpi[g] + gnpi[g];
    }
    int64_t maxlen = 1;
    for (int r = 0; r < c->nranks; ++r) maxlen = std::max(maxlen, rlen[r]);
    for (int g = 0; g < Ng; ++g) poff[g] += (int64_t)c->sub_rank[g] * maxlen;
    for (int i = 0; i < N; ++i) {
      VB_REQUIRE(gnpi[c->sub_gid[i]] == c->h_sub[i].npi, VB_EINVAL, "internal: coarse piece size mismatch");
      lpoff[i] = poff[c->sub_gid[i]] - (int64_t)c->rank * maxlen;
    }
    DBuf<double> mine, gathered;
    DBuf<int64_t> dlpoff, dpoff, dpimoff, dpimap;
    DBuf<int> dgnpi;
    mine.alloc(maxlen);
    mine.zero(s);
    dlpoff.upload(lpoff, s);
    coarse_piece_kernel<<<dim3(8, N), 256, 0, s>>>(c->d_sub.p, c->d_K.p, c->d_b0T.p, dlpoff.p, mine.p);
    VB_STAGE();
    sync(c);
    c->d_K.release();   // the dense subdomain matrices are not needed by the solve (frees ~48 MB per subdomain)
    double nubar = 0, volO = 0;
    for (int64_t K = 0; K < c->nK; ++K) nubar += c->nu[K];
    nubar /= c->nK;
    for (int g = 0; g < Ng; ++g) volO += c->gsub_vol[g];
    // augmentation of the p_0 block for the gauge sum vol_i p0_i = 0; none with Neumann faces (A35)
    const double gam_c = c->neumann ? 0.0 : 1.0 / (nubar * volO);
    if (c->cdis) {
      coarse_dissection(c, mine, lpoff, gnpi, pimoff, pimap, gam_c, blocks);
    } else {
      // C4: every rank gathers every subdomain's (S_c, b~0) and assembles/factors the same matrix
      const double *pieces = mine.p;
      if (c->nranks > 1) {
        gathered.alloc((size_t)maxlen * c->nranks);
        c->comm->allgather(mine.p, gathered.p, maxlen, s);
        pieces = gathered.p;
      }
      dpoff.upload(poff, s);
      dgnpi.upload(gnpi, s);
      dpimoff.upload(pimoff, s);
      if (pimap.empty()) pimap.push_back(0);
      dpimap.upload(pimap, s);
      DBuf<double> Kc, gvol;
      const int64_t ldC = ld4((int)Nc);   // 32-byte aligned columns (16-byte copies in the DMMA GEMM)
      Kc.alloc(ldC * Nc);
      Kc.zero(s);
      std::vector<std::vector<int>> colors(c->ncolors);
      for (int g = 0; g < Ng; ++g) colors[c->gsub_color[g]].push_back(g);
      for (auto &col : colors) {
        if (col.empty()) continue;
        DBuf<int> dcol;
        dcol.upload(col, s);
        coarse_assemble_kernel2<<<dim3(8, col.size()), 256, 0, s>>>(dcol.p, dpoff.p, dgnpi.p, dpimoff.p, dpimap.p,
                                                                   pieces, Kc.p, ldC, c->NPi_g);
        VB_STAGE();
        sync(c);
      }
      gvol.upload(c->gsub_vol, s);
      coarse_augment_kernel<<<(int)std::min<int64_t>(((int64_t)Ng * Ng + 255) / 256, 4096), 256, 0, s>>>(
          gvol.p, Ng, gam_c, Kc.p, ldC, c->NPi_g);
      VB_STAGE();
      STAGE_T("  coarse pieces + assembly (C4)");
      cd_dump(c, "kc", Kc.p, Nc, Nc, ldC);
      c->d_info.zero(s);
      std::vector<MatDesc> cm{MatDesc{Kc.p, (int)Nc, (int)ldC, (int)Nc}};
      cm[0].npos = (int)c->NPi_g;   // [u_Pi | p_0 (augmented)]: velocity > 0, pressure < 0
      ldl_partial_batched(cm, c->d_info.p, s);
      check_info(c, 1, "coarse saddle LDL^T (A5)");
      STAGE_T("  coarse LDL^T");
      coarse_inverse_pack(c, Kc, ldC, Nc);
    }
  }
  sync(c);
  double fv;
  memcpy(&fv, &vv, 8);
  c->flux_violation = fv;
}

// VB_FACTOR_TIMES=1: wall time of each factor stage on stderr (the stages synchronise)
void factor_device(vb_ctx *c) {
  cudaStream_t s = c->stream;
  g_gemm_flops = 0.0;
  g_gemm_timing = getenv("VB_KERNEL_TIMING") && atoi(getenv("VB_KERNEL_TIMING"));
  gemm_timing_collect(s);
  const double alloc0 = g_malloc_s + g_free_s;
  stage_time(c, nullptr);
  stage_dirichlet(c);
  stage_time(c, "dirichlet (A1/A2)");
  DBuf<double> sidebuf, sumbuf;
  const double tau = c->cons.adaptive_tau;
  c->extra_rows.assign(c->ents.size(), std::vector<double>());
  c->n_adaptive = 0;
  c->adaptive_margin = INFINITY;
  if (tau > 0) {
    // keep S_G: the interface stage overwrites it with S_T, and the enriched pass starts again from S_G
    DBuf<double> SG;
    SG.alloc(c->len_X);
    for (int i = 0; i < c->N; ++i) {
      const SubDev &S = c->h_sub[i];
      VB_CUDA(cudaMemcpy2DAsync(SG.p + S.off_X, S.nG * 8, c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), (size_t)S.ldk * 8,
                                S.nG * 8, S.nG, cudaMemcpyDeviceToDevice, s));
    }
    stage_interface(c, sidebuf, sumbuf);
    stage_time(c, "interface (A3/A4)");
    adaptive_enrich(c, tau, sidebuf);           // A6: face GEVPs -> c->extra_rows
    stage_time(c, "adaptive (A6)");
    for (int i = 0; i < c->N; ++i) {
      const SubDev &S = c->h_sub[i];
      VB_CUDA(cudaMemcpy2DAsync(c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), (size_t)S.ldk * 8, SG.p + S.off_X, S.nG * 8,
                                S.nG * 8, S.nG, cudaMemcpyDeviceToDevice, s));
    }
    sync(c);
  }
  stage_interface(c, sidebuf, sumbuf);
  stage_time(c, "interface (A3/A4)");
  stage_dual(c, sidebuf, sumbuf);
  stage_time(c, "dual + coarse (A3-A5)");
  c->factor_flops = g_gemm_flops;
  c->factor_alloc_s = g_malloc_s + g_free_s - alloc0;
  c->factor_gemm_s = g_gemm_timing ? gemm_timing_collect(s) : 0.0;
  g_gemm_timing = false;
}

}  // namespace vb
