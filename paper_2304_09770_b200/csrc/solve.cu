// Solve stage: rhs condensation, the PCG loop on the interface saddle problem
// Eq.(globInt) with the BDDC preconditioner Eq.(BDDCprec), back-substitution
// and the element-by-element saddle operator.
//
// PCG vectors live in transformed interface coordinates x = [dual coords per entity | u_Pi | p_0];
// T_G is orthogonal, so Euclidean norms, CG coefficients and the stopping test equal those of the
// original coordinates.
#include <mutex>
#include <map>
#include <algorithm>
#include <cmath>
#include "dense.cuh"
#include "setup.h"
#include "exchange.h"

namespace vb {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Programmatic dependent launch (PDL): a kernel of the PCG step waits for its predecessor grid to
// complete before touching memory, and lets its successor be scheduled as soon as all of its own
// CTAs have started (the successor's CTAs fill this kernel's last wave and wait in turn).
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

// ------------------------------------------------------------------ packed symmetric GEMV (K3)
// Work item: one CTA multiplies the tile rows [r0, r1) of one packed symmetric matrix with x and
// writes a full-length partial result.  Row contributions of a tile row are reduced in fixed warp
// order; column contributions of one tile row go to distinct tile columns (one warp each), so the
// accumulation order is fixed: the kernel is deterministic.
struct GemvWork {
  const double *M;        // packed tiles; tile (I, J) at M + ptile_off(n, I, J) - moff
  const int64_t *map;     // x gather map (or null: x contiguous at xsrc)
  const double *xsrc;
  double *out;            // partial output (length n)
  int n, r0, r1, pad;
  int64_t moff;           // offset of the stored slice in the full packed layout (a rank's coarse rows)
};

#ifndef GV_WARPS_CFG
#define GV_WARPS_CFG 4
#endif
constexpr int GV_WARPS = GV_WARPS_CFG;   // subdomain matrices (several CTAs per SM)
constexpr int GV_WARPS_C = 8;    // the single coarse matrix (one CTA per SM)

// BIG: vectors too long for shared memory (large coarse problems, very large subdomains): x is read through the L2 (it is
// small next to the streamed matrix) and the partial output accumulates in the CTA's own global
// partial vector (each column J is owned by one warp, so there are no races).
// PAIR: each warp streams two tiles per step (twice the loads in flight; for the coarse matrix,
// which runs one CTA per SM)
template <int GV_WARPS, bool BIG = false, bool PAIR = false>
__global__ void __launch_bounds__(GV_WARPS * 32) sym_gemv_kernel(const GemvWork *__restrict__ work) {
  pdl_prologue();
  extern __shared__ double sm[];
  const GemvWork W = work[blockIdx.x];
  const int n = W.n, nt = (n + 31) / 32;
  const int npad = nt * 32;
  double *xs = BIG ? nullptr : sm;              // npad
  double *ys = BIG ? W.out : sm + npad;         // npad (BIG: n, guarded)
  double *rowred = BIG ? sm : sm + 2 * npad;    // GV_WARPS * 32
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto X = [&](int j) -> double {
    if (BIG) return j < n ? (W.map ? __ldg(W.xsrc + __ldg(W.map + j)) : __ldg(W.xsrc + j)) : 0.0;
    return xs[j];
  };
  if (BIG) {
    for (int j = tid; j < n; j += blockDim.x) ys[j] = 0.0;
  } else {
    for (int j = tid; j < npad; j += blockDim.x) {
      double v = 0.0;
      if (j < n) v = W.map ? W.xsrc[W.map[j]] : W.xsrc[j];
      xs[j] = v;
      ys[j] = 0.0;
    }
  }
  __syncthreads();
  for (int I = W.r0; I < W.r1; ++I) {
    const int rows = (I == nt - 1) ? n - 32 * (nt - 1) : 32;    // short last tile row
    double rsum[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) rsum[r] = 0.0;
    const double xI_lane = X(32 * I + lane);
    for (int J = warp; J <= I; J += (PAIR ? 2 : 1) * GV_WARPS) {
      const double *T = W.M + (ptile_off(n, I, J) - W.moff);
      double t[32];
      if (rows == 32) {
#pragma unroll
        for (int r = 0; r < 32; ++r) t[r] = __ldg(T + r * 32 + lane);
      } else {   // short last tile row
#pragma unroll
        for (int r = 0; r < 32; ++r) t[r] = r < rows ? __ldg(T + r * 32 + lane) : 0.0;
      }
      const int J2 = J + GV_WARPS;
      double t2[PAIR ? 32 : 1];
      if (PAIR) {
        const double *T2 = W.M + (ptile_off(n, I, J2 <= I ? J2 : J) - W.moff);
#pragma unroll
        for (int r = 0; r < 32; ++r) t2[r] = (J2 <= I && r < rows) ? __ldg(T2 + r * 32 + lane) : 0.0;
      }
      const double xJ = X(32 * J + lane);
      double csum = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        rsum[r] += t[r] * xJ;
        csum += t[r] * __shfl_sync(FULL, xI_lane, r);
      }
      if (J < I && (!BIG || 32 * J + lane < n)) ys[32 * J + lane] += csum;   // transpose part, one warp per J
      if (PAIR && J2 <= I) {
        const double xJ2 = X(32 * J2 + lane);
        double csum2 = 0.0;
#pragma unroll
        for (int r = 0; r < 32; ++r) {
          rsum[r] += t2[r] * xJ2;
          csum2 += t2[r] * __shfl_sync(FULL, xI_lane, r);
        }
        if (J2 < I && (!BIG || 32 * J2 + lane < n)) ys[32 * J2 + lane] += csum2;
      }
    }
    // transpose-reduce rsum across lanes: lane l ends with sum over lanes of rsum[l]
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      const bool up = (lane & s) != 0;
#pragma unroll
      for (int r = 0; r < s; ++r) {
        double send = up ? rsum[r] : rsum[r + s];
        double keep = up ? rsum[r + s] : rsum[r];
        rsum[r] = keep + __shfl_xor_sync(FULL, send, s);
      }
    }
    rowred[warp * 32 + lane] = rsum[0];
    __syncthreads();
    if (warp == 0) {
      double v = 0.0;
#pragma unroll
      for (int w = 0; w < GV_WARPS; ++w) v += rowred[w * 32 + lane];
      if (!BIG || 32 * I + lane < n) ys[32 * I + lane] += v;
    }
    __syncthreads();
  }
  if (!BIG)
    for (int j = tid; j < n; j += blockDim.x) W.out[j] = ys[j];
}

static size_t gemv_smem(int nmax, int warps = GV_WARPS) {
  return (size_t)(2 * ((nmax + 31) / 32) * 32 + warps * 32) * sizeof(double);
}

// split a packed matrix of n into P chunks of tile rows balanced by tile count
// split a packed matrix of n into P chunks of tile rows balanced by cost = tiles + row_cost per tile
// row (the per-row reduction and barriers cost about row_cost tiles of streaming)
static void split_rows(int n, int P, std::vector<std::pair<int, int>> &out, double row_cost = 0.0) {
  int nt = (n + 31) / 32;
  auto cum = [&](int r) { return (double)r * (r + 1) / 2 + row_cost * r; };   // cost of rows [0, r)
  const double total = cum(nt);
  out.clear();
  int r = 0;
  for (int p = 0; p < P && r < nt; ++p) {
    const double target = total * (p + 1) / P;
    int r1 = r;
    while (r1 < nt && cum(r1 + 1) <= target) ++r1;
    if (r1 == r) r1 = r + 1;
    if (p == P - 1) r1 = nt;
    out.push_back({r, r1});
    r = r1;
  }
  while ((int)out.size() < P) out.push_back({nt, nt});
}

// ------------------------------------------------------------------ small kernels of the loop
// direct peer stores (SlotExchange::p2p): local position j's value also goes to every peer
// address routed to j (NVLink stores into the peers' receive areas, overlapping the rest of the
// producing kernel); a stream barrier follows the kernel.  rptr == nullptr: no routes.
__device__ __forceinline__ void peer_store(const int *__restrict__ rptr, double *const *__restrict__ rdst,
                                           int64_t j, double v) {
  if (!rptr) return;
  const int q1 = rptr[j + 1];
  for (int q = rptr[j]; q < q1; ++q) rdst[q][0] = v;
}

// per local subdomain: s_j = sum over the P partial chunks of the packed GEMV (fixed order), plus
// the b0 coupling on the primal coordinates: s_Pi += b~0 p0_i (Eq.(globInt) row 1); and
// q0_i = b~0 . u_Pi^(i) (row 2), written to the rank-local p0 position of q.
__global__ void chunk_sum_b0_kernel(const SubDev *__restrict__ subs, const double *__restrict__ part, int64_t stride,
                                    int P, const double *__restrict__ b0T, const int64_t *__restrict__ loc2x,
                                    const double *__restrict__ p, int64_t p0off, double *sbuf, double *q,
                                    const int *__restrict__ rptr, double *const *__restrict__ rdst) {
  pdl_prologue();
  const SubDev S = subs[blockIdx.y];
  const double p0 = p[p0off + blockIdx.y];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < S.nG; j += gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < P; ++c) v += part[c * stride + S.off_G + j];
    if (j >= S.nd) v += b0T[S.off_Pi + (j - S.nd)] * p0;
    sbuf[S.off_G + j] = v;
    peer_store(rptr, rdst, S.off_G + j, v);
  }
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    double acc = 0.0;
    for (int a = threadIdx.x; a < S.npi; a += 32) acc += b0T[S.off_Pi + a] * p[loc2x[S.off_G + S.nd + a]];
    acc = warp_sum(acc);
    if (threadIdx.x == 0) q[p0off + blockIdx.y] = acc;
  }
}

// out[g] = sum over the CSR sources of g (fixed order: sharers in global subdomain order)
__global__ void gather_src_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                  const double *__restrict__ src, int64_t n, double *out) {
  pdl_prologue();
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t q = ptr[g]; q < ptr[g + 1]; ++q) v += src[idx[q]];
    out[g] = v;
  }
}

// block partial dot products (fixed grid) -> part[blockIdx]
// mask (multi-rank): 1 on the coordinates this rank owns, 0 on ghost copies
__global__ void dot_partial_kernel(const double *__restrict__ a, const double *__restrict__ b,
                                   const double *__restrict__ mask, int64_t n, double *part) {
  __shared__ double red[32];
  double v = 0.0;
  if (mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      v += mask[i] * (a[i] * b[i]);
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      v += a[i] * b[i];
  }
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void dot_final_kernel(const double *__restrict__ part, int nb, double *dst) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) v += part[i];
  v = warp_sum(v);
  if (threadIdx.x == 0) *dst = v;
}

// scal: [0] rz, [1] pq, [2] rr, [3] rz_new, [4] alpha, [5] beta

// p = z + beta p (beta = rz_new / rz); unless first, the last block to finish then records beta and
// rotates rz <- rz_new (every block has read both by then)
__global__ void update_p_kernel(double *p, const double *z, int64_t n, double *scal, int first, double *hist,
                                unsigned *ticket) {
  pdl_prologue();
  if (first) {   // p_0 = z_0 (p holds no previous direction: never read it, it may hold NaN bits)
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      p[i] = z[i];
    return;
  }
  const double beta = scal[3] / scal[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
      const int it = (int)scal[6];   // counts this step already
      if (it >= 1 && it <= 4096) hist[2 * (it - 1) + 1] = beta;
      scal[0] = scal[3];
      *ticket = 0u;
    }
  }
}

// ---- single-launch deterministic reductions: block partials, the last block to finish sums them
// in block order (threadfence + ticket), then resets the ticket for the next use.
__device__ __forceinline__ bool block_reduce_last(double v, double *part, unsigned *ticket, double *dst) {
  __shared__ double red[32];
  __shared__ bool last;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x < 32) {
    __threadfence();
    double t = 0.0;
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) t += ((volatile double *)part)[i];
    t = warp_sum(t);
    if (threadIdx.x == 0) { *dst = t; *ticket = 0u; }
  }
  return last && threadIdx.x == 0;   // the thread that wrote *dst
}

__global__ void dot_kernel(const double *__restrict__ a, const double *__restrict__ b, const double *__restrict__ mask,
                           int64_t n, double *part, unsigned *ticket, double *dst) {
  pdl_prologue();
  double v = 0.0;
  if (mask) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      v += mask[i] * (a[i] * b[i]);
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
      v += a[i] * b[i];
  }
  block_reduce_last(v, part, ticket, dst);
}

// r.z with the coarse tail of z filled on the way: z[n0 + j] = u_c[zmap[j]] (primal and p0 coordinates
// of z = M^-1 r, B7), same arithmetic and order as dot_kernel
__global__ void dot_ztail_kernel(const double *__restrict__ r, double *z, const double *__restrict__ uc,
                                 const int64_t *__restrict__ zmap, int64_t n0, const double *__restrict__ mask,
                                 int64_t n, double *part, unsigned *ticket, double *dst) {
  pdl_prologue();
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double zi;
    if (i >= n0) {
      zi = uc[zmap[i - n0]];
      z[i] = zi;
    } else {
      zi = z[i];
    }
    v += mask ? mask[i] * (r[i] * zi) : r[i] * zi;
  }
  block_reduce_last(v, part, ticket, dst);
}

// one rank (no cross-rank copies): chunk_sum_b0 and gather_src_dot in one pass.  Every copy of an x
// coordinate is formed as chunk_sum_b0 forms it (the P chunk partials in order, then + b~0 p0_i on
// the primal coordinates: bcoef / bsub expand b~0 and the subdomain over the local Gamma positions)
// and the copies are summed as gather_src sums them, so q is bitwise the two-kernel q; the p0 rows
// q0_i = b~0 . u_Pi^(i) by one warp per subdomain as in chunk_sum_b0.  p.q -> dst (its partials in
// another order than gather_src_dot's).
__global__ void chunk_gather_dot_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                        const double *__restrict__ part, int64_t stride, int P,
                                        const double *__restrict__ bcoef, const int *__restrict__ bsub,
                                        const double *__restrict__ p, int64_t p0off, int64_t n, double *q,
                                        const SubDev *__restrict__ subs, int N, const double *__restrict__ b0T,
                                        const int64_t *__restrict__ loc2x, double *dpart, unsigned *ticket,
                                        double *dst) {
  pdl_prologue();
  double acc = 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = blockIdx.x * nw + warp; i < N; i += gridDim.x * nw) {
    const SubDev S = subs[i];
    double a = 0.0;
    for (int t = lane; t < S.npi; t += 32) a += b0T[S.off_Pi + t] * p[loc2x[S.off_G + S.nd + t]];
    a = warp_sum(a);
    if (lane == 0) {
      q[p0off + i] = a;
      acc += p[p0off + i] * a;
    }
  }
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t k = ptr[g]; k < ptr[g + 1]; ++k) {
      const int64_t j = idx[k];
      double t = 0.0;
      for (int c = 0; c < P; ++c) t += part[c * stride + j];
      const int sb = bsub[j];
      if (sb >= 0) t += bcoef[j] * p[p0off + sb];
      v += t;
    }
    q[g] = v;
    acc += p[g] * v;
  }
  block_reduce_last(acc, dpart, ticket, dst);
}

// bcoef / bsub of chunk_gather_dot_kernel: per local Gamma position, b~0 and the subdomain on the
// primal coordinates, 0 / -1 on the dual ones
__global__ void b0_expand_kernel(const SubDev *__restrict__ subs, const double *__restrict__ b0T, double *bcoef,
                                 int *bsub) {
  const SubDev S = subs[blockIdx.x];
  for (int j = threadIdx.x; j < S.nG; j += blockDim.x) {
    const bool prim = j >= S.nd;
    bcoef[S.off_G + j] = prim ? b0T[S.off_Pi + (j - S.nd)] : 0.0;
    bsub[S.off_G + j] = prim ? (int)blockIdx.x : -1;
  }
}

// x += alpha p, r -= alpha q (alpha = rz / pq), fused with the partial of r.r -> dst
// p0 block of the condensed rhs: the compatibility sum_i g0_i = 0 must hold up to
// rounding (checked on the host against acc[1] = sum over all pressure DOFs of |c_j g_pj|, the
// terms g0 is summed from: VB_EINVAL otherwise); remove the rounding (mode 0: local sum and
// abs-sum into acc[0], acc[1]; mode 1: subtract acc[0] / n_total from every entry, reading A30)
__global__ void p0_compat_kernel(double *p0, int n, double *acc, int mode, int n_total, const double *g0abs) {
  if (mode == 0) {
    double v = 0.0, a = 0.0;
    for (int i = threadIdx.x; i < n; i += 32) { v += p0[i]; a += g0abs[i]; }
    v = warp_sum(v);
    a = warp_sum(a);
    if (threadIdx.x == 0) { acc[0] = v; acc[1] = a; }
  } else {
    const double mean = *acc / n_total;
    for (int i = threadIdx.x; i < n; i += 32) p0[i] -= mean;
  }
}

// |b_0^(i) x_Gamma^(i)| per local subdomain (reported on VB_EBREAKDOWN; b~0 vanishes
// on the dual coordinates, so only the primal ones enter), one warp per subdomain; the max over
// subdomains by an atomic max on the bit patterns (order-independent for non-negative doubles; out[0]
// zeroed before the launch)
__global__ void flux_violation_kernel(const SubDev *__restrict__ subs, int N, const double *__restrict__ b0T,
                                      const int64_t *__restrict__ loc2x, const double *__restrict__ x,
                                      double *out) {
  const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (i >= N) return;
  const SubDev S = subs[i];
  double acc = 0.0;
  for (int a = lane; a < S.npi; a += 32) acc += b0T[S.off_Pi + a] * x[loc2x[S.off_G + S.nd + a]];
  acc = warp_sum(acc);
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long *>(out), (unsigned long long)__double_as_longlong(fabs(acc)));
}

// scal: [0] rz [1] pq [2] rr [3] rz_new [4] r0n [5] rtol*r0n [6] it [7] status [8] maxit
//  status: 0 running, 1 converged, 2 breakdown (p.Sp <= 0 or r.z <= 0), 3 maxit
__global__ void pcg_init_kernel(double *scal, double rtol, int maxit) {
  const double r0n = sqrt(scal[2]);
  scal[4] = r0n; scal[5] = rtol * r0n; scal[6] = 0.0; scal[8] = maxit;
  scal[7] = (r0n <= rtol * r0n) ? 1.0 : (maxit <= 0 ? 3.0 : 0.0);
}

__device__ void pcg_check(double *scal, double *hist, cudaGraphConditionalHandle hw, int use_graph) {
  const double rz = scal[0], pq = scal[1];
  int it = (int)scal[6];
  double status = 0.0;
  if (!(pq > 0) || !(rz > 0)) {
    status = 2.0;
  } else {
    if (it < 4096) hist[2 * it] = rz / pq;
    ++it;
    scal[6] = it;
    if (sqrt(scal[2]) <= scal[5]) status = 1.0;
    else if (it >= (int)scal[8]) status = 3.0;
  }
  scal[7] = status;
  if (use_graph) cudaGraphSetConditional(hw, status == 0.0 ? 1u : 0u);
}

__global__ void pcg_check_kernel(double *scal, double *hist, cudaGraphConditionalHandle hw, int use_graph) {
  pdl_prologue();
  pcg_check(scal, hist, hw, use_graph);
}

// check >= 0: one rank -- the last block also runs the stopping test (check = use_graph)
__global__ void update_xr_rr_kernel(double *x, double *r, const double *p, const double *q, const double *mask,
                                    int64_t n, double *scal, double *part, unsigned *ticket, double *dst,
                                    double *hist, cudaGraphConditionalHandle hw, int check) {
  pdl_prologue();
  const double alpha = scal[0] / scal[1];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    v += mask ? mask[i] * (ri * ri) : ri * ri;
  }
  if (block_reduce_last(v, part, ticket, dst) && check >= 0) pcg_check(scal, hist, hw, check);
}

// q[g] = sum over the CSR sources of g, fused with the partial of p.q (C3 after the launch)
__global__ void gather_src_dot_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                      const double *__restrict__ src, int64_t n, double *out,
                                      const double *__restrict__ p, const double *__restrict__ mask, int64_t n_all,
                                      double *part, unsigned *ticket, double *dst) {
  pdl_prologue();
  double acc = 0.0;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n_all; g += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (g < n) {
      for (int64_t q = ptr[g]; q < ptr[g + 1]; ++q) v += src[idx[q]];
      out[g] = v;
    } else {
      v = out[g];      // the p0 rows, written by chunk_sum_b0
    }
    acc += mask ? mask[g] * (p[g] * v) : p[g] * v;
  }
  block_reduce_last(acc, part, ticket, dst);
}

// c_i = Phi^_i^T r_i = Phi_i^T D^T r_i (coarse rhs pieces, Phi^ = D Phi, r_i = the dual coordinates of
// subdomain i gathered from r): phit_split CTAs per subdomain (4 at 512 subdomains, more when there
// are few large subdomains), warp per primal column
__global__ void __launch_bounds__(256) phit_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Phi,
                            const int64_t *__restrict__ loc2x, const double *__restrict__ r, double *cpart) {
  pdl_prologue();
  extern __shared__ double x[];
  const SubDev S = subs[blockIdx.y];
  const double *F = Phi + S.off_Phi;
  for (int j = threadIdx.x; j < S.nd; j += blockDim.x) x[j] = r[loc2x[S.off_G + j]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int a = blockIdx.x * nw + warp; a < S.npi; a += gridDim.x * nw) {
    const double *col = F + (int64_t)a * S.nd;
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
    int j = lane;
    for (; j + 96 < S.nd; j += 128) {
      v0 += col[j] * x[j]; v1 += col[j + 32] * x[j + 32]; v2 += col[j + 64] * x[j + 64]; v3 += col[j + 96] * x[j + 96];
    }
    for (; j < S.nd; j += 32) v0 += col[j] * x[j];
    double v = warp_sum((v0 + v1) + (v2 + v3));
    if (lane == 0) cpart[S.off_Pi + a] = v;
  }
}

// p0 projections of the coarse problem (gauge sum vol_i p0_i = 0, A5):
// mode 0 (input):  rc_p0 -= vol * (sum rc_p0) / sum vol ;  mode 1 (output): uc_p0 -= (vol . uc_p0)/sum vol
__global__ void coarse_p0_project_kernel(const double *__restrict__ vol, int N, double *v, int mode) {
  pdl_prologue();
  __shared__ double red[32];
  double a = 0.0, w = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    a += mode == 0 ? v[i] : vol[i] * v[i];
    w += vol[i];
  }
  a = warp_sum(a); w = warp_sum(w);
  __shared__ double ra[32], rw[32];
  if ((threadIdx.x & 31) == 0) { ra[threadIdx.x >> 5] = a; rw[threadIdx.x >> 5] = w; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0, Wt = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { A += ra[q]; Wt += rw[q]; }
    red[0] = A / Wt;
  }
  __syncthreads();
  const double mean = red[0];
  for (int i = threadIdx.x; i < N; i += blockDim.x) v[i] -= mode == 0 ? vol[i] * mean : mean;
}

// coarse extension DPhi_i u_Pi^(i) of subdomain i (thread per row of column-major DPhi, 4
// accumulators): runs on the coarse stream right after the coarse solve, concurrently with the
// local dual GEMV, so its DPhi read leaves the critical path
__global__ void __launch_bounds__(128) coarse_ext_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Phi,
                              const int64_t *__restrict__ pi_glob, const double *__restrict__ uc, double *wc) {
  pdl_prologue();
  const SubDev S = subs[blockIdx.y];
  const double *F = Phi + S.off_Phi;
  extern __shared__ double us[];
  for (int a = threadIdx.x; a < S.npi; a += blockDim.x) us[a] = uc[pi_glob[S.off_Pi + a]];
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S.nd) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int a = 0;
  for (; a + 3 < S.npi; a += 4) {
    a0 += F[j + (int64_t)a * S.nd] * us[a];
    a1 += F[j + (int64_t)(a + 1) * S.nd] * us[a + 1];
    a2 += F[j + (int64_t)(a + 2) * S.nd] * us[a + 2];
    a3 += F[j + (int64_t)(a + 3) * S.nd] * us[a + 3];
  }
  for (; a < S.npi; ++a) a0 += F[j + (int64_t)a * S.nd] * us[a];
  wc[S.off_Dv + j] = (a0 + a1) + (a2 + a3);
}

// one rank (no cross-rank copies): local2 and the entity sum in one pass -- z_e[i] = sum over the
// sharer slots q (EntitySum order) of (sum over the P chunks of y[off_q + i]) + wc[off_q + i], the
// same additions in the same order as local2_kernel followed by entity_sum_kernel (bitwise equal)
__global__ void local2_entity_sum_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ off,
                                         const int64_t *__restrict__ out_off, const int *__restrict__ len,
                                         const double *__restrict__ part, int64_t part_stride, int P,
                                         const double *__restrict__ wc, double *out) {
  pdl_prologue();
  const int e = blockIdx.x;
  const int n = len[e];
  const int64_t q0 = ptr[e], q1 = ptr[e + 1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = 0.0;
    for (int64_t q = q0; q < q1; ++q) {
      const int64_t j = off[q] + i;
      double t = 0.0;
      for (int c = 0; c < P; ++c) t += part[c * part_stride + j];
      v += t + wc[j];
    }
    out[out_off[e] + i] = v;
  }
}

// t_i = sum_chunks y_i + DPhi_i u_Pi^(i) = D (S_DD^-1 D^T r_i + Phi_i u_Pi^(i)), the scaled
// extension product of subdomain i (its coarse part from coarse_ext_kernel)
__global__ void local2_kernel(const double *__restrict__ part, int64_t part_stride, int P,
                              const double *__restrict__ wc, int64_t n, double *w,
                              const int *__restrict__ rptr, double *const *__restrict__ rdst) {
  pdl_prologue();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < P; ++c) v += part[c * part_stride + j];
    const double t = v + wc[j];
    w[j] = t;
    peer_store(rptr, rdst, j, t);
  }
}

// ------------------------------------------------------------------ B0 / B8
// B0 (GEMV form): b_D = [b_I ; Pi^T b_P] and g0_i = c^T b_P (p0 rhs, A5)
__global__ void rhs_D_kernel(const SubDev *__restrict__ subs, const int64_t *__restrict__ Ifree,
                             const int64_t *__restrict__ Pglob, const double *__restrict__ cvec,
                             const double *__restrict__ mvec, const double *__restrict__ rhs, int64_t nvf,
                             double *bD, double *g0, double *g0abs) {
  __shared__ double red[2][32];
  const SubDev S = subs[blockIdx.x];
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  double *b = bD + S.off_Dn;
  for (int j = tid; j < S.nI; j += blockDim.x) b[j] = rhs[Ifree[S.off_I + j]];
  double s = 0.0, sa = 0.0;
  for (int a = tid; a < S.nP; a += blockDim.x) {
    const double t = cvec[S.off_P + a] * rhs[nvf + Pglob[S.off_P + a]];
    s += t;
    sa += fabs(t);
  }
  s = warp_sum(s);
  sa = warp_sum(sa);
  if ((tid & 31) == 0) { red[0][tid >> 5] = s; red[1][tid >> 5] = sa; }
  __syncthreads();
  double g = 0.0, ga = 0.0;
  for (int w = 0; w < nw; ++w) { g += red[0][w]; ga += red[1][w]; }
  if (tid == 0) { g0[blockIdx.x] = g; g0abs[blockIdx.x] = ga; }
  for (int a = tid; a < S.nP; a += blockDim.x)
    b[S.nI + a] = rhs[nvf + Pglob[S.off_P + a]] - mvec[S.off_P + a] * g / S.vol;
}

// B0 / B8 coupling blocks applied element by element (no dense K_GD K_DD^-1 is stored): the
// coupling of the assembled, pressure-projected subdomain matrix (assemble_kernel) is
//   K_GI = sum_K A^K[G, I],   K_GP = sum_K B^K[P, G]^T - b0 m^T / vol   (the Pi^T projection of the
//   pressure rows; b0 = c^T B[P, G] is the stored flux row), K_DG = K_GD^T.
// MODE 0 (B0): zG = -(K_GI x_I + K_GP x_P)   with x_D = K_DD^-1 b_D  (= -K_GD K_DD^-1 b_D)
// MODE 1 (B8): t  = [K_IG u_G ; K_PG u_G]    with u_G gathered from the free-DOF vector
// Three deterministic passes: the per-subdomain projection scalar (m . x_P or b0 . u_G), the element
// rows (warp per row, one CTA per cell, into a per-(cell, row) buffer), and a gather of each output
// row over its (cell, row) contributions in cell order (CSR built on the host) with the projection.
template <int MODE>
__global__ void coupling_scalar_kernel(const SubDev *__restrict__ subs, const double *__restrict__ mvec,
                                       const double *__restrict__ b0all, const double *__restrict__ xin,
                                       const int64_t *__restrict__ Gfree, double *scal) {
  __shared__ double red[32];
  const SubDev S = subs[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double v = 0.0;
  if (MODE == 0)
    for (int a = threadIdx.x; a < S.nP; a += blockDim.x) v += mvec[S.off_P + a] * xin[S.off_Dn + S.nI + a];
  else
    for (int g = threadIdx.x; g < S.nG; g += blockDim.x) v += b0all[S.off_G + g] * xin[Gfree[S.off_G + g]];
  v = warp_sum(v);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += red[w];
    scal[blockIdx.x] = t / S.vol;
  }
}

template <int MODE>
__global__ void __launch_bounds__(128) coupling_cell_kernel(
    const int *__restrict__ cell_sub, const SubDev *__restrict__ subs, const int *__restrict__ cell_loc,
    const int *__restrict__ cell_nv, const double *__restrict__ elA, const double *__restrict__ elB, int nvmax, int np,
    const double *__restrict__ xin, const int64_t *__restrict__ Gfree, double *ycell) {
  const int cell = blockIdx.x;
  const SubDev S = subs[cell_sub[cell]];
  const int nI = S.nI, nIP = S.nI + S.nP;
  const int nv = cell_nv[cell], stride = nvmax + np;
  const int *loc = cell_loc + (int64_t)cell * stride;
  const double *A = elA + (int64_t)cell * nvmax * nvmax;
  const double *B = elB + (int64_t)cell * np * nvmax;
  const double *xD = xin + S.off_Dn;
  double *y = ycell + (int64_t)cell * stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int a = warp; a < nv + np; a += nw) {
    const bool pres = a >= nv;
    const int la = pres ? loc[nvmax + (a - nv)] : loc[a];
    double v = 0.0;
    if (MODE == 0) {            // interface velocity rows
      if (pres || la < nIP) continue;
      for (int b = lane; b < nv; b += 32) {
        const int lb = loc[b];
        if (lb >= 0 && lb < nI) v += A[(int64_t)a * nv + b] * xD[lb];
      }
      for (int p = lane; p < np; p += 32) v += B[(int64_t)p * nv + a] * xD[loc[nvmax + p]];
    } else {                    // interior velocity rows and pressure rows
      if (!pres && (la < 0 || la >= nI)) continue;
      const double *row = pres ? B + (int64_t)(a - nv) * nv : A + (int64_t)a * nv;
      for (int b = lane; b < nv; b += 32) {
        const int lb = loc[b];
        if (lb >= nIP) v += row[b] * __ldg(xin + __ldg(Gfree + S.off_G + (lb - nIP)));
      }
    }
    v = warp_sum(v);
    if (lane == 0) y[pres ? nvmax + (a - nv) : a] = v;
  }
}

// out[r] = sum of its (cell, row) contributions in order, with the projection and (MODE 0) the sign
template <int MODE>
__global__ void coupling_gather_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ src,
                                       const int *__restrict__ rsub, const SubDev *__restrict__ subs,
                                       const double *__restrict__ ycell, const double *__restrict__ mvec,
                                       const double *__restrict__ b0all, const double *__restrict__ scal, int64_t n,
                                       double *out) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t q = ptr[r]; q < ptr[r + 1]; ++q) v += ycell[src[q]];
    const int i = rsub[r];
    if (MODE == 0) {
      out[r] = -(v - b0all[r] * scal[i]);
    } else {
      const SubDev S = subs[i];
      const int64_t l = r - S.off_Dn;
      out[r] = l >= S.nI ? v - mvec[S.off_P + (l - S.nI)] * scal[i] : v;
    }
  }
}

// B8: x_D = y_D - sum over the GEMV chunks of K_DD^-1 t (fixed chunk order)
__global__ void xd_update_kernel(double *xD, const double *__restrict__ part, int64_t stride, int P, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int c = 0; c < P; ++c) v += part[c * stride + i];
    xD[i] -= v;
  }
}

// B8: pressure p = p_aug - c (m^T p_aug)/vol + p0 c (Q_I projection + Q_0 part); scatter to x
__global__ void xout_kernel(const SubDev *__restrict__ subs, const double *__restrict__ xD,
                            const int64_t *__restrict__ Ifree, const int64_t *__restrict__ Pglob,
                            const double *__restrict__ cvec, const double *__restrict__ mvec,
                            const double *__restrict__ p0, int64_t nvf, double *xout) {
  __shared__ double red[32];
  const SubDev S = subs[blockIdx.x];
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  const double *t = xD + S.off_Dn;
  double s = 0.0;
  for (int a = tid; a < S.nP; a += blockDim.x) s += mvec[S.off_P + a] * t[S.nI + a];
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  double mp = 0.0;
  for (int w = 0; w < nw; ++w) mp += red[w];
  const double shift = p0[blockIdx.x] - mp / S.vol;
  for (int j = tid; j < S.nI; j += blockDim.x) xout[Ifree[S.off_I + j]] = t[j];
  for (int a = tid; a < S.nP; a += blockDim.x) xout[nvf + Pglob[S.off_P + a]] = t[S.nI + a] + shift * cvec[S.off_P + a];
}

// per entity: r_x = T_e^T ghat_e, ghat_e = b_e + sum_m zG^(m)[e] (entity-major, gathered before)
__global__ void gamma_rhs_kernel(const EntDev *__restrict__ ents, const double *__restrict__ T,
                                 const double *__restrict__ ghat, int64_t NDelta, double *r) {
  const EntDev E = ents[blockIdx.x];
  const int n = E.n;
  const double *gh = ghat + E.off_gam;
  const double *Te = T + E.off_T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw) {
    double v = 0.0;
    for (int j = lane; j < n; j += 32) v += Te[j + (int64_t)i * n] * gh[j];
    v = warp_sum(v);
    if (lane == 0) {
      if (i < E.nd) r[E.off_xd + i] = v;
      else r[NDelta + E.off_pl + (i - E.nd)] = v;
    }
  }
}

// per entity: u_e = T_e x_e (back to original coordinates) -> x_free (interface entries)
__global__ void gamma_back_kernel(const EntDev *__restrict__ ents, const int64_t *__restrict__ gam_free,
                                  const double *__restrict__ T, const double *__restrict__ x, int64_t NDelta,
                                  double *gam, double *xout) {
  const EntDev E = ents[blockIdx.x];
  const int n = E.n;
  const double *Te = T + E.off_T;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = 0.0;
    for (int i = 0; i < n; ++i) {
      const double xi = i < E.nd ? x[E.off_xd + i] : x[NDelta + E.off_pl + (i - E.nd)];
      v += Te[j + (int64_t)i * n] * xi;
    }
    gam[E.off_gam + j] = v;
    xout[gam_free[E.off_gam + j]] = v;
  }
}

// global zero-mean pressure (Q_{h,0}): p -= c_K * (sum_K vol_K p_K0) / vol_Omega
// acc: [2 * nb block partials | folded (sum vol p0, sum vol)]; nb = the phase-0 grid size
__global__ void pressure_mean_kernel(const double *__restrict__ cellgeo, const int64_t *__restrict__ gid,
                                     int geo_stride, int np, int64_t nK, double *p, int phase, double *acc,
                                     int nb) {
  if (phase == 0) {
    __shared__ double red[2][32];
    double a = 0.0, w = 0.0;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nK; K += (int64_t)gridDim.x * blockDim.x) {
      const double vol = cellgeo[K * geo_stride];
      a += vol * p[gid[K] * np];
      w += vol;
    }
    a = warp_sum(a); w = warp_sum(w);
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = a; red[1][threadIdx.x >> 5] = w; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double A = 0, Wt = 0;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { A += red[0][q]; Wt += red[1][q]; }
      acc[2 * blockIdx.x] = A; acc[2 * blockIdx.x + 1] = Wt;
    }
  } else if (phase == 1) {   // fold the block partials: acc[2 nb], acc[2 nb + 1]
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      double A = 0, Wt = 0;
      for (int b = 0; b < nb; ++b) { A += acc[2 * b]; Wt += acc[2 * b + 1]; }
      acc[2 * nb] = A; acc[2 * nb + 1] = Wt;
    }
  } else {
    const double mean = acc[2 * nb] / acc[2 * nb + 1];
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nK; K += (int64_t)gridDim.x * blockDim.x)
      for (int a = 0; a < np; ++a) p[gid[K] * np + a] -= mean * cellgeo[K * geo_stride + 5 + a];
  }
}

// ------------------------------------------------------------------ K7: element-by-element operator
// y_K = [A_K B_K^T; B_K 0] x_K per element, then a deterministic per-DOF gather-sum.
// K7 on packed symmetric element matrices: A^K stored as its lower triangle row by row
// (nv (nv + 1) / 2 doubles: the algorithmic bytes of SURVEY §8(d), half of the dense A^K).
// One CTA per cell, K7_WARPS warps, rows interleaved over the warps.  Warp w reads row i once
// (coalesced over j <= i) and uses it twice: y_i += A_ij x_j (row part, warp sum) and
// t_w[j] += A_ij x_i for j < i (transpose part, lane-owned entries of the warp's shared-memory
// partial vector t_w).  y_i = row_i + sum_w t_w[i] in fixed warp order: no atomics, deterministic.
constexpr int K7_WARPS = 4;
__global__ void __launch_bounds__(K7_WARPS * 32) elem_apply_packed_kernel(
    const double *__restrict__ elAp, int64_t slotA, const double *__restrict__ elB,
    const int64_t *__restrict__ l2g, const int64_t *__restrict__ vel2free, const int *__restrict__ cell_nv,
    const int64_t *__restrict__ gid, int nvmax, int np, int64_t nK, int64_t nvf, const double *__restrict__ x,
    double *yel) {
  const int64_t K = blockIdx.x;
  if (K >= nK) return;
  extern __shared__ double k7s[];
  double *xs = k7s;                          // nv + np gathered inputs
  double *rowv = xs + nvmax + np;            // row parts
  double *tw = rowv + nvmax;                 // K7_WARPS partial transpose vectors (nvmax each)
  const int nv = cell_nv[K];
  const int stride = nvmax + np;
  for (int j = threadIdx.x; j < nv; j += blockDim.x) {
    const int64_t f = vel2free[l2g[K * nvmax + j]];
    xs[j] = f >= 0 ? x[f] : 0.0;
  }
  for (int a = threadIdx.x; a < np; a += blockDim.x) xs[nv + a] = x[nvf + gid[K] * np + a];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double *t = tw + warp * nvmax;
  for (int j = lane; j < nv; j += 32) t[j] = 0.0;
  __syncthreads();
  const double *A = elAp + K * slotA;
  const double *B = elB + K * np * nvmax;
  for (int i = warp; i < nv; i += K7_WARPS) {
    const double *row = A + (int64_t)i * (i + 1) / 2;
    const double xi = xs[i];
    double v = 0.0;
    for (int j = lane; j <= i; j += 32) {
      const double a = __ldg(row + j);
      v += a * xs[j];
      if (j < i) t[j] += a * xi;
    }
    for (int q = lane; q < np; q += 32) v += B[(int64_t)q * nv + i] * xs[nv + q];
    v = warp_sum(v);
    if (lane == 0) rowv[i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    double v = rowv[i];
    for (int w = 0; w < K7_WARPS; ++w) v += tw[w * nvmax + i];
    yel[K * stride + i] = v;
  }
  for (int q = warp; q < np; q += K7_WARPS) {   // pressure rows: B x
    double v = 0.0;
    for (int j = lane; j < nv; j += 32) v += B[(int64_t)q * nv + j] * xs[j];
    v = warp_sum(v);
    if (lane == 0) yel[K * stride + nvmax + q] = v;
  }
}

// K7 with the element matrices staged by the bulk-copy engine: one cp.async.bulk of the cell's packed
// lower triangle (~26 KB for k = 2 hexahedra) and one of B^K into shared memory per CTA, signalled
// on an mbarrier, while the threads gather the cell's inputs; rows then come from shared memory
// (the streaming kernel above waits on one global-memory row segment at a time), a lane pair per
// row summing its row and its column of the lower triangle over interleaved columns (round 1-2:
// one thread per row, a serial 85-term FMA chain, 0.52 of HBM on c5).  Needs
// (nv_max (nv_max+1)/2 + np nv_max) doubles of shared memory: used while that fits (k = 2
// hexahedra and small polyhedra).
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// K7B_TPR threads per row (default 2, CTA of 256; VB_K7_TPR / VB_K7_THREADS experiment knobs)
template <int K7B_TPR>
__global__ void __launch_bounds__(512) elem_apply_bulk_kernel(
    const double *__restrict__ elAp, int64_t slotA, const double *__restrict__ elB,
    const int64_t *__restrict__ l2g, const int64_t *__restrict__ vel2free, const int *__restrict__ cell_nv,
    const int64_t *__restrict__ gid, int nvmax, int np, int64_t nK, int64_t nvf, const double *__restrict__ x,
    double *yel) {
  const int64_t K = blockIdx.x;
  if (K >= nK) return;
  extern __shared__ __align__(16) double k7b[];
  __shared__ __align__(8) uint64_t bar;
  const int nv = cell_nv[K];
  const int64_t lenA = (int64_t)nv * (nv + 1) / 2;
  const int lenA16 = (int)((lenA + 1) & ~1LL);            // 16-byte multiple
  double *As = k7b;                                      // packed lower triangle
  double *Bs = As + ((slotA + 1) & ~1LL);                // np x nv
  double *xs = Bs + (int64_t)np * nvmax;                 // nv + np inputs
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned bA = 8u * lenA16, bB = 8u * (unsigned)(np * nv);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bA + bB)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(As)),
                 "l"(elAp + K * slotA), "r"(bA), "r"(smem_u32(&bar))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(Bs)),
                 "l"(elB + K * np * nvmax), "r"(bB), "r"(smem_u32(&bar))
                 : "memory");
  }
  const int stride = nvmax + np;
  for (int j = threadIdx.x; j < nv; j += blockDim.x) {   // overlaps with the bulk copies
    const int64_t f = vel2free[l2g[K * nvmax + j]];
    xs[j] = f >= 0 ? x[f] : 0.0;
  }
  for (int a = threadIdx.x; a < np; a += blockDim.x) xs[nv + a] = x[nvf + gid[K] * np + a];
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(&bar))
      : "memory");
  __syncthreads();
  // K7B_TPR threads per row (lane pairs, interleaved columns, two accumulators each -> four
  // independent FMA chains per row), partials combined in a fixed order by shuffles:
  // y_i = sum_{j <= i} L_ij x_j + sum_{k > i} L_ki x_k + (B^T p)_i
  const int sub = threadIdx.x % K7B_TPR, rpp = blockDim.x / K7B_TPR, nrows = nv + np;
  for (int base = 0; base < nrows; base += rpp) {       // uniform trip count (full-mask shuffles)
    const int i = base + threadIdx.x / K7B_TPR;
    double v0 = 0.0, v1 = 0.0;
    if (i < nv) {
      const double *row = As + (int64_t)i * (i + 1) / 2;
      int j = sub;
      for (; j + K7B_TPR <= i; j += 2 * K7B_TPR) {
        v0 += row[j] * xs[j];
        v1 += row[j + K7B_TPR] * xs[j + K7B_TPR];
      }
      if (j <= i) v0 += row[j] * xs[j];
      int k = i + 1 + sub;
      const double *col = As + (int64_t)k * (k + 1) / 2 + i;   // L_ki, k > i: next at + (k + 1), + (k + 2), ...
      for (; k + K7B_TPR < nv; k += 2 * K7B_TPR) {
        const double *col1 = col + (int64_t)K7B_TPR * k + K7B_TPR * (K7B_TPR + 1) / 2;
        v0 += col[0] * xs[k];
        v1 += col1[0] * xs[k + K7B_TPR];
        col = col1 + (int64_t)K7B_TPR * (k + K7B_TPR) + K7B_TPR * (K7B_TPR + 1) / 2;
      }
      if (k < nv) v0 += col[0] * xs[k];
      for (int q = sub; q < np; q += K7B_TPR) v1 += Bs[q * nv + i] * xs[nv + q];
    } else if (i < nrows) {
      const double *brow = Bs + (i - nv) * nv;
      int j = sub;
      for (; j + K7B_TPR < nv; j += 2 * K7B_TPR) {
        v0 += brow[j] * xs[j];
        v1 += brow[j + K7B_TPR] * xs[j + K7B_TPR];
      }
      if (j < nv) v0 += brow[j] * xs[j];
    }
    double v = v0 + v1;
#pragma unroll
    for (int o = K7B_TPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (sub == 0 && i < nrows) yel[K * stride + (i < nv ? i : nvmax + (i - nv))] = v;
  }
}

// K7, persistent and warp specialised (round 2, the default while two stages fit in shared
// memory): the one-cell-per-CTA kernel above moves 3.1 TB/s on c5 whatever its compute shape
// (profiles/r02z_k7_sweep.txt) -- every CTA pays launch, the l2g -> vel2free -> x gather chain, one
// bulk-copy round trip and its compute back to back.  Here each CTA walks cells
// blockIdx.x, + gridDim.x, ... through a ring of nst stages [A^K packed | B^K | inputs]: the
// cells' inputs are gathered beforehand by elem_xgather_kernel into contiguous per-cell vectors (a
// producer that walked the gather chain itself, one cell at a time, capped the first version at
// 5 us per cell and CTA); one producer lane waits for a free stage and issues three cp.async.bulk
// copies (complete_tx on the stage's full barrier); K7P_CONSUMERS threads wait on the full
// barrier, compute the rows as above (lane pairs) and release the stage through its empty barrier.
constexpr int K7P_MAXST = 8;   // consumers = blockDim.x - 32 (the last warp produces)
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}

// one lane's share (columns sub, sub + TPR, ...) of row i of [A^K B^K^T; B^K 0] x from the staged cell:
// four accumulators, loads of four terms issued ahead of their FMAs (shared-memory latency, not
// FP64 throughput, bounds this loop: 8 consumer warps took 2 us per cell with a single chain)
template <int TPR>
__device__ __forceinline__ double k7_row_share(const double *As, const double *Bs, const double *xs, int i, int nv,
                                               int np, int sub) {
  double v0 = 0.0, v1 = 0.0, v2 = 0.0, v3 = 0.0;
  if (i < nv) {
    const double *row = As + ((i * (i + 1)) >> 1);
    int j = sub;
    for (; j + 3 * TPR <= i; j += 4 * TPR) {
      const double a0 = row[j], a1 = row[j + TPR], a2 = row[j + 2 * TPR], a3 = row[j + 3 * TPR];
      const double x0 = xs[j], x1 = xs[j + TPR], x2 = xs[j + 2 * TPR], x3 = xs[j + 3 * TPR];
      v0 += a0 * x0, v1 += a1 * x1, v2 += a2 * x2, v3 += a3 * x3;
    }
    for (; j <= i; j += TPR) v0 += row[j] * xs[j];
    int k = i + 1 + sub;
    const double *col = As + i;
    for (; k + 3 * TPR < nv; k += 4 * TPR) {
      const int k1 = k + TPR, k2 = k + 2 * TPR, k3 = k + 3 * TPR;
      const double a0 = col[(k * (k + 1)) >> 1], a1 = col[(k1 * (k1 + 1)) >> 1], a2 = col[(k2 * (k2 + 1)) >> 1],
                   a3 = col[(k3 * (k3 + 1)) >> 1];
      const double x0 = xs[k], x1 = xs[k1], x2 = xs[k2], x3 = xs[k3];
      v0 += a0 * x0, v1 += a1 * x1, v2 += a2 * x2, v3 += a3 * x3;
    }
    for (; k < nv; k += TPR) v1 += col[(k * (k + 1)) >> 1] * xs[k];
    for (int a = sub; a < np; a += TPR) v2 += Bs[a * nv + i] * xs[nv + a];
  } else if (i < nv + np) {
    const double *brow = Bs + (i - nv) * nv;
    int j = sub;
    for (; j + 3 * TPR < nv; j += 4 * TPR) {
      const double a0 = brow[j], a1 = brow[j + TPR], a2 = brow[j + 2 * TPR], a3 = brow[j + 3 * TPR];
      const double x0 = xs[j], x1 = xs[j + TPR], x2 = xs[j + 2 * TPR], x3 = xs[j + 3 * TPR];
      v0 += a0 * x0, v1 += a1 * x1, v2 += a2 * x2, v3 += a3 * x3;
    }
    for (; j < nv; j += TPR) v0 += brow[j] * xs[j];
  }
  return (v0 + v1) + (v2 + v3);
}

__global__ void elem_xgather_kernel(const int64_t *__restrict__ l2g, const int64_t *__restrict__ vel2free,
                                    const int *__restrict__ cell_nv, const int64_t *__restrict__ gid, int nvmax,
                                    int np, int64_t nK, int64_t nvf, int xstride, const double *__restrict__ x,
                                    double *__restrict__ xel) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nK * xstride;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t K = e / xstride;
    const int j = (int)(e - K * xstride), nv = cell_nv[K];
    double v = 0.0;
    if (j < nv) {
      const int64_t f = vel2free[l2g[K * nvmax + j]];
      if (f >= 0) v = x[f];
    } else if (j < nv + np) {
      v = x[nvf + gid[K] * np + (j - nv)];
    }
    xel[e] = v;
  }
}

template <int K7P_TPR>
__global__ void __launch_bounds__(544) elem_apply_pipe_kernel(
    const double *__restrict__ elAp, int64_t slotA, const double *__restrict__ elB,
    const double *__restrict__ xel, const int *__restrict__ cell_nv, int nvmax, int np, int64_t nK, double *yel,
    int nst, int stage_dbl, int nocompute) {
  extern __shared__ __align__(16) double k7b[];
  __shared__ __align__(8) uint64_t full[K7P_MAXST], empty[K7P_MAXST];
  const int offB = (int)((slotA + 1) & ~1LL), offX = offB + ((np * nvmax + 1) & ~1);
  const int stride = nvmax + np, K7P_CONSUMERS = blockDim.x - 32;
  if (threadIdx.x == 0) {
    for (int q = 0; q < nst; ++q) {
      mbar_init(&full[q], 1);                     // the producer lane's expect_tx arrival
      mbar_init(&empty[q], K7P_CONSUMERS / 32);   // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t first = blockIdx.x;
  const int64_t cnt = first < nK ? (nK - first + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x >= K7P_CONSUMERS) {   // producer warp: one lane issues the bulk copies
    if (threadIdx.x != K7P_CONSUMERS || cnt == 0) return;
    const int xstride = (stride + 1) & ~1;
    int nv_next = cell_nv[first];
    for (int64_t n = 0; n < cnt; ++n) {
      const int q = (int)(n % nst);
      const unsigned round = (unsigned)(n / nst);
      const int64_t K = first + n * gridDim.x;
      double *As = k7b + (int64_t)q * stage_dbl, *Bs = As + offB, *xs = As + offX;
      const int nv = nv_next;
      if (n + 1 < cnt) nv_next = cell_nv[K + gridDim.x];   // in flight during the wait below
      mbar_wait(&empty[q], (round & 1u) ^ 1u);             // passes at once in the first round
      const int64_t lenA = (int64_t)nv * (nv + 1) / 2;
      const unsigned bA = 8u * (unsigned)((lenA + 1) & ~1LL), bB = 8u * (unsigned)(np * nv), bX = 8u * xstride;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[q])),
                   "r"(bA + bB + bX)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(As)),
                   "l"(elAp + K * slotA), "r"(bA), "r"(smem_u32(&full[q]))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(Bs)),
                   "l"(elB + K * np * nvmax), "r"(bB), "r"(smem_u32(&full[q]))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(xs)),
                   "l"(xel + K * xstride), "r"(bX), "r"(smem_u32(&full[q]))
                   : "memory");
    }
    return;
  }
  const int sub = threadIdx.x % K7P_TPR, rpp = K7P_CONSUMERS / K7P_TPR;
  int nv_next = cnt > 0 ? cell_nv[first] : 0;
  for (int64_t n = 0; n < cnt; ++n) {
    const int q = (int)(n % nst);
    const unsigned round = (unsigned)(n / nst);
    const int64_t K = first + n * gridDim.x;
    const double *As = k7b + (int64_t)q * stage_dbl, *Bs = As + offB, *xs = As + offX;
    const int nv = nv_next, nrows = nv + np;
    if (n + 1 < cnt) nv_next = cell_nv[K + gridDim.x];   // a global load per cell: one cell ahead, off the critical path
    mbar_wait(&full[q], round & 1u);
    for (int base = 0; base < nrows; base += rpp) {
      const int i = base + threadIdx.x / K7P_TPR;
      double v = nocompute ? xs[0] : k7_row_share<K7P_TPR>(As, Bs, xs, i, nv, np, sub);   // nocompute: load-only probe
#pragma unroll
      for (int o = K7P_TPR / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (sub == 0 && i < nrows) yel[K * stride + (i < nv ? i : nvmax + (i - nv))] = v;
    }
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[q]);
  }
}

// K7, warp-per-row consumers (VB_K7_PIPE=2; cells with nv <= 32 MX): the lane-pair kernel above is
// bound by shared-memory wavefronts (every L_ij is read twice, rows with 2-way bank conflicts, x from
// shared memory: ~1,900 cycles per cell and SM whatever the thread shape).  Here warp w owns rows
// w, w + W, ...: lanes read a row contiguously (conflict free), x_j lives in registers, each L_ij is
// read once and used for y_i (row sum, shuffle reduction, four rows interleaved) and y_j (per-lane
// column partials, summed over the warps in fixed order after one named barrier).
template <int MX, int W>
__global__ void __launch_bounds__(W * 32 + 32, 3) elem_apply_pipe2_kernel(
    const double *__restrict__ elAp, int64_t slotA, const double *__restrict__ elB,
    const double *__restrict__ xel, const int *__restrict__ cell_nv, int nvmax, int np, int64_t nK, double *yel,
    int nst, int stage_dbl) {
  extern __shared__ __align__(16) double k7b[];
  __shared__ __align__(8) uint64_t full[K7P_MAXST], empty[K7P_MAXST];
  const int offB = (int)((slotA + 1) & ~1LL), offX = offB + ((np * nvmax + 1) & ~1);
  constexpr int ncons = W * 32, RW = (32 * MX + W - 1) / W;   // rows per warp, all in registers
  const int stride = nvmax + np;
  double *red = k7b + (int64_t)nst * stage_dbl;   // 2 x [y rows (stride) | W column partial vectors (nvmax each)]
  const int red_dbl = stride + W * nvmax;
  if (threadIdx.x == 0) {
    for (int q = 0; q < nst; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], W);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t first = blockIdx.x;
  const int64_t cnt = first < nK ? (nK - first + gridDim.x - 1) / gridDim.x : 0;
  if (threadIdx.x >= ncons) {   // producer warp: one lane issues the bulk copies
    if (threadIdx.x != ncons || cnt == 0) return;
    const int xstride = (stride + 1) & ~1;
    int nv_next = cell_nv[first];
    for (int64_t n = 0; n < cnt; ++n) {
      const int q = (int)(n % nst);
      const unsigned round = (unsigned)(n / nst);
      const int64_t K = first + n * gridDim.x;
      double *As = k7b + (int64_t)q * stage_dbl, *Bs = As + offB, *xs = As + offX;
      const int nv = nv_next;
      if (n + 1 < cnt) nv_next = cell_nv[K + gridDim.x];
      mbar_wait(&empty[q], (round & 1u) ^ 1u);
      const int64_t lenA = (int64_t)nv * (nv + 1) / 2;
      const unsigned bA = 8u * (unsigned)((lenA + 1) & ~1LL), bB = 8u * (unsigned)(np * nv), bX = 8u * xstride;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[q])),
                   "r"(bA + bB + bX)
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(As)),
                   "l"(elAp + K * slotA), "r"(bA), "r"(smem_u32(&full[q]))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(Bs)),
                   "l"(elB + K * np * nvmax), "r"(bB), "r"(smem_u32(&full[q]))
                   : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_u32(xs)),
                   "l"(xel + K * xstride), "r"(bX), "r"(smem_u32(&full[q]))
                   : "memory");
    }
    return;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int nv_next = cnt > 0 ? cell_nv[first] : 0;
  for (int64_t n = 0; n < cnt; ++n) {
    const int q = (int)(n % nst);
    const unsigned round = (unsigned)(n / nst);
    const int64_t K = first + n * gridDim.x;
    const double *As = k7b + (int64_t)q * stage_dbl, *Bs = As + offB, *xs = As + offX;
    double *ysm = red + (n & 1) * red_dbl, *tw = ysm + stride;
    const int nv = nv_next;
    if (n + 1 < cnt) nv_next = cell_nv[K + gridDim.x];
    mbar_wait(&full[q], round & 1u);
    double xr[MX], yc[MX];
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int j = lane + 32 * m;
      xr[m] = j < nv ? xs[j] : 0.0;
      yc[m] = 0.0;
    }
    double p[RW];   // this warp's row sums (lane partials), reduced together: RW independent shuffle chains
#pragma unroll
    for (int r = 0; r < RW; ++r) {
      const int i = w + r * W;
      p[r] = 0.0;
      if (i < nv) {
        const double *row = As + ((i * (i + 1)) >> 1);
        const double xi = xs[i];
#pragma unroll
        for (int m = 0; m < MX; ++m) {
          const int j = lane + 32 * m;
          if (32 * m <= i && j <= i) {
            const double a = row[j];
            p[r] += a * xr[m];
            if (j < i) yc[m] += a * xi;
          }
        }
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int r = 0; r < RW; ++r) p[r] += __shfl_xor_sync(0xffffffffu, p[r], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int r = 0; r < RW; ++r)
        if (w + r * W < nv) ysm[w + r * W] = p[r];
    }
    for (int a = w; a < np; a += W) {   // pressure rows: (B x_v)_a
      double pb = 0.0;
#pragma unroll
      for (int m = 0; m < MX; ++m) {
        const int j = lane + 32 * m;
        if (j < nv) pb += Bs[a * nv + j] * xr[m];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) pb += __shfl_xor_sync(0xffffffffu, pb, o);
      if (lane == 0) ysm[nv + a] = pb;
    }
#pragma unroll
    for (int m = 0; m < MX; ++m) {
      const int j = lane + 32 * m;
      if (j < nv) tw[w * nvmax + j] = yc[m];
    }
    asm volatile("bar.sync 1, %0;" ::"r"(ncons) : "memory");
    for (int t = threadIdx.x; t < nv + np; t += ncons) {
      double v = ysm[t];
      if (t < nv) {
        double c0 = 0.0, c1 = 0.0;
#pragma unroll
        for (int ww = 0; ww < W; ww += 2) c0 += tw[ww * nvmax + t], c1 += tw[(ww + 1) * nvmax + t];
        double b0 = 0.0, b1 = 0.0;   // np is even (4, 10, 20)
        for (int a = 0; a < np; a += 2) b0 += Bs[a * nv + t] * xs[nv + a], b1 += Bs[(a + 1) * nv + t] * xs[nv + a + 1];
        v += (c0 + c1) + (b0 + b1);
        yel[K * stride + t] = v;
      } else {
        yel[K * stride + nvmax + (t - nv)] = v;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[q]);
  }
}

__global__ void pack_element_lower_kernel(const double *__restrict__ elA, const int *__restrict__ cell_nv, int nvmax,
                                          int64_t slotA, double *elAp) {
  const int64_t K = blockIdx.y;
  const int nv = cell_nv[K];
  const int64_t n = (int64_t)nv * (nv + 1) / 2;
  const double *A = elA + K * (int64_t)nvmax * nvmax;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    // row i, column j <= i of packed index e = i (i + 1) / 2 + j
    int64_t i = (int64_t)((sqrt(8.0 * (double)e + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= e) ++i;
    while (i * (i + 1) / 2 > e) --i;
    const int64_t j = e - i * (i + 1) / 2;
    elAp[K * slotA + e] = A[i * nv + j];
  }
}

// per free DOF: sum of its local cells' contributions (cell order); pressure rows of local cells
__global__ void elem_gather_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                   const int64_t *__restrict__ gid, const double *__restrict__ yel, int64_t nvf,
                                   int64_t nK, int np, int stride, int nvmax, double *y) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nvf + nK * np;
       f += (int64_t)gridDim.x * blockDim.x) {
    if (f < nvf) {
      double v = 0.0;
      for (int64_t q = ptr[f]; q < ptr[f + 1]; ++q) v += yel[idx[q]];
      y[f] = v;
    } else {
      const int64_t pidx = f - nvf, K = pidx / np, a = pidx % np;
      y[nvf + gid[K] * np + a] = yel[K * stride + nvmax + a];
    }
  }
}

// ------------------------------------------------------------------ host side
// out[i] = sum_c part[c][i]: block = 32 outputs x 8 warps (warp w sums chunks w, w+8, ...), then
// the 8 warp partials are added in fixed order.
// distributed coarse: u_c = sum over ranks (in rank order) of the gathered partial vectors
__global__ void rank_sum_vec_kernel(const double *__restrict__ g, int R, int64_t n, double *out) {
  pdl_prologue();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < R; ++r) v += g[r * n + i];
    out[i] = v;
  }
}

// f1 coarse dissection (factor.cu coarse_dissection): root rhs g_S = rc[root] - sum_r t_r (the
// gathered F^T g_I of every rank, rank order), then the gauge projection of its p_0 part (mode 0)
__global__ void cd_root_rhs_kernel(const int64_t *__restrict__ rptr, const int64_t *__restrict__ ridx,
                                   const double *__restrict__ tg, const double *__restrict__ rc,
                                   const int64_t *__restrict__ root, int64_t nroot, double *g) {
  pdl_prologue();
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nroot; j += (int64_t)gridDim.x * blockDim.x) {
    double v = rc[root[j]];
    for (int64_t q = rptr[j]; q < rptr[j + 1]; ++q) v -= tg[ridx[q]];
    g[j] = v;
  }
}

// root solution: gauge projection of its p_0 part (sum vol_i p0_i = 0, mode 1 of
// coarse_p0_project_kernel), then scattered to its global coarse positions (one CTA)
__global__ void cd_root_finish_kernel(const double *__restrict__ vol, int Ng, int64_t nsep, const double *__restrict__ x,
                                      const int64_t *__restrict__ root, int64_t nroot, double *uc) {
  pdl_prologue();
  __shared__ double ra[32], rw[32], mean;
  double a = 0.0, w = 0.0;
  for (int i = threadIdx.x; i < Ng; i += blockDim.x) {
    a += vol[i] * x[nsep + i];
    w += vol[i];
  }
  a = warp_sum(a); w = warp_sum(w);
  if ((threadIdx.x & 31) == 0) { ra[threadIdx.x >> 5] = a; rw[threadIdx.x >> 5] = w; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double A = 0, Wt = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { A += ra[q]; Wt += rw[q]; }
    mean = Ng > 0 ? A / Wt : 0.0;   // Ng = 0: no gauge (Neumann faces)
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < nroot; j += blockDim.x) uc[root[j]] = j >= nsep ? x[j] - mean : x[j];
}

// dissection pass 1 per owned part j (blockIdx.y): the P1 chunk partials of [[E, .], [F^T, 0]] [g_I; 0]
// summed in fixed order, y_I = E g_I to Y, t = F^T g_I to T[j maxS ...]
__global__ void cd_sum_parts_kernel(const CdPart *__restrict__ parts, const double *__restrict__ part1, double *Y,
                                    double *T, int64_t maxS, const double *__restrict__ addT) {
  pdl_prologue();
  const CdPart D = parts[blockIdx.y];
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < D.nloc; a += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < D.P1; ++q) v += part1[D.p1off + q * D.nloc + a];
    if (a < D.nIp) Y[D.yoff + a] = v;
    else T[blockIdx.y * maxS + (a - D.nIp)] = addT ? v + addT[a - D.nIp] : v;   // two levels: + the blocks' part
  }
}

// two levels: the rank-level input from the blocks' t vectors (CSR over level-1 positions, block
// order): X[a] = rc[RS[a]] - sum (a < nRS; the GEMV input [g_RS; 0]); C[q] = sum at S position q
__global__ void cd_l2_input_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                   const double *__restrict__ T1, const double *__restrict__ rc,
                                   const int64_t *__restrict__ RS, int64_t nRS, int64_t nRSp, int64_t nl,
                                   double *X, double *C) {
  pdl_prologue();
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < nl; a += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t k = ptr[a]; k < ptr[a + 1]; ++k) v += T1[idx[k]];
    if (a < nRS) X[a] = rc[RS[a]] - v;
    else if (a >= nRSp) C[a - nRSp] = v;
  }
}

// interior coarse values x_I = y_I - F x_S per owned part (F x_S: the transpose part of the second
// GEMV pass, summed over its chunks in fixed order)
__global__ void cd_interior_kernel(const CdPart *__restrict__ parts, const double *__restrict__ part2,
                                   const double *__restrict__ Y, const int64_t *__restrict__ Iall, double *uc) {
  pdl_prologue();
  const CdPart D = parts[blockIdx.y];
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < D.nI; a += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < D.P2; ++q) v += part2[D.p2off + q * D.nloc + a];
    uc[Iall[D.ioff + a]] = Y[D.yoff + a] - v;
  }
}

__global__ void __launch_bounds__(256) sum_chunks_kernel(const double *__restrict__ part, int64_t stride, int P,
                                                         int64_t n, double *out) {
  pdl_prologue();
  __shared__ double red[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32 + lane;
  double v = 0.0;
  if (i < n)
    for (int c = warp; c < P; c += 8) v += part[c * stride + i];
  red[warp][lane] = v;
  __syncthreads();
  if (warp == 0 && i < n) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w][lane];
    out[i] = s;
  }
}

struct SolveState {
  DBuf<GemvWork> w_op, w_loc, w_c;
  DBuf<GemvWork> w_kd;
  int nw_op = 0, nw_loc = 0, nw_c = 0, nw_kd = 0, max_nd = 1;
  int phit_split = 4;                // CTAs per subdomain of phit_kernel
  bool big_c = false;                // coarse vectors exceed shared memory: BIG GEMV variant
  bool big_op = false, big_loc = false, big_kd = false;   // the same for the subdomain matrices
  bool pair_sub = false;             // subdomain GEMVs with two tiles per warp step (sym_gemv PAIR)
  size_t sm_op = 0, sm_loc = 0, sm_c = 0, sm_ex = 0, sm_kd = 0;
  DBuf<int64_t> xptr, xidx;          // B2: x coordinate <- copies (local s or received), sharer order
  DBuf<int64_t> pptr, pidx;          // B6: global coarse index <- coarse pieces, fixed order
  DBuf<int64_t> cpack, zmap;         // coarse piece packing (r0, owned r_Pi); z tail <- u_c
  DBuf<double> hist, mask, gvol;
  DBuf<double> sx;                   // [s (len_G) | received copies]
  DBuf<double> cbuf, cgath;          // coarse pieces (local), gathered (nranks x cmax)
  DBuf<double> ucp, ucg;             // distributed coarse: this rank's partial u_c; gathered (R x N_c)
  DBuf<double> bcoef;                // one rank: b~0 expanded over the local Gamma positions (chunk_gather_dot)
  DBuf<int> bsub;
  // f1 coarse dissection: GEMV passes over the local packed [[E, .], [F^T, 0]] (pass 1: all tile
  // rows, x = [g_I; 0]; pass 2: the S tile rows, x = [0; x_S]), root rhs / solution
  DBuf<GemvWork> w_cd1, w_cd2;
  int nw_cd1 = 0, nw_cd2 = 0;
  size_t sm_cd = 0;
  bool big_cd = false;
  DBuf<int64_t> cd_map1, cd_map2, cd_Iall, cd_root, cd_rptr, cd_ridx;
  DBuf<double> cd_part1, cd_part2, cd_Y, cd_T, cd_tg, cd_groot, cd_xroot;
  DBuf<CdPart> cd_parts;
  int cd_no = 0;
  int64_t cd_maxloc = 1, cd_maxI = 1;
  // two levels: the blocks' t (T1, stride maxS0), the rank-level GEMV input X2, the blocks' part
  // of the rank's root contribution C, the level-1 passes
  DBuf<double> cd_T1, cd_X2, cd_C, cd2_part1, cd2_part2, cd2_Y;
  DBuf<int64_t> cd2_map2, cd2_RS, cd2_ptr, cd2_idx;
  DBuf<CdPart> cd2_desc;
  DBuf<GemvWork> w_cd21, w_cd22;
  int nw_cd21 = 0, nw_cd22 = 0;
  DBuf<double> gam2, gbuf, hbuf;     // B0: entity-major b_e; [zG | received]; DOF halo receive
  int64_t cmax = 0;
  SlotExchange XS, XE, XB, XH, XR;   // apply_S copies, extension products, B0 zG, DOF halo, rank partials
  EntitySum ESE, ESB, ESR;
  DBuf<int64_t> gh_dst;              // DOF halo: destination free ids of received owner values
  DBuf<int64_t> cp_ptr[2], cp_src[2];   // B0 (zG rows) / B8 (D rows) coupling gathers: (cell, row) slots
  DBuf<int> cp_rsub[2], cell_sub;
  DBuf<double> ycell, cscal;
  int64_t n_gh = 0;
  bool ready = false;
  bool graph_broken = false;
  DBuf<double> g0abs;                // per local subdomain: sum_j |c_j g_pj| (rhs compatibility scale)         // capture/instantiate failed once: host-driven iterations
  DBuf<unsigned> ticket;             // single-launch reductions
  cudaStream_t s2 = nullptr;         // coarse branch of M^-1, concurrent with the local solves
  int prio_hi = 0;                   // its (higher) scheduling priority
  cudaStream_t sg = nullptr;         // stream the iteration graph is captured on and launched on
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // the PCG iteration as a CUDA graph: WHILE(status == 0) { S-part; check; IF(status == 0) M-part }
  cudaGraphExec_t gexec = nullptr;
  bool capturing = false;
  bool pdl = true;                   // programmatic dependent launch inside the PCG step
  // optional per-kernel timing (VB_KERNEL_TIMING=1, host-driven iterations): event pairs per
  // launch category
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_cat;
  int nev = 0;
  ~SolveState() {
    for (auto e : ev) cudaEventDestroy(e);
    if (gexec) cudaGraphExecDestroy(gexec);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (s2) cudaStreamDestroy(s2);
    if (sg) cudaStreamDestroy(sg);
  }
};

// launch with the PDL attribute when enabled (kernels of the PCG step start with pdl_prologue)
template <typename... KArgs, typename... Args>
static void launch_k(const SolveState *st, bool pdl, void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t s,
                     Args &&...args);

template <typename... KArgs, typename... Args>
static void launch_pdl(const SolveState *st, void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t s,
                       Args &&...args) {
  launch_k(st, true, k, g, b, sm, s, std::forward<Args>(args)...);
}

// the first kernel after a cross-stream event wait (fork / join of the coarse branch) is launched
// without the programmatic-serialisation attribute: its launch must wait for the event, not only
// for the previous kernel of its own stream
template <typename... KArgs, typename... Args>
static void launch_after_event(const SolveState *st, void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t s,
                               Args &&...args) {
  launch_k(st, false, k, g, b, sm, s, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
static void launch_k(const SolveState *st, bool pdl, void (*k)(KArgs...), dim3 g, dim3 b, size_t sm, cudaStream_t s,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = sm;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (st->pdl && pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (s == st->s2 && st->prio_hi != 0) {
    // the coarse branch of M^-1 ahead of the queued CTAs of the local GEMV (it is on the critical path)
    at[na].id = cudaLaunchAttributePriority;
    at[na].val.priority = st->prio_hi;
    ++na;
  }
  cfg.attrs = na ? at : nullptr;
  cfg.numAttrs = na;
  VB_CUDA(cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...));
}

// packed GEMV over a subdomain work list; BIG when the vectors do not fit in shared memory
static void run_sub_gemv(const SolveState *st, const GemvWork *w, int nw, size_t sm, bool big, cudaStream_t s) {
  if (nw <= 0) return;
  if (big)
    launch_pdl(st, sym_gemv_kernel<GV_WARPS, true>, dim3(nw), dim3(GV_WARPS * 32), GV_WARPS * 32 * sizeof(double), s, w);
  else if (st->pair_sub)   // two tiles per warp step: twice the loads in flight when smem limits the CTAs per SM
    launch_pdl(st, sym_gemv_kernel<GV_WARPS, false, true>, dim3(nw), dim3(GV_WARPS * 32), sm, s, w);
  else
    launch_pdl(st, sym_gemv_kernel<GV_WARPS>, dim3(nw), dim3(GV_WARPS * 32), sm, s, w);
}

static const char *kCatNames[] = {"sym_gemv S_T (operator, B1)", "sym_gemv S_DD^-1 (local, B5)",
                                  "sym_gemv coarse inverse (B6)", "apply_S total (B1-B2)",
                                  "apply_M total (B4-B7)", "elem_apply K7 (packed element matrices)"};
constexpr int N_CAT = 6;

static void tick(vb_ctx *c, SolveState *st, int cat, bool begin, cudaStream_t strm = nullptr) {
  if (!c->timing) return;
  if (!strm) strm = c->stream;
  if (st->nev + 1 >= (int)st->ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      VB_CUDA(cudaEventCreate(&e));
      st->ev.push_back(e);
      st->ev_cat.push_back(-1);
    }
  }
  VB_CUDA(cudaEventRecord(st->ev[st->nev], strm));
  st->ev_cat[st->nev] = begin ? cat : -1 - cat;
  st->nev++;
}

static void collect_times(vb_ctx *c, SolveState *st) {
  if (!c->timing) return;
  c->ktime_ms.assign(N_CAT, 0.0);
  c->ktime_count.assign(N_CAT, 0);
  VB_CUDA(cudaStreamSynchronize(c->stream));
  int open[N_CAT];
  for (int q = 0; q < N_CAT; ++q) open[q] = -1;
  for (int i = 0; i < st->nev; ++i) {
    const int code = st->ev_cat[i];
    if (code >= 0) { open[code] = i; continue; }
    const int cat = -1 - code;
    if (open[cat] < 0) continue;
    float ms = 0;
    VB_CUDA(cudaEventElapsedTime(&ms, st->ev[open[cat]], st->ev[i]));
    c->ktime_ms[cat] += ms;
    c->ktime_count[cat]++;
    open[cat] = -1;
  }
  st->nev = 0;

}

const char *kernel_time_name(int i) { return (i >= 0 && i < N_CAT) ? kCatNames[i] : ""; }

#ifndef DOT_BLOCKS_CFG
#define DOT_BLOCKS_CFG 296
#endif
constexpr int DOT_BLOCKS = DOT_BLOCKS_CFG;
// scalar slots of w_dots (2 DOT_BLOCKS + 256 doubles) AFTER the block-partial region [0, DOT_BLOCKS)
// that every fused dot's last-block reduction writes
constexpr int W_P0 = 2 * DOT_BLOCKS;            // p0 compatibility: sum, abs-sum
constexpr int W_TRACE = 2 * DOT_BLOCKS + 4;     // VB_PCG_TRACE norms
constexpr int W_FLUX = 2 * DOT_BLOCKS + 6;      // max_i |b0 x_Gamma|
constexpr int W_PM = 2 * DOT_BLOCKS + 8;        // pressure mean: 2 PM_BLOCKS partials + 2 folded
constexpr int PM_BLOCKS = 64;
constexpr double kCompatRel = 1e-8;             // |sum g0| <= kCompatRel * sum |g0|
static_assert(W_PM + 2 * PM_BLOCKS + 2 <= 2 * DOT_BLOCKS + 256, "w_dots scalar slots");

static SolveState *get_state(vb_ctx *c) {
  if (!c->solve_state) c->solve_state = new SolveState();
  return (SolveState *)c->solve_state;
}

// C3: block partials -> rank partial -> fixed-order sum over ranks
static void dot(vb_ctx *c, const double *a, const double *b, int64_t n, double *dst) {
  SolveState *st = get_state(c);
  launch_pdl(st, dot_kernel, dim3(DOT_BLOCKS), dim3(256), 0, c->stream, a, b, c->nranks > 1 ? st->mask.p : nullptr, n, c->w_dots.p,
                                                st->ticket.p, dst);
  allreduce_sum_fixed(c, dst, 1);
}

// rz = r.z after apply_M(..., false): fills z's coarse tail in the same pass (C3 follows)
static void dot_rz(vb_ctx *c, SolveState *st, double *dst) {
  VB_REQUIRE(c->nx - c->n_delta_glob == (int64_t)st->zmap.n || (c->nx == c->n_delta_glob && st->zmap.n <= 1),
             VB_EINVAL, "internal: z tail layout");
  launch_pdl(st, dot_ztail_kernel, dim3(DOT_BLOCKS), dim3(256), 0, c->stream, c->w_r.p, c->w_z.p, c->w_uc.p,
             st->zmap.p, c->n_delta_glob, c->nranks > 1 ? st->mask.p : nullptr, c->nx, c->w_dots.p, st->ticket.p, dst);
  allreduce_sum_fixed(c, dst, 1);
}

static int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)); }

static void apply_S(vb_ctx *c, SolveState *st, bool with_pq = false) {   // q = S^ p  (B1, B2) [+ p.q]
  cudaStream_t s = c->stream;
  tick(c, st, 3, true);
  tick(c, st, 0, true);
  run_sub_gemv(st, st->w_op.p, st->nw_op, st->sm_op, st->big_op, s);
  tick(c, st, 0, false);
  int maxnG = 1;
  for (auto &S : c->h_sub) maxnG = std::max(maxnG, S.nG);
  if (with_pq && c->nranks == 1 && st->bsub.n && !c->debug && c->P_op <= 8) {   // one pass: q, p0 rows, p.q
    const int64_t nxp1 = c->n_delta_glob + c->NPi;
    launch_pdl(st, chunk_gather_dot_kernel, dim3(DOT_BLOCKS), dim3(256), 0, s, st->xptr.p, st->xidx.p, c->w_part.p,
               c->len_G, c->P_op, st->bcoef.p, st->bsub.p, c->w_p.p, nxp1, nxp1, c->w_q.p, c->d_sub.p, c->N,
               c->d_b0T.p, c->d_loc2x.p, c->w_dots.p, st->ticket.p, c->w_scal.p + 1);
    tick(c, st, 3, false);
    VB_STAGE();
    return;
  }
  // peer stores only where a collective (the p.q sum) separates this receive from the next write
  const bool p2p = with_pq && st->XS.p2p;
  launch_pdl(st, chunk_sum_b0_kernel, dim3((maxnG + 255) / 256, c->N), dim3(256), 0, s, c->d_sub.p, c->w_part.p, c->len_G, c->P_op,
                                                                     c->d_b0T.p, c->d_loc2x.p, c->w_p.p,
                                                                     c->n_delta_glob + c->NPi, st->sx.p, c->w_q.p,
                                                                     p2p ? st->XS.p2p_ptr.p : nullptr,
                                                                     p2p ? st->XS.p2p_dst.p : nullptr);
  if (p2p)
    c->comm->barrier(s);                                             // C1 (peer stores done)
  else
    run_slot_exchange(c, st->XS, st->sx.p, st->sx.p + c->len_G);    // C1 (cross-rank copies)
  int64_t nxp = c->n_delta_glob + c->NPi;
  if (with_pq) {   // q and the partial of p.q in one pass (C3 follows)
    launch_pdl(st, gather_src_dot_kernel, dim3(DOT_BLOCKS), dim3(256), 0, s, st->xptr.p, st->xidx.p, st->sx.p, nxp,
               c->w_q.p, c->w_p.p, c->nranks > 1 ? st->mask.p : nullptr, c->nx, c->w_dots.p, st->ticket.p,
               c->w_scal.p + 1);
    allreduce_sum_fixed(c, c->w_scal.p + 1, 1);
  } else {
    launch_pdl(st, gather_src_kernel, dim3(grid_for(nxp)), dim3(256), 0, s, st->xptr.p, st->xidx.p, st->sx.p, nxp,
               c->w_q.p);
  }
  tick(c, st, 3, false);
  VB_STAGE();
}

// debugging aid (VB_PCG_TRACE=2): squared norm of a vector, summed over ranks unless replicated
static void trace_norm(vb_ctx *c, const char *name, const double *v, int64_t n, bool replicated) {
  static const bool on = getenv("VB_PCG_TRACE") && atoi(getenv("VB_PCG_TRACE")) >= 2;
  if (!on) return;
  double *d = c->w_dots.p + W_TRACE;
  dot_partial_kernel<<<DOT_BLOCKS, 256, 0, c->stream>>>(v, v, nullptr, n, c->w_dots.p);
  dot_final_kernel<<<1, 32, 0, c->stream>>>(c->w_dots.p, DOT_BLOCKS, d);
  if (!replicated) allreduce_sum_fixed(c, d, 1);
  double h;
  VB_CUDA(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, c->stream));
  VB_CUDA(cudaStreamSynchronize(c->stream));
  fprintf(stderr, "[vb rank %d] %s %.17g\n", c->rank, name, h);
}

// z = M^-1 r  (B4-B7); fill_tail = false leaves z's coarse tail to dot_rz (fused with r.z)
static void apply_M(vb_ctx *c, SolveState *st, bool fill_tail = true) {
  cudaStream_t s = c->stream, s2 = st->s2;
  // peer stores only inside the PCG step, where the r.z sum separates this receive from the next write
  const bool p2p = !fill_tail && st->XE.p2p;
  tick(c, st, 4, true);
  // fork: the coarse branch (B6) runs on s2 while the local dual solves (B5) stream on s
  VB_CUDA(cudaEventRecord(st->ev_fork, s));
  VB_CUDA(cudaStreamWaitEvent(s2, st->ev_fork, 0));
  tick(c, st, 1, true);
  run_sub_gemv(st, st->w_loc.p, st->nw_loc, st->sm_loc, st->big_loc, s);
  tick(c, st, 1, false);
  // coarse pieces (C2): [Phi_i^T rD_i per local subdomain | r0_i | r_Pi of the owned entities]
  launch_after_event(st, phit_kernel, dim3(st->phit_split, c->N), dim3(256), st->max_nd * sizeof(double), s2, c->d_sub.p, c->d_Phi.p,
             c->d_loc2x.p, c->w_r.p, st->cbuf.p);
  dev_gather(c->w_r.p, st->cpack.p, (int64_t)st->cpack.n, st->cbuf.p + c->len_Pi, s2);
  const double *pieces = st->cbuf.p;
  if (c->nranks > 1) {
    c->comm->allgather(st->cbuf.p, st->cgath.p, st->cmax, s2);
    pieces = st->cgath.p;
  }
  launch_pdl(st, gather_src_kernel, dim3(grid_for(c->Nc)), dim3(256), 0, s2, st->pptr.p, st->pidx.p, pieces, c->Nc, c->w_rc.p);
  if (!c->neumann)   // the gauge of the p_0 block (none with Neumann faces, DESIGN A35)
    launch_pdl(st, coarse_p0_project_kernel, dim3(1), dim3(256), 0, s2, st->gvol.p, c->Ng, c->w_rc.p + c->NPi_g, 0);
  tick(c, st, 2, true, s2);
  auto coarse_gemv = [&](const GemvWork *w, int nw, size_t sm, bool big) {
    if (big)
      launch_pdl(st, sym_gemv_kernel<GV_WARPS_C, true, true>, dim3(nw), dim3(GV_WARPS_C * 32), GV_WARPS_C * 32 * sizeof(double), s2, w);
    else
      launch_pdl(st, sym_gemv_kernel<GV_WARPS_C, false, true>, dim3(nw), dim3(GV_WARPS_C * 32), sm, s2, w);
  };
  // f1 dissection: local pass 1 (y_I = E g_I, t = F^T g_I), root rhs from every rank's t
  const int64_t nC = c->cdis ? c->Nroot : c->Nc;       // order of the (root or whole) inverse
  double *ucout = c->cdis ? st->cd_xroot.p : c->w_uc.p;
  if (c->cdis) {
    if (st->nw_cd1) {
      coarse_gemv(st->w_cd1.p, st->nw_cd1, st->sm_cd, st->big_cd);
      launch_pdl(st, cd_sum_parts_kernel, dim3((unsigned)((st->cd_maxloc + 255) / 256), st->cd_no), dim3(256), 0, s2,
                 st->cd_parts.p, st->cd_part1.p, st->cd_Y.p, c->cd_two ? st->cd_T1.p : st->cd_T.p,
                 c->cd_two ? c->cd_maxS0 : c->cd_maxS, (const double *)nullptr);
    }
    if (c->cd_two) {   // the rank level: its input from the blocks, pass 1, its root contribution
      const CdPart &d2 = c->cd2_part;
      launch_pdl(st, cd_l2_input_kernel, dim3(grid_for(d2.nloc)), dim3(256), 0, s2, st->cd2_ptr.p, st->cd2_idx.p,
                 st->cd_T1.p, c->w_rc.p, st->cd2_RS.p, d2.nI, d2.nIp, d2.nloc, st->cd_X2.p, st->cd_C.p);
      if (st->nw_cd21) coarse_gemv(st->w_cd21.p, st->nw_cd21, st->sm_cd, st->big_cd);
      launch_pdl(st, cd_sum_parts_kernel, dim3((unsigned)((d2.nloc + 255) / 256), 1), dim3(256), 0, s2,
                 st->cd2_desc.p, st->cd2_part1.p, st->cd2_Y.p, st->cd_T.p, c->cd_maxS, (const double *)st->cd_C.p);
    }
    const double *tg = st->cd_T.p;
    if (c->nranks > 1) {
      c->comm->allgather(st->cd_T.p, st->cd_tg.p, c->cd_maxS, s2);
      tg = st->cd_tg.p;
    }
    launch_pdl(st, cd_root_rhs_kernel, dim3(grid_for(c->Nroot)), dim3(256), 0, s2, st->cd_rptr.p, st->cd_ridx.p, tg,
               c->w_rc.p, st->cd_root.p, c->Nroot, st->cd_groot.p);
    if (!c->neumann)
      launch_pdl(st, coarse_p0_project_kernel, dim3(1), dim3(256), 0, s2, st->gvol.p, c->Ng, st->cd_groot.p + c->cd_nsep, 0);
  }
  // the packed inverse (all of it on one rank; this rank's tile rows otherwise)
  coarse_gemv(st->w_c.p, st->nw_c, st->sm_c, st->big_c);
  tick(c, st, 2, false, s2);
  if (c->nranks > 1) {
    // this rank's partial, then the rank-order sum of all partials (C2)
    launch_pdl(st, sum_chunks_kernel, dim3((nC + 31) / 32), dim3(256), 0, s2, c->w_ucp.p, nC, st->nw_c, nC, st->ucp.p);
    c->comm->allgather(st->ucp.p, st->ucg.p, nC, s2);
    launch_pdl(st, rank_sum_vec_kernel, dim3(grid_for(nC)), dim3(256), 0, s2, st->ucg.p, c->nranks, nC, ucout);
  } else {
    launch_pdl(st, sum_chunks_kernel, dim3((nC + 31) / 32), dim3(256), 0, s2, c->w_ucp.p, nC, st->nw_c, nC, ucout);
  }
  if (c->cdis) {
    // x_S (gauge-projected) to its global positions; pass 2: x_I = y_I - F x_S
    launch_pdl(st, cd_root_finish_kernel, dim3(1), dim3(1024), 0, s2, st->gvol.p, c->neumann ? 0 : c->Ng, c->cd_nsep,
               st->cd_xroot.p, st->cd_root.p, c->Nroot, c->w_uc.p);
    if (c->cd_two && st->nw_cd22) {   // x_RS = y_RS - F2 x_S before the blocks' pass 2 reads it
      coarse_gemv(st->w_cd22.p, st->nw_cd22, st->sm_cd, st->big_cd);
      launch_pdl(st, cd_interior_kernel, dim3((unsigned)((c->cd2_part.nI + 255) / 256), 1), dim3(256), 0, s2,
                 st->cd2_desc.p, st->cd2_part2.p, st->cd2_Y.p, st->cd2_RS.p, c->w_uc.p);
    }
    if (st->nw_cd2) {
      coarse_gemv(st->w_cd2.p, st->nw_cd2, st->sm_cd, st->big_cd);
      launch_pdl(st, cd_interior_kernel, dim3((unsigned)((st->cd_maxI + 255) / 256), st->cd_no), dim3(256), 0, s2,
                 st->cd_parts.p, st->cd_part2.p, st->cd_Y.p, st->cd_Iall.p, c->w_uc.p);
    }
  } else if (!c->neumann) {
    launch_pdl(st, coarse_p0_project_kernel, dim3(1), dim3(256), 0, s2, st->gvol.p, c->Ng, c->w_uc.p + c->NPi_g, 1);
  }
  launch_pdl(st, coarse_ext_kernel, dim3((st->max_nd + 127) / 128, c->N), dim3(128), c->max_npi * sizeof(double), s2,
             c->d_sub.p, c->d_Phi.p, c->d_pi_glob.p, c->w_uc.p, c->w_locC.p);
  VB_CUDA(cudaEventRecord(st->ev_join, s2));
  VB_CUDA(cudaStreamWaitEvent(s, st->ev_join, 0));
  trace_norm(c, "uc", c->w_uc.p, c->Nc, true);
  // (the fused kernel sums the P chunks serially per output: kept for few chunks, e.g. P = 4 at 512
  // subdomains; at P = 32 (64 large subdomains, config 3) the two-kernel path is faster)
  if (c->nranks == 1 && st->ESE.n && !c->debug && c->P_loc <= 8) {
    launch_after_event(st, local2_entity_sum_kernel, dim3(st->ESE.n), dim3(st->ESE.maxlen > 64 ? 256 : 64), 0, s,
                       st->ESE.ptr.p, st->ESE.off.p, st->ESE.out_off.p, st->ESE.len.p, c->w_locY.p, c->len_Dv,
                       c->P_loc, c->w_locC.p, c->w_z.p);
  } else {
    launch_after_event(st, local2_kernel, dim3(grid_for(c->len_Dv)), dim3(256), 0, s, c->w_locY.p, c->len_Dv, c->P_loc,
                       c->w_locC.p, c->len_Dv, c->w_locD.p, p2p ? st->XE.p2p_ptr.p : nullptr,
                       p2p ? st->XE.p2p_dst.p : nullptr);
    trace_norm(c, "t", c->w_locD.p, c->len_Dv, false);
    if (p2p)
      c->comm->barrier(s);                                                  // C1 (peer stores done)
    else
      run_slot_exchange(c, st->XE, c->w_locD.p, c->w_locD.p + c->len_Dv);  // C1 (cross-rank products)
    run_entity_sum(c, st->ESE, c->w_locD.p, c->w_z.p);
  }
  trace_norm(c, "zdual", c->w_z.p, c->n_delta_glob, false);
  if (fill_tail) dev_gather(c->w_uc.p, st->zmap.p, c->NPi + c->N, c->w_z.p + c->n_delta_glob, s);
  tick(c, st, 4, false);
  VB_STAGE();
}

void destroy_solve_state(vb_ctx *c) {
  delete (SolveState *)c->solve_state;
  c->solve_state = nullptr;
}

static void build_csr(int64_t nrows, const std::vector<std::pair<int64_t, int64_t>> &pairs, DBuf<int64_t> &ptr,
                      DBuf<int64_t> &idx, cudaStream_t s) {
  std::vector<int64_t> p(nrows + 1, 0), ix(std::max<size_t>(pairs.size(), 1));
  for (auto &q : pairs) p[q.first + 1]++;
  for (int64_t i = 0; i < nrows; ++i) p[i + 1] += p[i];
  std::vector<int64_t> fill(p.begin(), p.end() - 1);
  for (auto &q : pairs) ix[fill[q.first]++] = q.second;   // pairs arrive in the required order per row
  ptr.upload(p, s);
  idx.upload(ix, s);
}

void prepare_solve(vb_ctx *c) {
  SolveState *st = get_state(c);
  if (st->ready) return;
  // row chunks per subdomain matrix for the packed GEMVs: about 2048 work items in all (4 per
  // subdomain at 512 subdomains, more when there are few large subdomains, e.g. config 3);
  // tuning knobs VB_P_OP / VB_P_LOC
  {
    const int P = std::max(4, std::min(32, (2048 + c->N - 1) / std::max(c->N, 1)));
    c->P_op = c->P_loc = c->P_kd = P;
  }
  st->phit_split = std::max(4, std::min(32, (2048 + c->N - 1) / std::max(c->N, 1)));
  if (getenv("VB_P_OP")) c->P_op = std::max(1, atoi(getenv("VB_P_OP")));
  if (getenv("VB_P_LOC")) c->P_loc = std::max(1, atoi(getenv("VB_P_LOC")));
  if (getenv("VB_P_C")) c->P_c = std::max(1, atoi(getenv("VB_P_C")));   // coarse GEMV chunks (experiment knob)
  cudaStream_t s = c->stream;
  const int N = c->N;
  const int64_t nx = c->nx;
  c->w_x.alloc(nx); c->w_r.alloc(nx); c->w_z.alloc(nx); c->w_p.alloc(nx); c->w_q.alloc(nx);
  c->w_part.alloc((int64_t)c->P_op * std::max<int64_t>(c->len_G, 1));
  c->w_locD.alloc(std::max<int64_t>(c->len_Dv, 1));
  c->w_locC.alloc(std::max<int64_t>(c->len_Dv, 1));
  c->w_locY.alloc((int64_t)c->P_loc * std::max<int64_t>(c->len_Dv, 1));
  // w_rc[Nc] = w_uc[Nc] = 0: the gather target of the zero blocks of the dissection GEMV inputs
  c->w_uc.alloc(c->Nc + 1); c->w_rc.alloc(c->Nc + 1);
  c->w_uc.zero(s); c->w_rc.zero(s);
  const int64_t nC = c->cdis ? c->Nroot : c->Nc;   // order of the (root or whole) coarse inverse
  if (c->nranks > 1) { st->ucp.alloc(nC); st->ucg.alloc(nC * c->nranks); }
  c->w_scal.alloc(16); c->w_scal.zero(s);
  st->ticket.alloc(4); st->ticket.zero(s);
  st->pdl = !(getenv("VB_NO_PDL") && atoi(getenv("VB_NO_PDL")));
  if (!st->s2) {
    int lo = 0, hi = 0;
    VB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    st->prio_hi = (getenv("VB_NO_PRIO") && atoi(getenv("VB_NO_PRIO"))) ? 0 : hi;
    VB_CUDA(cudaStreamCreateWithPriority(&st->s2, cudaStreamNonBlocking, st->prio_hi));
    VB_CUDA(cudaStreamCreateWithFlags(&st->sg, cudaStreamNonBlocking));
    VB_CUDA(cudaEventCreateWithFlags(&st->ev_fork, cudaEventDisableTiming));
    VB_CUDA(cudaEventCreateWithFlags(&st->ev_join, cudaEventDisableTiming));
  }
  if (c->nranks > 1) c->w_red.alloc((size_t)c->nranks * 8);
  c->w_dots.alloc(DOT_BLOCKS * 2 + 256);
  c->w_gam.alloc(std::max<int64_t>(c->nGamma, 1));
  c->w_bD.alloc(std::max<int64_t>(c->len_Dn, 1));
  c->w_zG.alloc(std::max<int64_t>(c->len_G, 1));
  st->hist.alloc(2 * 4096);
  // packed GEMV work lists
  std::vector<GemvWork> wl;
  std::vector<std::pair<int, int>> rows;
  size_t nmaxG = 1, nmaxD = 1;
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    nmaxG = std::max<size_t>(nmaxG, S.nG);
    split_rows(S.nG, c->P_op, rows);
    for (int q = 0; q < c->P_op; ++q)
      wl.push_back(GemvWork{c->d_STp.p + S.off_STp, c->d_loc2x.p + S.off_G, c->w_p.p,
                            c->w_part.p + (int64_t)q * c->len_G + S.off_G, S.nG, rows[q].first, rows[q].second, 0});
  }
  st->w_op.upload(wl, s); st->nw_op = wl.size(); st->sm_op = gemv_smem(nmaxG);
  wl.clear();
  for (int i = 0; i < N; ++i) {
    const SubDev &S = c->h_sub[i];
    if (!S.nd) continue;
    nmaxD = std::max<size_t>(nmaxD, S.nd);
    split_rows(S.nd, c->P_loc, rows);
    for (int q = 0; q < c->P_loc; ++q)
      wl.push_back(GemvWork{c->d_SDi.p + S.off_SDi, c->d_loc2x.p + S.off_G, c->w_r.p,
                            c->w_locY.p + (int64_t)q * c->len_Dv + S.off_Dv, S.nd, rows[q].first, rows[q].second, 0});
  }
  // sub-domains with nd = 0 still need zero partials
  c->w_locY.zero(s);
  st->w_loc.upload(wl, s); st->nw_loc = wl.size(); st->sm_loc = gemv_smem(nmaxD);
  wl.clear();
  // coarse work list: the tile rows [tlo, thi) of the packed inverse (all of them on one rank) --
  // of the whole coarse matrix, or of the dissection root
  // split the tile rows [tlo, thi) of a packed matrix of order n into Pc chunks balanced by tiles +
  // row cost (as split_rows over the slice); chunk q writes the partial vector out + q n
  auto slice_work = [&](const double *M, int64_t moff, const int64_t *map, const double *x, double *out, int64_t n,
                        int64_t tlo, int64_t thi, int Pc) {
    auto cum = [&](int64_t r) { return (double)r * (r + 1) / 2 + 4.0 * r; };
    const double c0 = cum(tlo), tot = cum(thi) - c0;
    int64_t r = tlo;
    for (int q = 0; q < Pc; ++q) {
      int64_t r1 = r;
      while (r1 < thi && cum(r1 + 1) - c0 <= tot * (q + 1) / Pc) ++r1;
      if (r1 == r && r < thi) r1 = r + 1;
      if (q == Pc - 1) r1 = thi;
      wl.push_back(GemvWork{M, map, x, out + (int64_t)q * n, (int)n, (int)r, (int)r1, 0, moff});
      r = r1;
    }
  };
  const int64_t ntc = (nC + 31) / 32;
  const int64_t tlo = c->nranks > 1 ? c->coarse_tlo : 0, thi = c->nranks > 1 ? c->coarse_thi : ntc;
  const double *Kc0 = c->nranks > 1 ? c->d_Kcs.p : c->d_Kcp.p;
  const int64_t Kc_off = c->nranks > 1 ? ptile_row_start(tlo) : 0;   // the slice starts at tile row tlo
  int Pc = (int)std::max<int64_t>(1, std::min<int64_t>(c->P_c, thi - tlo));
  c->w_ucp.alloc(std::max<int64_t>((int64_t)Pc * nC, 1));
  c->w_ucp.zero(s);
  if (c->cdis) {
    st->cd_groot.alloc(nC); st->cd_xroot.alloc(nC);
  }
  slice_work(Kc0, Kc_off, nullptr, c->cdis ? st->cd_groot.p : c->w_rc.p, c->w_ucp.p, nC, tlo, thi, Pc);
  st->w_c.upload(wl, s); st->nw_c = wl.size(); st->sm_c = gemv_smem(nC, GV_WARPS_C);
  st->big_c = st->sm_c > 200 * 1024;
  wl.clear();
  if (c->cdis) {
    // f1 dissection: per owned part the packed [[E, .], [F^T, 0]] of order n_loc = nIp + nS
    std::vector<CdPart> D = c->cd_parts;
    const int no = D.size();
    int act = 0;
    for (auto &d : D) act += d.nIp > 0;
    const int Pper = std::max(1, c->P_c / std::max(act, 1));
    std::vector<int64_t> m1, m2, Iall;
    int64_t p1 = 0, p2 = 0, y = 0, maxloc = 1, maxI = 1;
    for (int j = 0; j < no; ++j) {
      CdPart &d = D[j];
      const int64_t ntl = (d.nloc + 31) / 32, tS = d.nIp / 32;
      d.P1 = d.nIp ? (int)std::min<int64_t>(ntl, Pper) : 0;
      d.P2 = d.nIp ? (int)std::min<int64_t>(ntl - tS, Pper) : 0;
      d.p1off = p1; p1 += (int64_t)d.P1 * d.nloc;
      d.p2off = p2; p2 += (int64_t)d.P2 * d.nloc;
      d.yoff = y; y += d.nIp;
      d.moff = m1.size();
      d.ioff = Iall.size();
      for (int64_t a = 0; a < d.nloc; ++a) {
        m1.push_back(a < d.nI ? c->cd_I[j][a] : c->Nc);
        m2.push_back(a >= d.nIp ? c->cd_S[j][a - d.nIp] : c->Nc);
      }
      Iall.insert(Iall.end(), c->cd_I[j].begin(), c->cd_I[j].end());
      maxloc = std::max(maxloc, d.nloc);
      maxI = std::max(maxI, d.nI);
    }
    st->cd_map1.upload(m1, s); st->cd_map2.upload(m2, s);
    st->cd_Iall.upload(Iall.empty() ? std::vector<int64_t>{0} : Iall, s);
    st->cd_root.upload(c->cd_root_glob, s);
    st->cd_rptr.upload(c->cd_rptr, s);
    st->cd_ridx.upload(c->cd_ridx.empty() ? std::vector<int64_t>{0} : c->cd_ridx, s);
    st->cd_Y.alloc(std::max<int64_t>(y, 1));
    st->cd_T.alloc((int64_t)(c->cd_two ? 1 : std::max(no, 1)) * c->cd_maxS); st->cd_T.zero(s);
    if (c->cd_two) { st->cd_T1.alloc((int64_t)std::max(no, 1) * c->cd_maxS0); st->cd_T1.zero(s); }
    if (c->nranks > 1) st->cd_tg.alloc(c->cd_maxS * c->nranks);
    st->cd_part1.alloc(std::max<int64_t>(p1, 1)); st->cd_part2.alloc(std::max<int64_t>(p2, 1));
    st->nw_cd1 = st->nw_cd2 = 0;
    for (int j = 0; j < no; ++j)
      if (D[j].P1) slice_work(c->d_Kloc.p + D[j].koff, 0, st->cd_map1.p + D[j].moff, c->w_rc.p, st->cd_part1.p + D[j].p1off,
                              D[j].nloc, 0, (D[j].nloc + 31) / 32, D[j].P1);
    st->w_cd1.upload(wl, s); st->nw_cd1 = wl.size(); wl.clear();
    for (int j = 0; j < no; ++j)
      if (D[j].P2) slice_work(c->d_Kloc.p + D[j].koff, 0, st->cd_map2.p + D[j].moff, c->w_uc.p, st->cd_part2.p + D[j].p2off,
                              D[j].nloc, D[j].nIp / 32, (D[j].nloc + 31) / 32, D[j].P2);
    st->w_cd2.upload(wl, s); st->nw_cd2 = wl.size(); wl.clear();
    st->cd_parts.upload(D, s);
    st->cd_no = no; st->cd_maxloc = maxloc; st->cd_maxI = maxI;
    c->cd_parts = D;
    if (c->cd_two) {
      CdPart d2 = c->cd2_part;
      const int64_t ntl = (d2.nloc + 31) / 32, tS = d2.nIp / 32;
      d2.P1 = d2.nIp ? (int)std::min<int64_t>(ntl, c->P_c) : 0;
      d2.P2 = d2.nIp ? (int)std::min<int64_t>(ntl - tS, c->P_c) : 0;
      d2.p1off = d2.p2off = d2.yoff = d2.moff = d2.ioff = 0;
      std::vector<int64_t> mp2(d2.nloc, c->Nc);
      for (int64_t q = 0; q < d2.nS; ++q) mp2[d2.nIp + q] = c->cd2_S[q];
      st->cd2_map2.upload(mp2, s);
      st->cd2_RS.upload(c->cd2_RS.empty() ? std::vector<int64_t>{0} : c->cd2_RS, s);
      st->cd2_ptr.upload(c->cd2_ptr, s);
      st->cd2_idx.upload(c->cd2_idx.empty() ? std::vector<int64_t>{0} : c->cd2_idx, s);
      st->cd_X2.alloc(std::max<int64_t>(d2.nloc, 1)); st->cd_X2.zero(s);
      st->cd_C.alloc(std::max<int64_t>(d2.nS, 1)); st->cd_C.zero(s);
      st->cd2_Y.alloc(std::max<int64_t>(d2.nIp, 1));
      st->cd2_part1.alloc(std::max<int64_t>((int64_t)d2.P1 * d2.nloc, 1));
      st->cd2_part2.alloc(std::max<int64_t>((int64_t)d2.P2 * d2.nloc, 1));
      if (d2.P1) slice_work(c->d_Kloc2.p, 0, nullptr, st->cd_X2.p, st->cd2_part1.p, d2.nloc, 0, ntl, d2.P1);
      st->w_cd21.upload(wl, s); st->nw_cd21 = wl.size(); wl.clear();
      if (d2.P2) slice_work(c->d_Kloc2.p, 0, st->cd2_map2.p, c->w_uc.p, st->cd2_part2.p, d2.nloc, tS, ntl, d2.P2);
      st->w_cd22.upload(wl, s); st->nw_cd22 = wl.size(); wl.clear();
      st->cd2_desc.upload(std::vector<CdPart>{d2}, s);
      c->cd2_part = d2;
      maxloc = std::max(maxloc, d2.nloc);
    }
    st->sm_cd = gemv_smem(maxloc, GV_WARPS_C);
    st->big_cd = st->sm_cd > 200 * 1024;
    if (!st->big_cd)
      raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS_C, false, true>, st->sm_cd);
  }
  // VB_GV_BIG=<bytes>: experiment knob, the BIG variant (x through the L2, partial output in global
  // memory, shared memory only for the row reduction) from that many bytes of staged vectors on
  static const int64_t gv_big = getenv("VB_GV_BIG") ? atoll(getenv("VB_GV_BIG")) : 200 * 1024;
  st->big_op = (int64_t)st->sm_op > gv_big;
  st->big_loc = (int64_t)st->sm_loc > gv_big;
  size_t smmax = std::max(st->big_op ? 0 : st->sm_op, st->big_loc ? 0 : st->sm_loc);
  raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS>, smmax);
  {
    const char *ep = getenv("VB_GV_PAIR");   // experiment knob: 1 on, 0 off
    st->pair_sub = ep ? atoi(ep) != 0 : false;
  }
  if (st->pair_sub) raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS, false, true>, smmax);
  if (!st->big_c)
    raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS_C, false, true>, st->sm_c);
  st->max_nd = nmaxD;
  if (st->max_nd * sizeof(double) > 48 * 1024)
    raise_smem_limit((const void *)phit_kernel, st->max_nd * sizeof(double));
  const int ne = c->ents.size();
  // ---------------- B2 (apply_S): copies of each x coordinate, local and received, in sharer order
  {
    auto L = [&](int e) { return (int64_t)c->h_ent[e].n; };
    auto pos = [&](int sl, std::vector<int64_t> &out) {
      const SlotDev &q = c->h_slot[sl];
      const SubDev &S = c->h_sub[q.sub];
      for (int t = 0; t < q.nd; ++t) out.push_back(S.off_G + q.offD + t);
      for (int t = 0; t < q.r; ++t) out.push_back(S.off_G + S.nd + q.offPi + t);
    };
    build_slot_exchange(c, st->XS, L, pos);
    st->sx.alloc(std::max<int64_t>(c->len_G + st->XS.recv_len, 1));
    std::vector<std::pair<int64_t, int64_t>> pr;
    for (int e = 0; e < ne; ++e) {
      const Entity &E = c->ents[e];
      const EntDev &D = c->h_ent[e];
      int li = 0;
      for (size_t k = 0; k < E.sharers.size(); ++k) {
        std::vector<int64_t> src;
        if (c->sub_lid[E.sharers[k]] >= 0) {
          pos(D.side_begin + li, src);
          ++li;
        } else {
          const int64_t ro = st->XS.recv_off[st->XS.ent_ptr[e] + k];
          for (int t = 0; t < D.n; ++t) src.push_back(c->len_G + ro + t);
        }
        for (int t = 0; t < D.nd; ++t) pr.push_back({D.off_xd + t, src[t]});
        for (int t = 0; t < D.r; ++t) pr.push_back({c->n_delta_glob + D.off_pl + t, src[D.nd + t]});
      }
    }
    // (build_csr keeps the generation order within each row)
    build_csr(c->n_delta_glob + c->NPi, pr, st->xptr, st->xidx, s);
    if (c->nranks == 1 && c->len_G > 0) {   // chunk_gather_dot_kernel's b~0 expansion
      st->bcoef.alloc(c->len_G);
      st->bsub.alloc(c->len_G);
      b0_expand_kernel<<<c->N, 256, 0, s>>>(c->d_sub.p, c->d_b0T.p, st->bcoef.p, st->bsub.p);
      VB_CHECK_LAUNCH();
    }
  }
  // ---------------- B7 (extension): per-slot scaled products (in w_locD, subdomain-major) and their
  // sums over all sharers
  {
    auto L = [&](int e) { return (int64_t)c->h_ent[e].nd; };
    auto tb = [&](int sl) { return c->h_sub[c->h_slot[sl].sub].off_Dv + c->h_slot[sl].offD; };
    build_slot_exchange(c, st->XE, L, [&](int sl, std::vector<int64_t> &out) {
      for (int t = 0; t < c->h_slot[sl].nd; ++t) out.push_back(tb(sl) + t);
    });
    c->w_locD.alloc(std::max<int64_t>(c->len_Dv + st->XE.recv_len, 1));
    build_entity_sum(c, st->ESE, st->XE, L, tb, c->len_Dv, [&](int e) { return c->h_ent[e].off_xd; });
  }
  // ---------------- B0: zG copies of each entity DOF, summed over all sharers after b_e
  {
    auto L = [&](int e) { return (int64_t)c->h_ent[e].n; };
    auto sb = [&](int sl) { return c->h_sub[c->h_slot[sl].sub].off_G + c->h_slot[sl].offG; };
    build_slot_exchange(c, st->XB, L, [&](int sl, std::vector<int64_t> &out) {
      const int64_t b = sb(sl);
      for (int t = 0; t < c->h_slot[sl].n; ++t) out.push_back(b + t);
    });
    st->gbuf.alloc(std::max<int64_t>(c->len_G + st->XB.recv_len, 1));
    st->gam2.alloc(std::max<int64_t>(c->nGamma, 1));
    std::function<int64_t(int)> gb = [&](int e) { return c->h_ent[e].off_gam; };
    build_entity_sum(c, st->ESB, st->XB, L, sb, c->len_G, gb, &gb);
  }
  // ---------------- free-DOF halo (owner -> holders) and rank partial sums (holders -> all)
  {
    auto L = [&](int e) { return (int64_t)c->h_ent[e].n; };
    auto pos = [&](int sl, std::vector<int64_t> &out) {
      const EntDev &D = c->h_ent[c->h_slot[sl].ent];
      for (int t = 0; t < D.n; ++t) out.push_back(D.off_gam + t);
    };
    build_slot_exchange(c, st->XH, L, pos, XCH_OWNER);
    build_slot_exchange(c, st->XR, L, pos, XCH_RANK);
    std::function<int64_t(int)> gb = [&](int e) { return c->h_ent[e].off_gam; };
    build_entity_sum(c, st->ESR, st->XR, L, [&](int sl) { return c->h_ent[c->h_slot[sl].ent].off_gam; }, c->nGamma,
                     gb, nullptr, XCH_RANK);
    // received owner values: destination positions (entity-major) of the ghost entity DOFs
    // (indexed by receive position: the receive area is peer-major, not entity-major)
    std::vector<int64_t> dst(st->XH.recv_len, -1);
    for (int e = 0; e < ne; ++e) {
      const int64_t ro = st->XH.recv_off.empty() ? -1 : st->XH.recv_off[st->XH.ent_ptr[e]];
      if (ro < 0) continue;
      for (int t = 0; t < c->h_ent[e].n; ++t) dst[ro + t] = c->h_ent[e].off_gam + t;
    }
    st->n_gh = dst.size();
    st->hbuf.alloc(std::max<int64_t>(st->XH.recv_len, 1));
    for (int64_t d : dst) VB_REQUIRE(d >= 0, VB_EINVAL, "internal: halo receive position without destination");
    if (dst.empty()) dst.push_back(0);
    st->gh_dst.upload(dst, s);
  }
  // ---------------- B6: coarse pieces, their global layout and the coarse rhs sources
  {
    const int R = c->nranks, me = c->rank;
    std::vector<int> gnpi(c->Ng, 0);
    for (int g = 0; g < c->Ng; ++g)
      for (int e : c->gsub_ents[g]) gnpi[g] += c->gents[e].r;
    // per rank: [cpart of its subdomains (in order) | r0 of its subdomains | r_Pi of its owned entities]
    std::vector<int64_t> lenPi(R, 0), nsub(R, 0), nown(R, 0), sub_cpos(c->Ng, 0), sub_r0(c->Ng, 0);
    for (int g = 0; g < c->Ng; ++g) {
      const int r = c->sub_rank[g];
      sub_cpos[g] = lenPi[r];
      lenPi[r] += gnpi[g];
      sub_r0[g] = nsub[r]++;
    }
    std::vector<int64_t> ent_own(c->gents.size(), 0);
    for (size_t e = 0; e < c->gents.size(); ++e) {
      const int r = c->sub_rank[c->gents[e].sharers[0]];
      ent_own[e] = nown[r];
      nown[r] += c->gents[e].r;
    }
    int64_t cmax = 1;
    for (int r = 0; r < R; ++r) cmax = std::max(cmax, lenPi[r] + nsub[r] + nown[r]);
    st->cmax = cmax;
    VB_REQUIRE(lenPi[me] == c->len_Pi, VB_EINVAL, "internal: coarse piece layout mismatch");
    st->cbuf.alloc(cmax);
    st->cbuf.zero(s);
    if (R > 1) st->cgath.alloc((size_t)cmax * R);
    auto base = [&](int r) { return (int64_t)r * (R > 1 ? cmax : 0); };
    // local packing: r0 of local subs, then r_Pi of owned local entities
    std::vector<int64_t> cpack;
    for (int i = 0; i < N; ++i) cpack.push_back(c->n_delta_glob + c->NPi + i);
    for (int e = 0; e < ne; ++e) {
      const Entity &E = c->ents[e];
      if (c->sub_rank[E.sharers[0]] != me) continue;
      for (int t = 0; t < E.r; ++t) cpack.push_back(c->n_delta_glob + E.off_pl + t);
    }
    st->cpack.upload(cpack, s);
    // sources of every global coarse index: owner's r_Pi, then each sharer's Phi^T r piece
    std::vector<std::pair<int64_t, int64_t>> pr;
    for (size_t e = 0; e < c->gents.size(); ++e) {
      const GEnt &G = c->gents[e];
      const int ro = c->sub_rank[G.sharers[0]];
      for (int t = 0; t < G.r; ++t) pr.push_back({G.off_pi + t, base(ro) + lenPi[ro] + nsub[ro] + ent_own[e] + t});
      for (int m : G.sharers) {
        const int rm = c->sub_rank[m];
        int64_t within = 0;   // position of e in m's primal layout (entities in id order)
        for (int e2 : c->gsub_ents[m]) { if (e2 == (int)e) break; within += c->gents[e2].r; }
        for (int t = 0; t < G.r; ++t) pr.push_back({G.off_pi + t, base(rm) + sub_cpos[m] + within + t});
      }
    }
    for (int g = 0; g < c->Ng; ++g) {
      const int r = c->sub_rank[g];
      pr.push_back({c->NPi_g + g, base(r) + lenPi[r] + sub_r0[g]});
    }
    // (build_csr keeps the generation order within each row)
    build_csr(c->Nc, pr, st->pptr, st->pidx, s);
    // z tail <- u_c: local primal coordinates, then the local p0
    std::vector<int64_t> zm(c->NPi + N, 0);
    for (int e = 0; e < ne; ++e)
      for (int t = 0; t < c->h_ent[e].r; ++t) zm[c->h_ent[e].off_pl + t] = c->h_ent[e].off_pi + t;
    for (int i = 0; i < N; ++i) zm[c->NPi + i] = c->NPi_g + c->sub_gid[i];
    st->zmap.upload(zm, s);
    st->gvol.upload(c->gsub_vol, s);
  }
  // ---------------- C3 mask: coordinates owned by this rank (entities whose lowest sharer is here)
  if (c->nranks > 1) {
    std::vector<double> mk(nx, 0.0);
    for (int e = 0; e < ne; ++e) {
      if (c->sub_rank[c->ents[e].sharers[0]] != c->rank) continue;
      const EntDev &D = c->h_ent[e];
      for (int t = 0; t < D.nd; ++t) mk[D.off_xd + t] = 1.0;
      for (int t = 0; t < D.r; ++t) mk[c->n_delta_glob + D.off_pl + t] = 1.0;
    }
    for (int i = 0; i < N; ++i) mk[c->n_delta_glob + c->NPi + i] = 1.0;
    st->mask.upload(mk, s);
    const int64_t nfg = c->n_free_vel + c->npres;
    c->w_rhsg.alloc(nfg);
    c->w_xg.alloc(nfg);
  }
  // B0/B8: packed K_DD^-1 GEMV work list (y_D = K_DD^-1 b_D) and buffers
  c->w_yDp.alloc((int64_t)c->P_kd * std::max<int64_t>(c->len_Dn, 1));
  c->w_xD.alloc(std::max<int64_t>(c->len_Dn, 1));
  {
    std::vector<GemvWork> wk;
    size_t nmaxDn = 1;
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      nmaxDn = std::max<size_t>(nmaxDn, S.nD);
      split_rows(S.nD, c->P_kd, rows);
      for (int q = 0; q < c->P_kd; ++q)
        wk.push_back(GemvWork{c->d_KDi.p + S.off_KDi, nullptr, c->w_bD.p + S.off_Dn,
                              c->w_yDp.p + (int64_t)q * c->len_Dn + S.off_Dn, S.nD, rows[q].first, rows[q].second, 0});
    }
    st->w_kd.upload(wk, s);
    st->nw_kd = wk.size();
    st->sm_kd = gemv_smem(nmaxDn);
    st->big_kd = (int64_t)st->sm_kd > gv_big;
    size_t smg = std::max(std::max(st->big_op ? 0 : st->sm_op, st->big_loc ? 0 : st->sm_loc), st->big_kd ? 0 : st->sm_kd);
    raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS>, smg);
    if (st->pair_sub) raise_smem_limit((const void *)sym_gemv_kernel<GV_WARPS, false, true>, smg);
  }
  // ---------------- B0 / B8 coupling gathers: output row <- (cell, element row) slots in cell order
  {
    const int stride = c->nv_max + c->np;
    std::vector<int> csub(std::max<int64_t>(c->nKl, 1), 0);
    std::vector<std::pair<int64_t, int64_t>> e0, e1;
    std::vector<int> rs0(std::max<int64_t>(c->len_G, 1), 0), rs1(std::max<int64_t>(c->len_Dn, 1), 0);
    std::vector<int> hcells;
    for (int i = 0; i < N; ++i) {
      const SubDev &S = c->h_sub[i];
      for (int g = 0; g < S.nG; ++g) rs0[S.off_G + g] = i;
      for (int d = 0; d < S.nD; ++d) rs1[S.off_Dn + d] = i;
      for (int cell : c->subs[i].cells) {
        csub[cell] = i;
        const int *loc = c->h_cell_loc.data() + (size_t)cell * stride;
        const int nv = c->cell_nv[c->cell_gid[cell]];
        for (int a = 0; a < nv; ++a) {
          const int la = loc[a];
          if (la >= S.nD) e0.push_back({S.off_G + (la - S.nD), (int64_t)cell * stride + a});
          else if (la >= 0 && la < S.nI) e1.push_back({S.off_Dn + la, (int64_t)cell * stride + a});
        }
        for (int p = 0; p < c->np; ++p) {
          const int lp = loc[c->nv_max + p];
          if (lp >= S.nI && lp < S.nD) e1.push_back({S.off_Dn + lp, (int64_t)cell * stride + c->nv_max + p});
        }
      }
    }
    // build_csr keeps the generation order (subdomain, then cell order) within each row
    build_csr(std::max<int64_t>(c->len_G, 1), e0, st->cp_ptr[0], st->cp_src[0], s);
    build_csr(std::max<int64_t>(c->len_Dn, 1), e1, st->cp_ptr[1], st->cp_src[1], s);
    st->cp_rsub[0].upload(rs0, s);
    st->cp_rsub[1].upload(rs1, s);
    st->cell_sub.upload(csub, s);
    st->ycell.alloc(std::max<int64_t>((int64_t)c->nKl * stride, 1));
    st->ycell.zero(s);
    st->cscal.alloc(std::max(N, 1));
  }
  st->g0abs.alloc(std::max(N, 1));
  // direct peer stores for the two per-iteration interface exchanges (vb_set_option("p2p") or
  // VB_P2P=1; collective: every rank factors with the same setting)
  const char *pe = getenv("VB_P2P");
  if ((c->opt_p2p || (pe && atoi(pe))) && c->nranks > 1) {
    build_slot_p2p(c, st->XS, st->sx.p, c->len_G, c->len_G);
    build_slot_p2p(c, st->XE, c->w_locD.p, c->len_Dv, c->len_Dv);
  }
  VB_CUDA(cudaStreamSynchronize(s));
  st->ready = true;
  // bytes per PCG iteration (model of the streamed operators)
  double b = 0;
  for (auto &S : c->h_sub) {
    b += 8.0 * packed_size(S.nG) + 8.0 * packed_size(S.nd) + 2 * 8.0 * S.nd * S.npi;
  }
  // (the deluxe blocks are folded into S_DD^-1 and Phi at factor time: no per-iteration D traffic)
  b += 8.0 * (c->nranks > 1 ? (double)c->d_Kcs.n : (double)packed_size(c->cdis ? c->Nroot : c->Nc));
  if (c->cdis) {   // dissection passes 1 (all of each part's matrix) and 2 (its S tile rows)
    std::vector<CdPart> all = c->cd_parts;
    if (c->cd_two) all.push_back(c->cd2_part);
    for (auto &d : all)
      if (d.nIp > 0) b += 8.0 * (2.0 * packed_size((int)d.nloc) - ptile_row_start(d.nIp / 32));
  }
  c->bytes_per_iter = b;
}

// owner values of the ghost interface DOFs (global free layout vector v, entity DOFs)
static void dof_halo(vb_ctx *c, SolveState *st, double *v) {
  if (c->nranks == 1) return;
  cudaStream_t s = c->stream;
  dev_gather(v, c->d_gam_free.p, c->nGamma, c->w_gam.p, s);
  run_slot_exchange(c, st->XH, c->w_gam.p, st->hbuf.p);
  if (st->n_gh) {
    // w_gam[dst[k]] = received[k], then back to the free layout
    dev_scatter(st->hbuf.p, st->gh_dst.p, st->n_gh, c->w_gam.p, s);
    dev_scatter(c->w_gam.p, c->d_gam_free.p, c->nGamma, v, s);
  }
}

// interface DOF sums across ranks of per-rank partial sums (global free layout vector v)
static void dof_rank_sum(vb_ctx *c, SolveState *st, double *v) {
  if (c->nranks == 1) return;
  cudaStream_t s = c->stream;
  dev_gather(v, c->d_gam_free.p, c->nGamma, c->w_gam.p, s);
  DBuf<double> comb;
  comb.alloc(std::max<int64_t>(c->nGamma + st->XR.recv_len, 1));
  VB_CUDA(cudaMemcpyAsync(comb.p, c->w_gam.p, c->nGamma * 8, cudaMemcpyDeviceToDevice, s));
  run_slot_exchange(c, st->XR, comb.p, comb.p + c->nGamma);
  run_entity_sum(c, st->ESR, comb.p, c->w_gam.p);
  dev_scatter(c->w_gam.p, c->d_gam_free.p, c->nGamma, v, s);
  VB_CUDA(cudaStreamSynchronize(s));
}

// element contributions -> free vector in the ABI layout (owned DOFs; all free DOFs for one rank)
void element_gather(vb_ctx *c, const double *yel, double *out) {
  const int stride = c->nv_max + c->np;
  const int64_t nf = c->n_free_vel + c->nKl * c->np;
  if (c->nranks > 1)
    VB_REQUIRE(get_state(c)->ready, VB_ESTATE, "multi-rank assembly needs vb_factor first (exchange plans)");
  double *dst = c->nranks > 1 ? c->w_rhsg.p : out;
  elem_gather_kernel<<<grid_for(nf), 256, 0, c->stream>>>(c->d_el_ptr.p, c->d_el_ent.p, c->d_cell_gid.p, yel,
                                                          c->n_free_vel, c->nKl, c->np, stride, c->nv_max, dst);
  VB_STAGE();
  if (c->nranks > 1) {
    dof_rank_sum(c, get_state(c), dst);
    dev_gather(dst, c->d_owned_free.p, (int64_t)c->owned_free.size(), out, c->stream);
  }
}

// per-cell slot of the packed element matrices: even (16-byte aligned cells for the bulk copies)
static int64_t k7_slot(int nvmax) { return (((int64_t)nvmax * (nvmax + 1) / 2) + 1) & ~1LL; }
constexpr size_t kK7BulkSmem = 100 * 1024;   // beyond: the streaming kernel (several CTAs per SM kept)

void apply_operator_device(vb_ctx *c, const double *x, double *y) {
  cudaStream_t s = c->stream;
  c->timing = getenv("VB_KERNEL_TIMING") && atoi(getenv("VB_KERNEL_TIMING"));
  const int stride = c->nv_max + c->np;
  const double *xin = x;
  if (c->nranks > 1) {
    SolveState *st = get_state(c);
    VB_REQUIRE(st->ready, VB_ESTATE, "multi-rank operator needs vb_factor first (exchange plans)");
    dev_scatter(x, c->d_owned_free.p, (int64_t)c->owned_free.size(), c->w_xg.p, s);
    dof_halo(c, st, c->w_xg.p);
    xin = c->w_xg.p;
  }
  if (!c->d_elAp.p) {   // packed lower triangles of the element matrices (once per context)
    const int64_t slot = k7_slot(c->nv_max);
    c->d_elAp.alloc(std::max<int64_t>((int64_t)c->nKl * slot, 1));
    if (c->nKl)
      pack_element_lower_kernel<<<dim3(16, c->nKl), 256, 0, s>>>(c->d_elA.p, c->d_cell_nv.p, c->nv_max, slot,
                                                                  c->d_elAp.p);
    VB_STAGE();
  }
  const int64_t slot = k7_slot(c->nv_max);
  const size_t smem = (size_t)(stride + c->nv_max + K7_WARPS * c->nv_max) * sizeof(double);
  const size_t smem_bulk = (size_t)(((slot + 1) & ~1LL) + (int64_t)c->np * c->nv_max + stride) * sizeof(double);
  SolveState *st = get_state(c);
  tick(c, st, 5, true);
  // pipelined persistent kernel: nst stages per CTA, ctas CTAs per SM (VB_K7_STAGES / VB_K7_CTAS /
  // VB_K7_PIPE=0 experiment knobs; default 2 stages x 3 CTAs per SM, 6 consumer warps, when they
  // fit, else fewer: profiles/r02z_k7_sweep.txt)
  const int stage_dbl = (int)(((slot + 1) & ~1LL) + (((int64_t)c->np * c->nv_max + 1) & ~1LL) + ((stride + 1) & ~1));
  const size_t stage_b = (size_t)stage_dbl * sizeof(double), smem_sm = 220 * 1024;
  int ctas = getenv("VB_K7_CTAS") ? std::max(1, atoi(getenv("VB_K7_CTAS"))) : 3;
  int nst = getenv("VB_K7_STAGES") ? std::max(1, atoi(getenv("VB_K7_STAGES"))) : 2;
  while (ctas > 1 && (size_t)ctas * (2 * stage_b + 1024) > smem_sm) --ctas;
  nst = (int)std::min<size_t>(std::min(nst, K7P_MAXST), (smem_sm / ctas - 1024) / stage_b);
  const bool stream_only = getenv("VB_K7_STREAM") && atoi(getenv("VB_K7_STREAM"));
  const bool pipe = !(getenv("VB_K7_PIPE") && !atoi(getenv("VB_K7_PIPE")));
  const int pipe_ver = getenv("VB_K7_PIPE") ? atoi(getenv("VB_K7_PIPE")) : 1;
  if (!stream_only && pipe_ver == 2 && c->nv_max <= 128) {
    const int mx = (c->nv_max + 31) / 32;
    const int cons2 = (mx == 4 || (getenv("VB_K7_CONS") && atoi(getenv("VB_K7_CONS")) >= 256)) ? 256 : 192;
    const size_t red_b = 2 * (size_t)(stride + (cons2 / 32) * c->nv_max) * sizeof(double);
    int ctas2 = getenv("VB_K7_CTAS") ? std::max(1, atoi(getenv("VB_K7_CTAS"))) : 3;
    while (ctas2 > 1 && (size_t)ctas2 * (2 * stage_b + red_b + 1024) > smem_sm) --ctas2;
    int nst2 = getenv("VB_K7_STAGES") ? std::max(1, atoi(getenv("VB_K7_STAGES"))) : 2;
    nst2 = (int)std::min<size_t>(std::min(nst2, K7P_MAXST), (smem_sm / ctas2 - 1024 - red_b) / stage_b);
    VB_REQUIRE(nst2 >= 1, VB_EINVAL, "K7 pipe2: a stage does not fit in shared memory");
    auto pk2 = mx == 4 ? elem_apply_pipe2_kernel<4, 8> : cons2 == 256 ? elem_apply_pipe2_kernel<3, 8> : elem_apply_pipe2_kernel<3, 6>;
    raise_smem_limit((const void *)pk2, nst2 * stage_b + red_b);
    const int64_t grid = std::min<int64_t>(c->nKl, (int64_t)148 * ctas2);
    const int xstride = (stride + 1) & ~1;
    elem_xgather_kernel<<<grid_for(c->nKl * xstride), 256, 0, s>>>(c->d_cell_l2g.p, c->d_vel2free.p, c->d_cell_nv.p,
                                                                   c->d_cell_gid.p, c->nv_max, c->np, c->nKl,
                                                                   c->n_free_vel, xstride, xin, c->w_elx.p);
    pk2<<<(unsigned)grid, cons2 + 32, nst2 * stage_b + red_b, s>>>(c->d_elAp.p, slot, c->d_elB.p, c->w_elx.p,
                                                                   c->d_cell_nv.p, c->nv_max, c->np, c->nKl,
                                                                   c->w_elt.p, nst2, stage_dbl);
  } else if (!stream_only && pipe && nst >= 2) {
    const int tpr = getenv("VB_K7_TPR") ? atoi(getenv("VB_K7_TPR")) : 2;
    const int cons = getenv("VB_K7_CONS") ? std::min(512, std::max(32, atoi(getenv("VB_K7_CONS")) / 32 * 32)) : 192;
    auto pk = tpr == 4 ? elem_apply_pipe_kernel<4> : tpr == 8 ? elem_apply_pipe_kernel<8> : elem_apply_pipe_kernel<2>;
    raise_smem_limit((const void *)pk, nst * stage_b);
    const int64_t grid = std::min<int64_t>(c->nKl, (int64_t)148 * ctas);   // B200: 148 SMs
    const int xstride = (stride + 1) & ~1;
    elem_xgather_kernel<<<grid_for(c->nKl * xstride), 256, 0, s>>>(c->d_cell_l2g.p, c->d_vel2free.p, c->d_cell_nv.p,
                                                                   c->d_cell_gid.p, c->nv_max, c->np, c->nKl,
                                                                   c->n_free_vel, xstride, xin, c->w_elx.p);
    pk<<<(unsigned)grid, cons + 32, nst * stage_b, s>>>(
        c->d_elAp.p, slot, c->d_elB.p, c->w_elx.p, c->d_cell_nv.p, c->nv_max, c->np, c->nKl, c->w_elt.p, nst,
        stage_dbl, getenv("VB_K7_NOCOMPUTE") && atoi(getenv("VB_K7_NOCOMPUTE")));
  } else if (smem_bulk <= kK7BulkSmem && !stream_only) {
    const int tpr = getenv("VB_K7_TPR") ? atoi(getenv("VB_K7_TPR")) : 2;
    const int thr = getenv("VB_K7_THREADS") ? std::min(512, std::max(32, atoi(getenv("VB_K7_THREADS")) / 32 * 32)) : 256;
    auto kern = tpr == 1 ? elem_apply_bulk_kernel<1> : tpr == 4 ? elem_apply_bulk_kernel<4> : elem_apply_bulk_kernel<2>;
    raise_smem_limit((const void *)kern, smem_bulk);
    kern<<<c->nKl, thr, smem_bulk, s>>>(
        c->d_elAp.p, slot, c->d_elB.p, c->d_cell_l2g.p, c->d_vel2free.p, c->d_cell_nv.p, c->d_cell_gid.p, c->nv_max,
        c->np, c->nKl, c->n_free_vel, xin, c->w_elt.p);
  } else {
    raise_smem_limit((const void *)elem_apply_packed_kernel, smem);
    elem_apply_packed_kernel<<<c->nKl, K7_WARPS * 32, smem, s>>>(c->d_elAp.p, slot, c->d_elB.p, c->d_cell_l2g.p,
                                                                 c->d_vel2free.p, c->d_cell_nv.p, c->d_cell_gid.p,
                                                                 c->nv_max, c->np, c->nKl, c->n_free_vel, xin,
                                                                 c->w_elt.p);
  }
  tick(c, st, 5, false);
  VB_STAGE();
  element_gather(c, c->w_elt.p, y);
  if (c->timing) collect_times(c, st);
}

void lanczos_extremes(const std::vector<double> &al, const std::vector<double> &be, double *lmin, double *lmax);

__global__ void residual_kernel(const double *__restrict__ b, double *y, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = b[i] - y[i];
}

// ||b - K x|| / ||b|| of the full saddle system through K7 (SURVEY §8(c) "true full-system
// residual"; vb_set_option "true_residual"); b, x in the ABI layout (owned free DOFs)
static double true_relative_residual(vb_ctx *c, const double *b, const double *x) {
  cudaStream_t s = c->stream;
  const int64_t n = (int64_t)c->owned_free.size();
  DBuf<double> y, nn;
  y.alloc(std::max<int64_t>(n, 1));
  nn.alloc(2);
  apply_operator_device(c, x, y.p);
  residual_kernel<<<grid_for(n), 256, 0, s>>>(b, y.p, n);
  DBuf<double> part;
  part.alloc(DOT_BLOCKS);
  dot_partial_kernel<<<DOT_BLOCKS, 256, 0, s>>>(y.p, y.p, nullptr, n, part.p);
  dot_final_kernel<<<1, 32, 0, s>>>(part.p, DOT_BLOCKS, nn.p);
  dot_partial_kernel<<<DOT_BLOCKS, 256, 0, s>>>(b, b, nullptr, n, part.p);
  dot_final_kernel<<<1, 32, 0, s>>>(part.p, DOT_BLOCKS, nn.p + 1);
  VB_STAGE();
  allreduce_sum_fixed(c, nn.p, 2);
  double h[2];
  VB_CUDA(cudaMemcpyAsync(h, nn.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaStreamSynchronize(s));
  return h[1] > 0 ? sqrt(h[0] / h[1]) : sqrt(h[0]);
}

// one PCG step up to the stopping test: q = S^ p, pq, x/r update fused with r.r, check (SURVEY O-15)
static void pcg_step(vb_ctx *c, SolveState *st, cudaGraphConditionalHandle hw, bool graph) {
  cudaStream_t s = c->stream;
  double *sc = c->w_scal.p;
  const int64_t nx = c->nx;
  apply_S(c, st, true);                                   // q = S^ p and p.q
  // x, r update fused with r.r; one rank: the last block also runs the stopping test
  const int check = c->nranks == 1 ? (graph ? 1 : 0) : -1;
  launch_pdl(st, update_xr_rr_kernel, dim3(DOT_BLOCKS), dim3(256), 0, s, c->w_x.p, c->w_r.p, c->w_p.p, c->w_q.p,
             c->nranks > 1 ? st->mask.p : nullptr, nx, sc, c->w_dots.p, st->ticket.p, sc + 2, st->hist.p, hw,
             check);
  if (check < 0) {
    allreduce_sum_fixed(c, sc + 2, 1);
    launch_pdl(st, pcg_check_kernel, dim3(1), dim3(1), 0, s, sc, st->hist.p, hw, graph ? 1 : 0);
  }
  VB_STAGE();
}

// the rest of the step: z = M^-1 r, rz, p update, beta and rz rotation
static void pcg_mstep(vb_ctx *c, SolveState *st) {
  cudaStream_t s = c->stream;
  double *sc = c->w_scal.p;
  const int64_t nx = c->nx;
  apply_M(c, st, false);
  dot_rz(c, st, sc + 3);
  launch_pdl(st, update_p_kernel, dim3(grid_for(nx)), dim3(256), 0, s, c->w_p.p, c->w_z.p, nx, sc, 0, st->hist.p,
             st->ticket.p);
  VB_STAGE();
}

// graphs need a capturable transport (no host synchronisation inside the iteration)
static bool use_graph(const vb_ctx *c) {
  if (getenv("VB_NO_GRAPH") && atoi(getenv("VB_NO_GRAPH"))) return false;
  if (c->timing) return false;   // event records are not allowed inside conditional graph bodies
  if (getenv("VB_PCG_TRACE") && atoi(getenv("VB_PCG_TRACE"))) return false;
  return c->nranks == 1 || c->comm->capturable();
}

// WHILE(status == 0) { z = M^-1 r, beta, p; q = S^ p, alpha, x, r, stopping test } -- the first
// S-part runs before the graph, so no step is wasted at convergence.
static void build_iteration_graph(vb_ctx *c, SolveState *st) {
  // capture on the library's own stream (the caller's may be the legacy default stream, which
  // cannot be captured); kernels launched on c->stream during capture go to sg
  cudaStream_t s = st->sg, user = c->stream;
  c->stream = s;
  cudaGraph_t g;
  VB_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  VB_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  VB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  st->capturing = true;
  try {
    VB_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    pcg_mstep(c, st);
    pcg_step(c, st, hw, true);
    VB_CUDA(cudaStreamEndCapture(s, &body));
  } catch (...) {
    st->capturing = false;
    c->stream = user;
    cudaGraph_t dummy;
    cudaStreamEndCapture(s, &dummy);
    (void)cudaGetLastError();
    cudaGraphDestroy(g);
    throw;
  }
  st->capturing = false;
  c->stream = user;
  cudaError_t e = cudaGraphInstantiate(&st->gexec, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess && st->pdl) {     // programmatic edges not accepted here: capture without them
    (void)cudaGetLastError();
    st->gexec = nullptr;
    st->pdl = false;
    build_iteration_graph(c, st);
    return;
  }
  VB_CUDA(e);
}

// B0 / B8 couplings (see coupling_cell_kernel): mode 0 zG = -K_GD x_D, mode 1 t = K_DG u_G
static void coupling(vb_ctx *c, SolveState *st, int mode, const double *xin, double *out) {
  cudaStream_t s = c->stream;
  if (mode == 0) {
    coupling_scalar_kernel<0><<<c->N, 256, 0, s>>>(c->d_sub.p, c->d_mvec.p, c->d_b0.p, xin, c->d_subG_free.p, st->cscal.p);
    if (c->nKl)
      coupling_cell_kernel<0><<<c->nKl, 128, 0, s>>>(st->cell_sub.p, c->d_sub.p, c->d_cell_loc.p, c->d_cell_nv.p, c->d_elA.p,
                                                     c->d_elB.p, c->nv_max, c->np, xin, c->d_subG_free.p, st->ycell.p);
    coupling_gather_kernel<0><<<grid_for(c->len_G), 256, 0, s>>>(st->cp_ptr[0].p, st->cp_src[0].p, st->cp_rsub[0].p, c->d_sub.p,
                                                                  st->ycell.p, c->d_mvec.p, c->d_b0.p, st->cscal.p, c->len_G, out);
  } else {
    coupling_scalar_kernel<1><<<c->N, 256, 0, s>>>(c->d_sub.p, c->d_mvec.p, c->d_b0.p, xin, c->d_subG_free.p, st->cscal.p);
    if (c->nKl)
      coupling_cell_kernel<1><<<c->nKl, 128, 0, s>>>(st->cell_sub.p, c->d_sub.p, c->d_cell_loc.p, c->d_cell_nv.p, c->d_elA.p,
                                                     c->d_elB.p, c->nv_max, c->np, xin, c->d_subG_free.p, st->ycell.p);
    coupling_gather_kernel<1><<<grid_for(c->len_Dn), 256, 0, s>>>(st->cp_ptr[1].p, st->cp_src[1].p, st->cp_rsub[1].p, c->d_sub.p,
                                                                   st->ycell.p, c->d_mvec.p, c->d_b0.p, st->cscal.p, c->len_Dn, out);
  }
  VB_CHECK_LAUNCH();
}

void pcg_device(vb_ctx *c, const double *rhs_in, double *x_out, double rtol, int maxit, vb_report *rep) {
  prepare_solve(c);
  SolveState *st = get_state(c);
  cudaStream_t s = c->stream;
  c->timing = getenv("VB_KERNEL_TIMING") && atoi(getenv("VB_KERNEL_TIMING"));
  const bool trace = getenv("VB_PCG_TRACE") && atoi(getenv("VB_PCG_TRACE"));
  st->nev = 0;
  const int N = c->N;
  const int64_t nx = c->nx, NDelta = c->n_delta_glob;
  const int64_t nvf = c->n_free_vel;
  // multi-rank: work on global-layout free vectors (owned values + ghost interface values)
  const double *rhs = rhs_in;
  double *x = x_out;
  if (c->nranks > 1) {
    dev_scatter(rhs_in, c->d_owned_free.p, (int64_t)c->owned_free.size(), c->w_rhsg.p, s);
    dof_halo(c, st, c->w_rhsg.p);
    rhs = c->w_rhsg.p;
    x = c->w_xg.p;
  }
  // ---------------- B0: condensed rhs in transformed coordinates
  int64_t maxnG = 1, maxnD = 1;
  for (auto &S : c->h_sub) { maxnG = std::max<int64_t>(maxnG, S.nG); maxnD = std::max<int64_t>(maxnD, S.nD); }
  c->w_r.zero(s);
  rhs_D_kernel<<<N, 256, 0, s>>>(c->d_sub.p, c->d_subI_free.p, c->d_subP_glob.p, c->d_cvec.p, c->d_mvec.p, rhs, nvf,
                                 c->w_bD.p, c->w_r.p + NDelta + c->NPi, st->g0abs.p);
  run_sub_gemv(st, st->w_kd.p, st->nw_kd, st->sm_kd, st->big_kd, s);   // x_D = K_DD^-1 b_D (chunks)
  sum_chunks_kernel<<<(unsigned)((c->len_Dn + 31) / 32), 256, 0, s>>>(c->w_yDp.p, c->len_Dn, c->P_kd, c->len_Dn, c->w_xD.p);
  coupling(c, st, 0, c->w_xD.p, st->gbuf.p);                             // zG = -K_GD x_D
  VB_STAGE();
  dev_gather(rhs, c->d_gam_free.p, c->nGamma, st->gam2.p, s);                // b_e (entity-major)
  run_slot_exchange(c, st->XB, st->gbuf.p, st->gbuf.p + c->len_G);          // C1 (cross-rank zG)
  run_entity_sum(c, st->ESB, st->gbuf.p, c->w_gam.p, st->gam2.p);             // ghat = b + sum_m zG^(m)
  if (!c->h_ent.empty())
    gamma_rhs_kernel<<<c->h_ent.size(), 512, 0, s>>>(c->d_ent.p, c->d_T.p, c->w_gam.p, NDelta, c->w_r.p);
  if (!c->neumann) {   // with Neumann faces the p_0 rows carry no compatibility condition (A35)
    p0_compat_kernel<<<1, 32, 0, s>>>(c->w_r.p + NDelta + c->NPi, N, c->w_dots.p + W_P0, 0, c->Ng, st->g0abs.p);
    allreduce_sum_fixed(c, c->w_dots.p + W_P0, 2);
    p0_compat_kernel<<<1, 32, 0, s>>>(c->w_r.p + NDelta + c->NPi, N, c->w_dots.p + W_P0, 1, c->Ng, st->g0abs.p);
  }
  VB_STAGE();
  // ---------------- PCG (SURVEY O-15), iterations driven on the device (scal[6] = it, scal[7] = status)
  c->w_x.zero(s);
  double *sc = c->w_scal.p;
  dot(c, c->w_r.p, c->w_r.p, nx, sc + 2);
  pcg_init_kernel<<<1, 1, 0, s>>>(sc, rtol, maxit);
  double h[9], compat[2];
  VB_CUDA(cudaMemcpyAsync(h, sc, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaMemcpyAsync(compat, c->w_dots.p + W_P0, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaStreamSynchronize(s));
  // flux compatibility of the rhs: sum_i g0_i = 0 up to rounding, else VB_EINVAL
  // scale: the terms g0 is summed from, plus ||r0|| (rounding-level pressure data, e.g. a lifted trace
  // with u.n = 0 on the boundary, makes both sides pure rounding)
  VB_REQUIRE(c->neumann || fabs(compat[0]) <= kCompatRel * (compat[1] + h[4]), VB_EINVAL,
             "flux-incompatible rhs: sum_i g0_i = " + std::to_string(compat[0]) + " (sum_i |g0_i| = " +
                 std::to_string(compat[1]) + "); the pressure rows must integrate to zero against constants");
  const double r0n = h[4];
  if (trace) fprintf(stderr, "[vb rank %d] rr0 %.17g\n", c->rank, h[2]);
  if (h[7] == 0.0) {
    apply_M(c, st, false);
    dot_rz(c, st, sc + 0);
    update_p_kernel<<<grid_for(nx), 256, 0, s>>>(c->w_p.p, c->w_z.p, nx, sc, 1, st->hist.p, st->ticket.p);
    VB_STAGE();
    const bool graph = use_graph(c);
    while (true) {
      pcg_step(c, st, cudaGraphConditionalHandle{}, false);
      VB_CUDA(cudaMemcpyAsync(h, sc, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
      VB_CUDA(cudaStreamSynchronize(s));
      if (trace)
        fprintf(stderr, "[vb rank %d] it %d rz %.17g pq %.17g rr %.17g\n", c->rank, (int)h[6], h[0], h[1], h[2]);
      if (h[7] != 0.0) break;
      if (graph && !st->graph_broken) {   // the remaining steps as one graph launch, stopping on the device
        if (!st->gexec) {
          try {
            build_iteration_graph(c, st);
          } catch (const Error &e) {
            // e.g. a transport whose calls cannot be captured into a conditional body: keep
            // iterating host-driven (same kernels, same order; one host check per step)
            (void)cudaGetLastError();
            st->graph_broken = true;
            st->gexec = nullptr;
            fprintf(stderr, "[vb rank %d] iteration graph unavailable (%s); host-driven iterations\n", c->rank,
                    e.msg.c_str());
          }
        }
        if (st->gexec) {
          VB_CUDA(cudaEventRecord(st->ev_fork, s));
          VB_CUDA(cudaStreamWaitEvent(st->sg, st->ev_fork, 0));
          VB_CUDA(cudaGraphLaunch(st->gexec, st->sg));
          VB_CUDA(cudaEventRecord(st->ev_join, st->sg));
          VB_CUDA(cudaStreamWaitEvent(s, st->ev_join, 0));
          break;
        }
      }
      pcg_mstep(c, st);
    }
  }
  VB_CUDA(cudaMemsetAsync(c->w_dots.p + W_FLUX, 0, sizeof(double), s));
  flux_violation_kernel<<<(N + 7) / 8, 256, 0, s>>>(c->d_sub.p, N, c->d_b0T.p, c->d_loc2x.p, c->w_x.p,
                                                    c->w_dots.p + W_FLUX);
  VB_STAGE();
  double flux = 0.0;
  if (c->nranks > 1) {   // max over ranks
    if (c->w_red.n < (size_t)c->nranks) c->w_red.alloc(std::max(c->nranks, 8));
    c->comm->allgather(c->w_dots.p + W_FLUX, c->w_red.p, 1, s);
    std::vector<double> fl(c->nranks);
    VB_CUDA(cudaMemcpyAsync(fl.data(), c->w_red.p, c->nranks * sizeof(double), cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    for (double v : fl) flux = std::max(flux, v);
  } else {
    VB_CUDA(cudaMemcpyAsync(&flux, c->w_dots.p + W_FLUX, sizeof(double), cudaMemcpyDeviceToHost, s));
  }
  VB_CUDA(cudaMemcpyAsync(h, sc, 9 * sizeof(double), cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaStreamSynchronize(s));
  const int it = (int)h[6];
  const double rn = sqrt(h[2]);
  const int status = h[7] == 2.0 ? VB_EBREAKDOWN : (h[7] == 3.0 ? VB_ENOTCONV : VB_OK);
  std::vector<double> alphas, betas;
  {
    std::vector<double> hh(2 * 4096);
    VB_CUDA(cudaMemcpyAsync(hh.data(), st->hist.p, hh.size() * 8, cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    for (int j = 0; j < it && j < 4096; ++j) alphas.push_back(hh[2 * j]);
    for (int j = 0; j + 1 < it && j < 4096; ++j) betas.push_back(hh[2 * j + 1]);
  }
  // ---------------- B8: back to original coordinates and back-substitution
  if (!c->h_ent.empty())
    gamma_back_kernel<<<c->h_ent.size(), 512, 0, s>>>(c->d_ent.p, c->d_gam_free.p, c->d_T.p, c->w_x.p, NDelta,
                                                    c->w_gam.p, x);
  VB_STAGE();
  // u_D = x_D - K_DD^-1 (K_DG u_G): the coupling element by element into w_bD (b_D is spent), the packed
  // K_DD^-1 GEMV over it (same work list), then the update of x_D
  coupling(c, st, 1, x, c->w_bD.p);                                      // t = K_DG u_G
  run_sub_gemv(st, st->w_kd.p, st->nw_kd, st->sm_kd, st->big_kd, s);
  xd_update_kernel<<<grid_for(c->len_Dn), 256, 0, s>>>(c->w_xD.p, c->w_yDp.p, c->len_Dn, c->P_kd, c->len_Dn);
  xout_kernel<<<N, 256, 0, s>>>(c->d_sub.p, c->w_xD.p, c->d_subI_free.p, c->d_subP_glob.p, c->d_cvec.p, c->d_mvec.p,
                                c->w_x.p + NDelta + c->NPi, nvf, x);
  VB_STAGE();
  double *pm = c->w_dots.p + W_PM;
  if (!c->neumann) {   // zero-mean pressure gauge; the pressure is unique with Neumann faces
  pressure_mean_kernel<<<PM_BLOCKS, 256, 0, s>>>(c->d_cellgeo.p, c->d_cell_gid.p, c->geo_stride, c->np, c->nKl,
                                                 x + nvf, 0, pm, PM_BLOCKS);
  pressure_mean_kernel<<<1, 32, 0, s>>>(c->d_cellgeo.p, c->d_cell_gid.p, c->geo_stride, c->np, c->nKl, x + nvf, 1,
                                        pm, PM_BLOCKS);
  allreduce_sum_fixed(c, pm + 2 * PM_BLOCKS, 2);
  pressure_mean_kernel<<<grid_for(c->nKl), 256, 0, s>>>(c->d_cellgeo.p, c->d_cell_gid.p, c->geo_stride, c->np,
                                                        c->nKl, x + nvf, 2, pm, PM_BLOCKS);
  }
  VB_STAGE();
  if (c->nranks > 1) dev_gather(x, c->d_owned_free.p, (int64_t)c->owned_free.size(), x_out, s);
  double true_rel = -1.0;
  if (c->opt_true_residual && rep) true_rel = true_relative_residual(c, rhs_in, x_out);
  VB_CUDA(cudaStreamSynchronize(s));
  c->last_iterations = it;
  collect_times(c, st);
  if (rep) {
    rep->iterations = it;
    rep->converged = status == VB_OK;
    rep->r0_norm = r0n;
    rep->r_final_norm = rn;
    rep->rel_residual = r0n > 0 ? rn / r0n : 0.0;
    rep->true_rel_residual = true_rel;
    // Lanczos T from the CG coefficients (SURVEY O-15 index convention): beta_j pairs alpha_j, alpha_{j+1}
    std::vector<double> bb(betas.begin(), betas.end());
    double lmin = 1, lmax = 1;
    lanczos_extremes(alphas, bb, &lmin, &lmax);
    rep->lambda_min = lmin; rep->lambda_max = lmax; rep->kappa = lmin > 0 ? lmax / lmin : INFINITY;
    rep->bytes_per_iter_model = c->bytes_per_iter;
    rep->flux_violation_max = flux;
    rep->n_primal = c->NPi_g; rep->n_coarse = c->Nc;
    rep->n_dofs_paper = c->nvel + c->npres;
    rep->n_adaptive = c->n_adaptive;
    rep->adaptive_margin = c->adaptive_margin;
  }
  if (status != VB_OK)
    throw Error{(vb_status)status, status == VB_ENOTCONV ? "PCG reached maxit without converging"
                                                          : "PCG breakdown: p^T S p <= 0 or r^T z <= 0"};
}

// Debug/parity entry: y = S^ x (which = 0) or y = M^-1 x (which = 1) in ORIGINAL interface
// coordinates (entity-major order of vb_interface_dofs) followed by the N p0 entries.
void debug_interface_op(vb_ctx *c, int which, const double *in, double *out) {
  prepare_solve(c);
  SolveState *st = get_state(c);
  cudaStream_t s = c->stream;
  const int64_t NDelta = c->n_delta_glob, ng = c->nGamma, N = c->N;
  DBuf<double> gin, gout, dummy;
  gin.alloc(ng + N);
  gout.alloc(ng + N);
  dummy.alloc(c->n_free_vel + 1);
  VB_CUDA(cudaMemcpyAsync(gin.p, in, (ng + N) * 8, cudaMemcpyHostToDevice, s));
  double *dst = which == 0 ? c->w_p.p : c->w_r.p;
  gamma_rhs_kernel<<<c->h_ent.size(), 128, 0, s>>>(c->d_ent.p, c->d_T.p, gin.p, NDelta, dst);
  VB_CUDA(cudaMemcpyAsync(dst + NDelta + c->NPi, gin.p + ng, N * 8, cudaMemcpyDeviceToDevice, s));
  VB_STAGE();
  const double *res;
  if (which == 0) { apply_S(c, st); res = c->w_q.p; }
  else { apply_M(c, st); res = c->w_z.p; }
  // back to original coordinates; gamma_back writes gam (entity-major) and a scatter we discard
  DBuf<int64_t> ident;
  std::vector<int64_t> id(ng);
  for (int64_t i = 0; i < ng; ++i) id[i] = i;
  ident.upload(id, s);
  gamma_back_kernel<<<c->h_ent.size(), 128, 0, s>>>(c->d_ent.p, ident.p, c->d_T.p, res, NDelta, gout.p, dummy.p);
  VB_STAGE();
  VB_CUDA(cudaMemcpyAsync(out, gout.p, ng * 8, cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaMemcpyAsync(out + ng, res + NDelta + c->NPi, N * 8, cudaMemcpyDeviceToHost, s));
  VB_CUDA(cudaStreamSynchronize(s));
}

// Parity/debug (setup-stage gates of SURVEY §8(c)): dense operators of local subdomain `sub` in
// ORIGINAL local interface coordinates (its entities in slot order, each entity's free velocity
// DOFs in increasing id; ids[] returns that order):
//   which 0: S_Gamma^(i) = T S_T T^T from the packed S_T (T orthogonal, reading A9);
//   which 1: the deluxe-scaled local dual operator N (D S_DD^-1 D^T) N^T from the packed
//            D S_DD^-1 D^T (basis invariant: any orthonormal dual basis N_G gives the same matrix).
// out: nG x nG column-major, or NULL to query *n (and ids).
void debug_subdomain_op(vb_ctx *c, int sub, int which, int64_t *ids, double *out, int64_t *n) {
  VB_REQUIRE(sub >= 0 && sub < c->N, VB_EINVAL, "subdomain index out of range");
  VB_REQUIRE(which == 0 || which == 1, VB_EINVAL, "which must be 0 (S_Gamma) or 1 (local dual operator)");
  const SubDev &S = c->h_sub[sub];
  const int nG = S.nG;
  *n = nG;
  if (ids)
    for (int q = S.slot_begin; q < S.slot_end; ++q) {
      const SlotDev &sl = c->h_slot[c->h_sub_slots[q]];
      const auto &dofs = c->ents[sl.ent].dofs;
      for (int a = 0; a < sl.n; ++a) ids[sl.offG + a] = dofs[a];
    }
  if (!out) return;
  cudaStream_t s = c->stream;
  const int m = which == 0 ? nG : S.nd;
  std::vector<double> pk(packed_size(m));
  const double *src = which == 0 ? c->d_STp.p + S.off_STp : c->d_SDi.p + S.off_SDi;
  VB_CUDA(cudaMemcpyAsync(pk.data(), src, pk.size() * 8, cudaMemcpyDeviceToHost, s));
  std::vector<double> M((size_t)m * m, 0.0), T((size_t)nG * m, 0.0);
  for (int q = S.slot_begin; q < S.slot_end; ++q) {
    const SlotDev &sl = c->h_slot[c->h_sub_slots[q]];
    std::vector<double> Te((size_t)sl.n * sl.n);
    VB_CUDA(cudaMemcpyAsync(Te.data(), c->d_T.p + sl.off_T, Te.size() * 8, cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    for (int a = 0; a < sl.n; ++a) {
      for (int j = 0; j < sl.nd; ++j) T[(size_t)(sl.offD + j) * nG + sl.offG + a] = Te[a + (size_t)j * sl.n];
      if (which == 0)
        for (int j = 0; j < sl.r; ++j)
          T[(size_t)(S.nd + sl.offPi + j) * nG + sl.offG + a] = Te[a + (size_t)(sl.nd + j) * sl.n];
    }
  }
  VB_CUDA(cudaStreamSynchronize(s));
  const int nt = (m + 31) / 32;
  for (int I = 0; I < nt; ++I)
    for (int J = 0; J <= I; ++J) {
      const double *t = pk.data() + ptile_off(m, I, J);
      const int rows = (I == nt - 1) ? m - 32 * (nt - 1) : 32;
      for (int r = 0; r < rows; ++r)
        for (int cc = 0; cc < 32; ++cc) {
          const int i = 32 * I + r, j = 32 * J + cc;
          if (j >= m || j > i) continue;
          M[(size_t)j * m + i] = M[(size_t)i * m + j] = t[r * 32 + cc];
        }
    }
  std::vector<double> TM((size_t)nG * m, 0.0);   // T M
  for (int j = 0; j < m; ++j)
    for (int k = 0; k < m; ++k) {
      const double mk = M[(size_t)j * m + k];
      if (mk == 0.0) continue;
      for (int i = 0; i < nG; ++i) TM[(size_t)j * nG + i] += T[(size_t)k * nG + i] * mk;
    }
  for (int j = 0; j < nG; ++j)   // out = (T M) T^T
    for (int i = 0; i < nG; ++i) {
      double v = 0.0;
      for (int k = 0; k < m; ++k) v += TM[(size_t)k * nG + i] * T[(size_t)k * nG + j];
      out[(size_t)j * nG + i] = v;
    }
}

// Extreme eigenvalues of the Lanczos tridiagonal (symmetric QL on the host; m <= maxit scalars).
void lanczos_extremes(const std::vector<double> &al, const std::vector<double> &be, double *lmin, double *lmax) {
  int m = al.size();
  if (m == 0) { *lmin = *lmax = 1; return; }
  std::vector<double> d(m), e(m, 0.0);
  for (int j = 0; j < m; ++j) {
    d[j] = 1.0 / al[j] + (j > 0 ? be[j - 1] / al[j - 1] : 0.0);
    if (j > 0) e[j - 1] = sqrt(be[j - 1]) / al[j - 1];
  }
  // implicit QL (tqli)
  for (int l = 0; l < m; ++l) {
    int iter = 0, mm;
    do {
      for (mm = l; mm < m - 1; ++mm) {
        double dd = fabs(d[mm]) + fabs(d[mm + 1]);
        if (fabs(e[mm]) <= 1e-15 * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? fabs(r) : -fabs(r)));
        double sn = 1.0, cs = 1.0, p = 0.0;
        int i;
        for (i = mm - 1; i >= l; --i) {
          double f = sn * e[i], b = cs * e[i];
          e[i + 1] = (r = hypot(f, g));
          if (r == 0.0) { d[i + 1] -= p; e[mm] = 0.0; break; }
          sn = f / r; cs = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * sn + 2.0 * cs * b;
          d[i + 1] = g + (p = sn * r);
          g = cs * r - b;
        }
        if (r == 0.0 && i >= l) continue;
        d[l] -= p; e[l] = g; e[mm] = 0.0;
      }
    } while (mm != l);
  }
  *lmin = *std::min_element(d.begin(), d.end());
  *lmax = *std::max_element(d.begin(), d.end());
}

}  // namespace vb
