// Solve stage: rhs condensation, the PCG loop on the interface saddle problem
// Eq.(globInt) with the BDDC preconditioner Eq.(BDDCprec), back-substitution
// and the element-by-element saddle operator.
//
// PCG vectors live in transformed interface coordinates x = [dual coords per entity | u_Pi | p_0];
// T_G is orthogonal, so Euclidean norms, CG coefficients and the stopping test equal those of the
// original coordinates.
#include <algorithm>
#include <cmath>
#include "dense.cuh"
#include "setup.h"

namespace vb {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// ------------------------------------------------------------------ packed symmetric GEMV (K3)
// Work item: one CTA multiplies the tile rows [r0, r1) of one packed symmetric matrix with x and
// writes a full-length partial result.  Row contributions of a tile row are reduced in fixed warp
// order; column contributions of one tile row go to distinct tile columns (one warp each), so the
// accumulation order is fixed: the kernel is deterministic.
struct GemvWork {
  const double *M;        // packed tiles
  const int64_t *map;     // x gather map (or null: x contiguous at xsrc)
  const double *xsrc;
  double *out;            // partial output (length n)
  int n, r0, r1, pad;
};

constexpr int GV_WARPS = 4;      // subdomain matrices (several CTAs per SM)
constexpr int GV_WARPS_C = 8;    // the single coarse matrix (one CTA per SM)

template <int GV_WARPS>
__global__ void __launch_bounds__(GV_WARPS * 32) sym_gemv_kernel(const GemvWork *__restrict__ work) {
  extern __shared__ double sm[];
  const GemvWork W = work[blockIdx.x];
  const int n = W.n, nt = (n + 31) / 32;
  const int npad = nt * 32;
  double *xs = sm;              // npad
  double *ys = sm + npad;       // npad
  double *rowred = ys + npad;   // GV_WARPS * 32
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < npad; j += blockDim.x) {
    double v = 0.0;
    if (j < n) v = W.map ? W.xsrc[W.map[j]] : W.xsrc[j];
    xs[j] = v;
    ys[j] = 0.0;
  }
  __syncthreads();
  for (int I = W.r0; I < W.r1; ++I) {
    const double *rowbase = W.M + ((int64_t)I * (I + 1) / 2) * 1024;
    double rsum[32];
#pragma unroll
    for (int r = 0; r < 32; ++r) rsum[r] = 0.0;
    const double xI_lane = xs[32 * I + lane];
    for (int J = warp; J <= I; J += GV_WARPS) {
      const double *T = rowbase + (int64_t)J * 1024;
      double t[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) t[r] = __ldg(T + r * 32 + lane);
      const double xJ = xs[32 * J + lane];
      double csum = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        rsum[r] += t[r] * xJ;
        csum += t[r] * __shfl_sync(FULL, xI_lane, r);
      }
      if (J < I) ys[32 * J + lane] += csum;   // transpose contribution, one warp per J
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
      ys[32 * I + lane] += v;
    }
    __syncthreads();
  }
  for (int j = tid; j < n; j += blockDim.x) W.out[j] = ys[j];
}

static size_t gemv_smem(int nmax, int warps = GV_WARPS) {
  return (size_t)(2 * ((nmax + 31) / 32) * 32 + warps * 32) * sizeof(double);
}

// split a packed matrix of n into P chunks of tile rows balanced by tile count
static void split_rows(int n, int P, std::vector<std::pair<int, int>> &out) {
  int nt = (n + 31) / 32;
  int64_t total = (int64_t)nt * (nt + 1) / 2;
  out.clear();
  int r = 0;
  for (int p = 0; p < P && r < nt; ++p) {
    int64_t target = total * (p + 1) / P;
    int r1 = r;
    while (r1 < nt && (int64_t)(r1 + 1) * (r1 + 2) / 2 <= target) ++r1;
    if (r1 == r) r1 = r + 1;
    if (p == P - 1) r1 = nt;
    out.push_back({r, r1});
    r = r1;
  }
  while ((int)out.size() < P) out.push_back({nt, nt});
}

// ------------------------------------------------------------------ small kernels of the loop
// q_x[g] = sum over local copies and over the P partial chunks (deterministic order)
__global__ void gather_sum_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                  const double *__restrict__ part, int64_t part_stride, int P, int64_t n,
                                  double *out) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int64_t q = ptr[g]; q < ptr[g + 1]; ++q) {
      const int64_t j = idx[q];
      for (int c = 0; c < P; ++c) v += part[c * part_stride + j];
    }
    out[g] = v;
  }
}

// b0 coupling: q_Pi += sum_i b0T_i p0_i  (into the partial of chunk 0), q0_i = b0T_i . u_Pi^(i)
__global__ void b0_apply_kernel(const SubDev *__restrict__ subs, const int64_t *__restrict__ loc2x,
                                const double *__restrict__ b0T, const double *__restrict__ p,
                                int64_t p0off, double *part0, double *q) {
  const SubDev S = subs[blockIdx.x];
  const double p0 = p[p0off + blockIdx.x];
  double acc = 0.0;
  for (int a = threadIdx.x; a < S.npi; a += 32) {
    const int64_t j = S.off_G + S.nd + a;
    const double b = b0T[S.off_Pi + a];
    part0[j] += b * p0;
    acc += b * p[loc2x[j]];
  }
  acc = warp_sum(acc);
  if (threadIdx.x == 0) q[p0off + blockIdx.x] = acc;
}

// block partial dot products (fixed grid) -> part[blockIdx]
__global__ void dot_partial_kernel(const double *__restrict__ a, const double *__restrict__ b, int64_t n, double *part) {
  __shared__ double red[32];
  double v = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) v += a[i] * b[i];
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
__global__ void update_xr_kernel(double *x, double *r, const double *p, const double *q, int64_t n, const double *scal) {
  const double alpha = scal[0] / scal[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    r[i] -= alpha * q[i];
  }
}

__global__ void update_p_kernel(double *p, const double *z, int64_t n, double *scal, int first) {
  const double beta = first ? 0.0 : scal[3] / scal[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

__global__ void rotate_rz_kernel(double *scal, double *hist, int it) {
  // record alpha_it, beta_it and rotate rz <- rz_new
  hist[2 * it + 0] = scal[0] / scal[1];
  hist[2 * it + 1] = scal[3] / scal[0];
  scal[0] = scal[3];
}

// restriction with deluxe scaling: rD^(sub)[offD+j] = sum_i D^(sub)[i, j] r_x[off_xd + i]  (D^T r).
// D is stored as row-major 32x32 tiles (zero padded): a warp streams one contiguous 8 KB tile with
// lane = tile column, so the column sums need no cross-lane reduction; per-warp partials are
// summed in fixed order (deterministic).  One CTA per active (entity, sharer) slot.
constexpr int DLX_WARPS = 4;
__global__ void __launch_bounds__(DLX_WARPS * 32) restrict_kernel(const SlotDev *__restrict__ slots,
                                const int *__restrict__ act, const EntDev *__restrict__ ents,
                                const SubDev *__restrict__ subs, const double *__restrict__ Dt,
                                const double *__restrict__ r, double *rD) {
  extern __shared__ double sh[];
  const SlotDev s = slots[act[blockIdx.x]];
  const int nd = s.nd;
  const int nt = (nd + 31) / 32, npad = nt * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *xs = sh;                  // npad
  double *part = sh + npad;         // nw * npad
  const double *D = Dt + s.off_Dt;
  const double *re = r + ents[s.ent].off_xd;
  for (int i = threadIdx.x; i < npad; i += blockDim.x) xs[i] = i < nd ? re[i] : 0.0;
  for (int i = threadIdx.x; i < nw * npad; i += blockDim.x) part[i] = 0.0;
  __syncthreads();
  for (int u = warp; u < nt * nt; u += nw) {
    const int I = u / nt, J = u % nt;
    const double *T = D + (int64_t)u * 1024;
    double t[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) t[rr] = __ldg(T + rr * 32 + lane);
    double acc = 0.0;
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) acc += t[rr] * xs[32 * I + rr];
    part[warp * npad + 32 * J + lane] += acc;
  }
  __syncthreads();
  double *out = rD + subs[s.sub].off_Dv + s.offD;
  for (int j = threadIdx.x; j < nd; j += blockDim.x) {
    double v = 0.0;
    for (int w = 0; w < nw; ++w) v += part[w * npad + j];
    out[j] = v;
  }
}

// c_i = Phi_i^T rD_i (coarse rhs pieces): PHIT_SPLIT CTAs per subdomain, warp per primal column
constexpr int PHIT_SPLIT = 4;
__global__ void __launch_bounds__(256) phit_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Phi,
                            const double *__restrict__ rD, double *cpart) {
  const SubDev S = subs[blockIdx.y];
  const double *F = Phi + S.off_Phi;
  const double *x = rD + S.off_Dv;
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

// rc[pi] = r_Pi[pi] + sum over copies c_i; rc[NPi + i] = r0_i
__global__ void coarse_rhs_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                  const double *__restrict__ cpart, const double *__restrict__ r,
                                  int64_t NDelta, int64_t NPi, int N, double *rc) {
  const int64_t n = NPi + N;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < n; g += (int64_t)gridDim.x * blockDim.x) {
    double v = r[NDelta + g];
    if (g < NPi)
      for (int64_t q = ptr[g]; q < ptr[g + 1]; ++q) v += cpart[idx[q]];
    rc[g] = v;
  }
}

// p0 projections of the coarse problem (gauge sum vol_i p0_i = 0, A5):
// mode 0 (input):  rc_p0 -= vol * (sum rc_p0) / sum vol ;  mode 1 (output): uc_p0 -= (vol . uc_p0)/sum vol
__global__ void coarse_p0_project_kernel(const SubDev *__restrict__ subs, int N, double *v, int mode) {
  __shared__ double red[32];
  double a = 0.0, w = 0.0;
  for (int i = threadIdx.x; i < N; i += blockDim.x) {
    a += mode == 0 ? v[i] : subs[i].vol * v[i];
    w += subs[i].vol;
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
  for (int i = threadIdx.x; i < N; i += blockDim.x) v[i] -= mode == 0 ? subs[i].vol * mean : mean;
}

// w_i = sum_chunks y_i + Phi_i u_Pi^(i)   (thread per row of column-major Phi, 4 accumulators)
__global__ void __launch_bounds__(128) local2_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Phi,
                              const double *__restrict__ part, int64_t part_stride, int P,
                              const int64_t *__restrict__ pi_glob, const double *__restrict__ uc, double *w) {
  const SubDev S = subs[blockIdx.y];
  const double *F = Phi + S.off_Phi;
  extern __shared__ double us[];
  for (int a = threadIdx.x; a < S.npi; a += blockDim.x) us[a] = uc[pi_glob[S.off_Pi + a]];
  __syncthreads();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= S.nd) return;
  double v = 0.0;
  for (int c = 0; c < P; ++c) v += part[c * part_stride + S.off_Dv + j];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int a = 0;
  for (; a + 3 < S.npi; a += 4) {
    a0 += F[j + (int64_t)a * S.nd] * us[a];
    a1 += F[j + (int64_t)(a + 1) * S.nd] * us[a + 1];
    a2 += F[j + (int64_t)(a + 2) * S.nd] * us[a + 2];
    a3 += F[j + (int64_t)(a + 3) * S.nd] * us[a + 3];
  }
  for (; a < S.npi; ++a) a0 += F[j + (int64_t)a * S.nd] * us[a];
  w[S.off_Dv + j] = v + ((a0 + a1) + (a2 + a3));
}

// extension with deluxe scaling: z_x[off_xd + i] = sum_m sum_j D^(m)[i, j] w^(m)[offD_m + j];
// warps stream (side, 32x32 row-major tile) units, lane = tile column; the row sums come from a
// transpose-reduce; per-warp row partials are summed in fixed order.  One CTA per active entity.
__global__ void __launch_bounds__(DLX_WARPS * 32) extend_kernel(const EntDev *__restrict__ ents,
                              const int *__restrict__ act, const SlotDev *__restrict__ slots,
                              const SubDev *__restrict__ subs, const double *__restrict__ Dt,
                              const double *__restrict__ w, double *z) {
  extern __shared__ double sh[];
  const EntDev E = ents[act[blockIdx.x]];
  const int nd = E.nd;
  const int nt = (nd + 31) / 32, npad = nt * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double *ws = sh;                        // nsides * npad
  double *part = sh + E.nsides * npad;    // nw * npad
  for (int q = 0; q < E.nsides; ++q) {
    const SlotDev s = slots[E.side_begin + q];
    const double *src = w + subs[s.sub].off_Dv + s.offD;
    for (int i = threadIdx.x; i < npad; i += blockDim.x) ws[q * npad + i] = i < nd ? src[i] : 0.0;
  }
  for (int i = threadIdx.x; i < nw * npad; i += blockDim.x) part[i] = 0.0;
  __syncthreads();
  for (int u = warp; u < E.nsides * nt * nt; u += nw) {
    const int q = u / (nt * nt), tile = u % (nt * nt), I = tile / nt, J = tile % nt;
    const double *T = Dt + slots[E.side_begin + q].off_Dt + (int64_t)tile * 1024;
    double p[32];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) p[rr] = __ldg(T + rr * 32 + lane);
    const double wc = ws[q * npad + 32 * J + lane];
#pragma unroll
    for (int rr = 0; rr < 32; ++rr) p[rr] *= wc;
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
      const bool up = (lane & sft) != 0;
#pragma unroll
      for (int k2 = 0; k2 < sft; ++k2) {
        double send = up ? p[k2] : p[k2 + sft];
        double keep = up ? p[k2 + sft] : p[k2];
        p[k2] = keep + __shfl_xor_sync(FULL, send, sft);
      }
    }
    part[warp * npad + 32 * I + lane] += p[0];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nd; i += blockDim.x) {
    double v = 0.0;
    for (int w2 = 0; w2 < nw; ++w2) v += part[w2 * npad + i];
    z[E.off_xd + i] = v;
  }
}

__global__ void copy_kernel(const double *a, double *b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

// ------------------------------------------------------------------ B0 / B8
// B0 (GEMV form): b_D = [b_I ; Pi^T b_P] and g0_i = c^T b_P (p0 rhs, A5)
__global__ void rhs_D_kernel(const SubDev *__restrict__ subs, const int64_t *__restrict__ Ifree,
                             const int64_t *__restrict__ Pglob, const double *__restrict__ cvec,
                             const double *__restrict__ mvec, const double *__restrict__ rhs, int64_t nvf,
                             double *bD, double *g0) {
  __shared__ double red[32];
  const SubDev S = subs[blockIdx.x];
  const int tid = threadIdx.x, nw = blockDim.x >> 5;
  double *b = bD + S.off_Dn;
  for (int j = tid; j < S.nI; j += blockDim.x) b[j] = rhs[Ifree[S.off_I + j]];
  double s = 0.0;
  for (int a = tid; a < S.nP; a += blockDim.x) s += cvec[S.off_P + a] * rhs[nvf + Pglob[S.off_P + a]];
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  __syncthreads();
  double g = 0.0;
  for (int w = 0; w < nw; ++w) g += red[w];
  if (tid == 0) g0[blockIdx.x] = g;
  for (int a = tid; a < S.nP; a += blockDim.x)
    b[S.nI + a] = rhs[nvf + Pglob[S.off_P + a]] - mvec[S.off_P + a] * g / S.vol;
}

// B0: z_G = -Psi^T b_D = -K_GD K_DD^-1 b_D (thread per interface row, column-major Psi^T)
__global__ void __launch_bounds__(128) zG_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Psi,
                                                 const double *__restrict__ bD, double *zG) {
  const SubDev S = subs[blockIdx.y];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= S.nG) return;
  const double *P = Psi + S.off_Psi;
  const double *b = bD + S.off_Dn;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int j = 0;
  for (; j + 3 < S.nD; j += 4) {
    a0 += P[i + (int64_t)j * S.nG] * b[j];
    a1 += P[i + (int64_t)(j + 1) * S.nG] * b[j + 1];
    a2 += P[i + (int64_t)(j + 2) * S.nG] * b[j + 2];
    a3 += P[i + (int64_t)(j + 3) * S.nG] * b[j + 3];
  }
  for (; j < S.nD; ++j) a0 += P[i + (int64_t)j * S.nG] * b[j];
  zG[S.off_G + i] = -((a0 + a1) + (a2 + a3));
}

// B8: x_D[j] = y_D[j] - sum_i Psi^T[i, j] x_G[i]  (y_D = K_DD^-1 b_D from the packed GEMV partials);
// warp per column j of Psi^T (contiguous), XD_SPLIT CTAs per subdomain.
constexpr int XD_SPLIT = 4;
__global__ void __launch_bounds__(256) xD_kernel(const SubDev *__restrict__ subs, const double *__restrict__ Psi,
                                                 const double *__restrict__ ypart, int64_t pstride, int P,
                                                 const int64_t *__restrict__ Gfree, const double *__restrict__ x_in,
                                                 double *xD) {
  extern __shared__ double xg[];
  const SubDev S = subs[blockIdx.y];
  for (int i = threadIdx.x; i < S.nG; i += blockDim.x) xg[i] = x_in[Gfree[S.off_G + i]];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double *Pm = Psi + S.off_Psi;
  for (int j = blockIdx.x * nw + warp; j < S.nD; j += gridDim.x * nw) {
    const double *col = Pm + (int64_t)j * S.nG;
    double v0 = 0.0, v1 = 0.0;
    int i = lane;
    for (; i + 32 < S.nG; i += 64) { v0 += col[i] * xg[i]; v1 += col[i + 32] * xg[i + 32]; }
    for (; i < S.nG; i += 32) v0 += col[i] * xg[i];
    const double v = warp_sum(v0 + v1);
    if (lane == 0) {
      double y = 0.0;
      for (int c = 0; c < P; ++c) y += ypart[c * pstride + S.off_Dn + j];
      xD[S.off_Dn + j] = y - v;
    }
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

// per entity: ghat_e = b_e + sum_m zG^(m)[e]; r_x = T_e^T ghat_e
__global__ void gamma_rhs_kernel(const EntDev *__restrict__ ents, const SlotDev *__restrict__ slots,
                                 const SubDev *__restrict__ subs, const int64_t *__restrict__ gam_free,
                                 const double *__restrict__ rhs, const double *__restrict__ zG,
                                 const double *__restrict__ T, int64_t NDelta, double *gtmp, double *r) {
  const EntDev E = ents[blockIdx.x];
  const int n = E.n;
  double *gh = gtmp + E.off_gam;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v = rhs[gam_free[E.off_gam + j]];
    for (int q = 0; q < E.nsides; ++q) {
      const SlotDev s = slots[E.side_begin + q];
      v += zG[subs[s.sub].off_G + s.offG + j];
    }
    gh[j] = v;
  }
  __syncthreads();
  const double *Te = T + E.off_T;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw) {
    double v = 0.0;
    for (int j = lane; j < n; j += 32) v += Te[j + (int64_t)i * n] * gh[j];
    v = warp_sum(v);
    if (lane == 0) {
      if (i < E.nd) r[E.off_xd + i] = v;
      else r[NDelta + E.off_pi + (i - E.nd)] = v;
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
      const double xi = i < E.nd ? x[E.off_xd + i] : x[NDelta + E.off_pi + (i - E.nd)];
      v += Te[j + (int64_t)i * n] * xi;
    }
    gam[E.off_gam + j] = v;
    xout[gam_free[E.off_gam + j]] = v;
  }
}

// global zero-mean pressure (Q_{h,0}): p -= c_K * (sum_K vol_K p_K0) / vol_Omega
__global__ void pressure_mean_kernel(const double *__restrict__ cellgeo, int geo_stride, int np, int64_t nK,
                                     double *p, int phase, double *acc) {
  if (phase == 0) {
    __shared__ double red[2][32];
    double a = 0.0, w = 0.0;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nK; K += (int64_t)gridDim.x * blockDim.x) {
      const double vol = cellgeo[K * geo_stride];
      a += vol * p[K * np];
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
  } else {
    double A = 0, Wt = 0;
    for (int b = 0; b < phase; ++b) { A += acc[2 * b]; Wt += acc[2 * b + 1]; }
    const double mean = A / Wt;
    for (int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; K < nK; K += (int64_t)gridDim.x * blockDim.x)
      for (int a = 0; a < np; ++a) p[K * np + a] -= mean * cellgeo[K * geo_stride + 5 + a];
  }
}

// ------------------------------------------------------------------ K7: element-by-element operator
// y_K = [A_K B_K^T; B_K 0] x_K per element, then a deterministic per-DOF gather-sum.
__global__ void elem_apply_kernel(const double *__restrict__ elA, const double *__restrict__ elB,
                                  const int64_t *__restrict__ l2g, const int64_t *__restrict__ vel2free,
                                  const int *__restrict__ cell_nv, int nvmax, int np, int64_t nK, int64_t nvf,
                                  const double *__restrict__ x, double *yel) {
  const int64_t K = blockIdx.x;
  if (K >= nK) return;
  extern __shared__ double xs[];
  const int nv = cell_nv[K];
  const int stride = nvmax + np;
  for (int j = threadIdx.x; j < nv; j += blockDim.x) {
    const int64_t f = vel2free[l2g[K * nvmax + j]];
    xs[j] = f >= 0 ? x[f] : 0.0;
  }
  for (int a = threadIdx.x; a < np; a += blockDim.x) xs[nvmax + a] = x[nvf + K * np + a];
  __syncthreads();
  const double *A = elA + K * nvmax * nvmax;
  const double *B = elB + K * np * nvmax;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < nv + np; i += nw) {
    double v = 0.0;
    if (i < nv) {
      for (int j = lane; j < nv; j += 32) v += A[(int64_t)i * nv + j] * xs[j];
      for (int a = lane; a < np; a += 32) v += B[(int64_t)a * nv + i] * xs[nvmax + a];
    } else {
      const int a = i - nv;
      for (int j = lane; j < nv; j += 32) v += B[(int64_t)a * nv + j] * xs[j];
    }
    v = warp_sum(v);
    if (lane == 0) yel[K * stride + (i < nv ? i : nvmax + (i - nv))] = v;
  }
}

__global__ void elem_gather_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ idx,
                                   const double *__restrict__ yel, int64_t nvf, int64_t nK, int np, int stride,
                                   int nvmax, double *y) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nvf + nK * np;
       f += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    if (f < nvf) {
      for (int64_t q = ptr[f]; q < ptr[f + 1]; ++q) v += yel[idx[q]];
    } else {
      const int64_t pidx = f - nvf, K = pidx / np, a = pidx % np;
      v = yel[K * stride + nvmax + a];
    }
    y[f] = v;
  }
}

__global__ void axpby_kernel(const double *a, const double *b, double *out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = a[i] - b[i];
}

// ------------------------------------------------------------------ host side
// out[i] = sum_c part[c][i]: block = 32 outputs x 8 warps (warp w sums chunks w, w+8, ...), then
// the 8 warp partials are added in fixed order.
__global__ void __launch_bounds__(256) sum_chunks_kernel(const double *__restrict__ part, int64_t stride, int P,
                                                         int64_t n, double *out) {
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

// z_Pi = u_Pi, z_p0 = p0 (copy of the coarse solution into the tail of z)
__global__ void coarse_to_z_kernel(const double *uc, int64_t n, double *z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) z[i] = uc[i];
}

struct SolveState {
  DBuf<GemvWork> w_op, w_loc, w_c;
  DBuf<GemvWork> w_kd;
  int nw_op = 0, nw_loc = 0, nw_c = 0, nw_kd = 0, max_nd = 1;
  size_t sm_op = 0, sm_loc = 0, sm_c = 0, sm_rx = 0, sm_ex = 0, sm_kd = 0;
  DBuf<int64_t> xptr, xidx, pptr, pidx, eptr, eidx;
  DBuf<double> hist;
  bool ready = false;
  // optional per-kernel timing (VB_KERNEL_TIMING=1): event pairs per launch category
  std::vector<cudaEvent_t> ev;
  std::vector<int> ev_cat;
  int nev = 0;
  ~SolveState() {
    for (auto e : ev) cudaEventDestroy(e);
  }
};

static const char *kCatNames[] = {"sym_gemv S_T (operator, B1)", "sym_gemv S_DD^-1 (local, B5)",
                                  "sym_gemv coarse inverse (B6)", "apply_S total (B1-B2)",
                                  "apply_M total (B4-B7)"};
constexpr int N_CAT = 5;

static void tick(vb_ctx *c, SolveState *st, int cat, bool begin) {
  if (!c->timing) return;
  if (st->nev + 1 >= (int)st->ev.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      VB_CUDA(cudaEventCreate(&e));
      st->ev.push_back(e);
      st->ev_cat.push_back(-1);
    }
  }
  VB_CUDA(cudaEventRecord(st->ev[st->nev], c->stream));
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

constexpr int DOT_BLOCKS = 296;

static void dot(vb_ctx *c, const double *a, const double *b, int64_t n, double *dst) {
  dot_partial_kernel<<<DOT_BLOCKS, 256, 0, c->stream>>>(a, b, n, c->w_dots.p);
  dot_final_kernel<<<1, 32, 0, c->stream>>>(c->w_dots.p, DOT_BLOCKS, dst);
}

static int grid_for(int64_t n) { return (int)std::min<int64_t>((n + 255) / 256, 148 * 8); }

static void apply_S(vb_ctx *c, SolveState *st) {   // q = S^ p  (B1, B2)
  cudaStream_t s = c->stream;
  tick(c, st, 3, true);
  tick(c, st, 0, true);
  sym_gemv_kernel<GV_WARPS><<<st->nw_op, GV_WARPS * 32, st->sm_op, s>>>(st->w_op.p);
  tick(c, st, 0, false);
  b0_apply_kernel<<<c->N, 32, 0, s>>>(c->d_sub.p, c->d_loc2x.p, c->d_b0T.p, c->w_p.p,
                                      c->n_delta_glob + c->NPi, c->w_part.p, c->w_q.p);
  int64_t nxp = c->n_delta_glob + c->NPi;
  gather_sum_kernel<<<grid_for(nxp), 256, 0, s>>>(st->xptr.p, st->xidx.p, c->w_part.p, c->len_G, c->P_op, nxp, c->w_q.p);
  tick(c, st, 3, false);
  VB_STAGE();
}

static void apply_M(vb_ctx *c, SolveState *st) {   // z = M^-1 r  (B4-B7)
  cudaStream_t s = c->stream;
  const int nslot = c->h_slot.size(), nent = c->h_ent.size();
  tick(c, st, 4, true);
  if (c->n_act_slots)
    restrict_kernel<<<c->n_act_slots, DLX_WARPS * 32, st->sm_rx, s>>>(c->d_slot.p, c->d_act_slots.p, c->d_ent.p,
                                                                     c->d_sub.p, c->d_Dt.p, c->w_r.p, c->w_locD.p);
  tick(c, st, 1, true);
  if (st->nw_loc) sym_gemv_kernel<GV_WARPS><<<st->nw_loc, GV_WARPS * 32, st->sm_loc, s>>>(st->w_loc.p);
  tick(c, st, 1, false);
  phit_kernel<<<dim3(PHIT_SPLIT, c->N), 256, 0, s>>>(c->d_sub.p, c->d_Phi.p, c->w_locD.p, c->w_locC.p);
  coarse_rhs_kernel<<<grid_for(c->Nc), 256, 0, s>>>(st->pptr.p, st->pidx.p, c->w_locC.p, c->w_r.p,
                                                    c->n_delta_glob, c->NPi, c->N, c->w_rc.p);
  coarse_p0_project_kernel<<<1, 256, 0, s>>>(c->d_sub.p, c->N, c->w_rc.p + c->NPi, 0);
  tick(c, st, 2, true);
  sym_gemv_kernel<GV_WARPS_C><<<st->nw_c, GV_WARPS_C * 32, st->sm_c, s>>>(st->w_c.p);
  tick(c, st, 2, false);
  sum_chunks_kernel<<<(c->Nc + 31) / 32, 256, 0, s>>>(c->w_ucp.p, c->Nc, st->nw_c, c->Nc, c->w_uc.p);
  coarse_p0_project_kernel<<<1, 256, 0, s>>>(c->d_sub.p, c->N, c->w_uc.p + c->NPi, 1);
  local2_kernel<<<dim3((st->max_nd + 127) / 128, c->N), 128, c->max_npi * sizeof(double), s>>>(
      c->d_sub.p, c->d_Phi.p, c->w_locY.p, c->len_Dv, c->P_loc, c->d_pi_glob.p, c->w_uc.p, c->w_locD.p);
  if (c->n_act_ents)
    extend_kernel<<<c->n_act_ents, DLX_WARPS * 32, st->sm_ex, s>>>(c->d_ent.p, c->d_act_ents.p, c->d_slot.p, c->d_sub.p,
                                                                   c->d_Dt.p, c->w_locD.p, c->w_z.p);
  coarse_to_z_kernel<<<grid_for(c->Nc), 256, 0, s>>>(c->w_uc.p, c->Nc, c->w_z.p + c->n_delta_glob);
  tick(c, st, 4, false);
  VB_STAGE();
}

static SolveState *get_state(vb_ctx *c) {
  if (!c->solve_state) c->solve_state = new SolveState();
  return (SolveState *)c->solve_state;
}

void destroy_solve_state(vb_ctx *c) {
  delete (SolveState *)c->solve_state;
  c->solve_state = nullptr;
}

static void build_csr(int64_t nrows, const std::vector<std::pair<int64_t, int64_t>> &pairs, DBuf<int64_t> &ptr,
                      DBuf<int64_t> &idx, cudaStream_t s) {
  std::vector<int64_t> p(nrows + 1, 0), ix(pairs.size());
  for (auto &q : pairs) p[q.first + 1]++;
  for (int64_t i = 0; i < nrows; ++i) p[i + 1] += p[i];
  std::vector<int64_t> fill(p.begin(), p.end() - 1);
  for (auto &q : pairs) ix[fill[q.first]++] = q.second;   // pairs are pre-sorted by (row, sub)
  ptr.upload(p, s);
  idx.upload(ix, s);
}

void prepare_solve(vb_ctx *c) {
  SolveState *st = get_state(c);
  if (st->ready) return;
  cudaStream_t s = c->stream;
  const int N = c->N;
  const int64_t nx = c->nx;
  c->w_x.alloc(nx); c->w_r.alloc(nx); c->w_z.alloc(nx); c->w_p.alloc(nx); c->w_q.alloc(nx);
  c->w_part.alloc((int64_t)c->P_op * std::max<int64_t>(c->len_G, 1));
  c->w_locD.alloc(std::max<int64_t>(c->len_Dv, 1));
  c->w_locY.alloc((int64_t)c->P_loc * std::max<int64_t>(c->len_Dv, 1));
  c->w_locC.alloc(std::max<int64_t>(c->len_Pi, 1));
  c->w_uc.alloc(c->Nc); c->w_rc.alloc(c->Nc);
  c->w_scal.alloc(16); c->w_scal.zero(s);
  c->w_dots.alloc(DOT_BLOCKS * 2);
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
      wl.push_back(GemvWork{c->d_SDi.p + S.off_SDi, nullptr, c->w_locD.p + S.off_Dv,
                            c->w_locY.p + (int64_t)q * c->len_Dv + S.off_Dv, S.nd, rows[q].first, rows[q].second, 0});
  }
  // sub-domains with nd = 0 still need zero partials
  c->w_locY.zero(s);
  st->w_loc.upload(wl, s); st->nw_loc = wl.size(); st->sm_loc = gemv_smem(nmaxD);
  wl.clear();
  int Pc = std::max(1, std::min<int>(c->P_c, (int)((c->Nc + 31) / 32)));
  c->w_ucp.alloc((int64_t)Pc * c->Nc);
  split_rows(c->Nc, Pc, rows);
  for (int q = 0; q < Pc; ++q)
    wl.push_back(GemvWork{c->d_Kcp.p, nullptr, c->w_rc.p, c->w_ucp.p + (int64_t)q * c->Nc, (int)c->Nc, rows[q].first, rows[q].second, 0});
  st->w_c.upload(wl, s); st->nw_c = wl.size(); st->sm_c = gemv_smem(c->Nc, GV_WARPS_C);
  size_t smmax = std::max(st->sm_op, st->sm_loc);
  VB_REQUIRE(smmax <= 227 * 1024 && st->sm_c <= 227 * 1024, VB_EINVAL,
             "packed GEMV vector exceeds shared memory (coarse too large)");
  VB_CUDA(cudaFuncSetAttribute(sym_gemv_kernel<GV_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smmax));
  VB_CUDA(cudaFuncSetAttribute(sym_gemv_kernel<GV_WARPS_C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st->sm_c));
  // deluxe restriction / extension shared memory (vectors + per-warp partials)
  int maxnd_e = 1, maxs = 1;
  for (auto &E : c->h_ent)
    if (E.nd) { maxnd_e = std::max(maxnd_e, E.nd); maxs = std::max(maxs, E.nsides); }
  const int npad = (maxnd_e + 31) / 32 * 32;
  st->sm_rx = (size_t)(1 + DLX_WARPS) * npad * sizeof(double);
  st->sm_ex = (size_t)(maxs + DLX_WARPS) * npad * sizeof(double);
  VB_REQUIRE(st->sm_ex <= 227 * 1024, VB_EINVAL, "deluxe entity too large for the extension kernel");
  VB_CUDA(cudaFuncSetAttribute(restrict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st->sm_rx));
  VB_CUDA(cudaFuncSetAttribute(extend_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)st->sm_ex));
  st->max_nd = nmaxD;
  // x coordinate -> local copies (ordered by subdomain), primal -> local Pi copies
  std::vector<int64_t> loc2x;
  c->d_loc2x.download(loc2x, s);
  VB_CUDA(cudaStreamSynchronize(s));
  std::vector<std::pair<int64_t, int64_t>> pr;
  pr.reserve(loc2x.size());
  for (int64_t j = 0; j < (int64_t)loc2x.size(); ++j) pr.push_back({loc2x[j], j});
  std::sort(pr.begin(), pr.end());
  build_csr(c->n_delta_glob + c->NPi, pr, st->xptr, st->xidx, s);
  std::vector<int64_t> pig;
  c->d_pi_glob.download(pig, s);
  VB_CUDA(cudaStreamSynchronize(s));
  pr.clear();
  for (int64_t j = 0; j < (int64_t)pig.size(); ++j) pr.push_back({pig[j], j});
  std::sort(pr.begin(), pr.end());
  build_csr(c->NPi, pr, st->pptr, st->pidx, s);
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
    VB_REQUIRE(st->sm_kd <= 227 * 1024, VB_EINVAL, "Dirichlet block too large for the packed GEMV");
    size_t smg = std::max(std::max(st->sm_op, st->sm_loc), st->sm_kd);
    VB_CUDA(cudaFuncSetAttribute(sym_gemv_kernel<GV_WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smg));
    int64_t mg = 1;
    for (auto &S : c->h_sub) mg = std::max<int64_t>(mg, S.nG);
    VB_CUDA(cudaFuncSetAttribute(xD_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(mg * 8)));
  }
  VB_CUDA(cudaStreamSynchronize(s));
  st->ready = true;
  // bytes per PCG iteration (model of the streamed operators)
  double b = 0;
  for (auto &S : c->h_sub) {
    b += 8.0 * packed_tiles(S.nG) * 1024 + 8.0 * packed_tiles(S.nd) * 1024 + 2 * 8.0 * S.nd * S.npi;
  }
  for (auto &sl : c->h_slot) b += 2 * 8.0 * sl.nd * sl.nd;
  b += 8.0 * packed_tiles(c->Nc) * 1024;
  c->bytes_per_iter = b;
}

void element_gather(vb_ctx *c, const double *yel, double *out) {
  const int stride = c->nv_max + c->np;
  const int64_t nf = c->n_free_vel + c->npres;
  elem_gather_kernel<<<grid_for(nf), 256, 0, c->stream>>>(c->d_el_ptr.p, c->d_el_ent.p, yel, c->n_free_vel, c->nK,
                                                          c->np, stride, c->nv_max, out);
  VB_STAGE();
}

void apply_operator_device(vb_ctx *c, const double *x, double *y) {
  cudaStream_t s = c->stream;
  const int stride = c->nv_max + c->np;
  elem_apply_kernel<<<c->nK, 128, stride * sizeof(double), s>>>(c->d_elA.p, c->d_elB.p, c->d_cell_l2g.p,
                                                                c->d_vel2free.p, c->d_cell_nv.p, c->nv_max, c->np,
                                                                c->nK, c->n_free_vel, x, c->w_elt.p);
  VB_STAGE();
  element_gather(c, c->w_elt.p, y);
}

static double read_scalar(vb_ctx *c, int i) {
  double v;
  VB_CUDA(cudaMemcpyAsync(&v, c->w_scal.p + i, 8, cudaMemcpyDeviceToHost, c->stream));
  VB_CUDA(cudaStreamSynchronize(c->stream));
  return v;
}

void lanczos_extremes(const std::vector<double> &al, const std::vector<double> &be, double *lmin, double *lmax);

void pcg_device(vb_ctx *c, const double *rhs, double *x, double rtol, int maxit, vb_report *rep) {
  prepare_solve(c);
  SolveState *st = get_state(c);
  cudaStream_t s = c->stream;
  c->timing = getenv("VB_KERNEL_TIMING") && atoi(getenv("VB_KERNEL_TIMING"));
  st->nev = 0;
  const int N = c->N;
  const int64_t nx = c->nx, NDelta = c->n_delta_glob;
  const int64_t nvf = c->n_free_vel;
  // ---------------- B0: condensed rhs in transformed coordinates
  int64_t maxnG = 1, maxnD = 1;
  for (auto &S : c->h_sub) { maxnG = std::max<int64_t>(maxnG, S.nG); maxnD = std::max<int64_t>(maxnD, S.nD); }
  c->w_r.zero(s);
  rhs_D_kernel<<<N, 256, 0, s>>>(c->d_sub.p, c->d_subI_free.p, c->d_subP_glob.p, c->d_cvec.p, c->d_mvec.p, rhs, nvf,
                                 c->w_bD.p, c->w_r.p + NDelta + c->NPi);
  sym_gemv_kernel<GV_WARPS><<<st->nw_kd, GV_WARPS * 32, st->sm_kd, s>>>(st->w_kd.p);   // y_D = K_DD^-1 b_D
  zG_kernel<<<dim3((maxnG + 127) / 128, N), 128, 0, s>>>(c->d_sub.p, c->d_Psi.p, c->w_bD.p, c->w_zG.p);
  VB_STAGE();
  gamma_rhs_kernel<<<c->h_ent.size(), 128, 0, s>>>(c->d_ent.p, c->d_slot.p, c->d_sub.p, c->d_gam_free.p, rhs,
                                                   c->w_zG.p, c->d_T.p, NDelta, c->w_gam.p, c->w_r.p);
  VB_STAGE();
  // ---------------- PCG (SURVEY O-15)
  c->w_x.zero(s);
  double *sc = c->w_scal.p;
  dot(c, c->w_r.p, c->w_r.p, nx, sc + 2);
  const double rr0 = read_scalar(c, 2);
  const double r0n = sqrt(rr0);
  apply_M(c, st);
  dot(c, c->w_r.p, c->w_z.p, nx, sc + 0);
  update_p_kernel<<<grid_for(nx), 256, 0, s>>>(c->w_p.p, c->w_z.p, nx, sc, 1);
  VB_STAGE();
  int it = 0;
  int status = VB_OK;
  double rn = r0n;
  std::vector<double> alphas, betas;
  while (true) {
    if (rn <= rtol * r0n) break;
    if (it >= maxit) { status = VB_ENOTCONV; break; }
    apply_S(c, st);
    dot(c, c->w_p.p, c->w_q.p, nx, sc + 1);
    update_xr_kernel<<<grid_for(nx), 256, 0, s>>>(c->w_x.p, c->w_r.p, c->w_p.p, c->w_q.p, nx, sc);
    dot(c, c->w_r.p, c->w_r.p, nx, sc + 2);
    double h[4];
    VB_CUDA(cudaMemcpyAsync(h, sc, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    const double rz = h[0], pq = h[1];
    if (!(pq > 0) || !(rz > 0)) { status = VB_EBREAKDOWN; break; }
    alphas.push_back(rz / pq);
    rn = sqrt(h[2]);
    ++it;
    if (rn <= rtol * r0n || it >= maxit) {
      if (rn > rtol * r0n) status = VB_ENOTCONV;
      break;
    }
    apply_M(c, st);
    dot(c, c->w_r.p, c->w_z.p, nx, sc + 3);
    update_p_kernel<<<grid_for(nx), 256, 0, s>>>(c->w_p.p, c->w_z.p, nx, sc, 0);
    rotate_rz_kernel<<<1, 1, 0, s>>>(sc, st->hist.p, std::min(it, 4095));
    VB_STAGE();
  }
  // betas from the recorded history
  {
    std::vector<double> hh(2 * 4096);
    VB_CUDA(cudaMemcpyAsync(hh.data(), st->hist.p, hh.size() * 8, cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    for (int j = 1; j < (int)alphas.size() && j < 4096; ++j) betas.push_back(hh[2 * j + 1]);
  }
  // ---------------- B8: back to original coordinates and back-substitution
  gamma_back_kernel<<<c->h_ent.size(), 128, 0, s>>>(c->d_ent.p, c->d_gam_free.p, c->d_T.p, c->w_x.p, NDelta,
                                                    c->w_gam.p, x);
  VB_STAGE();
  xD_kernel<<<dim3(XD_SPLIT, N), 256, maxnG * 8, s>>>(c->d_sub.p, c->d_Psi.p, c->w_yDp.p, c->len_Dn, c->P_kd,
                                                      c->d_subG_free.p, x, c->w_xD.p);
  xout_kernel<<<N, 256, 0, s>>>(c->d_sub.p, c->w_xD.p, c->d_subI_free.p, c->d_subP_glob.p, c->d_cvec.p, c->d_mvec.p,
                                c->w_x.p + NDelta + c->NPi, nvf, x);
  VB_STAGE();
  pressure_mean_kernel<<<64, 256, 0, s>>>(c->d_cellgeo.p, c->geo_stride, c->np, c->nK, x + nvf, 0, c->w_dots.p);
  pressure_mean_kernel<<<grid_for(c->nK), 256, 0, s>>>(c->d_cellgeo.p, c->geo_stride, c->np, c->nK, x + nvf, 64, c->w_dots.p);
  VB_STAGE();
  VB_CUDA(cudaStreamSynchronize(s));
  collect_times(c, st);
  c->last_iterations = it;
  if (rep) {
    rep->iterations = it;
    rep->converged = status == VB_OK;
    rep->r0_norm = r0n;
    rep->r_final_norm = rn;
    rep->rel_residual = r0n > 0 ? rn / r0n : 0.0;
    // Lanczos T from the CG coefficients (SURVEY O-15 index convention): beta_j pairs alpha_j, alpha_{j+1}
    std::vector<double> bb(betas.begin(), betas.end());
    double lmin = 1, lmax = 1;
    lanczos_extremes(alphas, bb, &lmin, &lmax);
    rep->lambda_min = lmin; rep->lambda_max = lmax; rep->kappa = lmin > 0 ? lmax / lmin : INFINITY;
    rep->bytes_per_iter_model = c->bytes_per_iter;
    rep->flux_violation_max = c->flux_violation;
    rep->n_primal = c->NPi; rep->n_coarse = c->Nc;
    rep->n_dofs_paper = c->nvel + c->npres;
  }
  if (status != VB_OK)
    throw Error{(vb_status)status, status == VB_ENOTCONV ? "PCG reached maxit without converging"
                                                          : "PCG breakdown: p^T S p <= 0 or r^T z <= 0"};
}

// original interface coordinates (entity-major) -> transformed x (T_e^T per entity)
__global__ void to_transformed_kernel(const EntDev *__restrict__ ents, const double *__restrict__ T,
                                      const double *__restrict__ g, int64_t NDelta, double *x) {
  const EntDev E = ents[blockIdx.x];
  const int n = E.n;
  const double *Te = T + E.off_T;
  const double *gh = g + E.off_gam;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = warp; i < n; i += nw) {
    double v = 0.0;
    for (int j = lane; j < n; j += 32) v += Te[j + (int64_t)i * n] * gh[j];
    v = warp_sum(v);
    if (lane == 0) {
      if (i < E.nd) x[E.off_xd + i] = v;
      else x[NDelta + E.off_pi + (i - E.nd)] = v;
    }
  }
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
  to_transformed_kernel<<<c->h_ent.size(), 128, 0, s>>>(c->d_ent.p, c->d_T.p, gin.p, NDelta, dst);
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
