// Batched dense FP64 kernels: grouped DMMA GEMM (gemm_dmma.cuh: mma.sync.m16n8k16.f64 -> SASS
// DMMA.8x8x4, the FP64 tensor path of sm_100a; tcgen05 has no f64 kind; per-kernel SASS
// counts in profiles/r02_sass_summary.txt), blocked partial LDL^T,
// triangular inverse, packing.  Used by the factor stage.
#include <algorithm>
#include <functional>
#include <map>
#include <mutex>
#include "dense.cuh"
#include "gemm_dmma.cuh"

namespace vb {

// ------------------------------------------------------------------ grouped GEMM (DMMA)
// gemm_dmma.cuh: CTA tile 64 x 64 x 16, 4 warps of 16 x 64 warp tiles (m16n8k16 f64 MMAs), 3-stage
// cp.async ring, 16-byte copies (pairs of 8-byte ones for unaligned problems), 4 CTAs per SM.  Chosen over
// 128 x 64 / 128 x 128 / 64 x 128 / 64 x 32 / 32 x 64 and 16 or 32-deep slabs by tools/gemm_proto.cu
// on the factor's shapes (profiles/r02_gemm_proto.txt).
using GCfg = g2::Cfg<64, 64, 16, 4, 1, 3, 4>;
constexpr int GBM = GCfg::BM, GBN = GCfg::BN, GBK = GCfg::BK;
#ifndef LDL_NB_CFG
#define LDL_NB_CFG 256
#endif
constexpr int LDL_NB = LDL_NB_CFG;   // wide-panel width of the blocked LDL^T (VB_NVCC_DEFINES knob)
#ifndef TRI_NB_CFG
#define TRI_NB_CFG 256
#endif
constexpr int TRI_NB = TRI_NB_CFG;   // wide-block width of the triangular inverse

// Raise (never lower) a kernel's dynamic shared-memory limit: the attribute is process-wide and
// several contexts / loopback ranks (threads) launch the same kernels.
void raise_smem_limit(const void *func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> cur;
  int dev = 0;
  VB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  size_t &c = cur[{func, dev}];
  if (bytes <= c) return;
  VB_CUDA(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  c = bytes;
}

template <bool DENSE, bool SCALED, bool TA, bool TB, bool VEC>
static void launch_gemm(dim3 grid, const GemmProb *probs, const int4 *segs, int seg0, int nseg, cudaStream_t s) {
  using S = g2::Smem<GCfg, TA, TB>;
  auto k = g2::gemm2_kernel<GCfg, DENSE, SCALED, TA, TB, VEC>;
  raise_smem_limit((const void *)k, S::BYTES);
  k<<<grid, GCfg::THREADS, S::BYTES, s>>>(probs, segs, seg0, nseg);
  VB_CHECK_LAUNCH();
}

template <bool DENSE, bool SCALED>
static void launch_gemm_cls(int cls, dim3 grid, const GemmProb *probs, const int4 *segs, int seg0, int nseg,
                            cudaStream_t s) {
  switch (cls) {
    case 0: launch_gemm<DENSE, SCALED, false, false, true>(grid, probs, segs, seg0, nseg, s); break;
    case 1: launch_gemm<DENSE, SCALED, true, false, true>(grid, probs, segs, seg0, nseg, s); break;
    case 2: launch_gemm<DENSE, SCALED, false, true, true>(grid, probs, segs, seg0, nseg, s); break;
    default: launch_gemm<DENSE, SCALED, true, true, true>(grid, probs, segs, seg0, nseg, s); break;
  }
}

static int trans_class(const GemmProb &p) { return (p.transA ? 1 : 0) + (p.transB ? 2 : 0); }

thread_local double g_gemm_flops = 0.0;   // DMMA GEMM flops issued by this thread (factor-stage accounting)
thread_local bool g_gemm_timing = false;  // record CUDA events around every GemmPlan::run (kernel time)
thread_local std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_gemm_events;

double gemm_timing_collect(cudaStream_t s) {
  double ms = 0.0;
  if (!g_gemm_events.empty()) VB_CUDA(cudaStreamSynchronize(s));
  for (auto &e : g_gemm_events) {
    float t = 0.0f;
    VB_CUDA(cudaEventElapsedTime(&t, e.first, e.second));
    ms += t;
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  g_gemm_events.clear();
  return ms / 1e3;
}

void GemmPlan::add(const GemmProb &p_in) {
  if (p_in.M <= 0 || p_in.N <= 0) return;
  GemmProb p = p_in;
  // triangular-operand K skipping (GemmProb.kz_on: a site bit, see factor.cu); VB_KZ=0 disables it,
  // VB_KZ=<bits> keeps only those sites (diagnostics)
  static const int kz_mask = getenv("VB_KZ") ? atoi(getenv("VB_KZ")) : -1;
  if (!allow_kz) p.kz_on = (p.kz_on & kz_mask) ? p.kz_on : 0;
  {
    double f = 2.0 * p.M * (double)p.N * p.K;
    if (p.lower) f *= 0.5 * (1.0 + 1.0 / std::max(1, std::min(p.M, p.N)));   // lower triangle (square C)
    if (p.kz_on) {   // executed work: per tile, the K slabs from its first non-zero one
      f = 0.0;
      const int tm = (p.M + GBM - 1) / GBM, tn = (p.N + GBN - 1) / GBN;
      for (int i = 0; i < tm; ++i)
        for (int j = 0; j < tn; ++j) {
          if (p.lower && (i * GBM + GBM - 1) < j * GBN) continue;
          const int64_t kb = std::min<int64_t>(p.K, std::max<int64_t>(0, std::max<int64_t>((int64_t)i * GBM + p.kzA,
                                                                                             (int64_t)j * GBN + p.kzB)) / GBK * GBK);
          const int rows = std::min(GBM, p.M - i * GBM), cols = std::min(GBN, p.N - j * GBN);
          f += 2.0 * rows * cols * (double)(p.K - kb);
        }
    }
    g_gemm_flops += f;
  }
  int pid = probs.size();
  probs.push_back(p);
  int tm = (p.M + GBM - 1) / GBM, tn = (p.N + GBN - 1) / GBN;
  if ((int64_t)tm * tn >= 4096 && tm < 65536) {   // large: a 2D grid instead of a tile list
    dense.back().push_back(pid);
    return;
  }
  if (p.d) scaled.back() = 1;
  auto &tl = ltiles.back()[trans_class(p)];
  auto &cnt = ltcount.back()[trans_class(p)];
  int64_t ntile = 0;   // tiles of this problem (lower: j <= i only, square tiles)
  for (int i = 0; i < tm; ++i) ntile += p.lower ? std::min(i + 1, tn) : tn;
  tl.push_back(make_int4(pid, (int)cnt, tn, p.lower ? 1 : 0));
  cnt += ntile;
  VB_REQUIRE(cnt < (1LL << 31), VB_EINVAL, "internal: grouped GEMM launch too large");
}

void GemmPlan::upload(cudaStream_t s) {
  std::vector<GemmProb> hp(probs);
  std::vector<int4> ht;
  lrange.assign(ltiles.size(), {});
  lntile.assign(ltiles.size(), {});
  for (size_t l = 0; l < ltiles.size(); ++l)
    for (int c = 0; c < 4; ++c) {
      lrange[l][c] = {(int)ht.size(), (int)ltiles[l][c].size()};
      lntile[l][c] = (int)ltcount[l][c];
      ht.insert(ht.end(), ltiles[l][c].begin(), ltiles[l][c].end());
    }
  d_probs.upload(hp, s);
  d_tiles.upload(ht, s);
  VB_CUDA(cudaStreamSynchronize(s));
}

void GemmPlan::run(int launch, cudaStream_t s) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (g_gemm_timing) {
    VB_CUDA(cudaEventCreate(&e0));
    VB_CUDA(cudaEventCreate(&e1));
    VB_CUDA(cudaEventRecord(e0, s));
  }
  for (int c = 0; c < 4; ++c) {
    const auto &R = lrange[launch][c];
    if (R.second <= 0) continue;
    const dim3 grid(lntile[launch][c]);
    if (scaled[launch])
      launch_gemm_cls<false, true>(c, grid, d_probs.p, d_tiles.p, R.first, R.second, s);
    else
      launch_gemm_cls<false, false>(c, grid, d_probs.p, d_tiles.p, R.first, R.second, s);
  }
  for (int pid : dense[launch]) {
    const GemmProb &p = probs[pid];
    dim3 grid((p.N + GBN - 1) / GBN, (p.M + GBM - 1) / GBM);
    if (p.d)
      launch_gemm_cls<true, true>(trans_class(p), grid, d_probs.p, d_tiles.p, pid, 0, s);
    else
      launch_gemm_cls<true, false>(trans_class(p), grid, d_probs.p, d_tiles.p, pid, 0, s);
  }
  if (g_gemm_timing) {
    VB_CUDA(cudaEventRecord(e1, s));
    g_gemm_events.push_back({e0, e1});
  }
}

void gemm_grouped(GemmPlan &plan, int launch, cudaStream_t s) { plan.run(launch, s); }

// ------------------------------------------------------------------ partial LDL^T
// max |diag A| of each matrix before the factorisation (scale of the relative pivot test)
__global__ void diag_absmax_kernel(const MatDesc *__restrict__ mats, double *scale) {
  const MatDesc M = mats[blockIdx.x];
  __shared__ double red[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < M.n; i += blockDim.x) v = fmax(v, fabs(M.A[(int64_t)i * (M.ld + 1)]));
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) v = fmax(v, red[w]);
    scale[blockIdx.x] = fmax(red[0], v);
  }
}

// Factor the nb x nb diagonal block D11 L11 at (j0, j0) of M into shared memory (unit-lower L11
// below the diagonal, dd = D11): one warp, right-looking over the 32 columns.  Pivot test as
// MatDesc::npos says; `report`: this CTA writes *info.
__device__ void ldl_diag32(const MatDesc &M, int j0, int nb, double (*L11)[33], double *dd, int *info, bool report,
                           double scale) {
  const int tid = threadIdx.x, lane = tid & 31;
  for (int idx = tid; idx < 1024; idx += blockDim.x) {
    const int i = idx & 31, j = idx >> 5;
    L11[i][j] = (i < nb && j < nb && i >= j) ? M.A[(j0 + i) + (int64_t)(j0 + j) * M.ld] : 0.0;
  }
  __syncthreads();
  if (tid < 32) {
    for (int j = 0; j < nb; ++j) {
      const double d = L11[j][j];
      if (lane == 0) {
        dd[j] = d;
        bool bad = !(fabs(d) > 1e-300) || !isfinite(d);
        if (M.npos >= 0) {
          const double tol = kPivRel * scale;
          bad = bad || (j0 + j < M.npos ? !(d > tol) : !(d < -tol));
        }
        if (bad && report && info) atomicCAS(info, 0, 1 + j0 + j);
      }
      __syncwarp();
      if (lane > j && lane < nb) L11[lane][j] /= d;
      __syncwarp();
      if (lane > j && lane < nb) {
        const double lij = L11[lane][j] * d;
        for (int t = j + 1; t <= lane; ++t) L11[lane][t] -= lij * L11[t][j];
      }
      __syncwarp();
    }
  }
  __syncthreads();
}

// Panel of the blocked LDL^T (ldl_partial_batched), two launches.  (a) one CTA per matrix: factor
// the nb x nb diagonal block D11 L11 (one warp, ldl_diag32), write it back, and form
// W = L11^{-T} D11^{-1} (lane j: column j, back substitution) into `wbuf`; (b) the rows below:
// L21 = A21 W as independent dot products (one thread per row; column-major rows are coalesced),
// W read once per CTA into shared memory.  The serial 32-step work is done once per matrix.
constexpr int PANEL_ROWS = 128;
__global__ void __launch_bounds__(128) ldl_panel_a_kernel(const MatDesc *__restrict__ mats, int j0, int *info,
                                                          const double *__restrict__ scale, double *wbuf) {
  const MatDesc M = mats[blockIdx.x];
  if (j0 >= M.m) return;
  const int nb = min(32, M.m - j0);
  __shared__ double L11[32][33], dd[32];
  ldl_diag32(M, j0, nb, L11, dd, info ? info + blockIdx.x : nullptr, true, scale[blockIdx.x]);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 1024; idx += blockDim.x) {
    const int i = idx & 31, j = idx >> 5;
    if (i < nb && j < nb && i >= j) M.A[(j0 + i) + (int64_t)(j0 + j) * M.ld] = (i == j) ? dd[i] : L11[i][j];
  }
  if (tid < 32) {   // W = U^{-1} D^{-1}, U = L11^T unit upper: lane j back-substitutes column j
    const int j = tid;
    double w[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) w[t] = 0.0;
    if (j < nb) {
      w[j] = 1.0 / dd[j];
#pragma unroll
      for (int t = 31; t >= 0; --t) {
        if (t < j) {
          double v = 0.0;
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (q > t && q <= j) v -= L11[q][t] * w[q];   // U[t][q] = L11[q][t]
          w[t] = v;
        }
      }
    }
    double *W = wbuf + (int64_t)blockIdx.x * 1024;   // W[t + 32 j]
#pragma unroll
    for (int t = 0; t < 32; ++t) W[t + 32 * j] = w[t];
  }
}

__global__ void __launch_bounds__(PANEL_ROWS) ldl_panel_b_kernel(const MatDesc *__restrict__ mats, int j0,
                                                                 const double *__restrict__ wbuf) {
  const MatDesc M = mats[blockIdx.y];
  if (j0 >= M.m) return;
  const int nb = min(32, M.m - j0);
  const int r0 = j0 + nb + PANEL_ROWS * blockIdx.x;
  if (r0 >= M.n) return;
  __shared__ double W[32][33];
  const double *Wg = wbuf + (int64_t)blockIdx.y * 1024;
  for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) W[idx & 31][idx >> 5] = Wg[idx];
  __syncthreads();
  const int row = r0 + threadIdx.x;
  if (row >= M.n) return;
  double a[32];
#pragma unroll
  for (int t = 0; t < 32; ++t) a[t] = t < nb ? M.A[row + (int64_t)(j0 + t) * M.ld] : 0.0;
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    if (j < nb) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t <= j; ++t) v += a[t] * W[t][j];
      M.A[row + (int64_t)(j0 + j) * M.ld] = v;
    }
  }
}

// Blocked right-looking LDL^T.  The columns are processed in wide panels of LDL_NB; inside a wide
// panel they are split recursively in halves (multiples of 32): factor the left half, update the
// right half's columns (all rows below) with K = the left half's width, factor the right half -- so
// the intra-panel updates run as K = 128 / 64 / 32 DMMA GEMMs instead of a sequence of K = 32 ones;
// the 32-column leaves are ldl_panel_a/b_kernel launches.  The trailing matrix is updated once per wide
// panel (K = LDL_NB).  Every step is one launch over all matrices of the batch.
void ldl_partial_batched(const std::vector<MatDesc> &mats, int *info_dev, cudaStream_t s) {
  if (mats.empty()) return;
  DBuf<MatDesc> dm;
  std::vector<MatDesc> hm(mats);
  dm.upload(hm, s);
  int maxm = 0, maxn = 0;
  for (auto &M : mats) { maxm = std::max(maxm, M.m); maxn = std::max(maxn, M.n); }
  GemmPlan plan;
  std::vector<std::pair<int, int>> ops;   // (0, j0): panel at j0; (1, launch): GEMM launch
  auto update = [&](int a, int mid, int b) {   // columns [mid, b) (rows mid..n) from columns [a, mid)
    const int lid = plan.begin_launch();
    for (auto &M : mats) {
      const int e = std::min(b, M.m);
      if (mid >= e) continue;
      GemmProb p{};
      p.A = M.A + mid + (int64_t)a * M.ld; p.lda = M.ld; p.transA = 0;
      p.B = p.A; p.ldb = M.ld; p.transB = 1;
      p.d = M.A + (int64_t)a * (M.ld + 1); p.dstride = M.ld + 1;
      p.C = M.A + (int64_t)mid * (M.ld + 1); p.ldc = M.ld;
      p.M = M.n - mid; p.N = e - mid; p.K = mid - a; p.alpha = -1.0; p.beta = 1.0; p.lower = 1;
      plan.add(p);
    }
    ops.push_back({1, lid});
  };
  std::function<void(int, int)> rec = [&](int a, int b) {
    if (b - a <= 32) {
      ops.push_back({0, a});
      return;
    }
    const int mid = a + ((b - a) / 2 + 31) / 32 * 32;
    rec(a, mid);
    update(a, mid, b);
    rec(mid, b);
  };
  for (int J0 = 0; J0 < maxm; J0 += LDL_NB) {
    rec(J0, std::min(J0 + LDL_NB, maxm));
    const int lid = plan.begin_launch();
    for (auto &M : mats) {
      if (J0 >= M.m) continue;
      const int Je = std::min(J0 + LDL_NB, M.m);
      const int rows = M.n - Je;
      if (rows <= 0) continue;
      GemmProb p{};
      p.A = M.A + Je + (int64_t)J0 * M.ld; p.lda = M.ld; p.transA = 0;
      p.B = p.A; p.ldb = M.ld; p.transB = 1;
      p.d = M.A + (int64_t)J0 * (M.ld + 1); p.dstride = M.ld + 1;
      p.C = M.A + (int64_t)Je * (M.ld + 1); p.ldc = M.ld;
      p.M = p.N = rows; p.K = Je - J0; p.alpha = -1.0; p.beta = 1.0; p.lower = 1;
      plan.add(p);
    }
    ops.push_back({1, lid});
  }
  plan.upload(s);
  DBuf<double> dscale, ddiag;
  dscale.alloc(mats.size());
  ddiag.alloc(mats.size() * 1024);
  diag_absmax_kernel<<<mats.size(), 256, 0, s>>>(dm.p, dscale.p);
  VB_CHECK_LAUNCH();
  for (auto &op : ops) {
    if (op.first == 0) {
      const int j0 = op.second;
      ldl_panel_a_kernel<<<mats.size(), 128, 0, s>>>(dm.p, j0, info_dev, dscale.p, ddiag.p);
      VB_CHECK_LAUNCH();
      dim3 grid(std::max(1, (maxn - j0 - 1) / PANEL_ROWS + 1), mats.size());
      ldl_panel_b_kernel<<<grid, PANEL_ROWS, 0, s>>>(dm.p, j0, ddiag.p);
      VB_CHECK_LAUNCH();
    } else {
      plan.run(op.second, s);
    }
  }
  VB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ triangular inverse
__global__ void set_identity_kernel(const TriDesc *mats) {
  const TriDesc T = mats[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T.m; i += gridDim.x * blockDim.x)
    T.X[i + (int64_t)i * T.ldx] = 1.0;
}

// Inverses of all 32 x 32 unit-lower diagonal blocks of L (known before the blocked inversion
// starts): CTA (J, matrix), lane j computes column j of L_JJ^{-1} by forward substitution in
// registers into linv[matrix offset + 1024 J] (column-major 32 x 32, zero above the diagonal).
__global__ void tri_diag_inv_kernel(const TriDesc *__restrict__ mats, const int64_t *__restrict__ off,
                                    double *linv) {
  const TriDesc T = mats[blockIdx.y];
  const int J = blockIdx.x, r0 = 32 * J;
  if (r0 >= T.m) return;
  const int nb = min(32, T.m - r0);
  __shared__ double L[32][33];
  for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
    const int i = idx & 31, j = idx >> 5;
    L[i][j] = (i < nb && j < nb && i > j) ? T.L[(r0 + i) + (int64_t)(r0 + j) * T.ldl] : 0.0;
  }
  __syncthreads();
  if (threadIdx.x >= 32) return;
  double *Li = linv + off[blockIdx.y] + 1024 * (int64_t)J;
  const int j = threadIdx.x;
  double col[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) col[i] = (i == j && j < nb) ? 1.0 : 0.0;
#pragma unroll
  for (int i = 1; i < 32; ++i) {
    if (i > j && i < nb) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q >= j && q < i) v -= L[i][q] * col[q];
      col[i] = v;
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) Li[i + 32 * j] = col[i];
}

// X_J <- L_JJ^{-1} X_J for the 32-row block J on the columns 0 .. 32 J + nb - 1, one thread per
// column (independent dot products with the precomputed inverse, read once per CTA).
constexpr int TRI_COLS = 128;
__global__ void __launch_bounds__(TRI_COLS) trsm_diag_kernel(const TriDesc *__restrict__ mats, int J,
                                                             const int64_t *__restrict__ off,
                                                             const double *__restrict__ linv) {
  const TriDesc T = mats[blockIdx.y];
  const int r0 = 32 * J;
  if (r0 >= T.m) return;
  const int nb = min(32, T.m - r0);
  if (TRI_COLS * (int)blockIdx.x >= r0 + nb) return;
  __shared__ double Li[32][33];
  const double *Lg = linv + off[blockIdx.y] + 1024 * (int64_t)J;
  for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) Li[idx & 31][idx >> 5] = Lg[idx];
  __syncthreads();
  const int col = TRI_COLS * blockIdx.x + threadIdx.x;
  if (col >= r0 + nb) return;
  double x[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) x[i] = i < nb ? T.X[(r0 + i) + (int64_t)col * T.ldx] : 0.0;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < nb) {
      double v = 0.0;
#pragma unroll
      for (int q = 0; q <= i; ++q) v += Li[i][q] * x[q];
      T.X[(r0 + i) + (int64_t)col * T.ldx] = v;
    }
  }
}

// X <- L^{-1} by blocked forward substitution: row blocks of 32 (trsm_diag_kernel) grouped into wide
// blocks of TRI_NB; inside a wide block the rows are split recursively in halves: invert the upper
// half, update the lower half's rows with K = the upper half's height (DMMA GEMM), invert the lower
// half; the rows below the wide block are updated once per wide block (K = TRI_NB).
void tri_inverse_batched(const std::vector<TriDesc> &mats, cudaStream_t s) {
  if (mats.empty()) return;
  DBuf<TriDesc> dm;
  std::vector<TriDesc> hm(mats);
  dm.upload(hm, s);
  int maxm = 0;
  for (auto &T : mats) maxm = std::max(maxm, T.m);
  if (maxm == 0) return;
  set_identity_kernel<<<dim3((maxm + 255) / 256, mats.size()), 256, 0, s>>>(dm.p);
  VB_CHECK_LAUNCH();
  GemmPlan plan;
  std::vector<std::pair<int, int>> ops;   // (0, J): diagonal block J; (1, launch): GEMM launch
  auto update = [&](int a, int mid, int b) {   // rows [mid, b) from rows [a, mid), columns 0 .. mid-1
    const int lid = plan.begin_launch();
    for (auto &T : mats) {
      const int e = std::min(b, T.m);
      if (mid >= e) continue;
      GemmProb p{};
      p.A = T.L + mid + (int64_t)a * T.ldl; p.lda = T.ldl; p.transA = 0;
      p.B = T.X + a; p.ldb = T.ldx; p.transB = 0;
      p.C = T.X + mid; p.ldc = T.ldx;
      p.M = e - mid; p.N = mid; p.K = mid - a;
      p.alpha = -1.0; p.beta = 1.0; p.lower = 0;
      plan.add(p);
    }
    ops.push_back({1, lid});
  };
  std::function<void(int, int)> rec = [&](int a, int b) {
    if (b - a <= 32) {
      ops.push_back({0, a / 32});
      return;
    }
    const int mid = a + ((b - a) / 2 + 31) / 32 * 32;
    rec(a, mid);
    update(a, mid, b);
    rec(mid, b);
  };
  for (int J0 = 0; J0 < maxm; J0 += TRI_NB) {
    rec(J0, std::min(J0 + TRI_NB, maxm));
    const int lid = plan.begin_launch();
    for (auto &T : mats) {
      if (J0 >= T.m) continue;
      const int Je = std::min(J0 + TRI_NB, T.m);
      const int rows = T.m - Je;
      if (rows <= 0) continue;
      GemmProb p{};
      p.A = T.L + Je + (int64_t)J0 * T.ldl; p.lda = T.ldl; p.transA = 0;
      p.B = T.X + J0; p.ldb = T.ldx; p.transB = 0;
      p.C = T.X + Je; p.ldc = T.ldx;
      p.M = rows; p.N = Je; p.K = Je - J0;
      p.alpha = -1.0; p.beta = 1.0; p.lower = 0;
      plan.add(p);
    }
    ops.push_back({1, lid});
  }
  plan.upload(s);
  std::vector<int64_t> off(mats.size());
  int64_t tot = 0;
  for (size_t b = 0; b < mats.size(); ++b) { off[b] = tot; tot += 1024 * (int64_t)((mats[b].m + 31) / 32); }
  DBuf<int64_t> doff;
  DBuf<double> linv;
  doff.upload(off, s);
  linv.alloc(std::max<int64_t>(tot, 1));
  tri_diag_inv_kernel<<<dim3((maxm + 31) / 32, mats.size()), 64, 0, s>>>(dm.p, doff.p, linv.p);
  VB_CHECK_LAUNCH();
  for (auto &op : ops) {
    if (op.first == 0) {
      const int J = op.second;
      dim3 grid((32 * J + 32 + TRI_COLS - 1) / TRI_COLS, mats.size());
      trsm_diag_kernel<<<grid, TRI_COLS, 0, s>>>(dm.p, J, doff.p, linv.p);
      VB_CHECK_LAUNCH();
    } else {
      plan.run(op.second, s);
    }
  }
  VB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ symmetrize / pack
__global__ void symmetrize_kernel(const MatDesc *__restrict__ mats) {
  const MatDesc M = mats[blockIdx.z];
  int i = blockIdx.y * 32 + threadIdx.y, j = blockIdx.x * 32 + threadIdx.x;   // write (i,j), i<j
  if (i < M.n && j < M.n && i < j) M.A[i + (int64_t)j * M.ld] = M.A[j + (int64_t)i * M.ld];
}

void symmetrize_lower_batched(const std::vector<MatDesc> &mats, cudaStream_t s) {
  if (mats.empty()) return;
  DBuf<MatDesc> dm;
  std::vector<MatDesc> hm(mats);
  dm.upload(hm, s);
  int maxn = 0;
  for (auto &M : mats) maxn = std::max(maxn, M.n);
  if (maxn == 0) return;
  int nt = (maxn + 31) / 32;
  symmetrize_kernel<<<dim3(nt, nt, mats.size()), dim3(32, 32), 0, s>>>(dm.p);
  VB_CHECK_LAUNCH();
  VB_CUDA(cudaStreamSynchronize(s));
}

__global__ void pack_tiles_kernel(const PackDesc *__restrict__ mats) {
  const PackDesc M = mats[blockIdx.z];
  const int I = blockIdx.y, J = blockIdx.x;
  if (J > I) return;
  if (32 * I >= M.n) return;
  const int rows = min(32, M.n - 32 * I);
  double *out = M.out + ptile_off(M.n, I, J);
  for (int idx = threadIdx.x; idx < rows * 32; idx += blockDim.x) {
    const int r = idx >> 5, cc = idx & 31;
    const int row = 32 * I + r, col = 32 * J + cc;
    double v = 0.0;
    if (row < M.n && col < M.n)
      v = row >= col ? M.A[row + (int64_t)col * M.ld] : M.A[col + (int64_t)row * M.ld];
    out[idx] = v;
  }
}

void pack_tiles_batched(const std::vector<PackDesc> &mats, cudaStream_t s) {
  if (mats.empty()) return;
  DBuf<PackDesc> dm;
  std::vector<PackDesc> hm(mats);
  dm.upload(hm, s);
  int maxn = 0;
  for (auto &M : mats) maxn = std::max(maxn, M.n);
  if (maxn == 0) return;
  int nt = (maxn + 31) / 32;
  pack_tiles_kernel<<<dim3(nt, nt, mats.size()), 256, 0, s>>>(dm.p);
  VB_CHECK_LAUNCH();
  VB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vb
