// Batched dense FP64 kernels: grouped DMMA GEMM (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4, the
// FP64 tensor path of sm_100a; tcgen05 has no f64 kind), blocked partial LDL^T,
// triangular inverse, packing.  Used by the factor stage.
#include <algorithm>
#include <map>
#include <mutex>
#include "dense.cuh"

namespace vb {

// ------------------------------------------------------------------ grouped GEMM (DMMA)
// CTA tile 128 x 64 x 16, 8 warps (4 along M x 2 along N), warp tile 32 x 32 = 2 x 4 tiles of
// mma.sync.m16n8k16.f64 (SASS DMMA.16816: 8x fewer tensor instructions than m8n8k4 for the same
// work).  K-slabs of 16 stream through a 3-stage cp.async shared-memory ring, one barrier per slab.
constexpr int GBM = 128, GBN = 64, GBK = 16;   // 128x128 measured slower (1 CTA/SM, padding on small N)
constexpr int GPAD = 4;
constexpr int GTHREADS = 256;
constexpr int LDL_NB = 256;        // wide-panel width of the blocked LDL^T
#ifndef TRI_NB_CFG
#define TRI_NB_CFG 256
#endif
constexpr int TRI_NB = TRI_NB_CFG;   // wide-block width of the triangular inverse
constexpr int GWARPS_N = GBN / 32, GWARPS_M = (GTHREADS / 32) / GWARPS_N;
constexpr int GMI = GBM / GWARPS_M / 16;        // m16n8k16 tiles per warp along M
constexpr int GA_PER = GBM * GBK / GTHREADS;
constexpr int GB_PER = GBK * GBN / GTHREADS;

// D(16x8) += A(16x16) B(16x8); fragments (PTX ISA, f64 m16n8k16; g = lane / 4, t = lane % 4):
//   a[v] = A(g + 8 (v % 2), t + 4 (v / 2)),  b[v] = B(t + 4 v, g),  c[v] = C(g + 8 (v / 2), 2 t + v % 2)
__device__ __forceinline__ void dmma_16x8x16(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

// ---- asynchronous K-slab loads: cp.async 8-byte copies into a 3-stage shared-memory ring
// (zero-filled outside the matrix); the diagonal scaling d of op(A)'s columns is applied to the A
// fragments, so A and B are copied unmodified.
constexpr int GSTAGES = 3;
struct GemmSmem {
  double A[GSTAGES][GBM][GBK + GPAD];
  double B[GSTAGES][GBK][GBN + GPAD];
  double D[GSTAGES][GBK];
};

__device__ __forceinline__ void cp_async8(void *smem, const void *gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int bytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Per-thread copy pattern of the K-slabs, fixed for the whole K loop (only k0 moves).  With 256
// threads, thread tid copies for slot q:
//   op(A) slab (i, kk):  A not transposed (i contiguous): i = tid % 128, kk = tid / 128 + 2 q
//                        A transposed (k contiguous):     kk = tid % 16,  i = tid / 16 + 16 q
//   op(B) slab (kk, j):  B not transposed (k contiguous): kk = tid % 16,  j = tid / 16 + 16 q
//                        B transposed (j contiguous):     j = tid % 64,   kk = tid / 64 + 4 q
// so consecutive threads read consecutive addresses in every case.
static_assert(GTHREADS == 256 && GBM == 128 && GBN == 64 && GBK == 16, "copy pattern assumes these");
template <bool TA> struct ACopy {
  static constexpr int DI = TA ? 16 : 0, DKK = TA ? 0 : 2;
  __device__ static int i0(int tid) { return TA ? tid / GBK : tid % GBM; }
  __device__ static int kk0(int tid) { return TA ? tid % GBK : tid / GBM; }
};
template <bool TB> struct BCopy {
  static constexpr int DJ = TB ? 0 : 16, DKK = TB ? 4 : 0;
  __device__ static int j0(int tid) { return TB ? tid % GBN : tid / GBK; }
  __device__ static int kk0(int tid) { return TB ? tid / GBN : tid % GBK; }
};

template <bool TA, bool TB>
__device__ __forceinline__ void issue_slab(const double *pa, const double *pb, int lda, int ldb, const double *A0,
                                           const double *B0, int rows_left, int cols_left, int k_left,
                                           const double *d, int dstride, int tid, GemmSmem &sm, int stage) {
  // pa / pb: this thread's slot-0 sources in the current slab; *_left: extents past the tile origin
  const int ai = ACopy<TA>::i0(tid), akk = ACopy<TA>::kk0(tid);
#pragma unroll
  for (int q = 0; q < GA_PER; ++q) {
    const int i = ai + q * ACopy<TA>::DI, kk = akk + q * ACopy<TA>::DKK;
    const bool ok = i < rows_left && kk < k_left;
    const int64_t off = TA ? (int64_t)(q * 16) * lda : (int64_t)(q * 2) * lda;
    cp_async8(&sm.A[stage][i][kk], ok ? pa + off : A0, ok);
  }
  const int bj = BCopy<TB>::j0(tid), bkk = BCopy<TB>::kk0(tid);
#pragma unroll
  for (int q = 0; q < GB_PER; ++q) {
    const int j = bj + q * BCopy<TB>::DJ, kk = bkk + q * BCopy<TB>::DKK;
    const bool ok = j < cols_left && kk < k_left;
    const int64_t off = TB ? (int64_t)(q * 4) * ldb : (int64_t)(q * 16) * ldb;
    cp_async8(&sm.B[stage][kk][j], ok ? pb + off : B0, ok);
  }
  if (d && tid < GBK) {
    const bool ok = tid < k_left;
    cp_async8(&sm.D[stage][tid], ok ? d + (int64_t)tid * dstride : d, ok);
  }
}

// DENSE: one large problem (id = tile0) on a 2D grid of tiles (no tile list).
// SCALED: some problem of the launch has a diagonal scaling d (else the multiply is compiled out).
// TA / TB: op(A) = A^T / op(B) = B^T for every problem of the launch.
template <bool DENSE, bool SCALED, bool TA, bool TB>
__global__ void __launch_bounds__(GTHREADS, 2) gemm_grouped_kernel(const GemmProb *__restrict__ probs,
                                                                  const int4 *__restrict__ tiles, int tile0) {
  const int4 t = DENSE ? make_int4(tile0, blockIdx.y, blockIdx.x, 0) : tiles[tile0 + blockIdx.x];
  __shared__ GemmProb Ps;                 // problem descriptor in shared memory (register pressure)
  if (threadIdx.x == 0) Ps = probs[t.x];
  __syncthreads();
  const GemmProb &P = Ps;
  const int m0 = t.y * GBM, n0 = t.z * GBN;
  if (DENSE && P.lower && m0 + GBM - 1 < n0) return;   // tile strictly above the diagonal
  extern __shared__ __align__(16) unsigned char gsm_raw[];
  GemmSmem &sm = *reinterpret_cast<GemmSmem *>(gsm_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wm = (warp / GWARPS_N) * (GBM / GWARPS_M), wn = (warp % GWARPS_N) * 32;
  const bool scaled = SCALED && P.d != nullptr;
  double acc[GMI][4][4];
#pragma unroll
  for (int i = 0; i < GMI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;
  const int lda = P.lda, ldb = P.ldb, K = P.K, dstride = P.dstride;
  const int rows_left = P.M - m0, cols_left = P.N - n0;
  const double *dvec = SCALED ? P.d : nullptr;
  // slot-0 sources at k0 = 0 and their advance per slab
  const double *pa = TA ? P.A + ACopy<TA>::kk0(tid) + (int64_t)(m0 + ACopy<TA>::i0(tid)) * lda
                        : P.A + (m0 + ACopy<TA>::i0(tid)) + (int64_t)ACopy<TA>::kk0(tid) * lda;
  const double *pb = TB ? P.B + (n0 + BCopy<TB>::j0(tid)) + (int64_t)BCopy<TB>::kk0(tid) * ldb
                        : P.B + BCopy<TB>::kk0(tid) + (int64_t)(n0 + BCopy<TB>::j0(tid)) * ldb;
  const int64_t astep = TA ? GBK : (int64_t)GBK * lda, bstep = TB ? (int64_t)GBK * ldb : GBK;
  const double *A0 = P.A, *B0 = P.B;
  int kb = 0;   // first K slab with non-zero products (triangular operands)
  if (P.kz_on) {
    kb = max(0, max(m0 + P.kzA, n0 + P.kzB)) / GBK * GBK;
    if (kb > K) kb = K;
    pa += (kb / GBK) * astep;
    pb += (kb / GBK) * bstep;
  }
  if (kb < K)
    issue_slab<TA, TB>(pa, pb, lda, ldb, A0, B0, rows_left, cols_left, K - kb,
                       dvec ? dvec + (int64_t)kb * dstride : nullptr, dstride, tid, sm, 0);
  cp_async_commit();
  if (kb + GBK < K)
    issue_slab<TA, TB>(pa + astep, pb + bstep, lda, ldb, A0, B0, rows_left, cols_left, K - kb - GBK,
                       dvec ? dvec + (int64_t)(kb + GBK) * dstride : nullptr, dstride, tid, sm, 1);
  cp_async_commit();
  pa += 2 * astep;
  pb += 2 * bstep;
  int st = 0;
  for (int k0 = kb; k0 < K; k0 += GBK) {
    cp_async_wait1();       // all groups but the newest are complete: this slab has landed
    __syncthreads();        // ... for every thread; and every thread is done with the previous slab
    {
      int nst = st + 2;
      if (nst >= GSTAGES) nst -= GSTAGES;   // = the stage of the previous slab, free again
      if (k0 + 2 * GBK < K)
        issue_slab<TA, TB>(pa, pb, lda, ldb, A0, B0, rows_left, cols_left, K - k0 - 2 * GBK,
                           dvec ? dvec + (int64_t)(k0 + 2 * GBK) * dstride : nullptr, dstride, tid, sm, nst);
      cp_async_commit();
      pa += astep;
      pb += bstep;
    }
#pragma unroll
    for (int i = 0; i < GMI; ++i) {
      double a[8];
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        a[v] = sm.A[st][wm + 16 * i + g + 8 * (v & 1)][tg + 4 * (v >> 1)];
        if (SCALED && scaled) a[v] *= sm.D[st][tg + 4 * (v >> 1)];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        double b[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) b[v] = sm.B[st][tg + 4 * v][wn + 8 * j + g];
        dmma_16x8x16(acc[i][j], a, b);
      }
    }
    if (++st == GSTAGES) st = 0;
  }
#pragma unroll
  for (int i = 0; i < GMI; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int gi = m0 + wm + 16 * i + g + 8 * (v >> 1);
        const int gj = n0 + wn + 8 * j + 2 * tg + (v & 1);
        if (gi < P.M && gj < P.N && (!P.lower || gi >= gj)) {
          double *c = P.C + gi + (int64_t)gj * P.ldc;
          *c = (P.beta == 0.0 ? 0.0 : P.beta * *c) + P.alpha * acc[i][j][v];
        }
      }
}

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

template <bool DENSE, bool SCALED, bool TA, bool TB>
static void launch_gemm(dim3 grid, const GemmProb *probs, const int4 *tiles, int tile0, cudaStream_t s) {
  raise_smem_limit((const void *)gemm_grouped_kernel<DENSE, SCALED, TA, TB>, sizeof(GemmSmem));
  gemm_grouped_kernel<DENSE, SCALED, TA, TB><<<grid, GTHREADS, sizeof(GemmSmem), s>>>(probs, tiles, tile0);
  VB_CHECK_LAUNCH();
}

template <bool DENSE, bool SCALED>
static void launch_gemm_cls(int cls, dim3 grid, const GemmProb *probs, const int4 *tiles, int tile0, cudaStream_t s) {
  switch (cls) {
    case 0: launch_gemm<DENSE, SCALED, false, false>(grid, probs, tiles, tile0, s); break;
    case 1: launch_gemm<DENSE, SCALED, true, false>(grid, probs, tiles, tile0, s); break;
    case 2: launch_gemm<DENSE, SCALED, false, true>(grid, probs, tiles, tile0, s); break;
    default: launch_gemm<DENSE, SCALED, true, true>(grid, probs, tiles, tile0, s); break;
  }
}

static int trans_class(const GemmProb &p) { return (p.transA ? 1 : 0) + (p.transB ? 2 : 0); }

thread_local double g_gemm_flops = 0.0;   // DMMA GEMM flops issued by this thread (factor-stage accounting)

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
  for (int i = 0; i < tm; ++i)
    for (int j = 0; j < tn; ++j) {
      if (p.lower && (i * GBM + GBM - 1) < j * GBN) continue;   // tile strictly above diagonal
      tl.push_back(make_int4(pid, i, j, 0));
    }
}

void GemmPlan::upload(cudaStream_t s) {
  std::vector<GemmProb> hp(probs);
  std::vector<int4> ht;
  lrange.assign(ltiles.size(), {});
  for (size_t l = 0; l < ltiles.size(); ++l)
    for (int c = 0; c < 4; ++c) {
      lrange[l][c] = {(int)ht.size(), (int)ltiles[l][c].size()};
      ht.insert(ht.end(), ltiles[l][c].begin(), ltiles[l][c].end());
    }
  d_probs.upload(hp, s);
  d_tiles.upload(ht, s);
  VB_CUDA(cudaStreamSynchronize(s));
}

void GemmPlan::run(int launch, cudaStream_t s) {
  for (int c = 0; c < 4; ++c) {
    const auto &R = lrange[launch][c];
    if (R.second <= 0) continue;
    if (scaled[launch])
      launch_gemm_cls<false, true>(c, dim3(R.second), d_probs.p, d_tiles.p, R.first, s);
    else
      launch_gemm_cls<false, false>(c, dim3(R.second), d_probs.p, d_tiles.p, R.first, s);
  }
  for (int pid : dense[launch]) {
    const GemmProb &p = probs[pid];
    dim3 grid((p.N + GBN - 1) / GBN, (p.M + GBM - 1) / GBM);
    if (p.d)
      launch_gemm_cls<true, true>(trans_class(p), grid, d_probs.p, d_tiles.p, pid, s);
    else
      launch_gemm_cls<true, false>(trans_class(p), grid, d_probs.p, d_tiles.p, pid, s);
  }
}

void gemm_grouped(GemmPlan &plan, int launch, cudaStream_t s) { plan.run(launch, s); }

// ------------------------------------------------------------------ partial LDL^T
// Phase 1 (blockIdx.x == 0 launch): factor the nb x nb diagonal block in place.
// Phase 2 (separate launch): panel rows below read the factored block (no read/write race).
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

__global__ void ldl_panel_kernel(const MatDesc *__restrict__ mats, int j0, int *info, int phase,
                                 const double *__restrict__ scale) {
  const MatDesc M = mats[blockIdx.y];
  if (j0 >= M.m) return;
  const int nb = min(32, M.m - j0);
  const int r0 = phase == 0 ? j0 : j0 + nb + 32 * blockIdx.x;
  if (r0 >= M.n) return;
  __shared__ double L11[32][33];
  __shared__ double dd[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double *A = M.A;
  const int64_t ld = M.ld;
  if (phase == 1) {
    for (int idx = tid; idx < 1024; idx += blockDim.x) {
      int i = idx & 31, j = idx >> 5;
      L11[i][j] = (i < nb && j < nb && i > j) ? A[(j0 + i) + (j0 + j) * ld] : 0.0;
    }
    if (tid < 32) dd[tid] = tid < nb ? A[(j0 + tid) * (ld + 1)] : 1.0;
    __syncthreads();
    if (warp == 0) {
      const int row = r0 + lane;
      if (row < M.n) {
        double l[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j < nb) {
            double v = A[row + (j0 + j) * ld];
            for (int t = 0; t < j; ++t) v -= l[t] * dd[t] * L11[j][t];
            l[j] = v / dd[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < nb) A[row + (j0 + j) * ld] = l[j];
      }
    }
    return;
  }
  for (int idx = tid; idx < 1024; idx += blockDim.x) {
    int i = idx & 31, j = idx >> 5;
    L11[i][j] = (i < nb && j < nb && i >= j) ? A[(j0 + i) + (j0 + j) * ld] : 0.0;
  }
  __syncthreads();
  if (warp == 0) {
    for (int j = 0; j < nb; ++j) {
      double d = L11[j][j];
      if (lane == 0) {
        dd[j] = d;
        bool bad = !(fabs(d) > 1e-300) || !isfinite(d);
        if (M.npos >= 0) {
          const double tol = kPivRel * scale[blockIdx.y];
          bad = bad || (j0 + j < M.npos ? !(d > tol) : !(d < -tol));
        }
        if (bad && info && blockIdx.x == 0) atomicCAS(&info[blockIdx.y], 0, 1 + j0 + j);
      }
      __syncwarp();
      if (lane > j && lane < nb) L11[lane][j] /= d;
      __syncwarp();
      if (lane > j && lane < nb) {
        double lij = L11[lane][j] * d;
        for (int t = j + 1; t <= lane; ++t) L11[lane][t] -= lij * L11[t][j];
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int idx = tid; idx < 1024; idx += blockDim.x) {
    int i = idx & 31, j = idx >> 5;
    if (i < nb && j < nb && i >= j) A[(j0 + i) + (j0 + j) * ld] = (i == j) ? dd[i] : L11[i][j];
  }
}

// Blocked right-looking LDL^T: 32-column panels factored by ldl_panel_kernel, grouped into wide
// panels of LDL_NB columns; inside a wide panel only its remaining columns are updated (K = 32), the
// trailing matrix once per wide panel with K = LDL_NB (DMMA GEMM, 4x fewer passes over the trailing
// matrix than a 32-column right-looking update).
void ldl_partial_batched(const std::vector<MatDesc> &mats, int *info_dev, cudaStream_t s) {
  if (mats.empty()) return;
  DBuf<MatDesc> dm;
  std::vector<MatDesc> hm(mats);
  dm.upload(hm, s);
  int maxm = 0, maxn = 0;
  for (auto &M : mats) { maxm = std::max(maxm, M.m); maxn = std::max(maxn, M.n); }
  GemmPlan plan;
  std::vector<int> intra_launch, trail_launch;   // per 32-panel step / per wide panel
  for (int J0 = 0; J0 < maxm; J0 += LDL_NB) {
    for (int j0 = J0; j0 < std::min(J0 + LDL_NB, maxm); j0 += 32) {
      intra_launch.push_back(plan.begin_launch());
      for (auto &M : mats) {
        if (j0 >= M.m) continue;
        const int nb = std::min(32, M.m - j0);
        const int Je = std::min(J0 + LDL_NB, M.m);
        const int rows = M.n - j0 - nb, cols = Je - j0 - nb;
        if (rows <= 0 || cols <= 0) continue;
        GemmProb p{};
        p.A = M.A + (j0 + nb) + (int64_t)j0 * M.ld; p.lda = M.ld; p.transA = 0;
        p.B = p.A; p.ldb = M.ld; p.transB = 1;
        p.d = M.A + (int64_t)j0 * (M.ld + 1); p.dstride = M.ld + 1;
        p.C = M.A + (int64_t)(j0 + nb) * (M.ld + 1); p.ldc = M.ld;
        p.M = rows; p.N = cols; p.K = nb; p.alpha = -1.0; p.beta = 1.0; p.lower = 1;
        plan.add(p);
      }
    }
    trail_launch.push_back(plan.begin_launch());
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
  }
  plan.upload(s);
  DBuf<double> dscale;
  dscale.alloc(mats.size());
  diag_absmax_kernel<<<mats.size(), 256, 0, s>>>(dm.p, dscale.p);
  VB_CHECK_LAUNCH();
  int step = 0, wide = 0;
  for (int J0 = 0; J0 < maxm; J0 += LDL_NB, ++wide) {
    for (int j0 = J0; j0 < std::min(J0 + LDL_NB, maxm); j0 += 32, ++step) {
      ldl_panel_kernel<<<dim3(1, mats.size()), 128, 0, s>>>(dm.p, j0, info_dev, 0, dscale.p);
      VB_CHECK_LAUNCH();
      dim3 grid((maxn - j0 + 31) / 32, mats.size());
      ldl_panel_kernel<<<grid, 32, 0, s>>>(dm.p, j0, info_dev, 1, dscale.p);
      VB_CHECK_LAUNCH();
      plan.run(intra_launch[step], s);
    }
    plan.run(trail_launch[wide], s);
  }
  VB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ triangular inverse
__global__ void set_identity_kernel(const TriDesc *mats) {
  const TriDesc T = mats[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < T.m; i += gridDim.x * blockDim.x)
    T.X[i + (int64_t)i * T.ldx] = 1.0;
}

// Solve L_JJ X_J = X_J (in place) for column block cb of block row J (unit lower L_JJ).
__global__ void trsm_diag_kernel(const TriDesc *__restrict__ mats, int J) {
  const TriDesc T = mats[blockIdx.y];
  const int r0 = 32 * J;
  if (r0 >= T.m) return;
  const int cb = blockIdx.x;
  if (cb > J) return;
  const int nb = min(32, T.m - r0);
  __shared__ double L[32][33];
  for (int idx = threadIdx.x; idx < 1024; idx += blockDim.x) {
    int i = idx & 31, j = idx >> 5;
    L[i][j] = (i < nb && j < nb && i > j) ? T.L[(r0 + i) + (int64_t)(r0 + j) * T.ldl] : 0.0;
  }
  __syncthreads();
  int col = 32 * cb + threadIdx.x;
  if (threadIdx.x < 32 && col < T.m) {
    double x[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < nb) {
        double v = T.X[(r0 + i) + (int64_t)col * T.ldx];
        for (int t = 0; t < i; ++t) v -= L[i][t] * x[t];
        x[i] = v;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < nb) T.X[(r0 + i) + (int64_t)col * T.ldx] = x[i];
  }
}

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
  // blocked like the LDL^T: 32-row diagonal solves, updates inside a 128-row wide block with K = 32,
  // the rows below the wide block once per wide block with K = 128
  int nblk = (maxm + 31) / 32;
  GemmPlan plan;
  std::vector<int> intra(nblk, -1), trail;
  for (int J0 = 0; J0 < maxm; J0 += TRI_NB) {
    for (int r0 = J0; r0 < std::min(J0 + TRI_NB, maxm); r0 += 32) {
      intra[r0 / 32] = plan.begin_launch();
      for (auto &T : mats) {
        if (r0 >= T.m) continue;
        const int nb = std::min(32, T.m - r0);
        const int Je = std::min(J0 + TRI_NB, T.m);
        const int rows = Je - r0 - nb;
        if (rows <= 0) continue;
        GemmProb p{};
        p.A = T.L + (r0 + nb) + (int64_t)r0 * T.ldl; p.lda = T.ldl; p.transA = 0;
        p.B = T.X + r0; p.ldb = T.ldx; p.transB = 0;
        p.C = T.X + (r0 + nb); p.ldc = T.ldx;
        p.M = rows; p.N = r0 + nb; p.K = nb;
        p.alpha = -1.0; p.beta = 1.0; p.lower = 0;
        plan.add(p);
      }
    }
    trail.push_back(plan.begin_launch());
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
  }
  plan.upload(s);
  int wide = 0;
  for (int J0 = 0; J0 < maxm; J0 += TRI_NB, ++wide) {
    for (int r0 = J0; r0 < std::min(J0 + TRI_NB, maxm); r0 += 32) {
      const int J = r0 / 32;
      trsm_diag_kernel<<<dim3(J + 1, mats.size()), 32, 0, s>>>(dm.p, J);
      VB_CHECK_LAUNCH();
      plan.run(intra[J], s);
    }
    plan.run(trail[wide], s);
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
