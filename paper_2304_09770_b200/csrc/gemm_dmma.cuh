// Grouped FP64 GEMM on the DMMA tensor path of sm_100a (mma.sync.m16n8k16.f64 -> SASS
// DMMA.8x8x4; tcgen05 has no f64 kind), second generation:
//   C_p = alpha op(A_p) diag(d_p) op(B_p) + beta C_p   for every tile (p, tm, tn) of a tile list
// (or one large problem on a 2-D grid), column-major operands.
//
// Design:
//  * CTA tile BM x BN, K-slabs of BK through a STAGES-deep cp.async ring (one barrier per slab);
//    warps WM x WN, each a (BM/WM) x (BN/WN) warp tile of m16n8k16 MMAs;
//  * the shared-memory layout of each operand follows its global contiguity (A not transposed:
//    [k][m]; transposed: [m][k]; B not transposed: [n][k]; transposed: [k][n]) with a pad of 4
//    doubles, so both the 16-byte global->shared copies and the fragment reads (two 16-lane
//    phases of 8-byte loads) are free of bank conflicts;
//  * 16-byte cp.async (VEC) for problems whose operand columns are 16-byte aligned, pairs of
//    8-byte copies with the same thread mapping for the others (decided per CTA); ragged edges
//    zero-filled through the copy's source size;
//  * the diagonal scaling multiplies whichever fragment set is smaller per thread.
#pragma once
#include <cstdint>
#include "internal.h"

namespace vb {
namespace g2 {

__device__ __forceinline__ void mma16816(double (&c)[4], const double (&a)[8], const double (&b)[4]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
      "{%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
        "d"(b[1]), "d"(b[2]), "d"(b[3]));
}

__device__ __forceinline__ void cp16(void *smem, const void *gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp8(void *smem, const void *gmem, int src_bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int THREADS = WM * WN * 32;
  static constexpr int WTM = BM / WM, WTN = BN / WN;
  static constexpr int MI = WTM / 16, NJ = WTN / 8;
  static_assert(WTM % 16 == 0 && WTN % 8 == 0 && BK % 16 == 0, "tile shape");
};

// one operand tile (rows x cols of the stored, column-major matrix) per stage
// CONTIG: extent along the global contiguous dimension; OTHER: along the strided one
template <int CONTIG, int OTHER>
struct Tile {
  static constexpr int LD = CONTIG + 4;     // shared row length (doubles)
  static constexpr int SIZE = OTHER * LD;
};

template <class C, bool TA, bool TB>
struct Smem {
  // A tile: !TA -> contiguous m (BM), other k (BK); TA -> contiguous k, other m
  using TAt = Tile<TA ? C::BK : C::BM, TA ? C::BM : C::BK>;
  // B tile: !TB -> contiguous k, other n; TB -> contiguous n, other k
  using TBt = Tile<TB ? C::BN : C::BK, TB ? C::BK : C::BN>;
  static constexpr int A_STAGE = TAt::SIZE, B_STAGE = TBt::SIZE;
  static constexpr int STAGE = A_STAGE + B_STAGE + C::BK;   // + the slab of d
  static constexpr size_t BYTES = (size_t)C::STAGES * STAGE * sizeof(double);
};

// Per-thread copy plan of one operand tile: chunk q of thread t covers contiguous elements
// [c0, c0 + W) of "row" o (W = 2 with 16-byte copies, 1 otherwise).
template <int CONTIG, int OTHER, int THREADS, bool VEC>
struct CopyPlan {
  static constexpr int W = VEC ? 2 : 1;
  static constexpr int PER_ROW = CONTIG / W;
  static constexpr int CHUNKS = CONTIG * OTHER / W;
  static_assert(CHUNKS % THREADS == 0 && THREADS % PER_ROW == 0, "copy plan");
  static constexpr int PER_THREAD = CHUNKS / THREADS;
  static constexpr int ROW_STEP = THREADS / PER_ROW;   // o advance per chunk of a thread
  __device__ static int c0(int t) { return (t % PER_ROW) * W; }
  __device__ static int o0(int t) { return t / PER_ROW; }
};

// Issue the copies of one operand slab.  g: global element (c0, o0) of this thread's first chunk
// for this slab; ld: stride between "rows" o; c_left / o_left: extents still inside the matrix
// measured from the tile origin; s: the stage's shared tile.
// With VEC, `al` (uniform per CTA) says whether this problem's operand columns are 16-byte
// aligned; if not, each 2-element chunk goes as two 8-byte copies (same thread mapping).
template <int CONTIG, int OTHER, int THREADS, bool VEC>
__device__ __forceinline__ void copy_tile(double *s, const double *g, const double *safe, int64_t ld, int tid,
                                          int c_left, int o_left, bool al = true) {
  using P = CopyPlan<CONTIG, OTHER, THREADS, VEC>;
  const int c = P::c0(tid), o = P::o0(tid);
  constexpr int LD = CONTIG + 4;
#pragma unroll
  for (int q = 0; q < P::PER_THREAD; ++q) {
    const int oo = o + q * P::ROW_STEP;
    const double *src = g + (int64_t)(q * P::ROW_STEP) * ld;
    double *dst = s + oo * LD + c;
    if (VEC) {
      const int nvalid = (oo < o_left) ? max(0, min(2, c_left - c)) : 0;
      if (al) {
        cp16(dst, nvalid ? src : safe, 8 * nvalid);
      } else {
        cp8(dst, nvalid > 0 ? src : safe, nvalid > 0 ? 8 : 0);
        cp8(dst + 1, nvalid > 1 ? src + 1 : safe, nvalid > 1 ? 8 : 0);
      }
    } else {
      const int bytes = (oo < o_left && c < c_left) ? 8 : 0;
      cp8(dst, bytes ? src : safe, bytes);
    }
  }
}

// Tile of a grouped launch: segs[0 .. nseg) = {problem, first tile index, tiles per row (tn), lower}
// in increasing first-tile order; a problem's tiles are row-major over its (tm x tn) tile grid, the
// lower ones (C on the diagonal, BM == BN) keeping only j <= i: min(i + 1, tn) tiles in row i.
__device__ __forceinline__ int4 seg_tile(const int4 *__restrict__ segs, int nseg, int bid) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&segs[mid].y) <= bid) lo = mid; else hi = mid - 1;
  }
  const int4 sg = segs[lo];
  const int idx = bid - sg.y, tn = sg.z;
  int i, j;
  if (sg.w) {
    const int tri = tn * (tn + 1) / 2;
    if (idx < tri) {
      i = (int)((sqrt(8.0 * idx + 1.0) - 1.0) * 0.5);
      while ((i + 1) * (i + 2) / 2 <= idx) ++i;
      while (i * (i + 1) / 2 > idx) --i;
      j = idx - i * (i + 1) / 2;
    } else {
      const int r = idx - tri;
      i = tn + r / tn;
      j = r % tn;
    }
  } else {
    i = idx / tn;
    j = idx % tn;
  }
  return make_int4(sg.x, i, j, 0);
}

template <class C, bool DENSE, bool SCALED, bool TA, bool TB, bool VEC>
__global__ void __launch_bounds__(C::THREADS, C::MINB) gemm2_kernel(const GemmProb *__restrict__ probs,
                                                                     const int4 *__restrict__ segs, int seg0,
                                                                     int nseg) {
  using S = Smem<C, TA, TB>;
  constexpr int BM = C::BM, BN = C::BN, BK = C::BK, T = C::THREADS;
  constexpr int ACONT = TA ? BK : BM, AOTH = TA ? BM : BK;
  constexpr int BCONT = TB ? BN : BK, BOTH = TB ? BK : BN;
  constexpr int ALD = ACONT + 4, BLD = BCONT + 4;
  static_assert(BM == BN, "lower-tile enumeration assumes square tiles");
  const int4 t = DENSE ? make_int4(seg0, blockIdx.y, blockIdx.x, 0) : seg_tile(segs + seg0, nseg, blockIdx.x);
  const GemmProb P = probs[t.x];
  const int m0 = t.y * BM, n0 = t.z * BN;
  if (DENSE && P.lower && m0 + BM - 1 < n0) return;   // tile strictly above the diagonal
  extern __shared__ __align__(16) double g2_smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wm = (warp / C::WN) * C::WTM, wn = (warp % C::WN) * C::WTN;
  const bool scaled = SCALED && P.d != nullptr;
  const int K = P.K;
  const int rows_left = P.M - m0, cols_left = P.N - n0;
  int kb = 0;   // first K slab with non-zero products (triangular operands)
  if (P.kz_on) {
    kb = max(0, max(m0 + P.kzA, n0 + P.kzB)) / BK * BK;
    if (kb > K) kb = K;
  }
  // this thread's first-chunk sources at k = kb
  using PA = CopyPlan<ACONT, AOTH, T, VEC>;
  using PB = CopyPlan<BCONT, BOTH, T, VEC>;
  const int ac = PA::c0(tid), ao = PA::o0(tid), bc = PB::c0(tid), bo = PB::o0(tid);
  // A element (m, k): !TA at A[m + k lda] (contig m), TA at A[k + m lda] (contig k)
  const double *ga = TA ? P.A + (kb + ac) + (int64_t)(m0 + ao) * P.lda : P.A + (m0 + ac) + (int64_t)(kb + ao) * P.lda;
  // B element (k, n): !TB at B[k + n ldb] (contig k), TB at B[n + k ldb] (contig n)
  const double *gb = TB ? P.B + (n0 + bc) + (int64_t)(kb + bo) * P.ldb : P.B + (kb + bc) + (int64_t)(n0 + bo) * P.ldb;
  const int64_t astep = TA ? BK : (int64_t)BK * P.lda, bstep = TB ? (int64_t)BK * P.ldb : BK;
  const double *dv = SCALED ? P.d : nullptr;
  // 16-byte copies need 16-byte aligned columns (aligned base, even leading dimension)
  const bool alA = ((reinterpret_cast<uintptr_t>(P.A) & 15) == 0) && !(P.lda & 1);
  const bool alB = ((reinterpret_cast<uintptr_t>(P.B) & 15) == 0) && !(P.ldb & 1);

  auto stage_ptr = [&](int st) { return g2_smem + st * S::STAGE; };
  auto issue = [&](int st, int k0) {   // slab starting at k0 (k0 - kb a multiple of BK)
    double *sA = stage_ptr(st), *sB = sA + S::A_STAGE, *sD = sB + S::B_STAGE;
    const int k_left = K - k0;
    const int64_t ks = (k0 - kb) / BK;
    if (TA)
      copy_tile<ACONT, AOTH, T, VEC>(sA, ga + ks * astep, P.A, P.lda, tid, k_left, rows_left, alA);
    else
      copy_tile<ACONT, AOTH, T, VEC>(sA, ga + ks * astep, P.A, P.lda, tid, rows_left, k_left, alA);
    if (TB)
      copy_tile<BCONT, BOTH, T, VEC>(sB, gb + ks * bstep, P.B, P.ldb, tid, cols_left, k_left, alB);
    else
      copy_tile<BCONT, BOTH, T, VEC>(sB, gb + ks * bstep, P.B, P.ldb, tid, k_left, cols_left, alB);
    if (SCALED && tid < BK) {
      const bool ok = scaled && tid < k_left;
      cp8(sD + tid, ok ? dv + (int64_t)(k0 + tid) * P.dstride : P.A, ok ? 8 : 0);
    }
  };
  double acc[C::MI][C::NJ][4];
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NJ; ++j)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[i][j][v] = 0.0;

  const int nslab = (K - kb + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < C::STAGES - 1; ++s) {
    if (s < nslab) issue(s, kb + s * BK);
    commit();
  }
  int st = 0;
  for (int sl = 0; sl < nslab; ++sl) {
    wait_group<C::STAGES - 2>();
    __syncthreads();
    {
      const int nx = sl + C::STAGES - 1;
      int nst = st + C::STAGES - 1;
      if (nst >= C::STAGES) nst -= C::STAGES;
      if (nx < nslab) issue(nst, kb + nx * BK);
      commit();
    }
    const double *sA = stage_ptr(st), *sB = sA + S::A_STAGE, *sD = sB + S::B_STAGE;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 16) {
      double b[C::NJ][4];
#pragma unroll
      for (int j = 0; j < C::NJ; ++j)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int k = kk + tg + 4 * v, n = wn + 8 * j + g;
          b[j][v] = TB ? sB[k * BLD + n] : sB[n * BLD + k];
          if (SCALED && C::NJ * 4 <= C::MI * 8 && scaled) b[j][v] *= sD[k];
        }
#pragma unroll
      for (int i = 0; i < C::MI; ++i) {
        double a[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const int m = wm + 16 * i + g + 8 * (v & 1), k = kk + tg + 4 * (v >> 1);
          a[v] = TA ? sA[m * ALD + k] : sA[k * ALD + m];
          if (SCALED && C::NJ * 4 > C::MI * 8 && scaled) a[v] *= sD[k];
        }
#pragma unroll
        for (int j = 0; j < C::NJ; ++j) mma16816(acc[i][j], a, b[j]);
      }
    }
    if (++st == C::STAGES) st = 0;
  }
  wait_group<0>();
  // epilogue: C = beta C + alpha acc (lower triangle only where asked)
#pragma unroll
  for (int i = 0; i < C::MI; ++i)
#pragma unroll
    for (int j = 0; j < C::NJ; ++j)
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

}  // namespace g2
}  // namespace vb
