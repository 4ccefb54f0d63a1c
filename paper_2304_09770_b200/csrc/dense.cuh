// Batched dense FP64 kernels for the factorisations.
#pragma once
#include <array>
#include "internal.h"

namespace vb {

struct MatDesc {      // column-major square matrix
  double *A;
  int n, ld, m;       // m = number of leading columns to eliminate
  // pivot test (SURVEY §8(b) VB_ESINGULAR): npos < 0 -> only |d| > 1e-300 and finite (blocks that
  // may be semidefinite); else pivots of columns < npos must be > kPivRel * max|diag A| and those
  // of columns >= npos < -kPivRel * max|diag A| (velocity-first saddle LDL^T: A_II SPD, the
  // pressure Schur complement negative definite, reading A5)
  int npos = -1;
};
constexpr double kPivRel = 1e-13;

// A sequence of grouped-GEMM launches planned on the host and uploaded once.  Within a launch the
// tiles are grouped by transpose class (op(A), op(B)) so each class runs the kernel specialised for
// its copy pattern.
struct GemmPlan {
  std::vector<GemmProb> probs;
  // per launch, per class: segments {problem, first tile, tiles per row, lower} (gemm_dmma.cuh seg_tile)
  std::vector<std::array<std::vector<int4>, 4>> ltiles;
  std::vector<std::array<int64_t, 4>> ltcount;             // tiles per launch and class
  std::vector<std::array<std::pair<int, int>, 4>> lrange;  // after upload: (segment_begin, segment_count)
  std::vector<std::array<int, 4>> lntile;                  // after upload: tiles (= grid size)
  std::vector<std::vector<int>> dense;        // per launch: large problems run as 2D grids
  std::vector<char> scaled;                   // per launch: some tile-list problem has d != null
  bool allow_kz = false;                      // honour GemmProb.kz_on regardless of VB_KZ (vb_debug_gemm)
  DBuf<GemmProb> d_probs;
  DBuf<int4> d_tiles;
  int begin_launch() {
    ltiles.push_back({});
    ltcount.push_back({0, 0, 0, 0});
    dense.push_back({});
    scaled.push_back(0);
    return ltiles.size() - 1;
  }
  void add(const GemmProb &p);             // adds tiles to the current launch
  void upload(cudaStream_t s);
  void run(int launch, cudaStream_t s);
};

void gemm_grouped(GemmPlan &plan, int launch, cudaStream_t s);
// process-wide kernel attribute, only ever raised (thread-safe; several contexts share kernels)
void raise_smem_limit(const void *func, size_t bytes);
extern thread_local double g_gemm_flops;   // flops of the GEMMs planned since the last reset
extern thread_local bool g_gemm_timing;    // VB_KERNEL_TIMING: CUDA events around every GEMM launch set
double gemm_timing_collect(cudaStream_t s);   // seconds of GEMM kernel time since the last collect

// Partial LDL^T (no pivoting, velocity-first quasi-definite ordering) of a batch:
// eliminates the first m columns; on exit the strictly lower part of those columns holds L, the
// diagonal holds D, and the lower triangle of the trailing block holds the Schur complement.
// `info[b]` receives 1 + the column of the first tiny/sign-inconsistent pivot, else 0.
// pivot_sign: +1 all pivots positive (SPD), 0 = any sign allowed.
void ldl_partial_batched(const std::vector<MatDesc> &mats, int *info_dev, cudaStream_t s);

// X <- L^{-1} for the unit lower triangle of the leading m x m block of each matrix (column-major,
// X with leading dimension ldx, overwritten; X must be pre-zeroed).
struct TriDesc {
  const double *L;
  int ldl;
  double *X;
  int ldx, m;
};
void tri_inverse_batched(const std::vector<TriDesc> &mats, cudaStream_t s);

// Fill the strictly upper triangle of an n x n block from its lower triangle.
void symmetrize_lower_batched(const std::vector<MatDesc> &mats, cudaStream_t s);

// Pack the lower triangle of a symmetric column-major n x n block into 32x32 row-major tiles.
struct PackDesc {
  const double *A;
  int n, ld;
  double *out;
};
void pack_tiles_batched(const std::vector<PackDesc> &mats, cudaStream_t s);

}  // namespace vb
