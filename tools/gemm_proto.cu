// Standalone A/B harness for the second-generation DMMA GEMM (csrc/gemm_dmma.cuh): correctness
// against a naive FP64 kernel on ragged shapes (every transpose class, scaling, lower, beta,
// triangular K skipping) and TFLOP/s on the factorisation's shapes, for several tile configs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. tools/gemm_proto.cu -o /tmp/gp
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <algorithm>
#include "../paper_2304_09770_b200/csrc/gemm_dmma.cuh"

using namespace vb;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void naive(const GemmProb p, double *out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x, j = blockIdx.y;
  if (i >= p.M || j >= p.N) return;
  double s = 0;
  for (int k = 0; k < p.K; ++k) {
    double a = p.transA ? p.A[k + (int64_t)i * p.lda] : p.A[i + (int64_t)k * p.lda];
    double b = p.transB ? p.B[j + (int64_t)k * p.ldb] : p.B[k + (int64_t)j * p.ldb];
    double d = p.d ? p.d[(int64_t)k * p.dstride] : 1.0;
    s += a * d * b;
  }
  double c = p.C[i + (int64_t)j * p.ldc];
  out[i + (int64_t)j * p.ldc] = (p.lower && i < j) ? c : (p.beta == 0.0 ? 0.0 : p.beta * c) + p.alpha * s;
}

// zero op(A)(i, k) for k < i + kzA and op(B)(k, j) for k < j + kzB (the triangular promise)
__global__ void kz_zero(GemmProb p) {
  const int k = blockIdx.y;
  for (int i = threadIdx.x; i < max(p.M, p.N); i += blockDim.x) {
    if (i < p.M && k < i + p.kzA) ((double *)p.A)[p.transA ? k + (int64_t)i * p.lda : i + (int64_t)k * p.lda] = 0.0;
    if (i < p.N && k < i + p.kzB) ((double *)p.B)[p.transB ? i + (int64_t)k * p.ldb : k + (int64_t)i * p.ldb] = 0.0;
  }
}

__global__ void fill(double *x, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)i * 2654435761u ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995; h ^= h >> 15;
    x[i] = (h & 0xffffff) / double(0x1000000) - 0.5;
  }
}

template <class C, bool SC, bool TA, bool TB, bool VEC>
void launch_list(const GemmProb *dp, const int4 *dt, int ntiles, cudaStream_t s) {
  using S = g2::Smem<C, TA, TB>;
  auto k = g2::gemm2_kernel<C, false, SC, TA, TB, VEC>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::BYTES));
  k<<<ntiles, C::THREADS, S::BYTES, s>>>(dp, dt, 0);
  CK(cudaGetLastError());
}

template <class C, bool SC, bool VEC>
void launch_cls(int cls, const GemmProb *dp, const int4 *dt, int nt, cudaStream_t s) {
  switch (cls) {
    case 0: launch_list<C, SC, false, false, VEC>(dp, dt, nt, s); break;
    case 1: launch_list<C, SC, true, false, VEC>(dp, dt, nt, s); break;
    case 2: launch_list<C, SC, false, true, VEC>(dp, dt, nt, s); break;
    default: launch_list<C, SC, true, true, VEC>(dp, dt, nt, s); break;
  }
}

struct Case { int M, N, K, batch, tA, tB, scaled, lower, kz; double beta; };

template <class C>
double run_case(const Case &cs, bool check, bool vec, const char *name) {
  const int M = cs.M, N = cs.N, K = cs.K, b = cs.batch;
  // 16-byte copies need even leading dimensions; the 8-byte path is exercised with odd ones
  auto ldfix = [&](int x) { return vec ? (x + 1) / 2 * 2 : (x | 1); };
  const int lda = ldfix(cs.tA ? K : M), ldb = ldfix(cs.tB ? N : K), ldc = M + 3;
  const size_t sa = (size_t)lda * (cs.tA ? M : K), sb = (size_t)ldb * (cs.tB ? K : N), sc = (size_t)ldc * N;
  double *A, *B, *Cm, *Cr, *d;
  CK(cudaMalloc(&A, sa * b * 8)); CK(cudaMalloc(&B, sb * b * 8)); CK(cudaMalloc(&Cm, sc * b * 8));
  CK(cudaMalloc(&Cr, sc * b * 8)); CK(cudaMalloc(&d, (size_t)K * 8));
  fill<<<1024, 256>>>(A, sa * b, 1); fill<<<1024, 256>>>(B, sb * b, 2); fill<<<1024, 256>>>(Cm, sc * b, 3);
  fill<<<64, 256>>>(d, K, 4);
  std::vector<GemmProb> ps;
  std::vector<int4> tl;
  for (int q = 0; q < b; ++q) {
    GemmProb p{};
    p.A = A + q * sa; p.B = B + q * sb; p.C = Cm + q * sc; p.d = cs.scaled ? d : nullptr; p.dstride = 1;
    p.lda = lda; p.ldb = ldb; p.ldc = ldc; p.M = M; p.N = N; p.K = K; p.alpha = -1.0; p.beta = cs.beta;
    p.transA = cs.tA; p.transB = cs.tB; p.lower = cs.lower; p.kz_on = cs.kz; p.kzA = 3; p.kzB = 5;
    ps.push_back(p);
    if (cs.kz) kz_zero<<<dim3(1, K), 256>>>(p);
    for (int i = 0; i < (M + C::BM - 1) / C::BM; ++i)
      for (int j = 0; j < (N + C::BN - 1) / C::BN; ++j) {
        if (cs.lower && i * C::BM + C::BM - 1 < j * C::BN) continue;
        tl.push_back(make_int4(q, i, j, 0));
      }
  }
  GemmProb *dp; int4 *dt;
  CK(cudaMalloc(&dp, ps.size() * sizeof(GemmProb))); CK(cudaMalloc(&dt, tl.size() * sizeof(int4)));
  CK(cudaMemcpy(dp, ps.data(), ps.size() * sizeof(GemmProb), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt, tl.data(), tl.size() * sizeof(int4), cudaMemcpyHostToDevice));
  const int cls = cs.tA + 2 * cs.tB;
  auto go = [&]() {
    if (cs.scaled) { if (vec) launch_cls<C, true, true>(cls, dp, dt, tl.size(), 0); else launch_cls<C, true, false>(cls, dp, dt, tl.size(), 0); }
    else { if (vec) launch_cls<C, false, true>(cls, dp, dt, tl.size(), 0); else launch_cls<C, false, false>(cls, dp, dt, tl.size(), 0); }
  };
  double res = 0;
  if (check) {
    CK(cudaMemcpy(Cr, Cm, sc * b * 8, cudaMemcpyDeviceToDevice));
    double *out; CK(cudaMalloc(&out, sc * b * 8));
    CK(cudaMemcpy(out, Cm, sc * b * 8, cudaMemcpyDeviceToDevice));
    for (int q = 0; q < b; ++q) {
      GemmProb p = ps[q]; p.C = Cr + q * sc;
      naive<<<dim3((M + 127) / 128, N), 128>>>(p, out + q * sc);
    }
    go();
    CK(cudaDeviceSynchronize());
    std::vector<double> h1(sc * b), h2(sc * b);
    CK(cudaMemcpy(h1.data(), Cm, sc * b * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(h2.data(), out, sc * b * 8, cudaMemcpyDeviceToHost));
    double mx = 0, ref = 0;
    for (size_t i = 0; i < h1.size(); ++i) { mx = std::max(mx, fabs(h1[i] - h2[i])); ref = std::max(ref, fabs(h2[i])); }
    res = mx / (ref * K);
    cudaFree(out);
  } else {
    go();
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); go(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
    }
    double f = 2.0 * M * (double)N * K * b * (cs.lower ? 0.5 : 1.0);
    res = f / (best * 1e-3) / 1e12;
  }
  cudaFree(A); cudaFree(B); cudaFree(Cm); cudaFree(Cr); cudaFree(d); cudaFree(dp); cudaFree(dt);
  return res;
}

template <class C>
void suite(const char *name) {
  using S0 = g2::Smem<C, false, false>;
  printf("== %s: BM %d BN %d BK %d warps %dx%d stages %d minB %d smem %zu B\n", name, C::BM, C::BN, C::BK, C::WM, C::WN,
         C::STAGES, C::MINB, S0::BYTES);
  Case checks[] = {{131, 97, 77, 3, 0, 0, 0, 0, 0, 1.0}, {131, 97, 77, 3, 1, 0, 1, 0, 0, 0.0}, {131, 97, 77, 3, 0, 1, 1, 1, 0, 1.0},
                   {131, 131, 77, 2, 1, 1, 0, 1, 1, 1.0}, {300, 200, 160, 2, 0, 1, 1, 0, 1, 1.0}};
  double worst = 0;
  for (auto &cs : checks)
    for (int v = 0; v < 2; ++v) {
      const double e = run_case<C>(cs, true, v, name);
      if (!(e < 1e-15)) printf("   FAIL M %d N %d K %d tA %d tB %d sc %d low %d kz %d vec %d: %.2e\n", cs.M, cs.N, cs.K, cs.tA, cs.tB,
                              cs.scaled, cs.lower, cs.kz, v, e);
      worst = std::max(worst, e);
    }
  printf("   correctness: max rel err %.2e %s\n", worst, worst < 1e-15 ? "OK" : "FAIL");
  Case perf[] = {{1285, 1285, 128, 512, 0, 1, 1, 0, 0, 1.0}, {1285, 1285, 256, 512, 0, 1, 1, 0, 0, 1.0},
                 {1285, 1285, 256, 512, 0, 1, 1, 1, 0, 1.0},
                 {1285, 224, 32, 512, 0, 1, 1, 0, 0, 1.0}, {1285, 32, 224, 512, 0, 1, 1, 0, 0, 1.0},
                 {1080, 1080, 1080, 128, 0, 0, 0, 0, 0, 0.0},
                 {1158, 1158, 1285, 64, 1, 0, 0, 0, 0, 0.0}, {4096, 4096, 4096, 1, 0, 0, 0, 0, 0, 0.0}};
  for (auto &cs : perf)
    printf("   M %5d N %5d K %5d b %4d tA %d tB %d sc %d low %d : %6.2f TF/s\n", cs.M, cs.N, cs.K, cs.batch, cs.tA, cs.tB,
           cs.scaled, cs.lower, run_case<C>(cs, false, true, name));
}

int main() {
#ifdef ONLY
  suite<g2::Cfg<ONLY>>("only");
#else
  suite<g2::Cfg<64, 64, 16, 2, 2, 3, 4>>("v7 64x64x16 4 warps st3 minB4");
  suite<g2::Cfg<64, 64, 16, 2, 2, 4, 4>>("v8 64x64x16 4 warps st4 minB4");
  suite<g2::Cfg<64, 64, 32, 2, 2, 3, 3>>("v9 64x64x32 4 warps st3 minB3");
  suite<g2::Cfg<64, 32, 16, 2, 1, 3, 6>>("v10 64x32x16 2 warps st3 minB6");
  suite<g2::Cfg<64, 64, 16, 4, 1, 3, 4>>("v11 64x64x16 4 warps 4x1 (16x64)");
  suite<g2::Cfg<32, 64, 16, 1, 2, 4, 6>>("v12 32x64x16 2 warps st4 minB6");
#endif
  return 0;
}
