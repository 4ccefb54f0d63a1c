// Microbenchmark: FP64 tensor (DMMA via mma.sync f64) and DFMA peaks on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dmma_m8n8k4(double *out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
  for (int j = 0; j < 8; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_m16n8k16(double *out, int iters) {
  double a[8], b[4], c[4][4];
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int j = 0; j < 4; ++j) b[j] = 1.0 + threadIdx.x * 1e-4 + j;
  for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) c[j][q] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int j = 0; j < 4; ++j) for (int q = 0; q < 4; ++q) s += c[j][q];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma(double *out, int iters) {
  double x[16]; double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
  for (int j = 0; j < 16; ++j) x[j] = j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0; for (int j = 0; j < 16; ++j) s += x[j];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double *d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 20000;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int rep = 0; rep < 2; ++rep) {
      dim3 g(sms * 4), b(32 * warps);
      cudaEventRecord(e0); dmma_m8n8k4<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double fl = double(g.x) * warps * iters * 8 * 512.0;
      if (rep) printf("DMMA m8n8k4  blocks=%d warps/blk=%d: %.2f TFLOP/s\n", g.x, warps, fl / ms / 1e9);
      cudaEventRecord(e0); dmma_m16n8k16<<<g, b>>>(d, iters / 4); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = double(g.x) * warps * (iters / 4) * 4 * (16 * 8 * 16 * 2.0);
      if (rep) printf("DMMA m16n8k16 blocks=%d warps/blk=%d: %.2f TFLOP/s\n", g.x, warps, fl / ms / 1e9);
      cudaEventRecord(e0); dfma<<<g, b>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      fl = double(g.x) * warps * 32 * iters * 16 * 2.0;
      if (rep) printf("DFMA         blocks=%d warps/blk=%d: %.2f TFLOP/s\n", g.x, warps, fl / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}
