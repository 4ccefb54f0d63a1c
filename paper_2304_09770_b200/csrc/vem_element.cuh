// K9: divergence-free VEM element operators on the device (§3).
// One thread per cell; matrices live in a global scratch arena laid out element-fastest (SoA) so
// that a warp's accesses are coalesced.  The construction follows the paper's definitions:
//   face space B^_k(f) + enhancement (iii) -> Pi^0_{k+1,f};
//   div v in P_{k-1} from the flux (D3 normal p=1 moments) and D5;
//   Pi^nabla_{k,K} via integration by parts with [P_{k-2}]^3 = grad P_{k-1} (+) x^[P_{k-3}]^3;
//   Pi^0_{k,K} via [P_k]^3 = grad P_{k+1} (+) x^[P_{k-1}]^3 and the super-enhancement;
//   Pi^0_{k-1} grad v; a_h^K = consistency + D-recipe stabilisation;
//   B^K = |K| * (coefficients of div phi_i) for the dual pressure basis.
// The x^ basis of each homogeneous degree d is {x^(m e1): x1 does not divide m} u {x^(m e2)} u
// {x^(m e3)} (|m| = d): an explicit basis of the same space the oracle spans by least squares.
#pragma once
#include "vem_device.cuh"

namespace vb {

struct SM {
  double *p;
  int64_t s;
  __device__ double &operator()(int64_t i) const { return p[i * s]; }
};

__host__ __device__ constexpr int d2(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) / 2; }
__host__ __device__ constexpr int d3(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) / 6; }

// exponent of the j-th 3D monomial (degree-major, x-power descending, then y descending)
__device__ inline void exp3(int j, int e[3]) {
  int d = 0;
  while (d3(d) <= j) ++d;
  int r = j - d3(d - 1);
  for (int a = d; a >= 0; --a) {
    int cnt = d - a + 1;
    if (r < cnt) { e[0] = a; e[1] = d - a - r; e[2] = r; return; }
    r -= cnt;
  }
}
__device__ inline int idx3(int a, int b, int c) {
  int d = a + b + c;
  int base = d3(d - 1);
  int off = 0;
  for (int aa = d; aa > a; --aa) off += d - aa + 1;
  return base + off + (d - a - b);
}
__device__ inline void exp2d(int j, int e[2]) {
  int d = 0;
  while (d2(d) <= j) ++d;
  int r = j - d2(d - 1);
  e[0] = d - r; e[1] = r;
}
__device__ inline int idx2(int p, int q) { return d2(p + q - 1) + q; }

__device__ inline void mono2(double xi, double eta, double h, int n, double *m, double (*g)[2]) {
  const double X = xi / h, Y = eta / h;
  double px[7], py[7];
  px[0] = py[0] = 1.0;
  for (int p = 1; p <= n; ++p) { px[p] = px[p - 1] * X; py[p] = py[p - 1] * Y; }
  int j = 0;
  for (int d = 0; d <= n; ++d)
    for (int p = d; p >= 0; --p) {
      const int q = d - p;
      m[j] = px[p] * py[q];
      if (g) {
        g[j][0] = p ? p * px[p - 1] * py[q] / h : 0.0;
        g[j][1] = q ? q * px[p] * py[q - 1] / h : 0.0;
      }
      ++j;
    }
}

__device__ inline void mono3g(const double x[3], const double xc[3], double h, int n, double *m, double (*g)[3]) {
  const double X[3] = {(x[0] - xc[0]) / h, (x[1] - xc[1]) / h, (x[2] - xc[2]) / h};
  double p[3][7];
  for (int c = 0; c < 3; ++c) { p[c][0] = 1.0; for (int q = 1; q <= n; ++q) p[c][q] = p[c][q - 1] * X[c]; }
  int j = 0;
  for (int d = 0; d <= n; ++d)
    for (int a = d; a >= 0; --a)
      for (int b = d - a; b >= 0; --b) {
        const int cc = d - a - b;
        m[j] = p[0][a] * p[1][b] * p[2][cc];
        if (g) {
          g[j][0] = a ? a * p[0][a - 1] * p[1][b] * p[2][cc] / h : 0.0;
          g[j][1] = b ? b * p[0][a] * p[1][b - 1] * p[2][cc] / h : 0.0;
          g[j][2] = cc ? cc * p[0][a] * p[1][b] * p[2][cc - 1] / h : 0.0;
        }
        ++j;
      }
}

// In-place Gaussian elimination with partial pivoting: A (n x n, row-major via acc) X = B (n x m).
template <class MA, class MB>
__device__ void lu_solve(MA A, int n, MB B, int m) {
  for (int j = 0; j < n; ++j) {
    int piv = j;
    double best = fabs(A(j * n + j));
    for (int i = j + 1; i < n; ++i) {
      double v = fabs(A(i * n + j));
      if (v > best) { best = v; piv = i; }
    }
    if (piv != j) {
      for (int q = 0; q < n; ++q) { double t = A(j * n + q); A(j * n + q) = A(piv * n + q); A(piv * n + q) = t; }
      for (int q = 0; q < m; ++q) { double t = B(j * m + q); B(j * m + q) = B(piv * m + q); B(piv * m + q) = t; }
    }
    const double inv = 1.0 / A(j * n + j);
    for (int i = j + 1; i < n; ++i) {
      const double f = A(i * n + j) * inv;
      if (f == 0.0) continue;
      for (int q = j + 1; q < n; ++q) A(i * n + q) -= f * A(j * n + q);
      for (int q = 0; q < m; ++q) B(i * m + q) -= f * B(j * m + q);
    }
  }
  for (int j = n - 1; j >= 0; --j) {
    const double inv = 1.0 / A(j * n + j);
    for (int q = 0; q < m; ++q) {
      double v = B(j * m + q);
      for (int t = j + 1; t < n; ++t) v -= A(j * n + t) * B(t * m + q);
      B(j * m + q) = v * inv;
    }
  }
}

struct LocalArr {   // thin accessor for thread-local arrays
  double *p;
  __device__ double &operator()(int64_t i) const { return p[i]; }
};

}  // namespace vb
