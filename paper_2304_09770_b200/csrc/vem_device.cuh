// Device-side VEM geometry helpers (cell descriptors, scaled monomials, collapsed quadrature).
#pragma once
#include "setup.h"

namespace vb {

// Gauss-Legendre tables on [0,1] for n = 1..8 (filled by the host in vem.cu)
__constant__ double c_glx[9][8];   // only vem.cu includes this header
__constant__ double c_glw[9][8];
__constant__ double c_lobx[5];   // Gauss-Lobatto nodes for k+1 points (k <= 4)
__constant__ double c_lobw[5];

struct CellGeo {
  int nv, ne, nf;
  double X[MAXV][3];
  int flen[MAXF], floop[MAXF][MAXL], fedge[MAXF][MAXL], ffwd[MAXF][MAXL];
  double fsign[MAXF];
  int ev[MAXE][2];
  double apex[3];
  int ntet;
  short tet_face[MAXT];
  short tet_i[MAXT];         // fan triangle (0, i, i+1) of the face loop
  double vol, xc[3], h;
};

__device__ inline void load_cell(const int *T, const double *xyz, CellGeo &g) {
  g.nv = T[0]; g.ne = T[1]; g.nf = T[2];
  g.apex[0] = g.apex[1] = g.apex[2] = 0.0;
  for (int i = 0; i < g.nv; ++i) {
    int v = T[TOPO_V + i];
    for (int q = 0; q < 3; ++q) { g.X[i][q] = xyz[3 * (int64_t)v + q]; g.apex[q] += g.X[i][q]; }
  }
  for (int q = 0; q < 3; ++q) g.apex[q] /= g.nv;
  for (int e = 0; e < g.ne; ++e) { g.ev[e][0] = T[TOPO_E + 2 * e]; g.ev[e][1] = T[TOPO_E + 2 * e + 1]; }
  g.ntet = 0;
  double vol = 0, m1[3] = {0, 0, 0};
  for (int f = 0; f < g.nf; ++f) {
    const int *F = T + TOPO_F + f * FACE_STRIDE;
    g.fsign[f] = F[0];
    g.flen[f] = F[1];
    for (int q = 0; q < F[1]; ++q) { g.floop[f][q] = F[2 + q]; g.fedge[f][q] = F[2 + MAXL + q]; g.ffwd[f][q] = F[2 + 2 * MAXL + q]; }
    for (int i = 1; i + 1 < F[1]; ++i) {
      g.tet_face[g.ntet] = f; g.tet_i[g.ntet] = i; ++g.ntet;
      const double *a = g.X[g.floop[f][0]];
      const double *b = g.X[g.floop[f][F[0] > 0 ? i : i + 1]];
      const double *c = g.X[g.floop[f][F[0] > 0 ? i + 1 : i]];
      double u[3], v[3], w[3];
      for (int q = 0; q < 3; ++q) { u[q] = a[q] - g.apex[q]; v[q] = b[q] - g.apex[q]; w[q] = c[q] - g.apex[q]; }
      double v6 = u[0] * (v[1] * w[2] - v[2] * w[1]) - u[1] * (v[0] * w[2] - v[2] * w[0]) + u[2] * (v[0] * w[1] - v[1] * w[0]);
      vol += v6 / 6.0;
      for (int q = 0; q < 3; ++q) m1[q] += v6 / 6.0 * (g.apex[q] + a[q] + b[q] + c[q]) / 4.0;
    }
  }
  g.vol = vol;
  for (int q = 0; q < 3; ++q) g.xc[q] = m1[q] / vol;
  double h2 = 0;
  for (int i = 0; i < g.nv; ++i)
    for (int j = i + 1; j < g.nv; ++j) {
      double d = 0;
      for (int q = 0; q < 3; ++q) d += (g.X[i][q] - g.X[j][q]) * (g.X[i][q] - g.X[j][q]);
      h2 = fmax(h2, d);
    }
  g.h = sqrt(h2);
}

// collapsed Gauss rule on the sub-tetrahedra (apex, fan triangle), exact to degree 2n-3
struct QuadTet {
  int n;
  __device__ QuadTet(int n_) : n(n_) {}
  __device__ int npts() const { return n * n * n; }
  __device__ void point(const CellGeo &g, int t, int q, double x[3], double *w) const {
    const int f = g.tet_face[t], i = g.tet_i[t];
    // outward-oriented fan triangle (P0, Pi, Pi+1) or (P0, Pi+1, Pi): same vertex order as the
    // sub-tetrahedra of DESIGN.md §Quadrature (the collapsed rule is not vertex-symmetric)
    const bool pos = g.fsign[f] > 0;
    const double *A = g.apex;
    const double *B = g.X[g.floop[f][0]];
    const double *C = g.X[g.floop[f][pos ? i : i + 1]];
    const double *D = g.X[g.floop[f][pos ? i + 1 : i]];
    const int a = q / (n * n), b = (q / n) % n, c = q % n;
    const double u = c_glx[n][a], v = c_glx[n][b], s = c_glx[n][c];
    const double su = u, tv = v * (1 - u), rr = s * (1 - u) * (1 - v);
    double e1[3], e2[3], e3[3];
    for (int d = 0; d < 3; ++d) { e1[d] = B[d] - A[d]; e2[d] = C[d] - A[d]; e3[d] = D[d] - A[d]; }
    const double v6 = fabs(e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) - e1[1] * (e2[0] * e3[2] - e2[2] * e3[0]) +
                           e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]));
    for (int d = 0; d < 3; ++d) x[d] = A[d] + su * e1[d] + tv * e2[d] + rr * e3[d];
    *w = c_glw[n][a] * c_glw[n][b] * c_glw[n][c] * (1 - u) * (1 - u) * (1 - v) * v6;
  }
};

// scaled monomials ((x - xc)/h)^a ordered by degree, then x-power descending
__device__ inline void mono3(const double x[3], const double xc[3], double h, int n, double *m) {
  const double X = (x[0] - xc[0]) / h, Y = (x[1] - xc[1]) / h, Z = (x[2] - xc[2]) / h;
  double px[6], py[6], pz[6];
  px[0] = py[0] = pz[0] = 1.0;
  for (int p = 1; p <= n; ++p) { px[p] = px[p - 1] * X; py[p] = py[p - 1] * Y; pz[p] = pz[p - 1] * Z; }
  int j = 0;
  for (int d = 0; d <= n; ++d)
    for (int a = d; a >= 0; --a)
      for (int b = d - a; b >= 0; --b) m[j++] = px[a] * py[b] * pz[d - a - b];
}

}  // namespace vb
