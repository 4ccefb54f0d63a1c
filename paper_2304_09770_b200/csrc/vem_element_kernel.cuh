// The K9 element kernel body (included once, from vem.cu).
#pragma once
#include "vem_element.cuh"

namespace vb {

struct FaceG {
  double area, n[3], t1[3], t2[3], xc[3], h;
};

__device__ inline void face_geo(const CellGeo &g, int f, FaceG &F) {
  const int len = g.flen[f];
  double av[3] = {0, 0, 0};
  for (int i = 0; i < len; ++i) {
    const double *p = g.X[g.floop[f][i]], *q = g.X[g.floop[f][(i + 1) % len]];
    av[0] += 0.5 * (p[1] * q[2] - p[2] * q[1]);
    av[1] += 0.5 * (p[2] * q[0] - p[0] * q[2]);
    av[2] += 0.5 * (p[0] * q[1] - p[1] * q[0]);
  }
  F.area = sqrt(av[0] * av[0] + av[1] * av[1] + av[2] * av[2]);
  for (int d = 0; d < 3; ++d) F.n[d] = av[d] / F.area;
  double cen[3] = {0, 0, 0}, asum = 0;
  const double *P0 = g.X[g.floop[f][0]];
  for (int i = 1; i + 1 < len; ++i) {
    const double *P1 = g.X[g.floop[f][i]], *P2 = g.X[g.floop[f][i + 1]];
    double u[3], v[3];
    for (int d = 0; d < 3; ++d) { u[d] = P1[d] - P0[d]; v[d] = P2[d] - P0[d]; }
    double cr[3] = {u[1] * v[2] - u[2] * v[1], u[2] * v[0] - u[0] * v[2], u[0] * v[1] - u[1] * v[0]};
    double ai = 0.5 * (cr[0] * F.n[0] + cr[1] * F.n[1] + cr[2] * F.n[2]);
    for (int d = 0; d < 3; ++d) cen[d] += ai * (P0[d] + P1[d] + P2[d]) / 3.0;
    asum += ai;
  }
  for (int d = 0; d < 3; ++d) F.xc[d] = cen[d] / asum;
  double h2 = 0;
  for (int i = 0; i < len; ++i)
    for (int j = i + 1; j < len; ++j) {
      double s = 0;
      for (int d = 0; d < 3; ++d) s += (g.X[g.floop[f][i]][d] - g.X[g.floop[f][j]][d]) * (g.X[g.floop[f][i]][d] - g.X[g.floop[f][j]][d]);
      h2 = fmax(h2, s);
    }
  F.h = sqrt(h2);
  const double *P1 = g.X[g.floop[f][1]];
  double l = 0;
  for (int d = 0; d < 3; ++d) { F.t1[d] = P1[d] - P0[d]; l += F.t1[d] * F.t1[d]; }
  l = sqrt(l);
  for (int d = 0; d < 3; ++d) F.t1[d] /= l;
  F.t2[0] = F.n[1] * F.t1[2] - F.n[2] * F.t1[1];
  F.t2[1] = F.n[2] * F.t1[0] - F.n[0] * F.t1[2];
  F.t2[2] = F.n[0] * F.t1[1] - F.n[1] * F.t1[0];
}

// i-th point of the collapsed rule (n per direction) on the fan triangles of face f
__device__ inline int face_npts(const CellGeo &g, int f, int n) { return (g.flen[f] - 2) * n * n; }
__device__ inline void face_point(const CellGeo &g, int f, int n, int q, double x[3], double *w) {
  const int tri = q / (n * n), r = q % (n * n);
  const double *A = g.X[g.floop[f][0]], *B = g.X[g.floop[f][tri + 1]], *C = g.X[g.floop[f][tri + 2]];
  const double u = c_glx[n][r / n], v = c_glx[n][r % n];
  const double s = u, t = v * (1 - u);
  double e1[3], e2[3];
  for (int d = 0; d < 3; ++d) { e1[d] = B[d] - A[d]; e2[d] = C[d] - A[d]; x[d] = A[d] + s * e1[d] + t * e2[d]; }
  double cr[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2], e1[0] * e2[1] - e1[1] * e2[0]};
  *w = c_glw[n][r / n] * c_glw[n][r % n] * (1 - u) * sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
}

// element-local DOF layout
struct Lay {
  int k, nV, nE, nF, nm, n4, n5, oE, oF, o4, o5, nv;
  __device__ Lay(const CellGeo &g, int k_) : k(k_) {
    nV = g.nv; nE = g.ne; nF = g.nf;
    nm = d2(k - 2); n4 = 3 * d3(k - 3) - d3(k - 4); n5 = d3(k - 1) - 1;
    oE = 3 * nV; oF = oE + 3 * (k - 1) * nE; o4 = oF + 3 * nm * nF; o5 = o4 + n4; nv = o5 + n5;
  }
  __device__ int vdof(int lv, int c) const { return 3 * lv + c; }
  __device__ int edof(int le, int j, int c) const { return oE + 3 * (k - 1) * le + 3 * j + c; }
  __device__ int fdof(int lf, int t, int a) const { return oF + lf * 3 * nm + t * nm + a; }
  __device__ int nfl(const CellGeo &g, int f) const { return g.flen[f] * k + 3 * nm; }
  // face-local dof l of (face f, component c) -> element dof
  __device__ int fl2e(const CellGeo &g, int f, int c, int l) const {
    const int len = g.flen[f];
    if (l < len) return vdof(g.floop[f][l], c);
    if (l < len * k) {
      const int idx = l - len, q = idx / (k - 1), j = idx % (k - 1);
      return edof(g.fedge[f][q], j, c);
    }
    const int idx = l - len * k;
    return fdof(f, idx / nm, idx % nm);
  }
};

}  // namespace vb
