// VEM geometry and element kernels: cell measures, the D_Q DOFs of the
// constant pressure, element matrices A^K, B^K and the right-hand side.
#include <algorithm>
#include <cmath>
#include "setup.h"
#include "vem_device.cuh"

namespace vb {

// per cell: [vol, xc(3), h, c(np)] with c_a = (1/|K|) int m_a (D_Q of q = 1)
__global__ void cell_geometry_kernel(const int *__restrict__ topo, const double *__restrict__ xyz, int64_t nK,
                                     int k, int np, int geo_stride, double *geo) {
  const int64_t K = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (K >= nK) return;
  CellGeo g;
  load_cell(topo + K * TOPO_STRIDE, xyz, g);
  double *out = geo + K * geo_stride;
  out[0] = g.vol; out[1] = g.xc[0]; out[2] = g.xc[1]; out[3] = g.xc[2]; out[4] = g.h;
  double acc[20];
  for (int a = 0; a < np; ++a) acc[a] = 0.0;
  QuadTet qt(3);
  for (int t = 0; t < g.ntet; ++t)
    for (int q = 0; q < qt.npts(); ++q) {
      double x[3], w;
      qt.point(g, t, q, x, &w);
      double m[20];
      mono3(x, g.xc, g.h, k - 1, m);
      for (int a = 0; a < np; ++a) acc[a] += w * m[a];
    }
  for (int a = 0; a < np; ++a) out[5 + a] = acc[a] / g.vol;
}

void init_quadrature_constants(int k) {
  double gx[9][8] = {}, gw[9][8] = {};
  for (int n = 1; n <= 8; ++n) gauss_legendre01(n, gx[n], gw[n]);
  double lx[5] = {}, lw[5] = {};
  gauss_lobatto01(k + 1, lx, lw);
  VB_CUDA(cudaMemcpyToSymbol(c_glx, gx, sizeof(gx)));
  VB_CUDA(cudaMemcpyToSymbol(c_glw, gw, sizeof(gw)));
  VB_CUDA(cudaMemcpyToSymbol(c_lobx, lx, sizeof(lx)));
  VB_CUDA(cudaMemcpyToSymbol(c_lobw, lw, sizeof(lw)));
}

void cell_geometry_device(vb_ctx *c) {
  init_quadrature_constants(c->k);
  c->geo_stride = 5 + c->np;
  c->d_cellgeo.alloc(c->nK * c->geo_stride);
  cell_geometry_kernel<<<(c->nK + 127) / 128, 128, 0, c->stream>>>(c->d_topo.p, c->d_xyz.p, c->nK, c->k, c->np,
                                                                    c->geo_stride, c->d_cellgeo.p);
  VB_CHECK_LAUNCH();
  VB_CUDA(cudaStreamSynchronize(c->stream));
}

void element_matrices_device(vb_ctx *c) {
  throw Error{VB_EINVAL, "device element generation (K9) not built yet; use vb_setup_from_elements"};
}

void build_rhs_device(vb_ctx *c, const vb_problem *p, double *rhs) {
  throw Error{VB_EINVAL, "device rhs not built yet"};
}

}  // namespace vb
