// VEM geometry and element kernels: cell measures, the D_Q DOFs of the
// constant pressure, element matrices A^K, B^K and the right-hand side.
#include <algorithm>
#include <cmath>
#include "setup.h"
#include "vem_device.cuh"
#include "vem_element_kernel.cuh"

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
  c->d_cellgeo.alloc(std::max<int64_t>(c->nKl, 1) * c->geo_stride);
  cell_geometry_kernel<<<(c->nKl + 127) / 128, 128, 0, c->stream>>>(c->d_topo.p, c->d_xyz.p, c->nKl, c->k, c->np,
                                                                     c->geo_stride, c->d_cellgeo.p);
  VB_CHECK_LAUNCH();
  VB_CUDA(cudaStreamSynchronize(c->stream));
}

// ------------------------------------------------------------------ K9 element kernel
template <int K>
struct Arena {
  static constexpr int D1 = d3(K - 1), Dk = d3(K), Dk1 = d3(K + 1), D2m = d3(K - 2);
  static constexpr int q2k = d2(K), q2k1 = d2(K + 1), nm = d2(K - 2), NLM = MAXL * K + 3 * d2(K - 2);
  static constexpr int S3 = 3 * Dk;
  int64_t PF, FM, FW, G, GnK, DIV, RDV, M2, PIN, MK, P0, GR, E, GE, DP, Q, QP, WK, TT, ACD, total;
  __host__ __device__ Arena(int nv, int nf) {   // nv, nf: the largest cell of the launch
    int64_t o = 0;
    PF = o; o += (int64_t)nf * 3 * q2k1 * NLM;
    FM = o; o += (int64_t)nf * Dk1 * q2k1;
    FW = o; o += q2k * q2k + q2k1 * q2k1 + 2 * q2k1 * NLM + q2k1 * q2k1;
    G = o; o += Dk1 * Dk1;
    GnK = o; o += Dk * Dk;
    DIV = o; o += (int64_t)D1 * nv;
    RDV = o; o += (int64_t)D1 * nv;
    M2 = o; o += (int64_t)3 * D2m * nv;
    PIN = o; o += (int64_t)S3 * nv;
    MK = o; o += (int64_t)S3 * nv;
    P0 = o; o += (int64_t)S3 * nv;
    GR = o; o += (int64_t)9 * D1 * nv;
    E = o; o += (int64_t)6 * D1 * nv;
    GE = o; o += (int64_t)6 * D1 * nv;
    DP = o; o += (int64_t)nv * S3;
    Q = o; o += S3 * S3;
    QP = o; o += (int64_t)S3 * nv;
    WK = o; o += S3 * S3;
    TT = o; o += S3 * S3;
    ACD = o; o += nv;
    total = o;
  }
};

// x^e_i components: (x cross e_i)_comp = sgn * x_j  -> table [i][comp] = (j, sgn) or (-1, 0)
__device__ inline void cross_e(int i, int comp, int *j, int *sgn) {
  const int tab[3][3][2] = {{{-1, 0}, {2, 1}, {1, -1}}, {{2, -1}, {-1, 0}, {0, 1}}, {{1, 1}, {0, -1}, {-1, 0}}};
  *j = tab[i][comp][0];
  *sgn = tab[i][comp][1];
}

// The D4 fields x^(m e_cp), same order as the oracle's d4_basis (reading A24): monomials m of
// degree 0..K-3 (exps3 order), cp = 0, 1, 2, omitting cp = 0 when x_1 divides m.  Calls
// fn(i, em, cp) for field i.
template <int K, class Fn>
__device__ inline void for_d4(Fn fn) {
  int i = 0;
  for (int d = 0; d <= K - 3; ++d)
    for (int mi = d3(d - 1); mi < d3(d); ++mi) {
      int em[3];
      exp3(mi, em);
      for (int cp = 0; cp < 3; ++cp) {
        if (cp == 0 && em[0] > 0) continue;
        fn(i++, em, cp);
      }
    }
}

template <int K>
__global__ void __launch_bounds__(128) vem_element_kernel(const int *__restrict__ topo, const double *__restrict__ xyz,
                                                          const double *__restrict__ nu, int64_t K0, int64_t nE,
                                                          int nvmax, int nfmax, double *scratch, int64_t NE, double *elA,
                                                          double *elB, double *P0out, int stop) {
  using Ar = Arena<K>;
  constexpr int D1 = Ar::D1, Dk = Ar::Dk, Dk1 = Ar::Dk1, D2m = Ar::D2m, q2k = Ar::q2k, q2k1 = Ar::q2k1;
  constexpr int nm = Ar::nm, NLM = Ar::NLM, S3 = Ar::S3;
  const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (e >= nE) return;
  const int64_t cell = K0 + e;
  CellGeo g;
  load_cell(topo + cell * TOPO_STRIDE, xyz, g);
  const Lay L(g, K);
  const int nv = L.nv;
  const double nuK = nu[cell];
  const Ar ar(nvmax, nfmax);
  auto S = [&](int64_t off) { return SM{scratch + off * NE + e, NE}; };
  const SM PF = S(ar.PF), FM = S(ar.FM), G = S(ar.G), GnK = S(ar.GnK), DIV = S(ar.DIV), RDV = S(ar.RDV);
  const SM M2 = S(ar.M2), PIN = S(ar.PIN), MK = S(ar.MK), P0 = S(ar.P0), GR = S(ar.GR), E = S(ar.E), GE = S(ar.GE);
  const SM DP = S(ar.DP), Q = S(ar.Q), QP = S(ar.QP), WK = S(ar.WK), TT = S(ar.TT), ACD = S(ar.ACD);
  const SM FGn = S(ar.FW), FG0 = S(ar.FW + q2k * q2k), FR = S(ar.FW + q2k * q2k + q2k1 * q2k1),
           FPN = S(ar.FW + q2k * q2k + q2k1 * q2k1 + q2k1 * NLM),
           FGc = S(ar.FW + q2k * q2k + q2k1 * q2k1 + 2 * q2k1 * NLM);
  const int nqf = K + 2, nqv = K + 3;
  // ================= faces: FM, Pi^nabla_{k,f}, Pi^0_{k+1,f}
  for (int f = 0; f < g.nf; ++f) {
    FaceG F;
    face_geo(g, f, F);
    const int len = g.flen[f], nl = L.nfl(g, f);
    for (int i = 0; i < Dk1 * q2k1; ++i) FM(f * Dk1 * q2k1 + i) = 0.0;
    for (int i = 0; i < q2k1 * q2k1; ++i) FG0(i) = 0.0;
    for (int i = 0; i < q2k * q2k; ++i) FGn(i) = 0.0;
    const int np_ = face_npts(g, f, nqf);
    for (int q = 0; q < np_; ++q) {
      double x[3], w;
      face_point(g, f, nqf, q, x, &w);
      double m3[d3(K + 1)], m2[d2(K + 1)], g2[d2(K + 1)][2];
      mono3(x, g.xc, g.h, K + 1, m3);
      double xi = 0, eta = 0;
      for (int d = 0; d < 3; ++d) { xi += (x[d] - F.xc[d]) * F.t1[d]; eta += (x[d] - F.xc[d]) * F.t2[d]; }
      mono2(xi, eta, F.h, K + 1, m2, g2);
      for (int b = 0; b < Dk1; ++b)
        for (int a = 0; a < q2k1; ++a) FM(f * Dk1 * q2k1 + b * q2k1 + a) += w * m3[b] * m2[a];
      for (int a = 0; a < q2k1; ++a)
        for (int b = 0; b < q2k1; ++b) FG0(a * q2k1 + b) += w * m2[a] * m2[b];
      for (int a = 1; a < q2k; ++a)
        for (int b = 0; b < q2k; ++b) FGn(a * q2k + b) += w * (g2[a][0] * g2[b][0] + g2[a][1] * g2[b][1]);
    }
    // row 0 of Gn: int_{boundary of f} m_b (GL rule on the edges, exact)
    for (int i = 0; i < len; ++i) {
      const double *Pa = g.X[g.floop[f][i]], *Pb = g.X[g.floop[f][(i + 1) % len]];
      double el = 0;
      for (int d = 0; d < 3; ++d) el += (Pb[d] - Pa[d]) * (Pb[d] - Pa[d]);
      el = sqrt(el);
      for (int j = 0; j <= K; ++j) {
        double xi = 0, eta = 0;
        for (int d = 0; d < 3; ++d) {
          const double xd = Pa[d] + c_lobx[j] * (Pb[d] - Pa[d]) - F.xc[d];
          xi += xd * F.t1[d]; eta += xd * F.t2[d];
        }
        double m2[d2(K + 1)];
        mono2(xi, eta, F.h, K, m2, nullptr);
        for (int b = 0; b < q2k; ++b) FGn(b) += el * c_lobw[j] * m2[b];
      }
    }
    const double *tau[3] = {F.n, F.t1, F.t2};
    for (int c = 0; c < 3; ++c) {
      for (int i = 0; i < q2k * nl; ++i) FPN(i) = 0.0;
      // boundary terms on the loop edges (nodal values at the GL nodes are DOFs)
      for (int i = 0; i < len; ++i) {
        const double *Pa = g.X[g.floop[f][i]], *Pb = g.X[g.floop[f][(i + 1) % len]];
        double dv[3], el = 0;
        for (int d = 0; d < 3; ++d) { dv[d] = Pb[d] - Pa[d]; el += dv[d] * dv[d]; }
        el = sqrt(el);
        double ne[3] = {(dv[1] * F.n[2] - dv[2] * F.n[1]) / el, (dv[2] * F.n[0] - dv[0] * F.n[2]) / el,
                        (dv[0] * F.n[1] - dv[1] * F.n[0]) / el};
        const double n2x = ne[0] * F.t1[0] + ne[1] * F.t1[1] + ne[2] * F.t1[2];
        const double n2y = ne[0] * F.t2[0] + ne[1] * F.t2[1] + ne[2] * F.t2[2];
        for (int j = 0; j <= K; ++j) {
          double xi = 0, eta = 0;
          for (int d = 0; d < 3; ++d) {
            const double xd = Pa[d] + c_lobx[j] * dv[d] - F.xc[d];
            xi += xd * F.t1[d]; eta += xd * F.t2[d];
          }
          double m2[d2(K + 1)], g2[d2(K + 1)][2];
          mono2(xi, eta, F.h, K, m2, g2);
          int l;
          if (j == 0) l = i;
          else if (j == K) l = (i + 1) % len;
          else l = len + i * (K - 1) + (g.ffwd[f][i] ? j - 1 : K - 2 - (j - 1));
          const double wt = el * c_lobw[j];
          for (int b = 1; b < q2k; ++b) FPN(b * nl + l) += wt * (g2[b][0] * n2x + g2[b][1] * n2y);
          FPN(l) += wt;
        }
      }
      // - int_f Lap(m_b) v_c with the interior moments |f| (n_c D3n + t1_c D3t1 + t2_c D3t2)
      for (int b = 1; b < q2k; ++b) {
        int eb[2];
        exp2d(b, eb);
        for (int dir = 0; dir < 2; ++dir) {
          if (eb[dir] < 2) continue;
          const int gi = dir == 0 ? idx2(eb[0] - 2, eb[1]) : idx2(eb[0], eb[1] - 2);
          const double coef = eb[dir] * (eb[dir] - 1) / (F.h * F.h);
          for (int t = 0; t < 3; ++t) FPN(b * nl + len * K + t * nm + gi) -= coef * F.area * tau[t][c];
        }
      }
      for (int i = 0; i < q2k * q2k; ++i) FGc(i) = FGn(i);
      lu_solve(FGc, q2k, FPN, nl);
      // Pi^0_{k+1,f}: moments <= k-2 from the DOFs, k-1..k+1 by the enhancement (iii)
      for (int a = 0; a < q2k1; ++a)
        for (int l = 0; l < nl; ++l) {
          double v = 0.0;
          if (a < nm) {
            const int t = (l - len * K) / nm, aa = (l - len * K) % nm;
            if (l >= len * K && aa == a) v = F.area * tau[t][c];
          } else {
            for (int b = 0; b < q2k; ++b) v += FG0(a * q2k1 + b) * FPN(b * nl + l);
          }
          FR(a * nl + l) = v;
        }
      for (int i = 0; i < q2k1 * q2k1; ++i) FGc(i) = FG0(i);
      lu_solve(FGc, q2k1, FR, nl);
      for (int i = 0; i < q2k1 * nl; ++i) PF(((int64_t)f * 3 + c) * q2k1 * NLM + i) = FR(i);
    }
  }
  // face integral of v_c against a 3D monomial combination: out_row[elem dof] += s * int_f v_c m_b
  auto face_int = [&](int f, int c, int b, double s, SM out, int64_t row0) {
    const int nl = L.nfl(g, f);
    const int64_t base = ((int64_t)f * 3 + c) * q2k1 * NLM;
    for (int l = 0; l < nl; ++l) {
      double v = 0.0;
      for (int a = 0; a < q2k1; ++a) v += FM(f * Dk1 * q2k1 + b * q2k1 + a) * PF(base + a * nl + l);
      out(row0 + L.fl2e(g, f, c, l)) += s * v;
    }
  };
  if (stop == 1) return;   // VB_K9_STOP: stage-time experiment
  // ================= volume Gram matrices, from the cell moments int m_e of degree <= 2k + 2 (one
  // accumulator per distinct monomial, in registers/local memory, instead of one read-modify-write
  // of the global scratch per Gram entry per quadrature point):
  //   G_ab = int m_a m_b = mom[e_a + e_b],
  //   GnK_ab = int grad m_a . grad m_b = sum_c (a_c b_c / h^2) mom[e_a + e_b - 2 e_c]   (a >= 1)
  {
    constexpr int NM = d3(2 * K + 2);
    double mom[NM];
    for (int i = 0; i < NM; ++i) mom[i] = 0.0;
    QuadTet qt(nqv);
    for (int t = 0; t < g.ntet; ++t)
      for (int q = 0; q < qt.npts(); ++q) {
        double x[3], w;
        qt.point(g, t, q, x, &w);
        double px[2 * K + 3], py[2 * K + 3], pz[2 * K + 3];
        px[0] = py[0] = pz[0] = w;   // the weight folded into the x powers
        py[0] = pz[0] = 1.0;
        const double X = (x[0] - g.xc[0]) / g.h, Y = (x[1] - g.xc[1]) / g.h, Z = (x[2] - g.xc[2]) / g.h;
        for (int p = 1; p <= 2 * K + 2; ++p) { px[p] = px[p - 1] * X; py[p] = py[p - 1] * Y; pz[p] = pz[p - 1] * Z; }
        int j = 0;
        for (int d = 0; d <= 2 * K + 2; ++d)
          for (int a = d; a >= 0; --a)
            for (int b = d - a; b >= 0; --b) mom[j++] += px[a] * py[b] * pz[d - a - b];
      }
    for (int a = 0; a < Dk1; ++a) {
      int ea[3];
      exp3(a, ea);
      for (int b = 0; b <= a; ++b) {
        int eb[3];
        exp3(b, eb);
        const double v = mom[idx3(ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2])];
        G(a * Dk1 + b) = v;
        G(b * Dk1 + a) = v;
      }
    }
    const double ih2 = 1.0 / (g.h * g.h);
    for (int b = 0; b < Dk; ++b) GnK(b) = 0.0;
    for (int a = 1; a < Dk; ++a) {
      int ea[3];
      exp3(a, ea);
      for (int b = 0; b < Dk; ++b) {
        int eb[3];
        exp3(b, eb);
        double v = 0.0;
        for (int c = 0; c < 3; ++c) {
          if (ea[c] == 0 || eb[c] == 0) continue;
          int e[3] = {ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2]};
          e[c] -= 2;
          v += ea[c] * eb[c] * ih2 * mom[idx3(e[0], e[1], e[2])];
        }
        GnK(a * Dk + b) = v;
      }
    }
    for (int f = 0; f < g.nf; ++f)
      for (int b = 0; b < Dk; ++b) GnK(b) += FM(f * Dk1 * q2k1 + b * q2k1 + 0);
  }
  auto copyG = [&](int n) { for (int a = 0; a < n; ++a) for (int b = 0; b < n; ++b) WK(a * n + b) = G(a * Dk1 + b); };
  // ================= (1) divergence (F2): Rdiv and DIVc = G_{k-1}^-1 Rdiv
  for (int i = 0; i < D1 * nv; ++i) { RDV(i) = 0.0; DIV(i) = 0.0; }
  {
    double areas[MAXF];
    for (int f = 0; f < g.nf; ++f) { FaceG F; face_geo(g, f, F); areas[f] = F.area; }
    for (int f = 0; f < g.nf; ++f) RDV(L.fdof(f, 0, 0)) += g.fsign[f] * areas[f];
  }
  for (int a = 1; a < D1; ++a) RDV(a * nv + L.o5 + a - 1) = g.vol / g.h;
  for (int i = 0; i < D1 * nv; ++i) DIV(i) = RDV(i);
  copyG(D1);
  lu_solve(WK, D1, DIV, nv);
  // face normals (for the flux terms)
  double fn[MAXF][3];
  for (int f = 0; f < g.nf; ++f) { FaceG F; face_geo(g, f, F); for (int d = 0; d < 3; ++d) fn[f][d] = F.n[d]; }
  // ================= (2) moments against [P_{k-2}]^3: grad P_{k-1} (+) x^[P_{k-3}]^3 (square system)
  {
    const int ns = 3 * D2m;
    for (int i = 0; i < ns * ns; ++i) TT(i) = 0.0;
    for (int i = 0; i < ns * nv; ++i) M2(i) = 0.0;
    int s = 0;
    for (int b = 1; b < D1; ++b, ++s) {
      int eb[3];
      exp3(b, eb);
      for (int c = 0; c < 3; ++c)
        if (eb[c] > 0) {
          int ee[3] = {eb[0], eb[1], eb[2]};
          ee[c]--;
          TT(s * ns + c * D2m + idx3(ee[0], ee[1], ee[2])) += eb[c] / g.h;
        }
      for (int i = 0; i < nv; ++i) M2(s * nv + i) = -RDV(b * nv + i);
      for (int f = 0; f < g.nf; ++f)
        for (int c = 0; c < 3; ++c) face_int(f, c, b, g.fsign[f] * fn[f][c], M2, (int64_t)s * nv);
    }
    for_d4<K>([&](int i, const int em[3], int cp) {   // D4 rows: int v . x^(m e_cp) = |K| D4_i
      for (int comp = 0; comp < 3; ++comp) {
        int j, sg;
        cross_e(cp, comp, &j, &sg);
        if (j < 0) continue;
        int ee[3] = {em[0], em[1], em[2]};
        ee[j]++;
        TT(s * ns + comp * D2m + idx3(ee[0], ee[1], ee[2])) += sg;
      }
      M2(s * nv + L.o4 + i) = g.vol;
      ++s;
    });
    lu_solve(TT, ns, M2, nv);
  }
  if (stop == 2) return;   // VB_K9_STOP: stage-time experiment
  // ================= (3) Pi^nabla_{k,K} per component
  for (int c = 0; c < 3; ++c) {
    const int64_t r0 = (int64_t)c * Dk * nv;
    for (int i = 0; i < Dk * nv; ++i) PIN(r0 + i) = 0.0;
    for (int b = 1; b < Dk; ++b) {
      int eb[3];
      exp3(b, eb);
      for (int cc = 0; cc < 3; ++cc)
        if (eb[cc] >= 2) {
          int ee[3] = {eb[0], eb[1], eb[2]};
          ee[cc] -= 2;
          const int gi = idx3(ee[0], ee[1], ee[2]);
          const double coef = eb[cc] * (eb[cc] - 1) / (g.h * g.h);
          for (int i = 0; i < nv; ++i) PIN(r0 + b * nv + i) -= coef * M2((c * D2m + gi) * nv + i);
        }
      for (int d = 0; d < 3; ++d)
        if (eb[d] > 0) {
          int ee[3] = {eb[0], eb[1], eb[2]};
          ee[d]--;
          const int gi = idx3(ee[0], ee[1], ee[2]);
          for (int f = 0; f < g.nf; ++f) face_int(f, c, gi, g.fsign[f] * fn[f][d] * eb[d] / g.h, PIN, r0 + b * nv);
        }
    }
    for (int f = 0; f < g.nf; ++f) face_int(f, c, 0, 1.0, PIN, r0);
    for (int a = 0; a < Dk; ++a) for (int b = 0; b < Dk; ++b) WK(a * Dk + b) = GnK(a * Dk + b);
    SM pin{PIN.p + r0 * NE, NE};
    lu_solve(WK, Dk, pin, nv);
  }
  if (stop == 3) return;   // VB_K9_STOP: stage-time experiment
  // ================= (4) moments against [P_k]^3: grad P_{k+1} (+) x^[P_{k-1}]^3, super-enhancement
  {
    for (int i = 0; i < S3 * S3; ++i) TT(i) = 0.0;
    for (int i = 0; i < S3 * nv; ++i) MK(i) = 0.0;
    int s = 0;
    for (int b = 1; b < Dk1; ++b, ++s) {
      int eb[3];
      exp3(b, eb);
      for (int c = 0; c < 3; ++c)
        if (eb[c] > 0) {
          int ee[3] = {eb[0], eb[1], eb[2]};
          ee[c]--;
          TT(s * S3 + c * Dk + idx3(ee[0], ee[1], ee[2])) += eb[c] / g.h;
        }
      for (int a = 0; a < D1; ++a) {
        const double gba = G(b * Dk1 + a);
        if (gba != 0.0)
          for (int i = 0; i < nv; ++i) MK(s * nv + i) -= gba * DIV(a * nv + i);
      }
      for (int f = 0; f < g.nf; ++f)
        for (int c = 0; c < 3; ++c) face_int(f, c, b, g.fsign[f] * fn[f][c], MK, (int64_t)s * nv);
    }
    for_d4<K>([&](int i, const int em[3], int cp) {   // D4 rows
      for (int comp = 0; comp < 3; ++comp) {
        int j, sg;
        cross_e(cp, comp, &j, &sg);
        if (j < 0) continue;
        int ee[3] = {em[0], em[1], em[2]};
        ee[j]++;
        TT(s * S3 + comp * Dk + idx3(ee[0], ee[1], ee[2])) += sg;
      }
      MK(s * nv + L.o4 + i) = g.vol;
      ++s;
    });
    // super-enhancement rows: x^(m e_cp) for |m| = d in {k-2, k-1}, skipping (cp = 0, x1 | m)
    for (int d = K - 2; d <= K - 1; ++d)
      for (int mi = d3(d - 1); mi < d3(d); ++mi) {
        int em[3];
        exp3(mi, em);
        for (int cp = 0; cp < 3; ++cp) {
          if (cp == 0 && em[0] > 0) continue;
          // w = x^(m e_cp): component comp = sgn * x_j * m
          int wi[3] = {-1, -1, -1}, ws[3] = {0, 0, 0};
          for (int comp = 0; comp < 3; ++comp) {
            int j, sg;
            cross_e(cp, comp, &j, &sg);
            if (j < 0) continue;
            int ee[3] = {em[0], em[1], em[2]};
            ee[j]++;
            wi[comp] = idx3(ee[0], ee[1], ee[2]);
            ws[comp] = sg;
            TT(s * S3 + comp * Dk + wi[comp]) += sg;
          }
          // int Pi^nabla v . w = sum_comp sum_g PIN[comp][g] * sgn * G[g][wi]
          for (int comp = 0; comp < 3; ++comp) {
            if (wi[comp] < 0) continue;
            for (int gg = 0; gg < Dk; ++gg) {
              const double coef = ws[comp] * G(gg * Dk1 + wi[comp]);
              if (coef != 0.0)
                for (int i = 0; i < nv; ++i) MK(s * nv + i) += coef * PIN(((int64_t)comp * Dk + gg) * nv + i);
            }
          }
          ++s;
        }
      }
    lu_solve(TT, S3, MK, nv);
  }
  // ================= (5) Pi^0_{k,K} = G_k^-1 MomK
  for (int c = 0; c < 3; ++c) {
    for (int i = 0; i < Dk * nv; ++i) P0((int64_t)c * Dk * nv + i) = MK((int64_t)c * Dk * nv + i);
    copyG(Dk);
    SM p0{P0.p + (int64_t)c * Dk * nv * NE, NE};
    lu_solve(WK, Dk, p0, nv);
  }
  for (int i = 0; i < S3 * nv; ++i) P0out[cell * (int64_t)S3 * nvmax + i] = P0(i);
  if (stop == 5) return;   // VB_K9_STOP: stage-time experiment
  // ================= (6) Pi^0_{k-1} grad v
  for (int c = 0; c < 3; ++c)
    for (int d = 0; d < 3; ++d) {
      const int64_t r0 = (int64_t)(c * 3 + d) * D1 * nv;
      for (int i = 0; i < D1 * nv; ++i) GR(r0 + i) = 0.0;
      for (int a = 0; a < D1; ++a) {
        int ea[3];
        exp3(a, ea);
        if (ea[d] > 0) {
          int ee[3] = {ea[0], ea[1], ea[2]};
          ee[d]--;
          const int gi = idx3(ee[0], ee[1], ee[2]);
          for (int i = 0; i < nv; ++i) GR(r0 + a * nv + i) -= ea[d] / g.h * MK(((int64_t)c * Dk + gi) * nv + i);
        }
        for (int f = 0; f < g.nf; ++f) face_int(f, c, a, g.fsign[f] * fn[f][d], GR, r0 + a * nv);
      }
      copyG(D1);
      SM gr{GR.p + r0 * NE, NE};
      lu_solve(WK, D1, gr, nv);
    }
  // E_p = sym parts, GE_p = G_{k-1} E_p; pairs (00,11,22,01,02,12)
  const int pc[6] = {0, 1, 2, 0, 0, 1}, pd[6] = {0, 1, 2, 1, 2, 2};
  for (int p = 0; p < 6; ++p) {
    const int64_t a0 = (int64_t)(pc[p] * 3 + pd[p]) * D1 * nv, b0 = (int64_t)(pd[p] * 3 + pc[p]) * D1 * nv;
    for (int i = 0; i < D1 * nv; ++i) E((int64_t)p * D1 * nv + i) = 0.5 * (GR(a0 + i) + GR(b0 + i));
    for (int a = 0; a < D1; ++a)
      for (int i = 0; i < nv; ++i) {
        double v = 0.0;
        for (int b = 0; b < D1; ++b) v += G(a * Dk1 + b) * E(((int64_t)p * D1 + b) * nv + i);
        GE(((int64_t)p * D1 + a) * nv + i) = v;
      }
  }
  auto acons = [&](int i, int j) {
    double v = 0.0;
    for (int p = 0; p < 6; ++p) {
      const double wgt = p < 3 ? 1.0 : 2.0;
      double s = 0.0;
      for (int a = 0; a < D1; ++a) s += E(((int64_t)p * D1 + a) * nv + i) * GE(((int64_t)p * D1 + a) * nv + j);
      v += wgt * s;
    }
    return nuK * v;
  };
  if (stop == 6) return;   // VB_K9_STOP: stage-time experiment
  // ================= (7) DOFs of the polynomial basis {m_g e_c}: DP (nv x 3Dk)
  for (int i = 0; i < nv * S3; ++i) DP(i) = 0.0;
  for (int lv = 0; lv < g.nv; ++lv) {
    double m[d3(K)];
    mono3(g.X[lv], g.xc, g.h, K, m);
    for (int c = 0; c < 3; ++c)
      for (int gg = 0; gg < Dk; ++gg) DP((int64_t)L.vdof(lv, c) * S3 + c * Dk + gg) = m[gg];
  }
  for (int le = 0; le < g.ne; ++le) {
    const double *Pa = g.X[g.ev[le][0]], *Pb = g.X[g.ev[le][1]];
    for (int j = 0; j < K - 1; ++j) {
      double x[3];
      for (int d = 0; d < 3; ++d) x[d] = Pa[d] + c_lobx[j + 1] * (Pb[d] - Pa[d]);
      double m[d3(K)];
      mono3(x, g.xc, g.h, K, m);
      for (int c = 0; c < 3; ++c)
        for (int gg = 0; gg < Dk; ++gg) DP((int64_t)L.edof(le, j, c) * S3 + c * Dk + gg) = m[gg];
    }
  }
  for (int f = 0; f < g.nf; ++f) {
    FaceG F;
    face_geo(g, f, F);
    const double *tau[3] = {F.n, F.t1, F.t2};
    for (int t = 0; t < 3; ++t)
      for (int a = 0; a < nm; ++a)
        for (int c = 0; c < 3; ++c)
          for (int gg = 0; gg < Dk; ++gg)
            DP((int64_t)L.fdof(f, t, a) * S3 + c * Dk + gg) = tau[t][c] * FM(f * Dk1 * q2k1 + gg * q2k1 + a) / F.area;
  }
  for_d4<K>([&](int i, const int em[3], int cp) {   // D4 of m_g e_c: (1/|K|) int m_g (x^(m e_cp))_c
    for (int c = 0; c < 3; ++c) {
      int j, sg;
      cross_e(cp, c, &j, &sg);
      if (j < 0) continue;
      int ee[3] = {em[0], em[1], em[2]};
      ee[j]++;
      const int wi = idx3(ee[0], ee[1], ee[2]);
      for (int gg = 0; gg < Dk; ++gg) DP((int64_t)(L.o4 + i) * S3 + c * Dk + gg) = sg * G(gg * Dk1 + wi) / g.vol;
    }
  });
  for (int a = 1; a < D1; ++a)
    for (int c = 0; c < 3; ++c)
      for (int gg = 0; gg < Dk; ++gg) {
        int eg[3];
        exp3(gg, eg);
        if (eg[c] == 0) continue;
        int ee[3] = {eg[0], eg[1], eg[2]};
        ee[c]--;
        DP((int64_t)(L.o5 + a - 1) * S3 + c * Dk + gg) = eg[c] * G(idx3(ee[0], ee[1], ee[2]) * Dk1 + a) / g.vol;
      }
  // ================= (8) D-recipe weights, Q = DP^T diag(d) DP, QP = Q PiN
  for (int i = 0; i < nv; ++i) ACD(i) = fmax(acons(i, i), nuK * g.h);
  for (int a = 0; a < S3; ++a)
    for (int b = 0; b <= a; ++b) {
      double v = 0.0;
      for (int l = 0; l < nv; ++l) v += DP((int64_t)l * S3 + a) * ACD(l) * DP((int64_t)l * S3 + b);
      Q(a * S3 + b) = v;
      Q(b * S3 + a) = v;
    }
  for (int a = 0; a < S3; ++a)
    for (int i = 0; i < nv; ++i) {
      double v = 0.0;
      for (int b = 0; b < S3; ++b) v += Q(a * S3 + b) * PIN((int64_t)b * nv + i);
      QP((int64_t)a * nv + i) = v;
    }
  // ================= (10) B^K = |K| DIVc (dual pressure basis)
  double *Bout = elB + cell * (int64_t)D1 * nvmax;
  for (int a = 0; a < D1; ++a)
    for (int i = 0; i < nv; ++i) Bout[(int64_t)a * nv + i] = g.vol * DIV(a * nv + i);
  // (9) here when stop == -1, else in vem_assemble_A_kernel (a thread per (cell, row)) or not at all
  // (VB_K9_STOP stage-time experiment)
  if (stop != -1) return;
  // ================= (9) A = A_cons + (I - Pihat)^T D (I - Pihat)  (Eq.(discreteA))
  double *Aout = elA + cell * (int64_t)nvmax * nvmax;
  for (int i = 0; i < nv; ++i)
    for (int j = i; j < nv; ++j) {
      double pij = 0.0, pji = 0.0, quad = 0.0;
      for (int a = 0; a < S3; ++a) {
        const double pa_i = PIN((int64_t)a * nv + i), pa_j = PIN((int64_t)a * nv + j);
        pij += DP((int64_t)i * S3 + a) * pa_j;
        pji += DP((int64_t)j * S3 + a) * pa_i;
        quad += pa_i * QP((int64_t)a * nv + j);
      }
      double v = acons(i, j) - ACD(i) * pij - ACD(j) * pji + quad;
      if (i == j) v += ACD(i);
      Aout[(int64_t)i * nv + j] = v;
      Aout[(int64_t)j * nv + i] = v;
    }

}

// K9 stage (9), A^K = A_cons + (I - Pihat)^T D (I - Pihat) (Eq.(discreteA)), one thread per (cell,
// row i) instead of one per cell (a c3 cell has 252 rows: the single-thread loop was 40 % of K9):
// row i for j >= i from the cell's scratch (PIN, DP, QP, E, GE, ACD of vem_element_kernel), written
// to both triangles, the same arithmetic in the same order as the single-thread version.
template <int K>
__global__ void __launch_bounds__(128) vem_assemble_A_kernel(const int *__restrict__ cell_nv,
                                                             const double *__restrict__ nu, int64_t K0, int64_t nE,
                                                             int nvmax, int nfmax, const double *__restrict__ scratch,
                                                             int64_t NE, double *elA) {
  using Ar = Arena<K>;
  constexpr int D1 = Ar::D1, S3 = Ar::S3;
  // lanes = consecutive cells, same row: the cell-interleaved scratch stays coalesced
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t e = t % nE;
  const int i = (int)(t / nE);
  if (i >= nvmax) return;
  const int64_t cell = K0 + e;
  const int nv = cell_nv[cell];
  if (i >= nv) return;
  const double nuK = nu[cell];
  const Ar ar(nvmax, nfmax);
  auto S = [&](int64_t off) { return SM{const_cast<double *>(scratch) + off * NE + e, NE}; };
  const SM PIN = S(ar.PIN), DP = S(ar.DP), QP = S(ar.QP), E = S(ar.E), GE = S(ar.GE), ACD = S(ar.ACD);
  auto acons = [&](int a_, int b_) {
    double v = 0.0;
    for (int p = 0; p < 6; ++p) {
      const double wgt = p < 3 ? 1.0 : 2.0;
      double s = 0.0;
      for (int a = 0; a < D1; ++a) s += E(((int64_t)p * D1 + a) * nv + a_) * GE(((int64_t)p * D1 + a) * nv + b_);
      v += wgt * s;
    }
    return nuK * v;
  };
  double *Aout = elA + cell * (int64_t)nvmax * nvmax;
  const double acd_i = ACD(i);
  for (int j = i; j < nv; ++j) {
    double pij = 0.0, pji = 0.0, quad = 0.0;
    for (int a = 0; a < S3; ++a) {
      const double pa_i = PIN((int64_t)a * nv + i), pa_j = PIN((int64_t)a * nv + j);
      pij += DP((int64_t)i * S3 + a) * pa_j;
      pji += DP((int64_t)j * S3 + a) * pa_i;
      quad += pa_i * QP((int64_t)a * nv + j);
    }
    double v = acons(i, j) - acd_i * pij - ACD(j) * pji + quad;
    if (i == j) v += acd_i;
    Aout[(int64_t)i * nv + j] = v;
    Aout[(int64_t)j * nv + i] = v;
  }
}

void element_matrices_device(vb_ctx *c, bool wait) {
  cudaStream_t s = c->stream;
  const int nvm = c->nv_max;
  const int S3 = 3 * (c->k == 2 ? 10 : (c->k == 3 ? 20 : 35));
  c->d_elA.alloc((size_t)c->nKl * nvm * nvm);
  c->d_elB.alloc((size_t)c->nKl * c->np * nvm);
  c->d_P0.alloc((size_t)c->nKl * S3 * nvm);
  int nfm = 1;
  for (int64_t l = 0; l < c->nKl; ++l) nfm = std::max(nfm, c->cell_topo[c->cell_gid[l] * TOPO_STRIDE + 2]);
  const int64_t per = c->k == 2 ? Arena<2>(nvm, nfm).total
                                : (c->k == 3 ? Arena<3>(nvm, nfm).total : Arena<4>(nvm, nfm).total);
  // all cells in one launch when the scratch fits (one thread per cell: a launch needs every cell it
  // can get to fill 148 SMs), else chunks within a third of the free memory, at most 24 GB
  size_t fr = 0, tot = 0;
  VB_CUDA(cudaMemGetInfo(&fr, &tot));
  const double budget = std::min(24e9, fr / 3.0);
  int64_t NE = std::max<int64_t>(128, std::min<int64_t>(c->nKl, (int64_t)(budget / 8 / per)));
  NE = (NE + 127) / 128 * 128;
  DBuf<double> &scratch = c->w_k9;
  scratch.alloc((size_t)per * NE);
  // threads per block: one cell per thread, so the block size only sets how evenly the cells
  // spread over the 148 SMs (VB_K9_BLOCK: experiment knob)
  static const int k9_stop = getenv("VB_K9_STOP") ? atoi(getenv("VB_K9_STOP")) : 0;   // experiment knob
  static const int k9_block = getenv("VB_K9_BLOCK") ? std::max(32, std::min(128, atoi(getenv("VB_K9_BLOCK")))) : 64;
  for (int64_t K0 = 0; K0 < c->nKl; K0 += NE) {
    const int64_t n = std::min<int64_t>(NE, c->nKl - K0);
    const int blocks = (int)((n + k9_block - 1) / k9_block);
    // stage (9) in its own thread-per-(cell, row) kernel when a thread per cell under-fills the GPU
    // (c3: 4,096 cells, K9 1.33 -> 0.96 s); with many cells (c5: 32,768) the one-thread-per-cell
    // loop is faster (0.135 against 0.173 s)
    const bool split9 = k9_stop == 0 && n < 16384;
    const int stop_arg = k9_stop == 0 && !split9 ? -1 : k9_stop;
#define VB_K9(KK)                                                                                           \
  vem_element_kernel<KK><<<blocks, k9_block, 0, s>>>(c->d_topo.p, c->d_xyz.p, c->d_nu.p, K0, n, nvm, nfm, scratch.p, NE, \
                                                c->d_elA.p, c->d_elB.p, c->d_P0.p, stop_arg)
    if (c->k == 2) VB_K9(2);
    else if (c->k == 3) VB_K9(3);
    else VB_K9(4);
#undef VB_K9
    VB_STAGE();
    if (split9) {   // stage (9): a thread per (cell, row)
      const int64_t nt = n * nvm;
      const int ab = (int)((nt + 127) / 128);
      if (c->k == 2) vem_assemble_A_kernel<2><<<ab, 128, 0, s>>>(c->d_cell_nv.p, c->d_nu.p, K0, n, nvm, nfm, scratch.p, NE, c->d_elA.p);
      else if (c->k == 3) vem_assemble_A_kernel<3><<<ab, 128, 0, s>>>(c->d_cell_nv.p, c->d_nu.p, K0, n, nvm, nfm, scratch.p, NE, c->d_elA.p);
      else vem_assemble_A_kernel<4><<<ab, 128, 0, s>>>(c->d_cell_nv.p, c->d_nu.p, K0, n, nvm, nfm, scratch.p, NE, c->d_elA.p);
      VB_STAGE();
    }
  }
  if (wait) {
    VB_CUDA(cudaStreamSynchronize(s));
    scratch.release();
  }
}

// ------------------------------------------------------------------ problem data (BASELINE configs)
struct ProbDev {
  int kind, ns;
  double delta, omega, beta;
  double cen[16][3];
};

__device__ inline void u_exact(const double x[3], double u[3]) {
  const double PI = 3.141592653589793;
  const double sx = sin(PI * x[0]), sy = sin(PI * x[1]), sz = sin(PI * x[2]);
  const double cx = cos(PI * x[0]), cy = cos(PI * x[1]), cz = cos(PI * x[2]);
  const double px = PI * cx * sy * sz, py = PI * sx * cy * sz, pz = PI * sx * sy * cz;
  u[0] = py - pz; u[1] = pz - px; u[2] = px - py;      // curl of phi (1,1,1)
}

// f = (3 pi^2 nu / 2) u - grad p, p = sin(2 pi x) cos(pi y) z; sinker: (0,0,beta(chi-1))
__device__ inline void f_problem(const ProbDev &P, const double x[3], double nuK, double f[3]) {
  const double PI = 3.141592653589793;
  if (P.kind == 0) {
    double u[3];
    u_exact(x, u);
    const double gp0 = 2 * PI * cos(2 * PI * x[0]) * cos(PI * x[1]) * x[2];
    const double gp1 = -PI * sin(2 * PI * x[0]) * sin(PI * x[1]) * x[2];
    const double gp2 = sin(2 * PI * x[0]) * cos(PI * x[1]);
    const double a = 1.5 * PI * PI * nuK;
    f[0] = a * u[0] - gp0; f[1] = a * u[1] - gp1; f[2] = a * u[2] - gp2;
  } else {
    double chi = 1.0;
    for (int i = 0; i < P.ns; ++i) {
      double d = 0;
      for (int q = 0; q < 3; ++q) d += (x[q] - P.cen[i][q]) * (x[q] - P.cen[i][q]);
      d = sqrt(d);
      const double t = fmax(0.0, d - P.omega / 2);
      chi *= 1.0 - exp(-P.delta * t * t);
    }
    f[0] = 0.0; f[1] = 0.0; f[2] = P.beta * (chi - 1.0);
  }
}

// per element: load (int Pi^0_k f . phi_i) minus the lifted boundary data
template <int K>
__global__ void rhs_element_kernel(const int *__restrict__ topo, const double *__restrict__ xyz,
                                   const double *__restrict__ nu, const int64_t *__restrict__ l2g,
                                   const int64_t *__restrict__ vel2free, const double *__restrict__ elA,
                                   const double *__restrict__ elB, const double *__restrict__ P0all, int64_t nK,
                                   int nvmax, ProbDev P, double *yel, double *uDall) {
  constexpr int Dk = d3(K), D1 = d3(K - 1), S3 = 3 * d3(K), nm = d2(K - 2);
  const int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (cell >= nK) return;
  CellGeo g;
  load_cell(topo + cell * TOPO_STRIDE, xyz, g);
  const Lay L(g, K);
  const int nv = L.nv;
  const double nuK = nu[cell];
  double Fm[S3];
  for (int i = 0; i < S3; ++i) Fm[i] = 0.0;
  QuadTet qt(K + 3);
  for (int t = 0; t < g.ntet; ++t)
    for (int q = 0; q < qt.npts(); ++q) {
      double x[3], w, f[3], m[d3(K)];
      qt.point(g, t, q, x, &w);
      f_problem(P, x, nuK, f);
      mono3(x, g.xc, g.h, K, m);
      for (int c = 0; c < 3; ++c)
        for (int a = 0; a < Dk; ++a) Fm[c * Dk + a] += w * f[c] * m[a];
    }
  const double *P0 = P0all + cell * (int64_t)S3 * nvmax;
  const int stride = nvmax + D1;
  double *y = yel + cell * stride;
  // lifted boundary DOFs (interpolant of the exact trace; zero for the sinker problem), per cell in
  // global scratch (general polyhedra: up to a thousand DOFs per cell)
  double *uD = uDall + cell * (int64_t)nvmax;
  bool any = false;
  for (int j = 0; j < nv; ++j) {
    uD[j] = 0.0;
    if (P.kind != 0 || vel2free[l2g[cell * nvmax + j]] >= 0) continue;
    any = true;
  }
  if (any) {
    for (int lv = 0; lv < g.nv; ++lv) {
      double u[3];
      u_exact(g.X[lv], u);
      for (int c = 0; c < 3; ++c)
        if (vel2free[l2g[cell * nvmax + L.vdof(lv, c)]] < 0) uD[L.vdof(lv, c)] = u[c];
    }
    for (int le = 0; le < g.ne; ++le) {
      const double *Pa = g.X[g.ev[le][0]], *Pb = g.X[g.ev[le][1]];
      for (int j = 0; j < K - 1; ++j) {
        double x[3], u[3];
        for (int d = 0; d < 3; ++d) x[d] = Pa[d] + c_lobx[j + 1] * (Pb[d] - Pa[d]);
        u_exact(x, u);
        for (int c = 0; c < 3; ++c)
          if (vel2free[l2g[cell * nvmax + L.edof(le, j, c)]] < 0) uD[L.edof(le, j, c)] = u[c];
      }
    }
    for (int f = 0; f < g.nf; ++f) {
      if (vel2free[l2g[cell * nvmax + L.fdof(f, 0, 0)]] >= 0) continue;
      FaceG F;
      face_geo(g, f, F);
      const double *tau[3] = {F.n, F.t1, F.t2};
      double mom[3][d2(2)];
      for (int t = 0; t < 3; ++t) for (int a = 0; a < nm; ++a) mom[t][a] = 0.0;
      const int npf = face_npts(g, f, K + 2);
      for (int q = 0; q < npf; ++q) {
        double x[3], w, u[3], m2[d2(4)];
        face_point(g, f, K + 2, q, x, &w);
        u_exact(x, u);
        double xi = 0, eta = 0;
        for (int d = 0; d < 3; ++d) { xi += (x[d] - F.xc[d]) * F.t1[d]; eta += (x[d] - F.xc[d]) * F.t2[d]; }
        mono2(xi, eta, F.h, K - 2, m2, nullptr);
        for (int t = 0; t < 3; ++t) {
          const double ut = u[0] * tau[t][0] + u[1] * tau[t][1] + u[2] * tau[t][2];
          for (int a = 0; a < nm; ++a) mom[t][a] += w * ut * m2[a];
        }
      }
      for (int t = 0; t < 3; ++t)
        for (int a = 0; a < nm; ++a) uD[L.fdof(f, t, a)] = mom[t][a] / F.area;
    }
  }
  const double *A = elA + cell * (int64_t)nvmax * nvmax;
  const double *B = elB + cell * (int64_t)D1 * nvmax;
  for (int i = 0; i < nv; ++i) {
    double v = 0.0;
    for (int r = 0; r < S3; ++r) v += P0[(int64_t)r * nv + i] * Fm[r];
    if (any)
      for (int j = 0; j < nv; ++j) v -= A[(int64_t)i * nv + j] * uD[j];
    y[i] = v;
  }
  for (int a = 0; a < D1; ++a) {
    double v = 0.0;
    if (any)
      for (int j = 0; j < nv; ++j) v -= B[(int64_t)a * nv + j] * uD[j];
    y[nvmax + a] = v;
  }
}

void build_rhs_device(vb_ctx *c, const vb_problem *p, double *rhs) {
  VB_REQUIRE(c->d_P0.p, VB_ESTATE, "vb_build_rhs needs device element operators (vb_setup)");
  VB_REQUIRE(p->kind == 0 || p->kind == 1, VB_EINVAL, "unknown problem kind");
  ProbDev P{};
  P.kind = p->kind;
  if (p->kind == 1) {
    VB_REQUIRE(p->n_sinkers >= 0 && p->n_sinkers <= 16 && p->centres, VB_EINVAL, "sinker centres");
    P.ns = p->n_sinkers; P.delta = p->delta; P.omega = p->omega; P.beta = p->beta;
    for (int i = 0; i < P.ns; ++i) for (int q = 0; q < 3; ++q) P.cen[i][q] = p->centres[3 * i + q];
  }
  cudaStream_t s = c->stream;
  const int blocks = (c->nKl + 127) / 128;
  DBuf<double> uD;
  uD.alloc(std::max<int64_t>((int64_t)c->nKl * c->nv_max, 1));
#define VB_RHS_K(KK)                                                                                        \
  rhs_element_kernel<KK><<<blocks, 128, 0, s>>>(c->d_topo.p, c->d_xyz.p, c->d_nu.p, c->d_cell_l2g.p,       \
                                                c->d_vel2free.p, c->d_elA.p, c->d_elB.p, c->d_P0.p, c->nKl, \
                                                c->nv_max, P, c->w_elt.p, uD.p)
  if (c->k == 2) VB_RHS_K(2);
  else if (c->k == 3) VB_RHS_K(3);
  else VB_RHS_K(4);
#undef VB_RHS_K
  VB_STAGE();
  element_gather(c, c->w_elt.p, rhs);   // owned layout (multi-rank: interface sums exchanged)
  VB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace vb
