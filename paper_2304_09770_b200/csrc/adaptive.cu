// Adaptive coarse space (§6).
//
// For every macro face F shared by subdomains i, j (after the first interface pass, with S_T and
// the deluxe side blocks available):
//   1. S~_F^(m) = Schur complement of S_T^(m) onto F's dual coordinates, eliminating every other
//      coordinate of Gamma_m (F' = Gamma_m minus F_Delta): a permuted copy of S_T and a
//      batched partial LDL^T (DMMA trailing updates, dense.cu);
//   2. parallel sums A = S~i : S~j and B = S_F^i : S_F^j, X:Y = X (X+Y)^-1 Y symmetrised;
//   3. generalized eigenproblem A psi = lambda B psi reduced with B = L D L^T to the
//      standard problem C = D^-1/2 L^-1 A L^-T D^-1/2, solved by a batched parallel (round-robin)
//      Jacobi eigensolver, one CTA per face (K10);
//   4. eigenvectors with lambda < 1/tau give new primal rows (B psi)^T N_F^T on F (in
//      original coordinates), appended to C_F; the caller redoes A3-A5 with them.
#include <algorithm>
#include <cmath>
#include "dense.cuh"
#include "setup.h"
#include "exchange.h"

namespace vb {

struct PermDesc {          // one (face, side): gather a permuted copy of the side's S_T
  const double *ST;        // S_T of the subdomain (column-major, leading dimension ld)
  int ld, nG, offD, nd;
  double *out;             // nG x nG column-major: [other coordinates | F's dual coordinates]
};

__global__ void permute_gather_kernel(const PermDesc *__restrict__ pd) {
  const PermDesc P = pd[blockIdx.y];
  const int n = P.nG, m = n - P.nd;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < (int64_t)n * n;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = idx % n, j = idx / n;
    const int pi = i < m ? (i < P.offD ? i : i + P.nd) : P.offD + (i - m);
    const int pj = j < m ? (j < P.offD ? j : j + P.nd) : P.offD + (j - m);
    P.out[idx] = P.ST[pi + (int64_t)pj * P.ld];
  }
}

struct CopyDesc {          // dst (n x n, ld n, full) <- symmetric matrix given by its lower triangle
  const double *src;
  int ld, n;
  double *dst;
};

__global__ void copy_sym_lower_kernel(const CopyDesc *__restrict__ cd) {
  const CopyDesc C = cd[blockIdx.y];
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < C.n * C.n; idx += gridDim.x * blockDim.x) {
    const int i = idx % C.n, j = idx / C.n;
    C.dst[idx] = i >= j ? C.src[i + (int64_t)j * C.ld] : C.src[j + (int64_t)i * C.ld];
  }
}

// elementwise on batches of n x n matrices at a common stride: op 0: out = a + b;
// op 1: out = (a + a^T)/2 (in place on a, out ignored)
__global__ void batch_elementwise_kernel(double *a, const double *b, double *out, int n, int64_t stride, int op) {
  double *A = a + blockIdx.y * stride;
  if (op == 0) {
    const double *B = b + blockIdx.y * stride;
    double *O = out + blockIdx.y * stride;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) O[idx] = A[idx] + B[idx];
  } else {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
      const int i = idx % n, j = idx / n;
      if (i > j) {
        const double v = 0.5 * (A[i + (int64_t)j * n] + A[j + (int64_t)i * n]);
        A[i + (int64_t)j * n] = v;
        A[j + (int64_t)i * n] = v;
      }
    }
  }
}

// d[i] = 1 / A_ii (mode 0) or 1 / sqrt(A_ii) (mode 1), batched at a common stride
__global__ void batch_diag_kernel(const double *A, int n, int64_t stride, double *d, int mode) {
  const double *M = A + blockIdx.y * stride;
  double *o = d + blockIdx.y * (int64_t)n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double v = M[i + (int64_t)i * n];
    o[i] = mode == 0 ? 1.0 / v : 1.0 / sqrt(v);
  }
}

// C_ij *= dh_i dh_j, then symmetrise
__global__ void batch_scale_sym_kernel(double *C, const double *dh, int n, int64_t stride) {
  double *M = C + blockIdx.y * stride;
  const double *d = dh + blockIdx.y * (int64_t)n;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    const int i = idx % n, j = idx / n;
    if (i >= j) {
      const double v = 0.5 * (M[i + (int64_t)j * n] + M[j + (int64_t)i * n]) * d[i] * d[j];
      M[i + (int64_t)j * n] = v;
      M[j + (int64_t)i * n] = v;
    }
  }
}

// ------------------------------------------------------------------ K10: parallel Jacobi
// Symmetric eigenproblem C v = lambda v for one n x n matrix per CTA (column-major, in global
// memory, overwritten). Round-robin (circle) ordering: each step applies m/2 disjoint rotations
// (m = n rounded up to even; pairs with the padding index are skipped), rows then columns, so one
// step is J^T C J for a block rotation J; V accumulates the rotations.  Threshold Jacobi: a rotation
// is skipped when |c_pq| <= 1e-15 sqrt(|c_pp c_qq|); the sweeps stop when a sweep rotates nothing.
constexpr int JAC_THREADS = 256;

__global__ void __launch_bounds__(JAC_THREADS) jacobi_eig_kernel(double *Call, double *Vall, double *lam, int n,
                                                                 int64_t stride, int max_sweeps) {
  double *A = Call + blockIdx.x * stride;
  double *V = Vall + blockIdx.x * stride;
  const int m = n + (n & 1);
  const int half = m / 2;
  __shared__ double cs[256], sn[256];
  __shared__ int P[256], Q[256];
  const int tid = threadIdx.x;
  for (int idx = tid; idx < n * n; idx += blockDim.x) V[idx] = (idx % n == idx / n) ? 1.0 : 0.0;
  __syncthreads();
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < m - 1; ++r) {
      for (int k = tid; k < half; k += blockDim.x) {
        int a, b;
        if (k == 0) { a = r; b = m - 1; }
        else { a = (r + k) % (m - 1); b = (r - k + m - 1) % (m - 1); }
        const int p = min(a, b), q = max(a, b);
        double c = 1.0, s = 0.0;
        if (q < n) {
          const double app = A[p + (int64_t)p * n], aqq = A[q + (int64_t)q * n], apq = A[p + (int64_t)q * n];
          if (fabs(apq) > 1e-300 && fabs(apq) > 1e-15 * sqrt(fabs(app * aqq))) {
            const double theta = (aqq - app) / (2.0 * apq);
            const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        P[k] = p; Q[k] = q < n ? q : p; cs[k] = c; sn[k] = s;
        rotated |= s != 0.0;
      }
      __syncthreads();
      // rows: C <- J^T C
      for (int idx = tid; idx < half * n; idx += blockDim.x) {
        const int k = idx / n, j = idx % n;
        const double s = sn[k];
        if (s == 0.0) continue;
        const double c = cs[k];
        const int p = P[k], q = Q[k];
        const double ap = A[p + (int64_t)j * n], aq = A[q + (int64_t)j * n];
        A[p + (int64_t)j * n] = c * ap - s * aq;
        A[q + (int64_t)j * n] = s * ap + c * aq;
      }
      __syncthreads();
      // columns: C <- C J, V <- V J
      for (int idx = tid; idx < half * n; idx += blockDim.x) {
        const int k = idx / n, i = idx % n;
        const double s = sn[k];
        if (s == 0.0) continue;
        const double c = cs[k];
        const int p = P[k], q = Q[k];
        const double ap = A[i + (int64_t)p * n], aq = A[i + (int64_t)q * n];
        A[i + (int64_t)p * n] = c * ap - s * aq;
        A[i + (int64_t)q * n] = s * ap + c * aq;
        const double vp = V[i + (int64_t)p * n], vq = V[i + (int64_t)q * n];
        V[i + (int64_t)p * n] = c * vp - s * vq;
        V[i + (int64_t)q * n] = s * vp + c * vq;
      }
      __syncthreads();
    }
    if (!__syncthreads_or(rotated)) break;
  }
  for (int i = tid; i < n; i += blockDim.x) lam[blockIdx.x * (int64_t)n + i] = A[i + (int64_t)i * n];
}

// new primal row of a selected eigenvector: z = L D^1/2 v (= B psi), row = N_F z (n entries)
struct RowDesc {
  const double *L;       // LDL^T of B (unit lower strictly below the diagonal, D on it), nd x nd
  const double *v;       // eigenvector (nd)
  const double *N;       // T_F, first nd columns = N_F (n x nd, column-major, ld n)
  int n, nd;
  double *row;           // out: n
};

__global__ void adaptive_row_kernel(const RowDesc *__restrict__ rd, int nd_max) {
  const RowDesc R = rd[blockIdx.x];
  extern __shared__ double sh[];
  double *w = sh, *z = sh + nd_max;
  for (int i = threadIdx.x; i < R.nd; i += blockDim.x) w[i] = sqrt(R.L[i + (int64_t)i * R.nd]) * R.v[i];
  __syncthreads();
  for (int i = threadIdx.x; i < R.nd; i += blockDim.x) {
    double v = w[i];
    for (int j = 0; j < i; ++j) v += R.L[i + (int64_t)j * R.nd] * w[j];
    z[i] = v;
  }
  __syncthreads();
  for (int a = threadIdx.x; a < R.n; a += blockDim.x) {
    double v = 0.0;
    for (int i = 0; i < R.nd; ++i) v += R.N[a + (int64_t)i * R.n] * z[i];
    R.row[a] = v;
  }
}

static void check_pivots(vb_ctx *c, int nmat, const char *what) {
  std::vector<int> info(nmat);
  VB_CUDA(cudaMemcpyAsync(info.data(), c->d_info.p, nmat * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  VB_CUDA(cudaStreamSynchronize(c->stream));
  for (int b = 0; b < nmat; ++b)
    if (info[b])
      throw Error{VB_ESINGULAR, std::string(what) + ": zero pivot at column " + std::to_string(info[b] - 1) +
                                    " of pencil " + std::to_string(b)};
}

template <class T>
static T *upload_desc(DBuf<T> &buf, const std::vector<T> &h, cudaStream_t s) {
  std::vector<T> copy(h);
  buf.upload(copy, s);
  return buf.p;
}

// G = V diag(f(lambda)), f = 1/lambda above rel_tol * max|lambda| of the matrix, else 0
__global__ void pinv_scale_kernel(const double *__restrict__ V, const double *__restrict__ lam, int n, int64_t stride,
                                  double rel_tol, double *G) {
  const double *L = lam + blockIdx.y * (int64_t)n;
  __shared__ double lmax;
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int i = 0; i < n; ++i) m = fmax(m, fabs(L[i]));
    lmax = m;
  }
  __syncthreads();
  const double *Vm = V + blockIdx.y * stride;
  double *Gm = G + blockIdx.y * stride;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < n * n; idx += gridDim.x * blockDim.x) {
    const double l = L[idx / n];
    Gm[idx] = l > rel_tol * lmax ? Vm[idx] / l : 0.0;
  }
}

// parallel sums with a pseudo-inverse, for pencils whose sum is singular: on faces between two
// floating subdomains S~i and S~j share the projected rigid modes as kernel, and X:Y is the limit
// X (X+Y)^+ Y (A:B = (A^-1 + B^-1)^-1 extended by continuity to semidefinite A, B)
static void parallel_sum_pinv_batched(vb_ctx *c, const double *X, const double *Y, double *out, int nb, int n) {
  cudaStream_t s = c->stream;
  const int64_t st = (int64_t)n * n;
  DBuf<double> S, V, G, lam, T1;
  S.alloc(nb * st); V.alloc(nb * st); G.alloc(nb * st); lam.alloc((int64_t)nb * n); T1.alloc(nb * st);
  const dim3 g(std::max(1, (int)std::min<int64_t>((st + 255) / 256, 64)), nb);
  batch_elementwise_kernel<<<g, 256, 0, s>>>((double *)X, Y, S.p, n, st, 0);
  batch_elementwise_kernel<<<g, 256, 0, s>>>(S.p, nullptr, nullptr, n, st, 1);
  VB_STAGE();
  jacobi_eig_kernel<<<nb, JAC_THREADS, 0, s>>>(S.p, V.p, lam.p, n, st, 60);
  VB_STAGE();
  pinv_scale_kernel<<<g, 256, 0, s>>>(V.p, lam.p, n, st, 1e-12, G.p);
  VB_STAGE();
  GemmPlan plan;
  int l0 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // S <- (X+Y)^+ = G V^T
    GemmProb p{};
    p.A = G.p + b * st; p.lda = n; p.B = V.p + b * st; p.ldb = n; p.transB = 1;
    p.C = S.p + b * st; p.ldc = n; p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0;
    plan.add(p);
  }
  int l1 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // T1 = (X+Y)^+ Y
    GemmProb p{};
    p.A = S.p + b * st; p.lda = n; p.B = Y + b * st; p.ldb = n; p.C = T1.p + b * st; p.ldc = n;
    p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0;
    plan.add(p);
  }
  int l2 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // out = X T1
    GemmProb p{};
    p.A = X + b * st; p.lda = n; p.B = T1.p + b * st; p.ldb = n; p.C = out + b * st; p.ldc = n;
    p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0;
    plan.add(p);
  }
  plan.upload(s);
  plan.run(l0, s);
  plan.run(l1, s);
  plan.run(l2, s);
  batch_elementwise_kernel<<<g, 256, 0, s>>>(out, nullptr, nullptr, n, st, 1);
  VB_STAGE();
  VB_CUDA(cudaStreamSynchronize(s));
}

// batched parallel sums out_b = X_b (X_b + Y_b)^-1 Y_b (symmetrised) for nb SPD-sum pencils of
// order n, X, Y, out at stride n*n
static void parallel_sum_batched(vb_ctx *c, const double *X, const double *Y, double *out, int nb, int n) {
  cudaStream_t s = c->stream;
  const int64_t st = (int64_t)n * n;
  DBuf<double> S, W, T1, d;
  S.alloc(nb * st); W.alloc(nb * st); T1.alloc(nb * st); d.alloc((int64_t)nb * n);
  const dim3 g(std::max(1, (int)std::min<int64_t>((st + 255) / 256, 64)), nb);
  batch_elementwise_kernel<<<g, 256, 0, s>>>((double *)X, Y, S.p, n, st, 0);
  VB_STAGE();
  std::vector<MatDesc> mats(nb);
  std::vector<TriDesc> td(nb);
  for (int b = 0; b < nb; ++b) {
    mats[b] = MatDesc{S.p + b * st, n, n, n};
    td[b] = TriDesc{S.p + b * st, n, W.p + b * st, n, n};
  }
  c->d_info.alloc(std::max<size_t>(c->d_info.n, nb + 1));
  c->d_info.zero(s);
  ldl_partial_batched(mats, c->d_info.p, s);
  check_pivots(c, nb, "adaptive parallel sum LDL^T (A6)");
  W.zero(s);
  tri_inverse_batched(td, s);
  batch_diag_kernel<<<dim3((n + 255) / 256, nb), 256, 0, s>>>(S.p, n, st, d.p, 0);
  VB_STAGE();
  GemmPlan plan;
  int l0 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // S <- (X+Y)^-1 = W^T D^-1 W (lower)
    GemmProb p{};
    p.A = W.p + b * st; p.lda = n; p.transA = 1; p.d = d.p + (int64_t)b * n; p.dstride = 1;
    p.B = W.p + b * st; p.ldb = n; p.C = S.p + b * st; p.ldc = n;
    p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0; p.lower = 1;
    plan.add(p);
  }
  int l1 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // T1 = (X+Y)^-1 Y
    GemmProb p{};
    p.A = S.p + b * st; p.lda = n; p.B = Y + b * st; p.ldb = n; p.C = T1.p + b * st; p.ldc = n;
    p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0;
    plan.add(p);
  }
  int l2 = plan.begin_launch();
  for (int b = 0; b < nb; ++b) {            // out = X T1
    GemmProb p{};
    p.A = X + b * st; p.lda = n; p.B = T1.p + b * st; p.ldb = n; p.C = out + b * st; p.ldc = n;
    p.M = p.N = p.K = n; p.alpha = 1.0; p.beta = 0.0;
    plan.add(p);
  }
  plan.upload(s);
  plan.run(l0, s);
  for (int b = 0; b < nb; ++b) mats[b] = MatDesc{S.p + b * st, n, n, 0};
  symmetrize_lower_batched(mats, s);
  plan.run(l1, s);
  plan.run(l2, s);
  batch_elementwise_kernel<<<g, 256, 0, s>>>(out, nullptr, nullptr, n, st, 1);
  VB_STAGE();
  VB_CUDA(cudaStreamSynchronize(s));
}

void adaptive_enrich(vb_ctx *c, double tau, const DBuf<double> &sidebuf) {
  cudaStream_t s = c->stream;
  // faces with a dual part (both sharers, local or not), grouped by their dual size
  std::vector<int> faces;
  std::vector<char> isface(c->h_ent.size(), 0);
  for (size_t e = 0; e < c->h_ent.size(); ++e) {
    const EntDev &E = c->h_ent[e];
    if (E.kind == 2 && E.nd > 0 && E.nsh == 2) { faces.push_back(e); isface[e] = 1; }
  }
  c->extra_rows.assign(c->ents.size(), std::vector<double>());
  c->n_adaptive = 0;
  c->adaptive_margin = INFINITY;
  int64_t owned_selected = 0;
  // ---------------- 1. S~_F^(m) of every LOCAL face slot: permuted S_T copies + partial LDL^T
  std::vector<int64_t> st_off(c->h_slot.size(), -1);
  int64_t st_len = 0;
  std::vector<int> fslots;
  for (int e : faces) {
    const EntDev &E = c->h_ent[e];
    for (int t = 0; t < E.nsides; ++t) {
      st_off[E.side_begin + t] = st_len;
      st_len += (int64_t)E.nd * E.nd;
      fslots.push_back(E.side_begin + t);
    }
  }
  DBuf<double> Stl;
  Stl.alloc(std::max<int64_t>(st_len, 1));
  {
    const int64_t budget = (int64_t)3 << 30;   // bytes of permuted copies per chunk
    size_t a = 0;
    while (a < fslots.size()) {
      std::vector<int64_t> off;
      int64_t tot = 0;
      size_t b = a;
      while (b < fslots.size()) {
        const SubDev &S = c->h_sub[c->h_slot[fslots[b]].sub];
        const int64_t sz = (int64_t)S.nG * S.nG;
        if (b > a && (tot + sz) * 8 > budget) break;
        off.push_back(tot);
        tot += sz;
        ++b;
      }
      DBuf<double> buf;
      buf.alloc(tot);
      std::vector<PermDesc> pd;
      std::vector<MatDesc> md;
      std::vector<CopyDesc> cd;
      for (size_t q = a; q < b; ++q) {
        const SlotDev &sl = c->h_slot[fslots[q]];
        const SubDev &S = c->h_sub[sl.sub];
        double *o = buf.p + off[q - a];
        pd.push_back(PermDesc{c->d_K.p + S.off_K + (int64_t)S.nD * (S.ldk + 1), S.ldk, S.nG, sl.offD, sl.nd, o});
        md.push_back(MatDesc{o, S.nG, S.nG, S.nG - sl.nd});
        cd.push_back(CopyDesc{o + (int64_t)(S.nG - sl.nd) * (S.nG + 1), S.nG, sl.nd, Stl.p + st_off[fslots[q]]});
      }
      DBuf<PermDesc> dpd;
      upload_desc(dpd, pd, s);
      permute_gather_kernel<<<dim3(64, pd.size()), 256, 0, s>>>(dpd.p);
      VB_STAGE();
      c->d_info.alloc(std::max<size_t>(c->d_info.n, md.size() + 1));
      c->d_info.zero(s);
      ldl_partial_batched(md, c->d_info.p, s);
      check_pivots(c, md.size(), "adaptive face Schur complement LDL^T (A6)");
      DBuf<CopyDesc> dcd;
      upload_desc(dcd, cd, s);
      copy_sym_lower_kernel<<<dim3(16, cd.size()), 256, 0, s>>>(dcd.p);
      VB_STAGE();
      VB_CUDA(cudaStreamSynchronize(s));
      a = b;
    }
  }
  // ---------------- faces shared with another rank: the other side's S~ and S_F blocks (C1)
  auto Lf = [&](int e) { return isface[e] ? (int64_t)c->h_ent[e].nd * c->h_ent[e].nd : (int64_t)0; };
  SlotExchange XT, XF;
  build_slot_exchange(c, XT, Lf, [&](int sl, std::vector<int64_t> &out) {
    const int e = c->h_slot[sl].ent;
    for (int64_t q = 0; q < Lf(e); ++q) out.push_back(st_off[sl] + q);
  });
  build_slot_exchange(c, XF, Lf, [&](int sl, std::vector<int64_t> &out) {
    const int e = c->h_slot[sl].ent;
    for (int64_t q = 0; q < Lf(e); ++q) out.push_back(c->h_slot[sl].off_side + q);
  });
  DBuf<double> RT, RF;
  RT.alloc(std::max<int64_t>(XT.recv_len, 1));
  RF.alloc(std::max<int64_t>(XF.recv_len, 1));
  run_slot_exchange(c, XT, Stl.p, RT.p);
  run_slot_exchange(c, XF, sidebuf.p, RF.p);
  VB_CUDA(cudaStreamSynchronize(s));
  std::sort(faces.begin(), faces.end(), [&](int a, int b) {
    return c->h_ent[a].nd != c->h_ent[b].nd ? c->h_ent[a].nd < c->h_ent[b].nd : a < b;
  });
  for (size_t f0 = 0; f0 < faces.size();) {
    const int nd = c->h_ent[faces[f0]].nd;
    size_t f1 = f0;
    while (f1 < faces.size() && c->h_ent[faces[f1]].nd == nd) ++f1;
    const int nf = f1 - f0;
    const int64_t st = (int64_t)nd * nd;
    VB_REQUIRE(nd <= 510, VB_EINVAL, "adaptive face pencil larger than the Jacobi kernel supports (nd <= 510)");
    // ---------------- 2. parallel sums: A = S~i : S~j, B = S_F^i : S_F^j (side 0 : side 1)
    DBuf<double> X, Y, AB;
    X.alloc(2 * nf * st); Y.alloc(2 * nf * st); AB.alloc(2 * nf * st);
    for (int q = 0; q < nf; ++q) {
      const int e = faces[f0 + q];
      const Entity &E = c->ents[e];
      int li = 0;
      for (int k = 0; k < 2; ++k) {
        const double *st_src, *sf_src;
        if (c->sub_lid[E.sharers[k]] >= 0) {
          const int sl = c->h_ent[e].side_begin + li++;
          st_src = Stl.p + st_off[sl];
          sf_src = sidebuf.p + c->h_slot[sl].off_side;
        } else {
          st_src = RT.p + XT.recv_off[XT.ent_ptr[e] + k];
          sf_src = RF.p + XF.recv_off[XF.ent_ptr[e] + k];
        }
        double *dA = (k == 0 ? X.p : Y.p) + q * st;
        double *dB = (k == 0 ? X.p : Y.p) + (nf + q) * st;
        VB_CUDA(cudaMemcpyAsync(dA, st_src, st * 8, cudaMemcpyDeviceToDevice, s));
        VB_CUDA(cudaMemcpyAsync(dB, sf_src, st * 8, cudaMemcpyDeviceToDevice, s));
      }
    }
    parallel_sum_pinv_batched(c, X.p, Y.p, AB.p, nf, nd);                    // A = S~i : S~j
    parallel_sum_batched(c, X.p + nf * st, Y.p + nf * st, AB.p + nf * st, nf, nd);   // B = S_F^i : S_F^j
    X.release(); Y.release();
    // ---------------- 3. reduce to C = D^-1/2 L^-1 A L^-T D^-1/2 (B = L D L^T), Jacobi
    DBuf<double> LB, W, G1, C, V, dh, lam;
    LB.alloc(nf * st); W.alloc(nf * st); G1.alloc(nf * st); C.alloc(nf * st); V.alloc(nf * st);
    dh.alloc((int64_t)nf * nd); lam.alloc((int64_t)nf * nd);
    VB_CUDA(cudaMemcpyAsync(LB.p, AB.p + nf * st, nf * st * 8, cudaMemcpyDeviceToDevice, s));
    {
      std::vector<MatDesc> md(nf);
      std::vector<TriDesc> td(nf);
      for (int q = 0; q < nf; ++q) {
        md[q] = MatDesc{LB.p + q * st, nd, nd, nd};
        td[q] = TriDesc{LB.p + q * st, nd, W.p + q * st, nd, nd};
      }
      c->d_info.alloc(std::max<size_t>(c->d_info.n, nf + 1));
      c->d_info.zero(s);
      ldl_partial_batched(md, c->d_info.p, s);
      check_pivots(c, nf, "adaptive pencil B LDL^T (A6)");
      W.zero(s);
      tri_inverse_batched(td, s);
      batch_diag_kernel<<<dim3((nd + 255) / 256, nf), 256, 0, s>>>(LB.p, nd, st, dh.p, 1);
      VB_STAGE();
      GemmPlan plan;
      int l0 = plan.begin_launch();
      for (int q = 0; q < nf; ++q) {          // G1 = A W^T
        GemmProb p{};
        p.A = AB.p + q * st; p.lda = nd; p.B = W.p + q * st; p.ldb = nd; p.transB = 1;
        p.C = G1.p + q * st; p.ldc = nd; p.M = p.N = p.K = nd; p.alpha = 1.0; p.beta = 0.0;
        plan.add(p);
      }
      int l1 = plan.begin_launch();
      for (int q = 0; q < nf; ++q) {          // C = W G1
        GemmProb p{};
        p.A = W.p + q * st; p.lda = nd; p.B = G1.p + q * st; p.ldb = nd;
        p.C = C.p + q * st; p.ldc = nd; p.M = p.N = p.K = nd; p.alpha = 1.0; p.beta = 0.0;
        plan.add(p);
      }
      plan.upload(s);
      plan.run(l0, s);
      plan.run(l1, s);
      batch_scale_sym_kernel<<<dim3(16, nf), 256, 0, s>>>(C.p, dh.p, nd, st);
      VB_STAGE();
      jacobi_eig_kernel<<<nf, JAC_THREADS, 0, s>>>(C.p, V.p, lam.p, nd, st, 60);
      VB_STAGE();
    }
    // ---------------- 4. selection lambda < 1/tau and the new rows (B psi)^T N_F^T
    std::vector<double> hl;
    lam.download(hl, s);
    VB_CUDA(cudaStreamSynchronize(s));
    std::vector<RowDesc> rd;
    std::vector<std::pair<int, int>> who;   // (entity, count)
    int64_t nrow_tot = 0;
    const double thr = 1.0 / tau;
    if (const char *dump = getenv("VB_ADAPTIVE_DUMP")) {   // debugging aid: per-face spectra
      FILE *fp = fopen(dump, "a");
      if (fp) {
        for (int q = 0; q < nf; ++q) {
          fprintf(fp, "%d %d", c->ents[faces[f0 + q]].gid, nd);
          for (int i = 0; i < nd; ++i) fprintf(fp, " %.17g", hl[(int64_t)q * nd + i]);
          fprintf(fp, "\n");
        }
        fclose(fp);
      }
    }
    for (int q = 0; q < nf; ++q) {
      const EntDev &E = c->h_ent[faces[f0 + q]];
      int cnt = 0;
      for (int i = 0; i < nd; ++i) {
        const double l = hl[(int64_t)q * nd + i];
        c->adaptive_margin = std::min(c->adaptive_margin, fabs(l - thr));
        if (l < thr) {
          rd.push_back(RowDesc{LB.p + q * st, V.p + q * st + (int64_t)i * nd, c->d_T.p + E.off_T, E.n, nd, nullptr});
          ++cnt;
        }
      }
      if (cnt) who.push_back({faces[f0 + q], cnt});
      if (c->sub_rank[c->ents[faces[f0 + q]].sharers[0]] == c->rank) owned_selected += cnt;
      nrow_tot += (int64_t)cnt * E.n;
    }
    if (!rd.empty()) {
      DBuf<double> rows;
      rows.alloc(nrow_tot);
      int64_t o = 0;
      for (auto &r : rd) { r.row = rows.p + o; o += r.n; }
      DBuf<RowDesc> drd;
      upload_desc(drd, rd, s);
      adaptive_row_kernel<<<rd.size(), 128, 2 * nd * sizeof(double), s>>>(drd.p, nd);
      VB_STAGE();
      std::vector<double> hr;
      rows.download(hr, s);
      VB_CUDA(cudaStreamSynchronize(s));
      o = 0;
      for (auto &w : who) {
        const int n = c->h_ent[w.first].n;
        c->extra_rows[w.first].assign(hr.begin() + o, hr.begin() + o + (int64_t)w.second * n);
        o += (int64_t)w.second * n;
      }
    }
    f0 = f1;
  }
  // global count (faces owned here, summed over ranks) and global margin
  c->n_adaptive = owned_selected;
  if (c->nranks > 1) {
    DBuf<double> v, g;
    std::vector<double> hv{(double)owned_selected, c->adaptive_margin};
    v.upload(hv, s);
    g.alloc(2 * c->nranks);
    c->comm->allgather(v.p, g.p, 2, s);
    std::vector<double> hg;
    g.download(hg, s);
    VB_CUDA(cudaStreamSynchronize(s));
    c->n_adaptive = 0;
    for (int r = 0; r < c->nranks; ++r) {
      c->n_adaptive += (int)hg[2 * r];
      c->adaptive_margin = std::min(c->adaptive_margin, hg[2 * r + 1]);
    }
  }
}

}  // namespace vb
