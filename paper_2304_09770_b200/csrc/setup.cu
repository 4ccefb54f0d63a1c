// Host-side structural setup of a vb_ctx: edges, DOF numbering, local cell
// topology, subdomain/interface classification and constraint rows.
// This is index bookkeeping and O(#interface DOFs) geometry; every O(n^2)/O(n^3) numeric step
// of the method runs on the device (vem.cu, dense.cu, factor.cu, solve.cu).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <map>
#include <unordered_map>
#include <numeric>
#include <chrono>
#include "internal.h"
#include "setup.h"

namespace vb {

// ------------------------------------------------------------------ quadrature nodes (host)
static double legendre(int n, double x, double *dp) {
  double p0 = 1, p1 = x;
  if (n == 0) { *dp = 0; return 1; }
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1; p1 = p2;
  }
  *dp = n * (x * p1 - p0) / (x * x - 1);
  return p1;
}

void gauss_legendre01(int n, double *x, double *w) {
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p = legendre(n, z, &dp);
      double dz = p / dp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    legendre(n, z, &dp);
    x[n - 1 - i] = 0.5 * (z + 1);
    w[n - 1 - i] = 1.0 / ((1 - z * z) * dp * dp);   // 2/((1-z^2)P'^2) scaled by 1/2
  }
}

void gauss_lobatto01(int npts, double *x, double *w) {
  int m = npts - 1;
  x[0] = 0; x[m] = 1;
  // interior nodes: roots of P'_m, found by Newton on P'_m using the GL roots of degree m-1 as guess
  for (int i = 1; i < m; ++i) {
    double z = -cos(M_PI * i / m);
    for (int it = 0; it < 200; ++it) {
      // P'_m and P''_m via Legendre ODE: (1-z^2)P'' = 2z P' - m(m+1)P
      double dp, p = legendre(m, z, &dp);
      double d2 = (2 * z * dp - m * (m + 1) * p) / (1 - z * z);
      double dz = dp / d2;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    x[i] = 0.5 * (z + 1);
  }
  for (int i = 0; i <= m; ++i) {
    double z = 2 * x[i] - 1, dp;
    double p = legendre(m, z, &dp);
    w[i] = 1.0 / (m * (m + 1) * p * p);   // (2/(m(m+1)P^2)) / 2
  }
}

static inline int dim2(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) / 2; }
static inline int dim3(int n) { return n < 0 ? 0 : (n + 1) * (n + 2) * (n + 3) / 6; }

static double wall_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
// VB_SETUP_TIMES=2: fine timers of the host setup passes
static void fine_time(const char *what, double &t) {
  static const bool on = getenv("VB_SETUP_TIMES") && atoi(getenv("VB_SETUP_TIMES")) >= 2;
  if (!on) return;
  const double now = wall_s();
  fprintf(stderr, "[vb setup]   %-30s %.3f s\n", what, now - t);
  t = now;
}

// ------------------------------------------------------------------ topology and numbering
void build_topology(vb_ctx *c, const vb_mesh *m) {
  int k = c->k;
  double tf = wall_s();
  c->nV = m->n_vertices; c->nF = m->n_faces; c->nK = m->n_cells;
  c->xyz.assign(m->xyz, m->xyz + 3 * c->nV);
  c->face_ptr.assign(m->face_ptr, m->face_ptr + c->nF + 1);
  c->face_vtx.assign(m->face_vtx, m->face_vtx + c->face_ptr[c->nF]);
  c->cell_ptr.assign(m->cell_ptr, m->cell_ptr + c->nK + 1);
  c->cell_face.assign(m->cell_face, m->cell_face + c->cell_ptr[c->nK]);
  c->cell_sign.assign(m->cell_face_sign, m->cell_face_sign + c->cell_ptr[c->nK]);
  c->face_bnd.assign(m->face_on_dirichlet, m->face_on_dirichlet + c->nF);
  // edges: unique (min,max) pairs of loop edges, lexicographic
  std::vector<int64_t> keys;
  keys.reserve(c->face_vtx.size());
  int64_t nV = c->nV;
  for (int64_t f = 0; f < c->nF; ++f) {
    int64_t s = c->face_ptr[f], e = c->face_ptr[f + 1];
    VB_REQUIRE(e - s >= 3 && e - s <= MAXL, VB_EINVAL, "face " + std::to_string(f) + " has an unsupported loop length");
    for (int64_t i = s; i < e; ++i) {
      int64_t a = c->face_vtx[i], b = c->face_vtx[i + 1 < e ? i + 1 : s];
      keys.push_back(std::min(a, b) * nV + std::max(a, b));
    }
  }
  std::sort(keys.begin(), keys.end());
  keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  c->nE = keys.size();
  fine_time("edges", tf);
  c->edges.resize(2 * c->nE);
  for (int64_t i = 0; i < c->nE; ++i) { c->edges[2 * i] = keys[i] / nV; c->edges[2 * i + 1] = keys[i] % nV; }
  // edges grouped by their smaller vertex (keys are sorted by (min, max)): an edge id is a search
  // among the few edges of one vertex instead of over all keys
  std::vector<int64_t> eptr(nV + 1, 0);
  for (int64_t i = 0; i < c->nE; ++i) ++eptr[c->edges[2 * i] + 1];
  for (int64_t v = 0; v < nV; ++v) eptr[v + 1] += eptr[v];
  auto edge_id = [&](int64_t a, int64_t b) {
    const int64_t lo = std::min(a, b), hi = std::max(a, b);
    int64_t i = eptr[lo];
    while (i < eptr[lo + 1] && c->edges[2 * i + 1] < hi) ++i;
    return i;
  };
  // numbering (identical convention to DESIGN.md §Layout)
  c->nm = dim2(k - 2);
  c->n4 = 3 * dim3(k - 3) - dim3(k - 4);
  c->n5 = dim3(k - 1) - 1;
  c->np = dim3(k - 1);
  c->oE = 3 * c->nV;
  c->oF = c->oE + 3 * (k - 1) * c->nE;
  c->oC = c->oF + 3 * (int64_t)c->nm * c->nF;
  c->nvel = c->oC + c->nK * (c->n4 + c->n5);
  c->npres = c->nK * c->np;
  // boundary DOFs: face_bnd 1 = Dirichlet (removed, lifted); 2 = Neumann (natural
  // condition): the DOFs of its closure stay free unless they also lie on a Dirichlet face, and are
  // marked so the subdomain interface includes them (DESIGN A35)
  std::vector<char> isb(c->nvel, 0);
  c->vel_on_neu.assign(c->nvel, 0);
  c->neumann = false;
  for (int64_t f = 0; f < c->nF; ++f) {
    if (c->face_bnd[f] != 2) continue;
    c->neumann = true;
    int64_t s = c->face_ptr[f], e = c->face_ptr[f + 1];
    for (int64_t i = s; i < e; ++i) {
      int64_t a = c->face_vtx[i], b = c->face_vtx[i + 1 < e ? i + 1 : s];
      for (int q = 0; q < 3; ++q) c->vel_on_neu[3 * a + q] = 1;
      int64_t ed = edge_id(a, b);
      for (int q = 0; q < 3 * (k - 1); ++q) c->vel_on_neu[c->oE + 3 * (k - 1) * ed + q] = 1;
    }
    for (int q = 0; q < 3 * c->nm; ++q) c->vel_on_neu[c->oF + 3 * c->nm * f + q] = 1;
  }
  for (int64_t f = 0; f < c->nF; ++f) {
    VB_REQUIRE(c->face_bnd[f] <= 2, VB_EINVAL, "face " + std::to_string(f) + ": face_on_dirichlet must be 0, 1 or 2");
    if (c->face_bnd[f] != 1) continue;
    int64_t s = c->face_ptr[f], e = c->face_ptr[f + 1];
    for (int64_t i = s; i < e; ++i) {
      int64_t a = c->face_vtx[i], b = c->face_vtx[i + 1 < e ? i + 1 : s];
      for (int q = 0; q < 3; ++q) isb[3 * a + q] = 1;
      int64_t ed = edge_id(a, b);
      for (int q = 0; q < 3 * (k - 1); ++q) isb[c->oE + 3 * (k - 1) * ed + q] = 1;
    }
    for (int q = 0; q < 3 * c->nm; ++q) isb[c->oF + 3 * c->nm * f + q] = 1;
  }
  c->vel2free.assign(c->nvel, -1);
  c->free2vel.clear();
  for (int64_t g = 0; g < c->nvel; ++g)
    if (!isb[g]) { c->vel2free[g] = c->free2vel.size(); c->free2vel.push_back(g); }
  c->n_free_vel = c->free2vel.size();
  fine_time("numbering", tf);
  // per-cell local topology (vertices / edges / faces in increasing global id)
  c->topo_stride = TOPO_STRIDE;
  c->cell_topo.assign((size_t)c->nK * TOPO_STRIDE, 0);
  c->cell_nv.resize(c->nK);
  c->cell_l2g_ptr.assign(c->nK + 1, 0);
  c->cell_l2g.clear();
  c->nv_max = 0;
  // pass 1 (threads over cells): sorted faces, vertices and edges of each cell, its packed topology
  // and DOF count; the global face / edge ids are kept for pass 2
  std::vector<int64_t> cface((size_t)c->nK * MAXF), cedge((size_t)c->nK * MAXE);
  std::vector<int> nvmax_part(64, 0);
  std::atomic<int> chunk_id{0};
  parallel_for(c->nK, [&](int64_t K0, int64_t K1) {
    const int my = chunk_id++;
    int nvm = 0;
    std::pair<int64_t, int> fl[MAXF];
    int64_t vs[MAXF * MAXL], es[MAXF * MAXL];
    for (int64_t K = K0; K < K1; ++K) {
      int64_t s = c->cell_ptr[K], e = c->cell_ptr[K + 1];
      int nf = e - s;
      VB_REQUIRE(nf >= 4 && nf <= MAXF, VB_EINVAL, "cell " + std::to_string(K) + " has an unsupported face count");
      for (int64_t j = s; j < e; ++j) fl[j - s] = {c->cell_face[j], (int)c->cell_sign[j]};
      std::sort(fl, fl + nf);
      int nvs = 0, nes = 0;
      for (int f = 0; f < nf; ++f) {
        int64_t a0 = c->face_ptr[fl[f].first], a1 = c->face_ptr[fl[f].first + 1];
        for (int64_t i = a0; i < a1; ++i) {
          vs[nvs++] = c->face_vtx[i];
          es[nes++] = edge_id(c->face_vtx[i], c->face_vtx[i + 1 < a1 ? i + 1 : a0]);
        }
      }
      std::sort(vs, vs + nvs); nvs = std::unique(vs, vs + nvs) - vs;
      std::sort(es, es + nes); nes = std::unique(es, es + nes) - es;
      VB_REQUIRE(nvs <= MAXV && nes <= MAXE, VB_EINVAL,
                 "cell " + std::to_string(K) + " exceeds the supported vertex/edge count");
      int ntri = 0;
      for (int f = 0; f < nf; ++f) ntri += (int)(c->face_ptr[fl[f].first + 1] - c->face_ptr[fl[f].first]) - 2;
      VB_REQUIRE(ntri <= MAXT, VB_EINVAL, "cell " + std::to_string(K) + " exceeds the supported fan-triangle count");
      int *T = &c->cell_topo[(size_t)K * TOPO_STRIDE];
      T[0] = nvs; T[1] = nes; T[2] = nf;
      for (int i = 0; i < nvs; ++i) T[TOPO_V + i] = (int)vs[i];
      auto lv = [&](int64_t g) { return (int)(std::lower_bound(vs, vs + nvs, g) - vs); };
      for (int i = 0; i < nes; ++i) {
        T[TOPO_E + 2 * i] = lv(c->edges[2 * es[i]]);
        T[TOPO_E + 2 * i + 1] = lv(c->edges[2 * es[i] + 1]);
      }
      for (int f = 0; f < nf; ++f) {
        int *F = T + TOPO_F + f * FACE_STRIDE;
        int64_t gf = fl[f].first, a0 = c->face_ptr[gf], a1 = c->face_ptr[gf + 1];
        F[0] = fl[f].second; F[1] = a1 - a0;
        for (int64_t i = a0; i < a1; ++i) {
          int64_t a = c->face_vtx[i], b = c->face_vtx[i + 1 < a1 ? i + 1 : a0];
          int q = i - a0;
          F[2 + q] = lv(a);
          F[2 + MAXL + q] = (int)(std::lower_bound(es, es + nes, edge_id(a, b)) - es);
          F[2 + 2 * MAXL + q] = a < b ? 1 : 0;
        }
        cface[(size_t)K * MAXF + f] = gf;
      }
      for (int i = 0; i < nes; ++i) cedge[(size_t)K * MAXE + i] = es[i];
      const int nv = 3 * nvs + 3 * (k - 1) * nes + 3 * c->nm * nf + c->n4 + c->n5;
      c->cell_nv[K] = nv;
      nvm = std::max(nvm, nv);
    }
    nvmax_part[my] = nvm;
  });
  for (int v : nvmax_part) c->nv_max = std::max(c->nv_max, v);
  fine_time("cell topology", tf);
  for (int64_t K = 0; K < c->nK; ++K) c->cell_l2g_ptr[K + 1] = c->cell_l2g_ptr[K] + c->cell_nv[K];
  // pass 2: local -> global velocity map (vertices, edges, faces, cell), in increasing global id
  c->cell_l2g.resize(c->cell_l2g_ptr[c->nK]);
  parallel_for(c->nK, [&](int64_t K0, int64_t K1) {
    for (int64_t K = K0; K < K1; ++K) {
      const int *T = &c->cell_topo[(size_t)K * TOPO_STRIDE];
      int64_t *o = c->cell_l2g.data() + c->cell_l2g_ptr[K];
      for (int i = 0; i < T[0]; ++i) for (int q = 0; q < 3; ++q) *o++ = 3 * (int64_t)T[TOPO_V + i] + q;
      for (int i = 0; i < T[1]; ++i)
        for (int q = 0; q < 3 * (k - 1); ++q) *o++ = c->oE + 3 * (k - 1) * cedge[(size_t)K * MAXE + i] + q;
      for (int f = 0; f < T[2]; ++f)
        for (int q = 0; q < 3 * c->nm; ++q) *o++ = c->oF + 3 * c->nm * cface[(size_t)K * MAXF + f] + q;
      for (int q = 0; q < c->n4 + c->n5; ++q) *o++ = c->oC + K * (c->n4 + c->n5) + q;
    }
  });
}

// ------------------------------------------------------------------ subdomains and entities
// Interface entities are classified GLOBALLY (every rank sees the whole mesh): classes
// of interface DOFs with equal sharer sets.  The context then keeps only its LOCAL subdomains
// (subdomain_rank == rank, renumbered 0..N-1 in global order), the cells of those subdomains
// (renumbered in global order) and the entities they touch (renumbered in global order).
void build_subdomains(vb_ctx *c, const int32_t *cell_sub, int Ng, const int32_t *sub_rank) {
  c->Ng = Ng;
  double tf = wall_s();
  c->cell_sub.assign(cell_sub, cell_sub + c->nK);
  c->sub_rank.assign(Ng, 0);
  if (sub_rank) c->sub_rank.assign(sub_rank, sub_rank + Ng);
  for (int i = 0; i < Ng; ++i)
    VB_REQUIRE(c->sub_rank[i] >= 0 && c->sub_rank[i] < c->nranks, VB_EINVAL, "subdomain_rank out of range");
  c->sub_gid.clear();
  c->sub_lid.assign(Ng, -1);
  for (int i = 0; i < Ng; ++i)
    if (c->sub_rank[i] == c->rank) { c->sub_lid[i] = c->sub_gid.size(); c->sub_gid.push_back(i); }
  const int N = c->N = c->sub_gid.size();
  VB_REQUIRE(N >= 1, VB_EINVAL, "rank " + std::to_string(c->rank) + " owns no subdomain");
  c->cell_lid.assign(c->nK, -1);
  c->cell_gid.clear();
  c->gsub_ncell.assign(Ng, 0);
  for (int64_t K = 0; K < c->nK; ++K) {
    VB_REQUIRE(cell_sub[K] >= 0 && cell_sub[K] < Ng, VB_EINVAL, "cell_subdomain out of range");
    c->gsub_ncell[cell_sub[K]]++;
    if (c->sub_lid[cell_sub[K]] >= 0) { c->cell_lid[K] = c->cell_gid.size(); c->cell_gid.push_back(K); }
  }
  for (int i = 0; i < Ng; ++i) VB_REQUIRE(c->gsub_ncell[i] > 0, VB_EINVAL, "empty subdomain " + std::to_string(i));
  c->nKl = c->cell_gid.size();
  c->subs.assign(N, Sub());
  for (int64_t l = 0; l < c->nKl; ++l) c->subs[c->sub_lid[cell_sub[c->cell_gid[l]]]].cells.push_back(l);
  // (free dof, subdomain) pairs -> sharer sets (global): counting sort by dof (O(cells x nv)), then
  // each dof's few subdomain ids sorted and de-duplicated
  std::vector<std::pair<int64_t, int>> ds;
  {
    std::vector<int64_t> cnt(c->n_free_vel + 1, 0);
    for (int64_t K = 0; K < c->nK; ++K)
      for (int64_t j = c->cell_l2g_ptr[K]; j < c->cell_l2g_ptr[K + 1]; ++j) {
        const int64_t f = c->vel2free[c->cell_l2g[j]];
        if (f >= 0) cnt[f + 1]++;
      }
    for (int64_t f = 0; f < c->n_free_vel; ++f) cnt[f + 1] += cnt[f];
    std::vector<int> subs_of(cnt[c->n_free_vel]);
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int64_t K = 0; K < c->nK; ++K)
      for (int64_t j = c->cell_l2g_ptr[K]; j < c->cell_l2g_ptr[K + 1]; ++j) {
        const int64_t f = c->vel2free[c->cell_l2g[j]];
        if (f >= 0) subs_of[pos[f]++] = cell_sub[K];
      }
    ds.reserve(c->n_free_vel + c->n_free_vel / 4);
    for (int64_t f = 0; f < c->n_free_vel; ++f) {
      int *b = subs_of.data() + cnt[f], *e = subs_of.data() + cnt[f + 1];
      std::sort(b, e);
      e = std::unique(b, e);
      for (int *q = b; q < e; ++q) ds.push_back({f, *q});
    }
  }
  fine_time("dof sharers", tf);
  // entity classes: DOFs with equal sharer sets (hash of the sorted sharer list; the lookup key is
  // a reused scratch vector, a new key is stored only for a new class)
  struct VecHash {
    size_t operator()(const std::vector<int> &v) const {
      uint64_t h = 1469598103934665603ull;
      for (int x : v) h = (h ^ (uint64_t)(uint32_t)x) * 1099511628211ull;
      return (size_t)h;
    }
  };
  std::unordered_map<std::vector<int>, int, VecHash> emap;
  emap.reserve(1 << 16);
  std::vector<std::vector<int>> ekeys;
  std::vector<std::vector<int64_t>> edofs;
  c->dof_owner_sub.assign(c->n_free_vel, -1);
  c->dof_nsh.assign(c->n_free_vel, 0);
  std::vector<int> sh;
  for (size_t i = 0; i < ds.size();) {
    size_t j = i;
    while (j < ds.size() && ds[j].first == ds[i].first) ++j;
    c->dof_owner_sub[ds[i].first] = ds[i].second;
    c->dof_nsh[ds[i].first] = j - i;
    const bool neu = c->neumann && c->vel_on_neu[c->free2vel[ds[i].first]];
    if (j - i > 1 || neu) {
      sh.clear();
      for (size_t q = i; q < j; ++q) sh.push_back(ds[q].second);
      if (neu) sh.push_back(-1);   // Neumann-boundary DOFs form classes of their own
      auto it = emap.find(sh);
      int e;
      if (it == emap.end()) { e = ekeys.size(); emap.emplace(sh, e); ekeys.push_back(sh); edofs.push_back({}); }
      else e = it->second;
      edofs[e].push_back(ds[i].first);
    }
    i = j;
  }
  fine_time("entity classes", tf);
  // global entities ordered by their smallest DOF
  std::vector<int> order(ekeys.size());
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) { return edofs[a][0] < edofs[b][0]; });
  const int nge = order.size();
  c->gents.assign(nge, GEnt());
  c->gsub_ents.assign(Ng, std::vector<int>());
  c->gent_lid.assign(nge, -1);
  c->ents.clear();
  c->nGamma = 0;
  for (int q = 0; q < nge; ++q) {
    GEnt &G = c->gents[q];
    G.sharers = ekeys[order[q]];
    const bool neu = G.sharers.back() < 0;
    if (neu) G.sharers.pop_back();
    G.n = edofs[order[q]].size();
    bool vert = true, has_face = false;
    int64_t v0 = c->free2vel[edofs[order[q]][0]] / 3;
    for (auto d : edofs[order[q]]) {
      int64_t g = c->free2vel[d];
      if (g >= c->oE || g / 3 != v0) vert = false;
      has_face |= g >= c->oF && g < c->oC;
    }
    // on the Neumann boundary a class is a face iff it holds face moments (a subdomain's Neumann
    // patch has one sharer), otherwise an edge (the lines where subdomains meet on it)
    G.kind = vert ? 0 : (neu ? (has_face ? 2 : 1) : (G.sharers.size() == 2 ? 2 : 1));
    for (int s : G.sharers) c->gsub_ents[s].push_back(q);
    bool local = false;
    for (int s : G.sharers) local |= c->sub_lid[s] >= 0;
    if (!local) continue;
    c->gent_lid[q] = c->ents.size();
    Entity E;
    E.gid = q;
    E.sharers = G.sharers;
    E.dofs = edofs[order[q]];
    E.n = G.n;
    E.kind = G.kind;
    c->nGamma += E.n;
    for (int s : E.sharers)
      if (c->sub_lid[s] >= 0) c->subs[c->sub_lid[s]].ents.push_back(c->ents.size());
    c->ents.push_back(std::move(E));
  }
  fine_time("entities", tf);
  // per-subdomain orderings (local subdomains; threads over subdomains, each writes only its own)
  parallel_for(N, [&](int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) {
    Sub &S = c->subs[i];
    const int gi = c->sub_gid[i];
    std::sort(S.ents.begin(), S.ents.end());
    std::vector<int64_t> fr;
    for (int l : S.cells) {
      const int64_t K = c->cell_gid[l];
      for (int64_t j = c->cell_l2g_ptr[K]; j < c->cell_l2g_ptr[K + 1]; ++j) {
        int64_t f = c->vel2free[c->cell_l2g[j]];
        if (f >= 0 && c->dof_nsh[f] == 1 && c->dof_owner_sub[f] == gi && !(c->neumann && c->vel_on_neu[c->cell_l2g[j]]))
          fr.push_back(f);
      }
      for (int q = 0; q < c->np; ++q) S.P.push_back(K * c->np + q);
    }
    std::sort(fr.begin(), fr.end()); fr.erase(std::unique(fr.begin(), fr.end()), fr.end());
    S.I = fr;
    std::sort(S.P.begin(), S.P.end());
    S.nI = S.I.size(); S.nP = S.P.size();
    S.nG = 0;
    for (int e : S.ents) { S.ent_offG.push_back(S.nG); S.nG += c->ents[e].n; }
    S.nD = S.nI + S.nP;
    S.n = S.nD + S.nG;
  }
  }, 16);
}

// ------------------------------------------------------------------ face geometry (host)
void face_frame(const vb_ctx *c, int64_t f, double *area, double n[3], double t1[3], double t2[3]) {
  int64_t s = c->face_ptr[f], e = c->face_ptr[f + 1];
  double av[3] = {0, 0, 0};
  for (int64_t i = s; i < e; ++i) {
    const double *p = &c->xyz[3 * c->face_vtx[i]];
    const double *q = &c->xyz[3 * c->face_vtx[i + 1 < e ? i + 1 : s]];
    av[0] += 0.5 * (p[1] * q[2] - p[2] * q[1]);
    av[1] += 0.5 * (p[2] * q[0] - p[0] * q[2]);
    av[2] += 0.5 * (p[0] * q[1] - p[1] * q[0]);
  }
  double a = sqrt(av[0] * av[0] + av[1] * av[1] + av[2] * av[2]);
  *area = a;
  for (int q = 0; q < 3; ++q) n[q] = av[q] / a;
  const double *p0 = &c->xyz[3 * c->face_vtx[s]], *p1 = &c->xyz[3 * c->face_vtx[s + 1]];
  double d[3] = {p1[0] - p0[0], p1[1] - p0[1], p1[2] - p0[2]};
  double l = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
  for (int q = 0; q < 3; ++q) t1[q] = d[q] / l;
  t2[0] = n[1] * t1[2] - n[2] * t1[1];
  t2[1] = n[2] * t1[0] - n[0] * t1[2];
  t2[2] = n[0] * t1[1] - n[1] * t1[0];
}

// Constraint rows C_G (SURVEY O-9 / A8) as dense rows over the entity's DOFs.
void build_constraint_rows(vb_ctx *c, std::vector<double> &rows_out) {
  int k = c->k;
  double xg[8], wg[8];
  gauss_lobatto01(k + 1, xg, wg);
  // face sign w.r.t. the first sharer: from any cell of that subdomain containing the face
  std::vector<int> fsgn_cell(c->nF * 2, 0);
  std::vector<int> fcell(c->nF * 2, -1);
  for (int64_t K = 0; K < c->nK; ++K)
    for (int64_t j = c->cell_ptr[K]; j < c->cell_ptr[K + 1]; ++j) {
      int64_t f = c->cell_face[j];
      int slot = fcell[2 * f] < 0 ? 0 : 1;
      fcell[2 * f + slot] = K;
      fsgn_cell[2 * f + slot] = c->cell_sign[j];
    }
  rows_out.clear();
  for (auto &E : c->ents) {
    int n = E.n;
    std::vector<std::vector<double>> R;
    auto pos = [&](int64_t gvel) {
      int64_t f = c->vel2free[gvel];
      auto it = std::lower_bound(E.dofs.begin(), E.dofs.end(), f);
      return (it != E.dofs.end() && *it == f) ? (int)(it - E.dofs.begin()) : -1;
    };
    if (c->cons.svd_rel_tol < 0) {  // internal: all DOFs primal (exact-limit test)
      for (int j = 0; j < n; ++j) { std::vector<double> r(n, 0.0); r[j] = 1; R.push_back(r); }
    } else if (E.kind == 0) {
      if (c->cons.vertex)
        for (int q = 0; q < 3; ++q) { std::vector<double> r(n, 0.0); r[q] = 1; R.push_back(r); }
    } else if (E.kind == 1) {
      if (c->cons.edge_avg) {
        std::vector<std::vector<double>> r3(3, std::vector<double>(n, 0.0));
        std::vector<int64_t> eids;
        for (auto d : E.dofs) { int64_t g = c->free2vel[d]; if (g >= c->oE && g < c->oF) eids.push_back((g - c->oE) / (3 * (k - 1))); }
        std::sort(eids.begin(), eids.end()); eids.erase(std::unique(eids.begin(), eids.end()), eids.end());
        for (auto ed : eids) {
          int64_t a = c->edges[2 * ed], b = c->edges[2 * ed + 1];
          double L = 0;
          for (int q = 0; q < 3; ++q) L += (c->xyz[3 * b + q] - c->xyz[3 * a + q]) * (c->xyz[3 * b + q] - c->xyz[3 * a + q]);
          L = sqrt(L);
          for (int d = 0; d < 3; ++d) {
            for (int j = 0; j < k - 1; ++j) r3[d][pos(c->oE + 3 * (k - 1) * ed + 3 * j + d)] += L * wg[j + 1];
            int pa = pos(3 * a + d), pb = pos(3 * b + d);
            if (pa >= 0) r3[d][pa] += L * wg[0];
            if (pb >= 0) r3[d][pb] += L * wg[k];
          }
        }
        for (int d = 0; d < 3; ++d) R.push_back(r3[d]);
      }
    } else {
      std::vector<std::vector<double>> avg(3, std::vector<double>(n, 0.0));
      std::vector<double> flux(n, 0.0);
      std::vector<int64_t> fids;
      for (auto d : E.dofs) { int64_t g = c->free2vel[d]; if (g >= c->oF && g < c->oC) fids.push_back((g - c->oF) / (3 * c->nm)); }
      std::sort(fids.begin(), fids.end()); fids.erase(std::unique(fids.begin(), fids.end()), fids.end());
      int s0 = E.sharers[0];
      for (auto f : fids) {
        double area, nn[3], t1[3], t2[3];
        face_frame(c, f, &area, nn, t1, t2);
        int sg = (fcell[2 * f] >= 0 && c->cell_sub[fcell[2 * f]] == s0) ? fsgn_cell[2 * f] : fsgn_cell[2 * f + 1];
        const double *tau[3] = {nn, t1, t2};
        for (int t = 0; t < 3; ++t) {
          int col = pos(c->oF + 3 * c->nm * f + t * c->nm);
          for (int d = 0; d < 3; ++d) avg[d][col] += area * tau[t][d];
        }
        flux[pos(c->oF + 3 * c->nm * f)] += sg * area;
      }
      if (c->cons.face_avg) for (int d = 0; d < 3; ++d) R.push_back(avg[d]);
      if (c->cons.face_flux) R.push_back(flux);
    }
    // adaptive rows (SURVEY O-12 step 5), appended after the standard constraints
    size_t eid = &E - &c->ents[0];
    if (eid < c->extra_rows.size() && !c->extra_rows[eid].empty()) {
      const std::vector<double> &X = c->extra_rows[eid];
      for (size_t q = 0; q + n <= X.size(); q += n) R.push_back(std::vector<double>(X.begin() + q, X.begin() + q + n));
    }
    E.nrows_C = R.size();
    E.off_C = rows_out.size();
    for (auto &r : R) rows_out.insert(rows_out.end(), r.begin(), r.end());
  }
}

}  // namespace vb
