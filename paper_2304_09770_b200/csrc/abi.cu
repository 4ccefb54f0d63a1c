// C ABI (include/vbddc.h) and the host layout of device data.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <map>
#include "setup.h"
#include "exchange.h"
#include "dense.cuh"

using namespace vb;

static thread_local std::string g_last_error;

static vb_status fail(vb_ctx *c, const Error &e) {
  g_last_error = e.msg;
  if (c) c->err = e.msg;
  if (c && c->comm) c->comm->abort();   // release peers waiting in an exchange (loopback)
  return e.st;
}

#define ABI_GUARD(ctx, ...)                                                                     \
  try {                                                                                         \
    ::vb::AllocStreamScope _alloc_scope(ctx_stream(ctx));                                       \
    __VA_ARGS__;                                                                                \
  } catch (const Error &e) {                                                                    \
    return fail(ctx, e);                                                                        \
  } catch (const std::exception &e) {                                                          \
    return fail(ctx, Error{VB_EINVAL, e.what()});                                               \
  }                                                                                             \
  return VB_OK;

static cudaStream_t ctx_stream(const vb_ctx *c) { return c ? c->stream : nullptr; }
static cudaStream_t ctx_stream(std::nullptr_t) { return nullptr; }

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

namespace vb {

// ------------------------------------------------------------------ layout before the ranks
void layout_phase_a(vb_ctx *c, cudaStream_t s_upload) {
  const int N = c->N;
  cudaStream_t s = s_upload ? s_upload : c->stream;
  c->h_sub.assign(N, SubDev{});
  std::vector<int> sub_cells;
  std::vector<double> lvol(N);
  int64_t K = 0, G = 0, P = 0, I = 0, Dn = 0, X = 0;
  for (int i = 0; i < N; ++i) {
    Sub &S = c->subs[i];
    SubDev &D = c->h_sub[i];
    D.nI = S.nI; D.nP = S.nP; D.nG = S.nG; D.nD = S.nD; D.n = S.n;
    D.cell_begin = sub_cells.size();
    for (int cell : S.cells) sub_cells.push_back(cell);
    D.cell_end = sub_cells.size();
    D.ldk = ld4(S.n);
    D.off_K = K; K += (int64_t)D.ldk * S.n;
    D.off_G = G; G += S.nG;
    D.off_P = P; P += S.nP;
    D.off_I = I; I += S.nI;
    D.off_Dn = Dn; Dn += S.nD;
    D.off_X = X; X += (int64_t)ld4(S.nG) * S.nG;
    double vol = 0, nus = 0;
    for (int cell : S.cells) { vol += c->cellgeo[(int64_t)cell * c->geo_stride]; nus += c->nu[c->cell_gid[cell]]; }
    D.vol = vol;
    S.vol = vol;
    lvol[i] = vol;
    D.gamma = 1.0 / ((nus / std::max<size_t>(S.cells.size(), 1)) * vol);
  }
  c->len_K = K; c->len_G = G; c->len_P = P; c->len_I = I; c->len_Dn = Dn; c->len_X = X;
  // volumes of all subdomains (C0: gathered once; every rank owns a set of subdomains)
  c->gsub_vol.assign(c->Ng, 0.0);
  if (c->nranks == 1) {
    c->gsub_vol = lvol;
  } else {
    int maxN = 0;
    std::vector<int> cnt(c->nranks, 0);
    for (int g = 0; g < c->Ng; ++g) cnt[c->sub_rank[g]]++;
    for (int r = 0; r < c->nranks; ++r) maxN = std::max(maxN, cnt[r]);
    std::vector<double> mine(maxN, 0.0);
    for (int i = 0; i < N; ++i) mine[i] = lvol[i];
    DBuf<double> dm, dg;
    dm.upload(mine, s);
    dg.alloc((size_t)maxN * c->nranks);
    c->comm->allgather(dm.p, dg.p, maxN, s);
    std::vector<double> all;
    dg.download(all, s);
    VB_CUDA(cudaStreamSynchronize(s));
    std::vector<int> seen(c->nranks, 0);
    for (int g = 0; g < c->Ng; ++g) { const int r = c->sub_rank[g]; c->gsub_vol[g] = all[(size_t)r * maxN + seen[r]++]; }
  }
  // entity-major slots: one per (local entity, LOCAL sharer)
  c->h_slot.clear();
  c->h_ent.assign(c->ents.size(), EntDev{});
  int64_t gam = 0;
  std::vector<std::vector<int>> sub_slot(N);
  for (size_t e = 0; e < c->ents.size(); ++e) {
    Entity &E = c->ents[e];
    EntDev &D = c->h_ent[e];
    D.n = E.n; D.kind = E.kind; D.nsh = E.sharers.size(); D.side_begin = c->h_slot.size();
    D.off_gam = gam; gam += E.n;
    for (int mg : E.sharers) {
      const int m = c->sub_lid[mg];
      if (m < 0) continue;
      Sub &S = c->subs[m];
      int j = std::lower_bound(S.ents.begin(), S.ents.end(), (int)e) - S.ents.begin();
      SlotDev sl{};
      sl.sub = m; sl.ent = e; sl.n = E.n; sl.offG = S.ent_offG[j];
      sub_slot[m].push_back(c->h_slot.size());
      c->h_slot.push_back(sl);
    }
    D.nsides = c->h_slot.size() - D.side_begin;
  }
  c->h_sub_slots.clear();
  for (int i = 0; i < N; ++i) {
    // subdomain slot order = its entity order (sorted by entity id = slot creation order)
    c->h_sub[i].slot_begin = c->h_sub_slots.size();
    for (int q : sub_slot[i]) c->h_sub_slots.push_back(q);
    c->h_sub[i].slot_end = c->h_sub_slots.size();
  }
  // index maps
  std::vector<int64_t> Ifree, Pglob, Gfree, gamfree;
  std::vector<double> cvec, mvec;
  for (int i = 0; i < N; ++i) {
    Sub &S = c->subs[i];
    Ifree.insert(Ifree.end(), S.I.begin(), S.I.end());
    Pglob.insert(Pglob.end(), S.P.begin(), S.P.end());
    for (int e : S.ents) Gfree.insert(Gfree.end(), c->ents[e].dofs.begin(), c->ents[e].dofs.end());
    for (int64_t p : S.P) {
      int64_t cell = c->cell_lid[p / c->np], a = p % c->np;
      cvec.push_back(c->cellgeo[cell * c->geo_stride + 5 + a]);
      mvec.push_back(a == 0 ? c->cellgeo[cell * c->geo_stride] : 0.0);
    }
  }
  for (auto &E : c->ents) gamfree.insert(gamfree.end(), E.dofs.begin(), E.dofs.end());
  c->d_subI_free.upload(Ifree, s);
  c->d_subP_glob.upload(Pglob, s);
  c->d_subG_free.upload(Gfree, s);
  c->d_gam_free.upload(gamfree, s);
  c->d_cvec.upload(cvec, s);
  c->d_mvec.upload(mvec, s);
  c->d_sub_cells.upload(sub_cells, s);
  c->d_sub_slots.upload(c->h_sub_slots, s);
  // local cell -> subdomain-matrix positions
  const int stride = c->nv_max + c->np;
  std::vector<int> loc((size_t)c->nKl * stride, -1);
  std::vector<int64_t> posI(c->n_free_vel, -1);
  // interface dof -> (local entity, position in the entity)
  std::vector<int> dof_ent(c->n_free_vel, -1), dof_epos(c->n_free_vel, -1);
  for (size_t e = 0; e < c->ents.size(); ++e)
    for (size_t a = 0; a < c->ents[e].dofs.size(); ++a) {
      dof_ent[c->ents[e].dofs[a]] = (int)e;
      dof_epos[c->ents[e].dofs[a]] = (int)a;
    }
  // threads over subdomains (interior DOFs and cells belong to one subdomain: disjoint writes)
  parallel_for(N, [&](int64_t i0, int64_t i1) {
  std::vector<int> ent_slot(c->ents.size(), -1);   // entity -> its index t in the current subdomain
  for (int64_t i = i0; i < i1; ++i) {
    Sub &S = c->subs[i];
    for (int j = 0; j < S.nI; ++j) posI[S.I[j]] = j;
    for (size_t t = 0; t < S.ents.size(); ++t) ent_slot[S.ents[t]] = (int)t;
    for (int cell : S.cells) {
      const int64_t Kg = c->cell_gid[cell];
      int *L = &loc[(size_t)cell * stride];
      for (int64_t j = c->cell_l2g_ptr[Kg]; j < c->cell_l2g_ptr[Kg + 1]; ++j) {
        int64_t f = c->vel2free[c->cell_l2g[j]];
        int q = j - c->cell_l2g_ptr[Kg];
        if (f < 0) continue;
        if (dof_ent[f] < 0) {
          VB_REQUIRE(posI[f] >= 0 && posI[f] < S.nI && S.I[posI[f]] == f, VB_EINVAL,
                     "internal: interior dof not in its subdomain");
          L[q] = posI[f];
        } else {
          const int t = ent_slot[dof_ent[f]];
          VB_REQUIRE(t >= 0 && S.ents[t] == dof_ent[f], VB_EINVAL, "internal: interface dof not found in its subdomain");
          L[q] = S.nD + S.ent_offG[t] + dof_epos[f];
        }
      }
      int64_t p0 = std::lower_bound(S.P.begin(), S.P.end(), Kg * c->np) - S.P.begin();
      for (int a = 0; a < c->np; ++a) L[c->nv_max + a] = S.nI + p0 + a;
    }
    for (size_t t = 0; t < S.ents.size(); ++t) ent_slot[S.ents[t]] = -1;
  }
  }, 16);
  c->d_cell_loc.upload(loc, s);
  c->h_cell_loc = loc;
  // element-by-element operator / rhs: free velocity dof -> contribution slots (local cells, in order)
  {
    // counting sort by dof; within a dof the slots stay in (cell, local dof) order
    std::vector<int64_t> ptr(c->n_free_vel + 1, 0);
    for (int64_t cell = 0; cell < c->nKl; ++cell) {
      const int64_t Kg = c->cell_gid[cell];
      for (int64_t j = c->cell_l2g_ptr[Kg]; j < c->cell_l2g_ptr[Kg + 1]; ++j) {
        const int64_t f = c->vel2free[c->cell_l2g[j]];
        if (f >= 0) ptr[f + 1]++;
      }
    }
    for (int64_t i = 0; i < c->n_free_vel; ++i) ptr[i + 1] += ptr[i];
    std::vector<int64_t> idx(ptr[c->n_free_vel]), fill(ptr.begin(), ptr.end() - 1);
    for (int64_t cell = 0; cell < c->nKl; ++cell) {
      const int64_t Kg = c->cell_gid[cell];
      for (int64_t j = c->cell_l2g_ptr[Kg]; j < c->cell_l2g_ptr[Kg + 1]; ++j) {
        const int64_t f = c->vel2free[c->cell_l2g[j]];
        if (f >= 0) idx[fill[f]++] = cell * stride + (j - c->cell_l2g_ptr[Kg]);
      }
    }
    c->d_el_ptr.upload(ptr, s);
    c->d_el_ent.upload(idx, s);
    c->w_elt.alloc((size_t)c->nKl * stride);
    c->w_elx.alloc((size_t)c->nKl * ((stride + 1) & ~1));   // K7 per-cell inputs, 16-byte aligned cells
  }
  // greedy colouring of the GLOBAL subdomain adjacency (shared entities) for the coarse assembly
  {
    std::vector<std::vector<int>> adj(c->Ng);
    for (auto &E : c->gents)
      for (int a : E.sharers)
        for (int b : E.sharers)
          if (a != b) adj[a].push_back(b);
    c->gsub_color.assign(c->Ng, 0);
    c->ncolors = 0;
    for (int i = 0; i < c->Ng; ++i) {
      std::vector<char> used(128, 0);
      for (int j : adj[i]) if (j < i && c->gsub_color[j] < 128) used[c->gsub_color[j]] = 1;
      int col = 0;
      while (used[col]) ++col;
      c->gsub_color[i] = col;
      c->ncolors = std::max(c->ncolors, col + 1);
    }
  }
  // ABI layout of the free vectors: owned velocity DOFs (lowest sharer on this rank), then the
  // pressure DOFs of the local cells; identical to the global free numbering for one rank
  c->owned_free.clear();
  for (int64_t f = 0; f < c->n_free_vel; ++f)
    if (c->dof_owner_sub[f] >= 0 && c->sub_rank[c->dof_owner_sub[f]] == c->rank) c->owned_free.push_back(f);
  {
    std::vector<int64_t> pl;
    for (int64_t l = 0; l < c->nKl; ++l)
      for (int a = 0; a < c->np; ++a) pl.push_back(c->n_free_vel + c->cell_gid[l] * c->np + a);
    std::sort(pl.begin(), pl.end());
    c->owned_free.insert(c->owned_free.end(), pl.begin(), pl.end());
  }
  c->d_owned_free.upload(c->owned_free, s);
  c->d_sub.upload(c->h_sub, s);
  c->d_slot.upload(c->h_slot, s);
  c->d_ent.upload(c->h_ent, s);
  VB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------------ maps needing the ranks
void build_transformed_maps(vb_ctx *c) {
  std::vector<int64_t> loc2x(c->len_G, -1), pig(std::max<int64_t>(c->len_Pi, 1), -1);
  c->max_npi = 0;
  for (int i = 0; i < c->N; ++i) {
    const SubDev &S = c->h_sub[i];
    c->max_npi = std::max(c->max_npi, S.npi);
    for (int q = S.slot_begin; q < S.slot_end; ++q) {
      const SlotDev &sl = c->h_slot[c->h_sub_slots[q]];
      const EntDev &E = c->h_ent[sl.ent];
      for (int j = 0; j < sl.nd; ++j) loc2x[S.off_G + sl.offD + j] = E.off_xd + j;
      for (int j = 0; j < sl.r; ++j) {
        loc2x[S.off_G + S.nd + sl.offPi + j] = c->n_delta_glob + E.off_pl + j;
        pig[S.off_Pi + sl.offPi + j] = E.off_pi + j;
      }
    }
  }
  c->d_loc2x.upload(loc2x, c->stream);
  c->d_pi_glob.upload(pig, c->stream);
  VB_CUDA(cudaStreamSynchronize(c->stream));
}

// ------------------------------------------------------------------ common setup
// VB_SETUP_TIMES=1: wall time of each setup stage on stderr
static void setup_time(const char *what, double &t) {
  static const bool on = getenv("VB_SETUP_TIMES") && atoi(getenv("VB_SETUP_TIMES"));
  if (!on) return;
  const double now = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  fprintf(stderr, "[vb setup] %-28s %8.3f s\n", what, now - t);
  t = now;
}

static void common_setup(vb_ctx *c, const vb_mesh *m, const int32_t *cell_sub, int32_t nsub,
                         const int32_t *sub_rank, const vb_constraints *cons, const double *nu,
                         const vb_dist *dist) {
  VB_REQUIRE(m && cell_sub && nu && cons, VB_EINVAL, "null argument");
  VB_REQUIRE(m->k >= 2 && m->k <= 4, VB_EINVAL, "k must be 2, 3 or 4");
  VB_REQUIRE(nsub >= 1, VB_EINVAL, "n_subdomains must be >= 1");
  c->k = m->k;
  c->cons = *cons;
  c->debug = getenv("VB_DEBUG") ? atoi(getenv("VB_DEBUG")) : 0;
  if (dist) {
    c->rank = dist->rank; c->nranks = dist->nranks; c->device = dist->device;
    c->stream = (cudaStream_t)dist->stream;
    g_alloc_stream = c->stream;
  }
  VB_REQUIRE(c->nranks >= 1 && c->rank >= 0 && c->rank < c->nranks, VB_EINVAL, "bad rank / nranks");
  VB_CUDA(cudaSetDevice(c->device));
  if (c->nranks > 1) {
    VB_REQUIRE(sub_rank, VB_EINVAL, "nranks > 1 needs subdomain_rank");
    if (dist->loopback_world) c->comm = make_loopback_comm(dist->loopback_world, c->rank);
    else c->comm = make_nccl_comm(c->rank, c->nranks, dist->nccl_unique_id, c->device);
    VB_REQUIRE(c->comm->nranks == c->nranks, VB_EINVAL, "communicator size differs from nranks");
  }
  double ts = std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
  build_topology(c, m);
  setup_time("topology", ts);
  c->nu.assign(nu, nu + c->nK);
  for (int64_t K = 0; K < c->nK; ++K) VB_REQUIRE(c->nu[K] > 0, VB_EINVAL, "viscosity must be positive (P:108)");
  build_subdomains(c, cell_sub, nsub, c->nranks > 1 ? sub_rank : nullptr);
  setup_time("subdomains / DOF maps", ts);
  cudaStream_t s = c->stream;
  // device copies of the LOCAL cells (topology, viscosity, dof maps); vertices and the dof status are global
  // (all cells local, one rank: the global arrays are uploaded as they are)
  const bool all_local = c->nKl == c->nK;
  std::vector<int> topo(all_local ? 0 : (size_t)c->nKl * TOPO_STRIDE);
  std::vector<double> nul(all_local ? 0 : c->nKl);
  std::vector<int> nvl(all_local ? 0 : c->nKl);
  std::vector<int64_t> l2g((size_t)c->nKl * c->nv_max);
  parallel_for(c->nKl, [&](int64_t l0, int64_t l1) {
    for (int64_t l = l0; l < l1; ++l) {
      const int64_t K = c->cell_gid[l];
      if (!all_local) {
        std::copy(c->cell_topo.begin() + K * TOPO_STRIDE, c->cell_topo.begin() + (K + 1) * TOPO_STRIDE,
                  topo.begin() + l * TOPO_STRIDE);
        nul[l] = c->nu[K];
        nvl[l] = c->cell_nv[K];
      }
      int64_t *o = l2g.data() + l * c->nv_max;
      const int64_t n = c->cell_l2g_ptr[K + 1] - c->cell_l2g_ptr[K];
      std::copy(c->cell_l2g.begin() + c->cell_l2g_ptr[K], c->cell_l2g.begin() + c->cell_l2g_ptr[K + 1], o);
      std::fill(o + n, o + c->nv_max, (int64_t)-1);
    }
  });
  c->d_xyz.upload(c->xyz, s);
  c->d_topo.upload(all_local ? c->cell_topo : topo, s);
  c->d_nu.upload(all_local ? c->nu : nul, s);
  c->d_cell_nv.upload(all_local ? c->cell_nv : nvl, s);
  c->d_vel2free.upload(c->vel2free, s);
  c->d_cell_l2g.upload(l2g, s);
  c->d_cell_gid.upload(c->cell_gid, s);
  VB_CUDA(cudaStreamSynchronize(s));
  setup_time("local copies + upload", ts);
  cell_geometry_device(c);
  c->d_cellgeo.download(c->cellgeo, s);
  VB_CUDA(cudaStreamSynchronize(s));
  setup_time("cell geometry (device)", ts);
}

}  // namespace vb

// ------------------------------------------------------------------ ABI
extern "C" {

vb_status vb_debug_nccl_selftest(int32_t device, double *result) {
  if (!result) return VB_EINVAL;
  ABI_GUARD(nullptr, {
    std::string msg;
    vb::nccl_selftest(device, result, msg);
    if (!msg.empty()) g_last_error = msg;
  })
}

vb_status vb_set_option(vb_ctx *c, const char *name, double value) {
  if (!c || !name) return VB_EINVAL;
  if (!strcmp(name, "true_residual")) {
    c->opt_true_residual = value != 0.0;
    return VB_OK;
  }
  if (!strcmp(name, "coarse_dissection")) {
    if (c->state >= 2) return fail(c, Error{VB_ESTATE, "option coarse_dissection is read by vb_factor: set it before"});
    c->opt_coarse_dis = value < 0 ? -1 : (value != 0.0);
    return VB_OK;
  }
  if (!strcmp(name, "coarse_blocks")) {
    if (c->state >= 2) return fail(c, Error{VB_ESTATE, "option coarse_blocks is read by vb_factor: set it before"});
    c->opt_coarse_blocks = value < 1 ? -1 : (int)value;
    return VB_OK;
  }
  if (!strcmp(name, "p2p")) {
    if (c->state >= 2) return fail(c, Error{VB_ESTATE, "option p2p is read by vb_factor: set it before"});
    c->opt_p2p = value != 0.0;
    return VB_OK;
  }
  return fail(c, Error{VB_EINVAL, std::string("unknown option ") + name});
}

vb_status vb_nccl_unique_id(void *out128) {
  if (!out128) return VB_EINVAL;
  ABI_GUARD(nullptr, { vb::nccl_unique_id(out128); })
}

vb_status vb_loopback_world_create(int32_t nranks, void **world) {
  if (!world || nranks < 1) return VB_EINVAL;
  *world = vb::loopback_world_create(nranks);
  return VB_OK;
}

vb_status vb_loopback_world_destroy(void *world) {
  if (!world) return VB_EINVAL;
  vb::loopback_world_destroy(world);
  return VB_OK;
}

vb_status vb_plan_exchange(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                           const int32_t *subdomain_rank, int32_t rank, int32_t nranks, int32_t mode,
                           int64_t *send_counts, int64_t *recv_counts, int64_t *n_owned_free) {
  if (!mesh || !cell_subdomain || !send_counts || !recv_counts || !n_owned_free || nranks < 1 || rank < 0 ||
      rank >= nranks || mode < XCH_ALL || mode > XCH_RANK || (nranks > 1 && !subdomain_rank))
    return VB_EINVAL;
  vb_ctx c;   // host bookkeeping only: no device work
  try {
    VB_REQUIRE(mesh->k >= 2 && mesh->k <= 4, VB_EINVAL, "k must be 2, 3 or 4");
    c.k = mesh->k;
    c.rank = rank;
    c.nranks = nranks;
    build_topology(&c, mesh);
    build_subdomains(&c, cell_subdomain, n_subdomains, nranks > 1 ? subdomain_rank : nullptr);
    std::vector<int64_t> snd, rcv;
    plan_slot_counts(&c, [&](int e) { return (int64_t)c.ents[e].n; }, mode, snd, rcv);
    for (int p = 0; p < nranks; ++p) { send_counts[p] = snd[p]; recv_counts[p] = rcv[p]; }
    int64_t own = c.nKl * c.np;
    for (int64_t f = 0; f < c.n_free_vel; ++f)
      if (c.dof_owner_sub[f] >= 0 && c.sub_rank[c.dof_owner_sub[f]] == rank) ++own;
    *n_owned_free = own;
  } catch (const Error &e) {
    return fail(nullptr, e);
  }
  return VB_OK;
}

vb_status vb_plan_coarse_dissection(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                                    const int32_t *subdomain_rank, int32_t rank, int32_t nranks,
                                    const int32_t *primal_per_kind, int64_t *out6) {
  if (!mesh || !cell_subdomain || !primal_per_kind || !out6 || nranks < 1 || rank < 0 || rank >= nranks ||
      (nranks > 1 && !subdomain_rank))
    return VB_EINVAL;
  vb_ctx c;   // host bookkeeping only: no device work
  try {
    VB_REQUIRE(mesh->k >= 2 && mesh->k <= 4, VB_EINVAL, "k must be 2, 3 or 4");
    for (int q = 0; q < 3; ++q) VB_REQUIRE(primal_per_kind[q] >= 0, VB_EINVAL, "negative primal count");
    c.k = mesh->k;
    c.rank = rank;
    c.nranks = nranks;
    build_topology(&c, mesh);
    build_subdomains(&c, cell_subdomain, n_subdomains, nranks > 1 ? subdomain_rank : nullptr);
    int64_t off = 0;
    for (auto &G : c.gents) {
      G.r = std::min(G.n, (int)primal_per_kind[G.kind]);
      G.off_pi = off;
      off += G.r;
    }
    c.NPi_g = off;
    const CoarsePlan P = plan_coarse_dissection(&c, c.sub_rank, nranks);
    const int64_t nI = P.I[rank].size(), nS = P.S[rank].size();
    const int64_t v[6] = {nI, nS, P.nsep, (int64_t)P.root.size(), (nI + 31) / 32 * 32 + nS, c.NPi_g};
    memcpy(out6, v, sizeof(v));
  } catch (const Error &e) {
    return fail(nullptr, e);
  }
  return VB_OK;
}

vb_status vb_setup(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                   const int32_t *subdomain_rank, const vb_constraints *cons, const double *cell_viscosity,
                   const vb_dist *dist, vb_ctx **out) {
  if (!out) return VB_EINVAL;
  *out = nullptr;
  vb_ctx *c = new vb_ctx();
  AllocStreamScope alloc_scope(nullptr);   // common_setup switches it to the context's stream
  try {
    double t0 = now_s();
    common_setup(c, mesh, cell_subdomain, n_subdomains, subdomain_rank, cons, cell_viscosity, dist);
    double ts = now_s();
    // one rank, plain allocator: the element kernel (K9) runs while the host builds the layout,
    // whose uploads go to a second stream (pageable copies on the K9 stream would wait for it)
    // (not with VB_POISON: its fill of each new allocation is queued on the K9 stream and would land
    // after the second stream's upload into it)
    const bool overlap = c->nranks == 1 && !g_use_pool && !g_poison &&
                         !(getenv("VB_NO_SETUP_OVERLAP") && atoi(getenv("VB_NO_SETUP_OVERLAP")));
    element_matrices_device(c, !overlap);
    if (!overlap) setup_time("element matrices K9 (device)", ts);
    cudaStream_t ss = nullptr;
    if (overlap) VB_CUDA(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
    try {
      layout_phase_a(c, ss);
    } catch (...) {
      if (ss) { cudaStreamSynchronize(c->stream); cudaStreamDestroy(ss); }
      throw;
    }
    if (overlap) {
      VB_CUDA(cudaStreamSynchronize(ss));
      VB_CUDA(cudaStreamDestroy(ss));
      VB_CUDA(cudaStreamSynchronize(c->stream));
      c->w_k9.release();
      setup_time("K9 (device) || layout (host)", ts);
    } else {
      setup_time("layout", ts);
    }
    c->t_setup = now_s() - t0;
    c->state = 1;
  } catch (const Error &e) {
    vb_status st = fail(c, e);
    delete c;
    return st;
  }
  *out = c;
  return VB_OK;
}

vb_status vb_setup_from_elements(const vb_mesh *mesh, const int32_t *cell_subdomain, int32_t n_subdomains,
                                 const int32_t *subdomain_rank, const vb_constraints *cons,
                                 const double *cell_viscosity, const vb_dist *dist, const int64_t *elem_ptr_A,
                                 const double *elem_A, const int64_t *elem_ptr_B, const double *elem_B,
                                 vb_ctx **out) {
  if (!out) return VB_EINVAL;
  *out = nullptr;
  vb_ctx *c = new vb_ctx();
  AllocStreamScope alloc_scope(nullptr);   // common_setup switches it to the context's stream
  try {
    double t0 = now_s();
    common_setup(c, mesh, cell_subdomain, n_subdomains, subdomain_rank, cons, cell_viscosity, dist);
    VB_REQUIRE(elem_ptr_A && elem_A && elem_ptr_B && elem_B, VB_EINVAL, "null element arrays");
    const int nvm = c->nv_max, np = c->np;
    std::vector<double> A((size_t)c->nKl * nvm * nvm, 0.0), B((size_t)c->nKl * np * nvm, 0.0);
    for (int64_t l = 0; l < c->nKl; ++l) {
      const int64_t K = c->cell_gid[l];
      const int nv = c->cell_nv[K];
      VB_REQUIRE(elem_ptr_A[K + 1] - elem_ptr_A[K] == (int64_t)nv * nv, VB_EINVAL, "element A size mismatch");
      VB_REQUIRE(elem_ptr_B[K + 1] - elem_ptr_B[K] == (int64_t)np * nv, VB_EINVAL, "element B size mismatch");
      std::copy(elem_A + elem_ptr_A[K], elem_A + elem_ptr_A[K + 1], A.begin() + (size_t)l * nvm * nvm);
      std::copy(elem_B + elem_ptr_B[K], elem_B + elem_ptr_B[K + 1], B.begin() + (size_t)l * np * nvm);
    }
    c->d_elA.upload(A, c->stream);
    c->d_elB.upload(B, c->stream);
    layout_phase_a(c);
    c->t_setup = now_s() - t0;
    c->state = 1;
  } catch (const Error &e) {
    vb_status st = fail(c, e);
    delete c;
    return st;
  }
  *out = c;
  return VB_OK;
}

vb_status vb_factor(vb_ctx *c) {
  if (!c) return VB_EINVAL;
  if (c->state < 1) return fail(c, Error{VB_ESTATE, "vb_factor before vb_setup"});
  ABI_GUARD(c, {
    double t0 = now_s();
    if (c->state >= 2) {   // re-factorisation: the solve state points into the old factors
      VB_CUDA(cudaStreamSynchronize(c->stream));
      destroy_solve_state(c);
    }
    factor_device(c);
    prepare_solve(c);
    if (getenv("VB_FACTOR_TIMES") && atoi(getenv("VB_FACTOR_TIMES")))
      fprintf(stderr, "[vb factor rank %d] total incl. solve preparation %8.3f s\n", c->rank, now_s() - t0);
    c->t_factor = now_s() - t0;
    c->state = 2;
  })
}

vb_status vb_build_rhs(vb_ctx *c, const vb_problem *prob, double *rhs_dev) {
  if (!c || !prob || !rhs_dev) return VB_EINVAL;
  if (c->state < 1) return fail(c, Error{VB_ESTATE, "vb_build_rhs before vb_setup"});
  ABI_GUARD(c, { build_rhs_device(c, prob, rhs_dev); })
}

vb_status vb_pcg_solve(vb_ctx *c, const double *rhs_dev, double *x_dev, double rtol, int32_t maxit, vb_report *rep) {
  if (!c || !rhs_dev || !x_dev) return VB_EINVAL;
  if (c->state < 2) return fail(c, Error{VB_ESTATE, "vb_pcg_solve before vb_factor"});
  if (!(rtol > 0)) return fail(c, Error{VB_EINVAL, "rtol must be positive"});
  if (rep) memset(rep, 0, sizeof(*rep));
  ABI_GUARD(c, {
    double t0 = now_s();
    pcg_device(c, rhs_dev, x_dev, rtol, maxit > 0 ? maxit : 2000, rep);
    if (rep) {
      rep->t_solve_s = now_s() - t0;
      rep->t_setup_s = c->t_setup;
      rep->t_factor_s = c->t_factor;
    }
  })
}

vb_status vb_pcg_solve_host(vb_ctx *c, const double *rhs_host, double *x_host, double rtol, int32_t maxit,
                            vb_report *rep) {
  if (!c || !rhs_host || !x_host) return VB_EINVAL;
  if (c->state < 2) return fail(c, Error{VB_ESTATE, "vb_pcg_solve_host before vb_factor"});
  ABI_GUARD(c, {
    // this rank's owned free DOFs (vb_num_free_dofs): the caller's host buffers hold only those
    const int64_t n = (int64_t)c->owned_free.size();
    if (c->w_hostio.n < (size_t)(2 * n)) c->w_hostio.alloc(2 * n);
    VB_CUDA(cudaMemcpyAsync(c->w_hostio.p, rhs_host, n * 8, cudaMemcpyHostToDevice, c->stream));
    vb_status st = vb_pcg_solve(c, c->w_hostio.p, c->w_hostio.p + n, rtol, maxit, rep);
    if (st != VB_OK) throw Error{st, c->err};
    VB_CUDA(cudaMemcpyAsync(x_host, c->w_hostio.p + n, n * 8, cudaMemcpyDeviceToHost, c->stream));
    VB_CUDA(cudaStreamSynchronize(c->stream));
  })
}

vb_status vb_apply_operator(vb_ctx *c, const double *x_dev, double *y_dev) {
  if (!c || !x_dev || !y_dev) return VB_EINVAL;
  if (c->state < 1) return fail(c, Error{VB_ESTATE, "vb_apply_operator before vb_setup"});
  ABI_GUARD(c, {
    apply_operator_device(c, x_dev, y_dev);
    VB_CUDA(cudaStreamSynchronize(c->stream));
  })
}

vb_status vb_debug_interface_op(vb_ctx *c, int32_t which, const double *in, double *out) {
  if (!c || !in || !out || (which != 0 && which != 1)) return VB_EINVAL;
  if (c->state < 2) return fail(c, Error{VB_ESTATE, "vb_debug_interface_op before vb_factor"});
  if (c->nranks != 1) return fail(c, Error{VB_EINVAL, "vb_debug_interface_op is single-rank only"});
  ABI_GUARD(c, { debug_interface_op(c, which, in, out); })
}

vb_status vb_debug_subdomain_op(vb_ctx *c, int32_t sub, int32_t which, int64_t *ids, double *out, int64_t *n) {
  if (!c || !n) return VB_EINVAL;
  if (c->state < 2) return fail(c, Error{VB_ESTATE, "vb_debug_subdomain_op before vb_factor"});
  ABI_GUARD(c, { debug_subdomain_op(c, sub, which, ids, out, n); })
}

vb_status vb_interface_dofs(const vb_ctx *c, int64_t *ids, int64_t *n) {
  if (!c || !n) return VB_EINVAL;
  *n = c->nGamma;
  if (ids) {
    int64_t q = 0;
    for (auto &E : c->ents)
      for (auto d : E.dofs) ids[q++] = d;
  }
  return VB_OK;
}

vb_status vb_num_free_dofs(const vb_ctx *c, int64_t *n_vel, int64_t *n_p) {
  if (!c || !n_vel || !n_p) return VB_EINVAL;
  *n_p = c->nKl * c->np;
  *n_vel = (int64_t)c->owned_free.size() - *n_p;
  return VB_OK;
}

vb_status vb_dof_layout(const vb_ctx *c, int64_t *ids) {
  if (!c || !ids) return VB_EINVAL;
  for (size_t i = 0; i < c->owned_free.size(); ++i) {
    const int64_t f = c->owned_free[i];
    ids[i] = f < c->n_free_vel ? c->free2vel[f] : c->nvel + (f - c->n_free_vel);
  }
  return VB_OK;
}

vb_status vb_cell_local_dofs(const vb_ctx *c, int64_t cell, int64_t *vel_ids, int32_t *n_vel, int64_t *p_ids,
                             int32_t *n_p) {
  if (!c || cell < 0 || cell >= c->nK) return VB_EINVAL;
  int nv = c->cell_nv[cell];
  if (n_vel) *n_vel = nv;
  if (n_p) *n_p = c->np;
  if (vel_ids)
    for (int j = 0; j < nv; ++j) vel_ids[j] = c->cell_l2g[c->cell_l2g_ptr[cell] + j];
  if (p_ids)
    for (int a = 0; a < c->np; ++a) p_ids[a] = cell * c->np + a;
  return VB_OK;
}

vb_status vb_get_element_matrices(const vb_ctx *c, int64_t gcell, double *A, double *B) {
  if (!c || gcell < 0 || gcell >= c->nK || c->cell_lid[gcell] < 0) return VB_EINVAL;
  const int nvm = c->nv_max, np = c->np, nv = c->cell_nv[gcell];
  const int64_t cell = c->cell_lid[gcell];
  try {
    if (A) VB_CUDA(cudaMemcpy(A, c->d_elA.p + cell * nvm * nvm, (size_t)nv * nv * 8, cudaMemcpyDeviceToHost));
    if (B) VB_CUDA(cudaMemcpy(B, c->d_elB.p + cell * np * nvm, (size_t)np * nv * 8, cudaMemcpyDeviceToHost));
  } catch (const Error &e) {
    return fail(const_cast<vb_ctx *>(c), e);
  }
  return VB_OK;
}

vb_status vb_stats(const vb_ctx *c, int64_t *o) {
  if (!c || !o) return VB_EINVAL;
  int64_t maxnG = 0, maxnd = 0, maxn = 0;
  for (auto &S : c->h_sub) { maxnG = std::max<int64_t>(maxnG, S.nG); maxnd = std::max<int64_t>(maxnd, S.nd); maxn = std::max<int64_t>(maxn, S.n); }
  int64_t pkG = 0, pkD = 0, ndsq = 0, ndpi = 0;
  for (auto &S : c->h_sub) { pkG += (int64_t)S.nG * (S.nG + 1) / 2; pkD += (int64_t)S.nd * (S.nd + 1) / 2; ndpi += (int64_t)S.nd * S.npi; }
  for (auto &sl : c->h_slot) ndsq += (int64_t)sl.nd * sl.nd;
  // coarse doubles streamed in the timed coarse window (the B6 kernel-time category): the inverse's
  // slice (or all of it), plus with the dissection the parts' packed matrices of pass 1
  int64_t cd_nloc = 0, pk_coarse = c->nranks > 1 ? (int64_t)c->d_Kcs.n : (int64_t)packed_size((int)(c->cdis ? c->Nroot : c->Nc));
  if (c->cdis) {
    std::vector<CdPart> all = c->cd_parts;
    if (c->cd_two) all.push_back(c->cd2_part);
    for (auto &d : all) {
      cd_nloc += d.nloc;
      if (d.nIp > 0) pk_coarse += packed_size((int)d.nloc);
    }
  }
  int64_t v[28] = {c->nvel + c->npres, c->n_free_vel, c->npres, c->N, (int64_t)c->ents.size(), c->nGamma,
                   c->NPi_g, c->Nc, c->n_delta_glob, maxn, maxnG, maxnd, c->nE, (int64_t)c->bytes_per_iter, c->nv_max,
                   c->ncolors, pkG, pkD, ndsq, ndpi, pk_coarse, c->last_iterations, c->nK,
                   (int64_t)c->factor_flops, (int64_t)(c->factor_alloc_s * 1e6), (int64_t)(c->factor_gemm_s * 1e6),
                   c->cdis ? c->Nroot : 0, cd_nloc};
  memcpy(o, v, sizeof(v));
  return VB_OK;
}

vb_status vb_kernel_times(const vb_ctx *c, double *ms, int32_t n_max, int32_t *n_out) {
  if (!c || !n_out) return VB_EINVAL;
  int n = std::min<int>(n_max, c->ktime_ms.size());
  for (int i = 0; i < n; ++i) ms[i] = c->ktime_count[i] ? c->ktime_ms[i] / c->ktime_count[i] : 0.0;
  *n_out = n;
  return VB_OK;
}

const char *vb_kernel_time_name(int32_t i) { return vb::kernel_time_name(i); }

const char *vb_last_error(const vb_ctx *c) { return c ? c->err.c_str() : g_last_error.c_str(); }

vb_status vb_debug_gemm(int32_t M, int32_t N, int32_t K, double alpha, const double *A, int32_t lda,
                        int32_t transA, const double *B, int32_t ldb, int32_t transB, const double *d,
                        double beta, double *C, int32_t ldc, int32_t batch, int64_t strideA,
                        int64_t strideB, int64_t strideC, void *stream, int32_t kz_on, int32_t kzA,
                        int32_t kzB) {
  if (M <= 0 || N <= 0 || K <= 0 || batch <= 0 || !A || !B || !C) return VB_EINVAL;
  if (lda < (transA ? K : M) || ldb < (transB ? N : K) || ldc < M) return VB_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  ABI_GUARD(nullptr, {
    AllocStreamScope scope(s);
    GemmPlan plan;
    plan.allow_kz = true;
    int l0 = plan.begin_launch();
    for (int b = 0; b < batch; ++b) {
      GemmProb p{};
      p.A = A + b * strideA; p.lda = lda; p.transA = transA != 0;
      p.B = B + b * strideB; p.ldb = ldb; p.transB = transB != 0;
      p.C = C + b * strideC; p.ldc = ldc;
      p.d = d; p.dstride = 1;
      p.M = M; p.N = N; p.K = K; p.alpha = alpha; p.beta = beta;
      p.kz_on = kz_on != 0; p.kzA = kzA; p.kzB = kzB;
      plan.add(p);
    }
    plan.upload(s);
    plan.run(l0, s);
    VB_CUDA(cudaStreamSynchronize(s));
  })
}

vb_status vb_destroy(vb_ctx *c) {
  if (!c) return VB_EINVAL;
  cudaStream_t s = c->stream;
  cudaStreamSynchronize(s);
  {
    AllocStreamScope alloc_scope(s);
    destroy_solve_state(c);
    delete c->comm;
    delete c;
  }
  pool_trim(s);   // return the context's device memory (other live contexts keep theirs)
  return VB_OK;
}

}  // extern "C"
