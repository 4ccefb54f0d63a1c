// Interface exchanges between ranks (exchange.h).
#include <algorithm>
#include "exchange.h"
#include "setup.h"

namespace vb {

__global__ void pack_kernel(const double *__restrict__ src, const int64_t *__restrict__ idx, int64_t n, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[idx[i]];
}

__global__ void scatter_idx_kernel(const double *__restrict__ src, const int64_t *__restrict__ idx, int64_t n, double *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = src[i];
}

void dev_gather(const double *src, const int64_t *idx, int64_t n, double *out, cudaStream_t s) {
  if (n <= 0) return;
  pack_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(src, idx, n, out);
  VB_CHECK_LAUNCH();
}

void dev_scatter(const double *src, const int64_t *idx, int64_t n, double *out, cudaStream_t s) {
  if (n <= 0) return;
  scatter_idx_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(src, idx, n, out);
  VB_CHECK_LAUNCH();
}

__global__ void rank_sum_kernel(const double *__restrict__ g, int R, int k, double *v) {
  const int i = threadIdx.x;
  if (i >= k) return;
  double s = 0.0;
  for (int r = 0; r < R; ++r) s += g[r * k + i];
  v[i] = s;
}

bool xch_sends(const vb_ctx *c, int e, int k, int mode) {
  const std::vector<int> &sh = c->ents[e].sharers;
  if (mode == XCH_ALL) return true;
  if (mode == XCH_OWNER) return k == 0;
  const int r = c->sub_rank[sh[k]];
  for (int q = 0; q < k; ++q)
    if (c->sub_rank[sh[q]] == r) return false;
  return true;
}

void plan_slot_counts(const vb_ctx *c, const std::function<int64_t(int)> &L, int mode, std::vector<int64_t> &send,
                      std::vector<int64_t> &recv) {
  send.assign(c->nranks, 0);
  recv.assign(c->nranks, 0);
  for (size_t e = 0; e < c->ents.size(); ++e) {
    const std::vector<int> &sh = c->ents[e].sharers;
    const int64_t Le = L(e);
    for (int p = 0; p < c->nranks; ++p) {
      if (p == c->rank) continue;
      bool shared = false;
      for (int m : sh) shared |= c->sub_rank[m] == p;
      if (!shared) continue;
      for (size_t k = 0; k < sh.size(); ++k) {
        if (!xch_sends(c, e, k, mode)) continue;
        if (c->sub_rank[sh[k]] == c->rank) send[p] += Le;
        if (c->sub_rank[sh[k]] == p) recv[p] += Le;
      }
    }
  }
}

void build_slot_exchange(vb_ctx *c, SlotExchange &X, const std::function<int64_t(int)> &L,
                         const std::function<void(int, std::vector<int64_t> &)> &pos, int mode) {
  const int R = c->nranks, me = c->rank;
  const int ne = c->ents.size();
  X.ent_ptr.assign(ne + 1, 0);
  for (int e = 0; e < ne; ++e) X.ent_ptr[e + 1] = X.ent_ptr[e] + c->ents[e].sharers.size();
  X.recv_off.assign(X.ent_ptr[ne], -1);
  X.xfers.clear();
  X.send_len = X.recv_len = 0;
  if (R == 1) return;
  std::vector<int64_t> sidx;
  int64_t roff = 0;
  for (int p = 0; p < R; ++p) {
    if (p == me) continue;
    PeerXfer x{p, (int64_t)sidx.size(), 0, roff, 0};
    for (int e = 0; e < ne; ++e) {
      const Entity &E = c->ents[e];
      bool shared = false;
      for (int m : E.sharers) shared |= c->sub_rank[m] == p;
      if (!shared) continue;
      const int64_t Le = L(e);
      int li = 0;   // index among the local sharers = slot offset from side_begin
      for (size_t k = 0; k < E.sharers.size(); ++k) {
        const int m = E.sharers[k];
        if (c->sub_rank[m] != me) continue;
        if (xch_sends(c, e, k, mode)) {
          const size_t before = sidx.size();
          pos(c->h_ent[e].side_begin + li, sidx);
          VB_REQUIRE((int64_t)(sidx.size() - before) == Le, VB_EINVAL, "internal: slot payload length mismatch");
        }
        ++li;
      }
      for (size_t k = 0; k < E.sharers.size(); ++k) {
        const int m = E.sharers[k];
        if (c->sub_rank[m] != p || !xch_sends(c, e, k, mode)) continue;
        X.recv_off[X.ent_ptr[e] + k] = roff;
        roff += Le;
      }
    }
    x.scount = sidx.size() - x.soff;
    x.rcount = roff - x.roff;
    if (x.scount || x.rcount) X.xfers.push_back(x);
  }
  X.send_len = sidx.size();
  X.recv_len = roff;
  std::vector<int64_t> ps, pr;
  plan_slot_counts(c, L, mode, ps, pr);
  for (const PeerXfer &x : X.xfers)
    VB_REQUIRE(x.scount == ps[x.peer] && x.rcount == pr[x.peer], VB_EINVAL, "internal: exchange differs from its plan");
  X.send_idx.upload(sidx, c->stream);
  X.h_send_idx = sidx;
  X.sendbuf.alloc(std::max<int64_t>(X.send_len, 1));
  VB_CUDA(cudaStreamSynchronize(c->stream));
}

void run_slot_exchange(vb_ctx *c, SlotExchange &X, const double *local, double *recv) {
  // every rank takes part, even with nothing to move: the loopback transport's exchange is a
  // collective (a rank skipping it would pair its next collective with the others' exchange);
  // the NCCL transport returns at once for an empty peer list (point-to-point semantics)
  if (c->nranks == 1) return;
  if (X.send_len) {
    const int grid = (int)std::min<int64_t>((X.send_len + 255) / 256, 148 * 8);
    pack_kernel<<<grid, 256, 0, c->stream>>>(local, X.send_idx.p, X.send_len, X.sendbuf.p);
    VB_CHECK_LAUNCH();
  }
  c->comm->exchange(X.xfers, X.sendbuf.p, recv, c->stream);
}

void build_slot_p2p(vb_ctx *c, SlotExchange &X, double *alloc, int64_t recv_at, int64_t local_len) {
  const int R = c->nranks, me = c->rank;
  X.p2p = false;
  if (R == 1) return;
  cudaStream_t s = c->stream;
  // table of every rank: [recv_at, receive offset of the payload from rank 0 .. R-1 (-1: none),
  // its length from rank 0 .. R-1]  (int64 bit patterns moved as doubles)
  const int W = 2 * R + 1;
  std::vector<int64_t> mine(W, -1), all((size_t)R * W);
  mine[0] = recv_at;
  for (int r = 0; r < R; ++r) mine[1 + R + r] = 0;
  for (const PeerXfer &x : X.xfers) {
    mine[1 + x.peer] = x.roff;
    mine[1 + R + x.peer] = x.rcount;
  }
  DBuf<double> t;
  t.alloc((size_t)(R + 1) * W);
  VB_CUDA(cudaMemcpyAsync(t.p + (size_t)R * W, mine.data(), W * 8, cudaMemcpyHostToDevice, s));
  c->comm->allgather(t.p + (size_t)R * W, t.p, W, s);
  VB_CUDA(cudaMemcpyAsync(all.data(), t.p, all.size() * 8, cudaMemcpyDeviceToHost, s));
  std::vector<void *> base;
  c->comm->share_buffer(alloc, base, s);   // (synchronises s)
  std::vector<std::pair<int64_t, double *>> route;
  for (const PeerXfer &x : X.xfers) {
    if (!x.scount) continue;
    const int64_t *T = all.data() + (size_t)x.peer * W;
    VB_REQUIRE(T[1 + me] >= 0 && T[1 + R + me] == x.scount && base[x.peer], VB_ENCCL,
               "peer-store plans disagree between ranks");
    double *dst = (double *)base[x.peer] + T[0] + T[1 + me];
    for (int64_t i = 0; i < x.scount; ++i) {
      const int64_t j = X.h_send_idx[x.soff + i];
      VB_REQUIRE(j >= 0 && j < local_len, VB_EINVAL, "internal: peer-store source outside the local buffer");
      route.push_back({j, dst + i});
    }
  }
  std::vector<int> ptr(local_len + 1, 0);
  for (auto &r : route) ++ptr[r.first + 1];
  for (int64_t j = 0; j < local_len; ++j) ptr[j + 1] += ptr[j];
  std::vector<double *> dst(std::max<size_t>(route.size(), 1), nullptr);
  std::vector<int> fill(ptr.begin(), ptr.end() - 1);
  for (auto &r : route) dst[fill[r.first]++] = r.second;
  X.p2p_ptr.upload(ptr, s);
  X.p2p_dst.upload(dst, s);
  VB_CUDA(cudaStreamSynchronize(s));
  X.p2p = true;
}

__global__ void entity_sum_kernel(const int64_t *__restrict__ ptr, const int64_t *__restrict__ off,
                                  const int64_t *__restrict__ out_off, const int64_t *__restrict__ init_off,
                                  const int *__restrict__ len, const double *__restrict__ src,
                                  const double *__restrict__ init, double *out) {
  const int e = blockIdx.x;
  const int n = len[e];
  const int64_t q0 = ptr[e], q1 = ptr[e + 1];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double v = init ? init[init_off[e] + i] : 0.0;
    for (int64_t q = q0; q < q1; ++q) v += src[off[q] + i];
    out[out_off[e] + i] = v;
  }
}

void build_entity_sum(vb_ctx *c, EntitySum &S, const SlotExchange &X, const std::function<int64_t(int)> &L,
                      const std::function<int64_t(int)> &slot_base, int64_t local_len,
                      const std::function<int64_t(int)> &out_base, const std::function<int64_t(int)> *init_base,
                      int mode) {
  const int ne = c->ents.size();
  std::vector<int64_t> ptr(1, 0), off, oo(ne), io(ne, 0);
  std::vector<int> len(ne);
  S.maxlen = 1;
  for (int e = 0; e < ne; ++e) {
    const Entity &E = c->ents[e];
    int li = 0;
    for (size_t k = 0; k < E.sharers.size(); ++k) {
      const bool local = c->sub_lid[E.sharers[k]] >= 0;
      if (local) {
        if (xch_sends(c, e, k, mode)) off.push_back(slot_base(c->h_ent[e].side_begin + li));
        ++li;
      } else if (!xch_sends(c, e, k, mode)) {
        continue;
      } else if (!X.recv_off.empty() && X.recv_off[X.ent_ptr[e] + k] >= 0) {
        off.push_back(local_len + X.recv_off[X.ent_ptr[e] + k]);
      } else {
        VB_REQUIRE(false, VB_EINVAL, "internal: remote sharer without received payload");
      }
    }
    ptr.push_back(off.size());
    oo[e] = out_base(e);
    if (init_base) io[e] = (*init_base)(e);
    len[e] = L(e);
    S.maxlen = std::max<int>(S.maxlen, len[e]);
  }
  S.n = ne;
  cudaStream_t s = c->stream;
  S.ptr.upload(ptr, s);
  if (off.empty()) off.push_back(0);
  S.off.upload(off, s);
  S.out_off.upload(oo, s);
  S.init_off.upload(io, s);
  S.len.upload(len, s);
  VB_CUDA(cudaStreamSynchronize(s));
}

void run_entity_sum(vb_ctx *c, const EntitySum &S, const double *src, double *out, const double *init) {
  if (!S.n) return;
  entity_sum_kernel<<<S.n, S.maxlen > 64 ? 256 : 64, 0, c->stream>>>(S.ptr.p, S.off.p, S.out_off.p, S.init_off.p, S.len.p, src,
                                                          init, out);
  VB_CHECK_LAUNCH();
}

void allreduce_sum_fixed(vb_ctx *c, double *v, int k) {
  if (c->nranks == 1) return;
  if (c->w_red.n < (size_t)(c->nranks * k)) c->w_red.alloc((size_t)c->nranks * std::max(k, 8));
  c->comm->allgather(v, c->w_red.p, k, c->stream);
  rank_sum_kernel<<<1, 32, 0, c->stream>>>(c->w_red.p, c->nranks, k, v);
  VB_CHECK_LAUNCH();
}

}  // namespace vb
