// Interface exchanges between ranks: data attached to (entity, sharer) pairs
// ("slots") of interface entities shared by subdomains on different ranks.
#pragma once
#include <functional>
#include "internal.h"

namespace vb {

// A planned exchange: every local slot of an entity with a sharer on another rank sends L_e values
// (gathered from a local buffer at per-slot positions) to every other rank holding a sharer of the
// entity; the receiver gets, for every remote sharer of each of its entities, L_e values.
// Both sides derive the same ordering from the global topology: per peer, entities in global id
// order, then the sending rank's sharers of the entity in global subdomain order.
struct SlotExchange {
  std::vector<PeerXfer> xfers;
  DBuf<int64_t> send_idx;            // gather positions (into the local buffer) of the send buffer
  DBuf<double> sendbuf;
  int64_t send_len = 0, recv_len = 0;
  // recv_off[ent_ptr[e] + k] = offset in the receive area of sharer k (position in E.sharers) of
  // local entity e, or -1 when that sharer is local
  std::vector<int64_t> ent_ptr, recv_off;
  std::vector<int64_t> h_send_idx;   // host copy of send_idx
  // direct peer stores (build_slot_p2p): the producing kernel stores local position j's value at
  // every address p2p_dst[p2p_ptr[j] .. p2p_ptr[j+1]) (inside peers' receive areas), then a
  // stream barrier replaces pack + send/recv
  bool p2p = false;
  DBuf<int> p2p_ptr;
  DBuf<double *> p2p_dst;
};

// L(e): payload length per slot of local entity e; pos(slot, out): the local buffer positions of
// the slot's L values (appended to out).  mode: which sharers send a payload --
//   XCH_ALL: every sharer;  XCH_OWNER: only the entity's lowest sharer;
//   XCH_RANK: only the lowest sharer on each rank (one payload per rank: rank partial sums).
enum { XCH_ALL = 0, XCH_OWNER = 1, XCH_RANK = 2 };
void build_slot_exchange(vb_ctx *c, SlotExchange &X, const std::function<int64_t(int)> &L,
                         const std::function<void(int, std::vector<int64_t> &)> &pos, int mode = XCH_ALL);
// Host-only plan of the same exchange: doubles sent to / received from every rank (size nranks).
// build_slot_exchange checks its transfers against this plan.
void plan_slot_counts(const vb_ctx *c, const std::function<int64_t(int)> &L, int mode, std::vector<int64_t> &send,
                      std::vector<int64_t> &recv);
// does sharer k of local entity e send under `mode`?
bool xch_sends(const vb_ctx *c, int e, int k, int mode);
// pack from `local`, exchange, receive into `recv` (recv_len doubles).  No-op for one rank.
void run_slot_exchange(vb_ctx *c, SlotExchange &X, const double *local, double *recv);
// Direct peer stores for X (collective): `alloc` is this rank's cudaMalloc allocation holding the
// receive area at element offset `recv_at`; local positions are < local_len.  Each rank learns
// where its payload lands in every peer's receive area (the peer's recv offset for it) and maps
// the peers' allocations (Comm::share_buffer).
void build_slot_p2p(vb_ctx *c, SlotExchange &X, double *alloc, int64_t recv_at, int64_t local_len);

// Per-entity sums over ALL sharers (global subdomain order) of slot payloads that live either in
// a local buffer (contiguous per slot) or in the receive area of a SlotExchange:
//   out[out_off[e] + i] = init[init_off[e] + i] (optional) + sum_k src[src_off[e][k] + i], i < len[e]
// where src = [local buffer (local_len) | receive area].
struct EntitySum {
  DBuf<int64_t> ptr, off, out_off, init_off;
  DBuf<int> len;
  int n = 0, maxlen = 0;
};
void build_entity_sum(vb_ctx *c, EntitySum &S, const SlotExchange &X, const std::function<int64_t(int)> &L,
                      const std::function<int64_t(int)> &slot_base, int64_t local_len,
                      const std::function<int64_t(int)> &out_base,
                      const std::function<int64_t(int)> *init_base = nullptr, int mode = XCH_ALL);
void run_entity_sum(vb_ctx *c, const EntitySum &S, const double *src, double *out, const double *init = nullptr);

// out[k] = src[idx[k]]  /  out[idx[k]] = src[k]   (k < n)
void dev_gather(const double *src, const int64_t *idx, int64_t n, double *out, cudaStream_t s);
void dev_scatter(const double *src, const int64_t *idx, int64_t n, double *out, cudaStream_t s);

// deterministic fixed-order sum of per-rank partial scalars (C3): v[0..k) <- sum over ranks
void allreduce_sum_fixed(vb_ctx *c, double *dev_vals, int k);

}  // namespace vb
