// Inter-rank transport of the multi-GPU path (C1 interface sums, C2 coarse-rhs
// gather, C3 dot partials, C4 local coarse matrices).  One rank per GPU.  Two transports:
//   * NCCL over NVLink/NVSwitch (the product path): libnccl is resolved at run time from the
//     process (torch already loaded it) so the library carries no link-time NCCL dependency;
//   * loopback: R ranks as R threads of ONE process sharing one GPU, exchanging through
//     host-synchronised device-to-device copies (test infrastructure: lets the partitioned data
//     path run against the oracle on a single GPU; no kernel ever waits on another rank).
#pragma once
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

namespace vb {

struct PeerXfer {          // one peer of a grouped point-to-point exchange (doubles)
  int peer;
  int64_t soff, scount;    // slice of the send buffer for this peer
  int64_t roff, rcount;    // slice of the receive buffer from this peer
};

struct Comm {
  int rank = 0, nranks = 1;
  virtual ~Comm() {}
  // grouped send/recv with every listed peer, on stream s (stream-ordered)
  virtual void exchange(const std::vector<PeerXfer> &x, const double *send, double *recv, cudaStream_t s) = 0;
  // every rank contributes `count` doubles; recv holds nranks * count in rank order
  virtual void allgather(const double *send, double *recv, int64_t count, cudaStream_t s) = 0;
  // stream-ordered barrier: work any rank enqueued on its stream before the barrier (including
  // stores into peer memory) is complete and visible before work any rank enqueues after it runs
  virtual void barrier(cudaStream_t s) = 0;
  // direct peer stores: out[r] = the address, usable from THIS rank's kernels, of the buffer
  // rank r passed as `mine` (a cudaMalloc allocation base; out[rank] = mine).  Collective.
  virtual void share_buffer(void *mine, std::vector<void *> &out, cudaStream_t s) = 0;
  virtual void abort() {}
  virtual bool capturable() const { return false; }   // may run inside CUDA stream capture
};

Comm *make_nccl_comm(int rank, int nranks, const void *unique_id128, int device);
Comm *make_loopback_comm(void *world, int rank);
void *loopback_world_create(int nranks);
void loopback_world_destroy(void *world);
int nccl_unique_id(void *out128);   // 0 on success
// vb_debug_nccl_selftest: result[4] = {eager ok, graph ok, graph iterations, max abs error}
void nccl_selftest(int device, double *result, std::string &msg);

}  // namespace vb
