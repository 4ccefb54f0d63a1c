// Transports of the multi-GPU path (comm.h).
#include <dlfcn.h>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include "comm.h"
#include "internal.h"

namespace vb {

// ------------------------------------------------------------------ NCCL (resolved at run time)
// Minimal NCCL ABI (nccl.h, stable since 2.7): opaque communicator, 128-byte unique id.
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclDouble = 8;

struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // prefer the copy already in the process (torch's), then the system one
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.h = h;
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  });
  VB_REQUIRE(api.h && api.GetUniqueId && api.CommInitRank && api.Send && api.Recv && api.AllGather &&
                 api.GroupStart && api.GroupEnd,
             VB_ENCCL, "libnccl.so.2 not found in the process (load torch first) or missing symbols");
  return api;
}

#define VB_NCCL(x)                                                                              \
  do {                                                                                          \
    ncclResult_t _r = (x);                                                                      \
    if (_r != 0)                                                                                \
      throw ::vb::Error{VB_ENCCL, std::string(#x) + ": " +                                      \
                                      (nccl().GetErrorString ? nccl().GetErrorString(_r) : "?")}; \
  } while (0)

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  bool capturable() const override { return true; }
  ~NcclComm() override {
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  void exchange(const std::vector<PeerXfer> &x, const double *send, double *recv, cudaStream_t s) override {
    if (x.empty()) return;
    NcclApi &a = nccl();
    VB_NCCL(a.GroupStart());
    for (const PeerXfer &p : x) {
      if (p.scount) VB_NCCL(a.Send(send + p.soff, p.scount, kNcclDouble, p.peer, comm, s));
      if (p.rcount) VB_NCCL(a.Recv(recv + p.roff, p.rcount, kNcclDouble, p.peer, comm, s));
    }
    VB_NCCL(a.GroupEnd());
  }
  void allgather(const double *send, double *recv, int64_t count, cudaStream_t s) override {
    if (count == 0) return;
    VB_NCCL(nccl().AllGather(send, recv, count, kNcclDouble, comm, s));
  }
};

int nccl_unique_id(void *out128) {
  ncclUniqueId id;
  VB_NCCL(nccl().GetUniqueId(&id));
  memcpy(out128, &id, 128);
  return 0;
}

Comm *make_nccl_comm(int rank, int nranks, const void *id128, int device) {
  VB_REQUIRE(id128, VB_EINVAL, "nranks > 1 needs the NCCL unique id from vb_nccl_unique_id (rank 0)");
  NcclApi &a = nccl();
  VB_CUDA(cudaSetDevice(device));
  ncclUniqueId id;
  memcpy(&id, id128, 128);
  NcclComm *c = new NcclComm();
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = a.CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    delete c;
    throw Error{VB_ENCCL, std::string("ncclCommInitRank: ") + (a.GetErrorString ? a.GetErrorString(r) : "?")};
  }
  return c;
}

// ------------------------------------------------------------------ loopback (threads, one GPU)
struct LoopWorld {
  int n = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  bool broken = false;
  std::vector<const double *> send;
  std::vector<const std::vector<PeerXfer> *> xfer;
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    if (broken) throw Error{VB_ENCCL, "loopback world broken by another rank's failure"};
    const int64_t gen = generation;
    if (++arrived == n) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen || broken; }) || broken) {
      broken = true;
      cv.notify_all();
      throw Error{VB_ENCCL, "loopback barrier timed out (a rank did not reach the exchange)"};
    }
  }
};

void *loopback_world_create(int nranks) {
  LoopWorld *w = new LoopWorld();
  w->n = nranks;
  w->send.assign(nranks, nullptr);
  w->xfer.assign(nranks, nullptr);
  return w;
}

void loopback_world_destroy(void *world) { delete (LoopWorld *)world; }

struct LoopComm : Comm {
  LoopWorld *w = nullptr;
  void abort() override {
    std::lock_guard<std::mutex> lk(w->m);
    w->broken = true;
    w->cv.notify_all();
  }
  void exchange(const std::vector<PeerXfer> &x, const double *send, double *recv, cudaStream_t s) override {
    VB_CUDA(cudaStreamSynchronize(s));
    w->send[rank] = send;
    w->xfer[rank] = &x;
    w->barrier();
    for (const PeerXfer &p : x) {
      if (!p.rcount) continue;
      const std::vector<PeerXfer> &px = *w->xfer[p.peer];
      const PeerXfer *mine = nullptr;
      for (const PeerXfer &q : px)
        if (q.peer == rank) mine = &q;
      VB_REQUIRE(mine && mine->scount == p.rcount, VB_ENCCL, "loopback exchange plans disagree between ranks");
      VB_CUDA(cudaMemcpyAsync(recv + p.roff, w->send[p.peer] + mine->soff, p.rcount * 8, cudaMemcpyDeviceToDevice, s));
    }
    VB_CUDA(cudaStreamSynchronize(s));
    w->barrier();
  }
  void allgather(const double *send, double *recv, int64_t count, cudaStream_t s) override {
    VB_CUDA(cudaStreamSynchronize(s));
    w->send[rank] = send;
    w->barrier();
    for (int r = 0; r < nranks; ++r)
      if (count) VB_CUDA(cudaMemcpyAsync(recv + (int64_t)r * count, w->send[r], count * 8, cudaMemcpyDeviceToDevice, s));
    VB_CUDA(cudaStreamSynchronize(s));
    w->barrier();
  }
};

Comm *make_loopback_comm(void *world, int rank) {
  LoopComm *c = new LoopComm();
  c->w = (LoopWorld *)world;
  c->rank = rank;
  c->nranks = c->w->n;
  return c;
}

}  // namespace vb
