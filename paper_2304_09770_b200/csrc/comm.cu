// Transports of the multi-GPU path (comm.h).
#include <dlfcn.h>
#include <chrono>
#include <condition_variable>
#include <cstring>
#include <cmath>
#include <memory>
#include <algorithm>
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
  ncclResult_t (*CommCount)(ncclComm_t, int *) = nullptr;
  ncclResult_t (*GetVersion)(int *) = nullptr;
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
    api.CommCount = (decltype(api.CommCount))dlsym(h, "ncclCommCount");
    api.GetVersion = (decltype(api.GetVersion))dlsym(h, "ncclGetVersion");
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
  DBuf<double> bar;                  // barrier operand (1 double per rank)
  std::vector<void *> opened;        // peer allocations mapped by share_buffer
  ~NcclComm() override {
    for (void *p : opened) cudaIpcCloseMemHandle(p);
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  // an allgather completes on a rank only after every rank has entered it, i.e. after every
  // rank's earlier stream work (kernel completion flushes its peer stores)
  void barrier(cudaStream_t s) override {
    VB_NCCL(nccl().AllGather(bar.p + nranks, bar.p, 1, kNcclDouble, comm, s));
  }
  // CUDA IPC: each rank exports its allocation, the handles travel by allgather, every peer's
  // allocation is mapped into this process (NVLink peer access enabled lazily by the driver)
  void share_buffer(void *mine, std::vector<void *> &out, cudaStream_t s) override {
    VB_REQUIRE(!g_use_pool, VB_EINVAL, "direct peer stores need cudaMalloc allocations (unset VB_POOL)");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    cudaIpcMemHandle_t h;
    VB_CUDA(cudaIpcGetMemHandle(&h, mine));
    DBuf<double> t;
    t.alloc((size_t)8 * (nranks + 1));
    VB_CUDA(cudaMemcpyAsync(t.p + 8 * nranks, &h, 64, cudaMemcpyHostToDevice, s));
    VB_NCCL(nccl().AllGather(t.p + 8 * nranks, t.p, 8, kNcclDouble, comm, s));
    std::vector<cudaIpcMemHandle_t> all(nranks);
    VB_CUDA(cudaMemcpyAsync(all.data(), t.p, 64 * (size_t)nranks, cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    out.assign(nranks, nullptr);
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) { out[r] = mine; continue; }
      VB_CUDA(cudaIpcOpenMemHandle(&out[r], all[r], cudaIpcMemLazyEnablePeerAccess));
      opened.push_back(out[r]);
    }
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
  // the PCG iteration graph captures the exchanges inside a conditional WHILE body, which takes
  // kernel/memcpy nodes only: keep NCCL from adding its graph-mixing event nodes (read at init;
  // a value set by the user wins)
  setenv("NCCL_GRAPH_MIXING_SUPPORT", "0", 0);
  ncclResult_t r = a.CommInitRank(&c->comm, nranks, id, rank);
  if (r != 0) {
    delete c;
    throw Error{VB_ENCCL, std::string("ncclCommInitRank: ") + (a.GetErrorString ? a.GetErrorString(r) : "?")};
  }
  int cnt = -1, ver = 0;
  if (a.CommCount) a.CommCount(c->comm, &cnt);
  if (a.GetVersion) a.GetVersion(&ver);
  fprintf(stderr, "[vb] NCCL communicator: rank %d nranks %d (ncclCommCount %d) device %d, NCCL %d\n", rank, nranks,
          cnt, device, ver);
  VB_REQUIRE(cnt < 0 || cnt == nranks, VB_ENCCL, "NCCL communicator size differs from nranks");
  c->bar.alloc(nranks + 1);   // (not inside a capture: barrier() may be captured)
  VB_CUDA(cudaMemset(c->bar.p, 0, (nranks + 1) * sizeof(double)));
  return c;
}

// ------------------------------------------------------------------ NCCL self-test (one GPU)
__global__ void selftest_step_kernel(double *a, int n, int *counter) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] += 1.0;
  if (threadIdx.x == 0) ++*counter;
}
__global__ void selftest_cond_kernel(const int *counter, int stop, cudaGraphConditionalHandle h) {
  cudaGraphSetConditional(h, *counter < stop ? 1u : 0u);
}

void nccl_selftest(int device, double *result, std::string &msg) {
  NcclApi &a = nccl();
  VB_CUDA(cudaSetDevice(device));
  result[0] = result[1] = result[2] = 0.0;
  result[3] = INFINITY;
  ncclUniqueId id;
  VB_NCCL(a.GetUniqueId(&id));
  NcclComm *cm = (NcclComm *)make_nccl_comm(0, 1, &id, device);
  std::unique_ptr<NcclComm> guard(cm);
  const int n = 4096;
  DBuf<double> buf;
  buf.alloc(3 * n);
  DBuf<int> counter;
  counter.alloc(1);
  cudaStream_t s;
  VB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::vector<double> h(3 * n);
  for (int i = 0; i < n; ++i) h[i] = 0.5 * i;
  VB_CUDA(cudaMemcpyAsync(buf.p, h.data(), n * 8, cudaMemcpyHostToDevice, s));
  counter.zero(s);
  const std::vector<PeerXfer> self{PeerXfer{0, 0, n, 0, n}};
  auto step = [&]() {   // a += 1; b <- a (send/recv to self); g <- allgather(a)
    selftest_step_kernel<<<1, 256, 0, s>>>(buf.p, n, counter.p);
    cm->exchange(self, buf.p, buf.p + n, s);
    cm->allgather(buf.p, buf.p + 2 * n, n, s);
    cm->barrier(s);
  };
  std::vector<void *> shared;   // IPC export of the buffer (the peer-store path's setup)
  cm->share_buffer(buf.p, shared, s);
  VB_REQUIRE(shared.size() == 1 && shared[0] == buf.p, VB_ENCCL, "share_buffer returned a wrong table");
  auto check = [&](int steps) {
    VB_CUDA(cudaMemcpyAsync(h.data(), buf.p, 3 * n * 8, cudaMemcpyDeviceToHost, s));
    VB_CUDA(cudaStreamSynchronize(s));
    double err = 0;
    for (int i = 0; i < n; ++i)
      err = std::max({err, fabs(h[i] - (0.5 * i + steps)), fabs(h[n + i] - h[i]), fabs(h[2 * n + i] - h[i])});
    return err;
  };
  step();
  double e1 = check(1);
  result[0] = e1 == 0.0;
  // the same step 3 times inside a conditional WHILE body (captured)
  cudaGraph_t g;
  VB_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hw;
  VB_CUDA(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp = {};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wnode;
  VB_CUDA(cudaGraphAddNode(&wnode, g, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphExec_t ge = nullptr;
  try {
    VB_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    try {
      step();
      selftest_cond_kernel<<<1, 1, 0, s>>>(counter.p, 4, hw);
    } catch (...) {
      cudaGraph_t dummy;
      cudaStreamEndCapture(s, &dummy);
      throw;
    }
    VB_CUDA(cudaStreamEndCapture(s, &body));
    VB_CUDA(cudaGraphInstantiate(&ge, g, 0));
    VB_CUDA(cudaGraphLaunch(ge, s));
    double e2 = check(4);
    int cnt = 0;
    VB_CUDA(cudaMemcpy(&cnt, counter.p, sizeof(int), cudaMemcpyDeviceToHost));
    result[1] = (e2 == 0.0 && cnt == 4) ? 1.0 : 0.0;
    result[2] = cnt - 1;
    result[3] = std::max(e1, e2);
  } catch (const Error &e) {
    (void)cudaGetLastError();
    msg = "NCCL capture in a conditional graph body failed: " + e.msg;
    result[3] = e1;
  }
  if (ge) cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
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
  std::vector<void *> shared;
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
  w->shared.assign(nranks, nullptr);
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
  void barrier(cudaStream_t s) override {
    VB_CUDA(cudaStreamSynchronize(s));
    w->barrier();
  }
  // all ranks live in one process on one device: the pointers themselves
  void share_buffer(void *mine, std::vector<void *> &out, cudaStream_t s) override {
    VB_CUDA(cudaStreamSynchronize(s));
    w->shared[rank] = mine;
    w->barrier();
    out = w->shared;
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
