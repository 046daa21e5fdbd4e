// comm.cu — NCCL (dlopen) and loopback implementations of Comm.
//
// The bin shuffle is the path's only partition point: an
// all-gather of the per-bin histograms, then a grouped ncclSend/ncclRecv
// all-to-allv of super-mer descriptors and payload over NVLink 5 / NVSwitch.
// NCCL is loaded at run time (the process may already hold torch's copy of
// libnccl.so.2; RTLD_NOLOAD picks that one first).
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <map>
#include <thread>
#include <memory>
#include <mutex>
#include <vector>

#include "comm.h"

namespace gerbil {
namespace {

// ---------------------------------------------------------------- NCCL ----
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*);  // optional
  ncclResult_t (*CommAbort)(ncclComm_t);                          // optional
};

NcclApi* nccl_api(std::string& err) {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SYM(n) api.n = reinterpret_cast<decltype(api.n)>(dlsym(h, "nccl" #n))
    SYM(GetUniqueId); SYM(CommInitRank); SYM(CommDestroy); SYM(AllGather); SYM(Send);
    SYM(Recv); SYM(GroupStart); SYM(GroupEnd); SYM(GetErrorString); SYM(CommGetAsyncError); SYM(CommAbort);
#undef SYM
    api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather &&
             api.Send && api.Recv && api.GroupStart && api.GroupEnd && api.GetErrorString;
  });
  if (!api.ok) {
    err = "libnccl.so.2 could not be loaded";
    return nullptr;
  }
  return &api;
}

class NcclComm : public Comm {
 public:
  NcclApi* api = nullptr;
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) api->CommDestroy(comm);
  }
  bool check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return true;
    err = std::string(what) + ": " + api->GetErrorString(r);
    return false;
  }
  // Wait for the collective on st, polling NCCL's asynchronous error state; a peer that never
  // arrives (dead rank) ends in a timeout (GERBIL_NCCL_TIMEOUT_S, default 600 s) and an abort,
  // so the call fails instead of hanging.
  bool wait(cudaStream_t st, const char* what) {
    static const double limit = [] {
      const char* e = getenv("GERBIL_NCCL_TIMEOUT_S");
      return (e && *e) ? atof(e) : 600.0;
    }();
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0;; ++spin) {
      const cudaError_t q = cudaStreamQuery(st);
      if (q == cudaSuccess) return true;
      if (q != cudaErrorNotReady) {
        err = std::string(what) + ": " + cudaGetErrorString(q);
        return false;
      }
      if (api->CommGetAsyncError) {
        ncclResult_t ae = ncclSuccess;
        if (api->CommGetAsyncError(comm, &ae) == ncclSuccess && ae != ncclSuccess && ae != ncclInProgress) {
          err = std::string(what) + ": asynchronous NCCL error: " + api->GetErrorString(ae);
          if (api->CommAbort) api->CommAbort(comm);
          comm = nullptr;
          return false;
        }
      }
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > limit) {
        err = std::string(what) + ": timed out waiting for the peers (GERBIL_NCCL_TIMEOUT_S)";
        if (api->CommAbort) api->CommAbort(comm);
        comm = nullptr;
        return false;
      }
      if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }
  bool allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    if (!comm) {
      err = "NCCL communicator aborted by an earlier error";
      return false;
    }
    if (!check(api->AllGather(s, r, bytes, ncclUint8, comm, st), "ncclAllGather")) return false;
    return wait(st, "ncclAllGather");
  }
  bool alltoallv(const void* s, const size_t* so, const size_t* sb, void* r, const size_t* ro,
                 const size_t* rb, cudaStream_t st) override {
    Xfer x{s, so, sb, r, ro, rb};
    return alltoallv_multi(&x, 1, st);
  }
  bool alltoallv_multi(const Xfer* x, int n, cudaStream_t st) override {
    if (!comm) {
      err = "NCCL communicator aborted by an earlier error";
      return false;
    }
    if (!check(api->GroupStart(), "ncclGroupStart")) return false;
    for (int p = 0; p < world; ++p)
      for (int b = 0; b < n; ++b) {
        const size_t sb = x[b].send_bytes[p], rb = x[b].recv_bytes[p];
        if (sb && !check(api->Send((const char*)x[b].send + x[b].send_off[p], sb, ncclUint8, p, comm, st),
                         "ncclSend")) {
          api->GroupEnd();
          return false;
        }
        if (rb && !check(api->Recv((char*)x[b].recv + x[b].recv_off[p], rb, ncclUint8, p, comm, st),
                         "ncclRecv")) {
          api->GroupEnd();
          return false;
        }
      }
    if (!check(api->GroupEnd(), "ncclGroupEnd")) return false;
    return wait(st, "grouped ncclSend/ncclRecv");
  }
};

// ------------------------------------------------------------ loopback ----
struct LoopGroup {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned gen = 0;
  std::vector<const void*> send;
  std::vector<const size_t*> soff, sbytes;
  explicit LoopGroup(int w) : world(w), send(w), soff(w), sbytes(w) {}
  // false when the peers did not all arrive within GERBIL_LOOPBACK_TIMEOUT_S (default 120 s):
  // a virtual rank that failed and left the collective must not hang the others
  bool barrier() {
    static const long tmo = [] {
      const char* e = getenv("GERBIL_LOOPBACK_TIMEOUT_S");
      const long v = e ? atol(e) : 0;
      return v > 0 ? v : 120L;
    }();
    std::unique_lock<std::mutex> lk(mu);
    unsigned g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return true;
    }
    return cv.wait_for(lk, std::chrono::seconds(tmo), [&] { return gen != g; });
  }
};

std::mutex g_reg_mu;
std::map<std::string, std::weak_ptr<LoopGroup>> g_registry;

class LoopComm : public Comm {
 public:
  std::shared_ptr<LoopGroup> g;
  bool allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    g->send[rank] = s;
    if (!g->barrier()) {
      err = "loopback allgather: timed out waiting for the peers";
      return false;
    }
    bool ok = true;
    for (int p = 0; p < world; ++p)
      ok &= cudaMemcpyAsync((char*)r + p * bytes, g->send[p], bytes, cudaMemcpyDeviceToDevice, st) ==
            cudaSuccess;
    ok &= cudaStreamSynchronize(st) == cudaSuccess;
    if (!g->barrier()) {
      err = "loopback allgather: timed out waiting for the peers";
      return false;
    }
    if (!ok) err = "loopback allgather copy failed";
    return ok;
  }
  bool alltoallv(const void* s, const size_t* so, const size_t* sb, void* r, const size_t* ro,
                 const size_t* rb, cudaStream_t st) override {
    Xfer x{s, so, sb, r, ro, rb};
    return alltoallv_multi(&x, 1, st);
  }
  bool alltoallv_multi(const Xfer* x, int n, cudaStream_t st) override {
    bool ok = true;
    for (int b = 0; b < n; ++b) {
      g->send[rank] = x[b].send;
      g->soff[rank] = x[b].send_off;
      g->sbytes[rank] = x[b].send_bytes;
      if (!g->barrier()) {
        err = "loopback alltoallv: timed out waiting for the peers";
        return false;
      }
      for (int p = 0; p < world; ++p) {
        const size_t m = g->sbytes[p][rank];
        if (m != x[b].recv_bytes[p]) ok = false;
        if (m && ok)
          ok &= cudaMemcpyAsync((char*)x[b].recv + x[b].recv_off[p], (const char*)g->send[p] + g->soff[p][rank], m,
                                cudaMemcpyDeviceToDevice, st) == cudaSuccess;
      }
      ok &= cudaStreamSynchronize(st) == cudaSuccess;
      if (!g->barrier()) {
        err = "loopback alltoallv: timed out waiting for the peers";
        return false;
      }
    }
    if (!ok) err = "loopback alltoallv size mismatch or copy failure";
    return ok;
  }
};

}  // namespace

Comm* make_comm(int backend, const void* id, int rank, int world, std::string& err) {
  if (backend == 1) {
    std::string key((const char*)id, 128);
    std::shared_ptr<LoopGroup> g;
    {
      std::lock_guard<std::mutex> lk(g_reg_mu);
      auto it = g_registry.find(key);
      if (it != g_registry.end()) g = it->second.lock();
      if (!g) {
        g = std::make_shared<LoopGroup>(world);
        g_registry[key] = g;
      }
    }
    if (g->world != world) {
      err = "loopback group world size mismatch";
      return nullptr;
    }
    LoopComm* c = new LoopComm();
    c->g = g;
    c->rank = rank;
    c->world = world;
    return c;
  }
  NcclApi* api = nccl_api(err);
  if (!api) return nullptr;
  NcclComm* c = new NcclComm();
  c->api = api;
  c->rank = rank;
  c->world = world;
  ncclUniqueId uid;
  memcpy(uid.internal, id, sizeof uid.internal);
  ncclResult_t r = api->CommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + api->GetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

bool nccl_get_unique_id(void* out, std::string& err) {
  NcclApi* api = nccl_api(err);
  if (!api) return false;
  ncclUniqueId uid;
  ncclResult_t r = api->GetUniqueId(&uid);
  if (r != ncclSuccess) {
    err = std::string("ncclGetUniqueId: ") + api->GetErrorString(r);
    return false;
  }
  memcpy(out, uid.internal, sizeof uid.internal);
  return true;
}

}  // namespace gerbil
