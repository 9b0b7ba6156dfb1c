// Rebalancing transports (see comm.h).
#include "comm.h"

#include <dlfcn.h>

#include "drb.h"

#include <condition_variable>
#include <map>
#include <mutex>

namespace dycl {
namespace {

// ---- NCCL, resolved at run time (ABI of nccl.h; enum values are part of NCCL's stable ABI)
typedef int ncclResult_t;       // 0 == ncclSuccess
typedef void* ncclComm_t;
enum { NCCL_INT8 = 0, NCCL_INT32 = 2 };
struct NcclUid {
  char internal[128];
};

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*GetUniqueId)(NcclUid*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, NcclUid, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // symmetric windows (NCCL >= 2.27; optional: only the device-initiated rebalancing needs them)
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*WindowRegister)(ncclComm_t, void*, size_t, void**, int) = nullptr;
  ncclResult_t (*WindowDeregister)(ncclComm_t, void*) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // the NCCL already mapped in this process (torch's) first: a borrowed communicator must be
    // driven by the library instance that created it
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
#define SYM(field, name)                                                      \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));          \
  if (!api.field) {                                                           \
    api.why = std::string("NCCL symbol missing: ") + name;                    \
    return;                                                                   \
  }
    SYM(AllGather, "ncclAllGather");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.MemAlloc = reinterpret_cast<decltype(api.MemAlloc)>(dlsym(h, "ncclMemAlloc"));
    api.MemFree = reinterpret_cast<decltype(api.MemFree)>(dlsym(h, "ncclMemFree"));
    api.WindowRegister = reinterpret_cast<decltype(api.WindowRegister)>(dlsym(h, "ncclCommWindowRegister"));
    api.WindowDeregister = reinterpret_cast<decltype(api.WindowDeregister)>(dlsym(h, "ncclCommWindowDeregister"));
    api.ok = true;
  });
  return api;
}

bool nccl_err(ncclResult_t r, const char* where, std::string* err) {
  if (r == 0) return true;
  *err = std::string(where) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error");
  return false;
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int* d_all = nullptr;
  int* h_all = nullptr;
  void* win_buf = nullptr;                         // ncclMemAlloc'd symmetric window
  void* win = nullptr;                             // its ncclWindow_t
  void** peers = nullptr;                          // device [world] LSA peer pointers
  size_t win_bytes = 0;

  ~NcclTransport() override {
    if (d_all) cudaFree(d_all);
    if (h_all) cudaFreeHost(h_all);
    if (win && nccl().WindowDeregister) nccl().WindowDeregister(comm, win);
    if (win_buf && nccl().MemFree) nccl().MemFree(win_buf);
    if (peers) cudaFree(peers);
  }
  bool window(size_t bytes, void** local, void*** peers_dev, std::string* err) override {
    const NcclApi& A = nccl();
    if (!win) {
      if (!A.MemAlloc || !A.WindowRegister) {
        *err = "device rebalancing needs NCCL symmetric windows (ncclMemAlloc / ncclCommWindowRegister)";
        return false;
      }
      if (!nccl_err(A.MemAlloc(&win_buf, bytes), "ncclMemAlloc", err)) return false;
      if (cudaMemset(win_buf, 0, bytes) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        *err = "window clear failed";
        return false;
      }
      if (!nccl_err(A.WindowRegister(comm, win_buf, bytes, &win, 1 /* NCCL_WIN_COLL_SYMMETRIC */),
                    "ncclCommWindowRegister", err))
        return false;
      if (cudaMalloc(reinterpret_cast<void**>(&peers), world * sizeof(void*)) != cudaSuccess ||
          drb_nccl_peers(win, world, peers, 0) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
        *err = "window peer table failed";
        return false;
      }
      win_bytes = bytes;
    } else if (bytes > win_bytes) {
      *err = "window size changed";
      return false;
    }
    *local = win_buf;
    *peers_dev = peers;
    return true;
  }
  bool allgather_int(const int* dev_val, int* host_out, cudaStream_t st, std::string* err) override {
    const NcclApi& A = nccl();
    if (!d_all) {
      if (cudaMalloc(&d_all, world * sizeof(int)) != cudaSuccess ||
          cudaMallocHost(&h_all, world * sizeof(int)) != cudaSuccess) {
        *err = "rebalance: allocation of the count buffers failed";
        return false;
      }
    }
    if (!nccl_err(A.AllGather(dev_val, d_all, 1, NCCL_INT32, comm, st), "ncclAllGather", err)) return false;
    cudaError_t e = cudaMemcpyAsync(h_all, d_all, world * sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      *err = std::string("rebalance count read: ") + cudaGetErrorString(e);
      return false;
    }
    for (int r = 0; r < world; ++r) host_out[r] = h_all[r];
    return true;
  }
  bool exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st,
                std::string* err) override {
    const NcclApi& A = nccl();
    if (!nccl_err(A.GroupStart(), "ncclGroupStart", err)) return false;
    for (const Msg& m : sends)
      if (m.bytes && !nccl_err(A.Send(m.ptr, m.bytes, NCCL_INT8, m.peer, comm, st), "ncclSend", err)) {
        A.GroupEnd();
        return false;
      }
    for (const Msg& m : recvs)
      if (m.bytes && !nccl_err(A.Recv(m.ptr, m.bytes, NCCL_INT8, m.peer, comm, st), "ncclRecv", err)) {
        A.GroupEnd();
        return false;
      }
    return nccl_err(A.GroupEnd(), "ncclGroupEnd", err);
  }
};

}  // namespace

// ---- in-process transport
struct LocalGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<int> ints;
  // (src, dst) -> that step's send buffers in posting order (matched to receives in order,
  // as NCCL matches several sends between one pair of ranks)
  std::map<std::pair<int, int>, std::vector<Transport::Msg>> posted;
  std::vector<void*> wins;                         // device windows (device-initiated rebalancing)
  std::vector<int> win_dev;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {
struct LocalTransport : Transport {
  LocalGroup* g = nullptr;
  void* win = nullptr;
  void** peers = nullptr;
  size_t win_bytes = 0;
  ~LocalTransport() override {
    if (win) cudaFree(win);
    if (peers) cudaFree(peers);
  }
  bool window(size_t bytes, void** local, void*** peers_dev, std::string* err) override {
    if (!win) {
      int dev = 0;
      cudaGetDevice(&dev);
      if (cudaMalloc(&win, bytes) != cudaSuccess || cudaMemset(win, 0, bytes) != cudaSuccess ||
          cudaDeviceSynchronize() != cudaSuccess) {
        *err = "local window allocation failed";
        return false;
      }
      {
        std::lock_guard<std::mutex> lk(g->mu);
        g->wins[rank] = win;
        g->win_dev[rank] = dev;
      }
      g->barrier();
      std::vector<void*> all;
      std::vector<int> devs;
      {
        std::lock_guard<std::mutex> lk(g->mu);
        all = g->wins;
        devs = g->win_dev;
      }
      for (int r = 0; r < world; ++r)
        if (devs[r] != dev) {
          const cudaError_t e = cudaDeviceEnablePeerAccess(devs[r], 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            *err = "local window: peer access";
            return false;
          }
          cudaGetLastError();
        }
      if (cudaMalloc(reinterpret_cast<void**>(&peers), world * sizeof(void*)) != cudaSuccess ||
          cudaMemcpy(peers, all.data(), world * sizeof(void*), cudaMemcpyHostToDevice) != cudaSuccess) {
        *err = "local window: peer table";
        return false;
      }
      win_bytes = bytes;
      g->barrier();
    } else if (bytes > win_bytes) {
      *err = "window size changed";
      return false;
    }
    *local = win;
    *peers_dev = peers;
    return true;
  }
  bool allgather_int(const int* dev_val, int* host_out, cudaStream_t st, std::string* err) override {
    int v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, dev_val, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      *err = std::string("local allgather: ") + cudaGetErrorString(e);
      return false;
    }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      g->ints[rank] = v;
    }
    g->barrier();
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (int r = 0; r < world; ++r) host_out[r] = g->ints[r];
    }
    g->barrier();                                   // nobody overwrites ints before all have read
    return true;
  }
  bool exchange(const std::vector<Msg>& sends, const std::vector<Msg>& recvs, cudaStream_t st,
                std::string* err) override {
    cudaError_t e = cudaStreamSynchronize(st);     // send buffers are complete
    if (e != cudaSuccess) {
      *err = std::string("local exchange: ") + cudaGetErrorString(e);
      return false;
    }
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (const Msg& m : sends) g->posted[{rank, m.peer}].push_back(m);
    }
    g->barrier();
    bool ok = true;
    std::map<int, size_t> next;                     // per source rank: next posted message
    for (const Msg& m : recvs) {
      Msg src{};
      {
        std::lock_guard<std::mutex> lk(g->mu);
        auto it = g->posted.find({m.peer, rank});
        const size_t k = next[m.peer]++;
        if (it == g->posted.end() || k >= it->second.size() || it->second[k].bytes != m.bytes) {
          *err = "local exchange: unmatched message";
          ok = false;
          break;
        }
        src = it->second[k];
      }
      if (m.bytes && cudaMemcpyAsync(m.ptr, src.ptr, m.bytes, cudaMemcpyDefault, st) != cudaSuccess) {
        *err = "local exchange: copy failed";
        ok = false;
        break;
      }
    }
    e = cudaStreamSynchronize(st);
    if (ok && e != cudaSuccess) {
      *err = std::string("local exchange: ") + cudaGetErrorString(e);
      ok = false;
    }
    g->barrier();                                   // all copies done: senders may reuse buffers
    {
      std::lock_guard<std::mutex> lk(g->mu);
      for (const Msg& m : sends) g->posted.erase({rank, m.peer});   // (idempotent per peer)
    }
    g->barrier();
    return ok;
  }
};
}  // namespace

Transport* make_nccl_transport(void* nccl_comm, int rank, int world, std::string* err) {
  if (!nccl().ok) {
    *err = nccl().why;
    return nullptr;
  }
  NcclTransport* t = new NcclTransport();
  t->comm = nccl_comm;
  t->rank = rank;
  t->world = world;
  return t;
}

LocalGroup* local_group_create(int world) {
  LocalGroup* g = new LocalGroup();
  g->world = world;
  g->ints.assign(world, 0);
  g->wins.assign(world, nullptr);
  g->win_dev.assign(world, 0);
  return g;
}
void local_group_destroy(LocalGroup* g) { delete g; }
int local_group_world(const LocalGroup* g) { return g->world; }

Transport* make_local_transport(LocalGroup* g, int rank) {
  LocalTransport* t = new LocalTransport();
  t->g = g;
  t->rank = rank;
  t->world = g->world;
  return t;
}

bool nccl_get_unique_id(uint8_t out[128], std::string* err) {
  if (!nccl().ok) {
    *err = nccl().why;
    return false;
  }
  NcclUid id{};
  if (!nccl_err(nccl().GetUniqueId(&id), "ncclGetUniqueId", err)) return false;
  for (int i = 0; i < 128; ++i) out[i] = (uint8_t)id.internal[i];
  return true;
}

bool nccl_comm_init_rank(const uint8_t idb[128], int rank, int world, void** comm, std::string* err) {
  if (!nccl().ok) {
    *err = nccl().why;
    return false;
  }
  NcclUid id{};
  for (int i = 0; i < 128; ++i) id.internal[i] = (char)idb[i];
  ncclComm_t c = nullptr;
  if (!nccl_err(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank", err)) return false;
  *comm = c;
  return true;
}

bool nccl_comm_destroy(void* comm, std::string* err) {
  if (!nccl().ok) {
    *err = nccl().why;
    return false;
  }
  return nccl_err(nccl().CommDestroy(comm), "ncclCommDestroy", err);
}

}  // namespace dycl
