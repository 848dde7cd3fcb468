// transport.cpp — collectives of the expert-parallel decode step (transport.h).
#include "transport.h"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>

#include "capi_util.h"

namespace ef {
namespace {

#define CKT(expr)                                                                         \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) throw CudaErr(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

struct LocalTransport : Transport {
  void allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    if (s != r) CKT(cudaMemcpyAsync(r, s, bytes, cudaMemcpyDeviceToDevice, st));
  }
  void alltoall(const void* s, void* r, size_t chunk, cudaStream_t st) override {
    if (s != r) CKT(cudaMemcpyAsync(r, s, chunk, cudaMemcpyDeviceToDevice, st));
  }
  const char* name() const override { return "local"; }
};

// ---- NCCL, resolved at run time: the ABI below is NCCL 2.x's (nccl.h);
// torch has already mapped its libnccl.so.2, so dlopen returns that copy.
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
enum { kNcclInt8 = 0, kNcclSuccess = 0 };
struct Nccl {
  int (*GetUniqueId)(ncclUniqueId*);
  int (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  int (*CommDestroy)(ncclComm_t);
  int (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t);
  int (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t);
  int (*GroupStart)();
  int (*GroupEnd)();
  const char* (*GetErrorString)(int);
};

const Nccl& nccl() {
  static Nccl n{};
  static bool loaded = false;
  if (loaded) return n;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw RuntimeErr(std::string("expert parallelism needs libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* s) {
    void* p = dlsym(h, s);
    if (!p) throw RuntimeErr(std::string("libnccl.so.2 lacks ") + s);
    return p;
  };
  n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
  n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
  n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
  n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
  n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
  n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
  n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
  n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
  n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  loaded = true;
  return n;
}

void nck(int r, const char* what) {
  if (r != kNcclSuccess)
    throw RuntimeErr(std::string(what) + ": " + nccl().GetErrorString(r));
}

struct NcclTransport : Transport {
  ncclComm_t comm = nullptr;
  int world, rank;
  NcclTransport(int w, int r, const void* id128) : world(w), rank(r) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    nck(nccl().CommInitRank(&comm, w, id, r), "ncclCommInitRank");
  }
  ~NcclTransport() override {
    if (comm) nccl().CommDestroy(comm);
  }
  void allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    nck(nccl().AllGather(s, r, bytes, kNcclInt8, comm, st), "ncclAllGather");
  }
  void alltoall(const void* s, void* r, size_t chunk, cudaStream_t st) override {
    const auto& n = nccl();
    nck(n.GroupStart(), "ncclGroupStart");
    for (int g = 0; g < world; ++g) {
      nck(n.Send(static_cast<const char*>(s) + g * chunk, chunk, kNcclInt8, g, comm, st), "ncclSend");
      nck(n.Recv(static_cast<char*>(r) + g * chunk, chunk, kNcclInt8, g, comm, st), "ncclRecv");
    }
    nck(n.GroupEnd(), "ncclGroupEnd");
  }
  const char* name() const override { return "nccl"; }
};

struct CallbackTransport : Transport {
  ef_collective_cb cb;
  void* user;
  CallbackTransport(ef_collective_cb c, void* u) : cb(c), user(u) {}
  void call(int op, const void* s, void* r, size_t n, cudaStream_t st) {
    if (cb(user, op, const_cast<void*>(s), r, (int64_t)n, st) != 0)
      throw RuntimeErr("expert-parallel collective callback failed");
  }
  void allgather(const void* s, void* r, size_t bytes, cudaStream_t st) override {
    call(EF_COLL_ALLGATHER, s, r, bytes, st);
  }
  void alltoall(const void* s, void* r, size_t chunk, cudaStream_t st) override {
    call(EF_COLL_ALLTOALL, s, r, chunk, st);
  }
  const char* name() const override { return "callback"; }
};

}  // namespace

std::unique_ptr<Transport> make_local_transport() { return std::make_unique<LocalTransport>(); }
std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const void* id128) {
  return std::make_unique<NcclTransport>(world, rank, id128);
}
std::unique_ptr<Transport> make_callback_transport(ef_collective_cb cb, void* user) {
  return std::make_unique<CallbackTransport>(cb, user);
}
void nccl_unique_id(void* out128) {
  ncclUniqueId id;
  nck(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

}  // namespace ef

extern "C" int ef_ep_nccl_unique_id(void* out128) {
  EF_TRY({ ef::nccl_unique_id(out128); });
}
