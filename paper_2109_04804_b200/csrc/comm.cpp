// comm.cpp -- NCCL and loopback transports of the element partition (comm.h).
#include "comm.h"

#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

namespace hbpdc {

// ============================================================================
// NCCL, resolved at run time (torch has normally loaded libnccl.so.2 already;
// dlopen by soname then returns that copy)
// ============================================================================
namespace {
struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* env = std::getenv("HBPDC_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("cannot dlopen libnccl.so.2 (set HBPDC_NCCL_LIB): ") + dlerror();
      return;
    }
#define SYM(name)                                                               \
  api.name = reinterpret_cast<decltype(api.name)>(dlsym(h, "nccl" #name));      \
  if (!api.name) {                                                              \
    api.why = "libnccl lacks nccl" #name;                                       \
    return;                                                                     \
  }
    SYM(GetUniqueId) SYM(CommInitRank) SYM(CommDestroy) SYM(AllReduce) SYM(Send) SYM(Recv) SYM(GroupStart)
    SYM(GroupEnd) SYM(GetErrorString)
#undef SYM
    api.ok = true;
  });
  return api;
}

#define NCK(call)                                                                 \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess) {                                                      \
      err = std::string("NCCL error: ") + nccl().GetErrorString(r_) + " at " #call; \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

class NcclComm final : public Comm {
 public:
  ncclComm_t comm = nullptr;
  ~NcclComm() override {
    if (comm) nccl().CommDestroy(comm);
  }
  int allreduce_sum(double* d, int n, cudaStream_t st, std::string& err) override {
    if (n <= 0) return 0;
    NCK(nccl().AllReduce(d, d, (size_t)n, ncclFloat64, ncclSum, comm, st));
    return 0;
  }
  int halo(const double* send, double* recv, const size_t off[4], const size_t len[4], const int nbr[4],
           const int active[4], cudaStream_t st, std::string& err) override {
    // sends in side order; receives in the order of the matching sends of a
    // peer that is our neighbour on both sides (px == 2 or a forced self halo):
    // recv slot s^1 for s = 0..3 (see comm.h)
    NCK(nccl().GroupStart());
    for (int s = 0; s < 4; ++s)
      if (active[s]) NCK(nccl().Send(send + off[s], len[s], ncclFloat64, nbr[s], comm, st));
    for (int s = 0; s < 4; ++s) {
      const int r = s ^ 1;
      if (active[r]) NCK(nccl().Recv(recv + off[r], len[r], ncclFloat64, nbr[r], comm, st));
    }
    NCK(nccl().GroupEnd());
    return 0;
  }
  const char* kind() const override { return "nccl"; }
};
}  // namespace

int nccl_unique_id(void* out128, std::string& err) {
  if (!nccl().ok) {
    err = nccl().why;
    return 1;
  }
  ncclUniqueId id;
  NCK(nccl().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out128, &id, sizeof(id));
  return 0;
}

Comm* make_nccl_comm(int rank, int nranks, const void* unique_id, std::string& err) {
  if (!nccl().ok) {
    err = nccl().why;
    return nullptr;
  }
  if (!unique_id) {
    err = "nccl_unique_id is NULL";
    return nullptr;
  }
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  auto* c = new NcclComm();
  ncclResult_t r = nccl().CommInitRank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + nccl().GetErrorString(r);
    c->comm = nullptr;
    delete c;
    return nullptr;
  }
  return c;
}

// ============================================================================
// Loopback: ranks are host threads of one process
// ============================================================================
struct LoopbackGroup {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long generation = 0;
  std::vector<const double*> send;          // published send buffers
  std::vector<std::vector<double>> slot;    // host copies for the all-reduce
  std::vector<double> sum;
  explicit LoopbackGroup(int n) : nranks(n), send(n, nullptr), slot(n) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long gen = generation;
    if (++arrived == nranks) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

LoopbackGroup* loopback_group_create(int nranks) { return nranks > 0 ? new LoopbackGroup(nranks) : nullptr; }
void loopback_group_destroy(LoopbackGroup* g) { delete g; }

namespace {
#define CCK(call)                                                              \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      err = std::string("CUDA error in loopback comm: ") + cudaGetErrorString(e_); \
      return 1;                                                                \
    }                                                                          \
  } while (0)

class LoopbackComm final : public Comm {
 public:
  LoopbackGroup* g;
  int rank;
  LoopbackComm(LoopbackGroup* g_, int r) : g(g_), rank(r) {}
  int allreduce_sum(double* d, int n, cudaStream_t st, std::string& err) override {
    if (n <= 0) return 0;
    auto& mine = g->slot[rank];
    mine.resize(n);
    CCK(cudaMemcpyAsync(mine.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    CCK(cudaStreamSynchronize(st));
    g->barrier();
    std::vector<double> s(n, 0.0);
    for (int r = 0; r < g->nranks; ++r)           // fixed rank order: identical on every rank
      for (int i = 0; i < n; ++i) s[i] += g->slot[r][i];
    g->barrier();                                  // everyone has read the slots
    CCK(cudaMemcpyAsync(d, s.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    CCK(cudaStreamSynchronize(st));
    return 0;
  }
  int halo(const double* send, double* recv, const size_t off[4], const size_t len[4], const int nbr[4],
           const int active[4], cudaStream_t st, std::string& err) override {
    CCK(cudaStreamSynchronize(st));                // our pack is complete
    g->send[rank] = send;
    g->barrier();
    for (int s = 0; s < 4; ++s)
      if (active[s])
        CCK(cudaMemcpyAsync(recv + off[s], g->send[nbr[s]] + off[s ^ 1], len[s] * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
    CCK(cudaStreamSynchronize(st));
    g->barrier();                                  // peers may reuse their send buffers
    return 0;
  }
  const char* kind() const override { return "loopback"; }
};
}  // namespace

Comm* make_loopback_comm(LoopbackGroup* g, int rank) {
  if (!g || rank < 0 || rank >= g->nranks) return nullptr;
  return new LoopbackComm(g, rank);
}

}  // namespace hbpdc
