// comm.h -- inter-rank communication of the element partition (P:626-630,
// SURVEY 8(e)): face-trace halo exchange before an operator, and sum
// all-reduces for the global norms / GMRES dot products.
//
// Three transports behind one interface:
//   NcclComm      -- one process per GPU, NCCL over NVLink/NVSwitch (libnccl is
//                    dlopen'ed, so the library loads and runs single-rank without it);
//   LoopbackComm  -- several ranks as host threads of ONE process (any devices,
//                    typically one GPU): halos by device-to-device copies, sums on
//                    the host in rank order.  Tests the whole partition path on a
//                    single GPU; no kernel ever waits on another rank's kernel
//                    (ranks meet at host barriers after synchronising their stream).
//   (nullptr)     -- a single rank without forced halos: no communication at all.
//
// Halo convention.  The send buffer holds 4 side segments (side 0 = -x, 1 = +x,
// 2 = -y, 3 = +y) at offsets off[s], each len[s] doubles, identical on every
// rank.  Receive slot s is filled with the segment opp(s) = s ^ 1 of the rank
// nbr[s] (the neighbour across side s sends the face it shares with us).  Only
// sides with active[s] != 0 take part.
#pragma once
#include <cstddef>
#include <string>
#include <cuda_runtime.h>

namespace hbpdc {

class Comm {
 public:
  virtual ~Comm() = default;
  // in-place sum over ranks of n doubles in device memory (enqueued on st);
  // returns 0 on success, else sets err
  virtual int allreduce_sum(double* d, int n, cudaStream_t st, std::string& err) = 0;
  virtual int halo(const double* send, double* recv, const size_t off[4], const size_t len[4], const int nbr[4],
                   const int active[4], cudaStream_t st, std::string& err) = 0;
  virtual const char* kind() const = 0;
};

// NCCL (rank, nranks, 128-byte unique id of rank 0); device must be current
Comm* make_nccl_comm(int rank, int nranks, const void* unique_id, std::string& err);
int nccl_unique_id(void* out128, std::string& err);

// loopback group shared by `nranks` host threads
struct LoopbackGroup;
LoopbackGroup* loopback_group_create(int nranks);
void loopback_group_destroy(LoopbackGroup* g);
Comm* make_loopback_comm(LoopbackGroup* g, int rank);

}  // namespace hbpdc
