// comm.cuh — the exchange step of the 1D vertex-sharded refinement
// (SURVEY §8(e)): a variable-size all-gather of device buffers between the
// ranks of one node. Two transports behind one interface:
//   NcclComm  : one process per GPU, NCCL over NVLink/NVSwitch (libnccl is
//               opened at run time; the communicator is built from a unique
//               id the Python side broadcasts with torch.distributed);
//   LocalComm : several "virtual ranks" (host threads, one context each) in
//               one process on one GPU -- the same sharded code path, used to
//               prove it bit-exact against the unsharded run where only one
//               GPU is available.
#pragma once
#include "common.cuh"
#include <condition_variable>
#include <mutex>
#include <vector>

namespace jet {

struct Comm {
  int rank = 0, size = 1;
  virtual ~Comm() = default;
  // Gathers every rank's `bytes` bytes at `dsend` (device, ordered on
  // c.stream) into `recv`, rank-major and compact; counts[r] = rank r's bytes.
  virtual void allgatherv(Ctx& c, const void* dsend, int64_t bytes, DBuf<uint8_t>& recv,
                          std::vector<int64_t>& counts) = 0;
  // Personalised exchange: scounts[r] bytes of `dsend` (rank-major, packed)
  // go to rank r; rank s's bytes for this rank arrive rank-major in `recv`,
  // rcounts[s] = their length.
  virtual void alltoallv(Ctx& c, const void* dsend, const std::vector<int64_t>& scounts,
                         DBuf<uint8_t>& recv, std::vector<int64_t>& rcounts) = 0;
  // In-place sum over ranks of a device array of 64-bit words (two's
  // complement: signed deltas sum correctly). NCCL: ncclAllReduce on the
  // context stream; the local group: gather + local sum.
  virtual void allreduce_sum(Ctx& c, unsigned long long* d, int64_t count);
  DBuf<uint8_t> red_buf;
};

struct LocalGroup {
  int size = 1;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<const void*> ptrs;
  std::vector<int64_t> bytes;
  std::vector<std::vector<int64_t>> sc;  // alltoallv: every rank's send counts
  explicit LocalGroup(int n) : size(n), ptrs(n, nullptr), bytes(n, 0), sc(n) {}
  void barrier();
};

struct LocalComm : Comm {
  LocalGroup* g;
  LocalComm(LocalGroup* grp, int r) : g(grp) {
    rank = r;
    size = grp->size;
  }
  void allgatherv(Ctx& c, const void* dsend, int64_t bytes, DBuf<uint8_t>& recv,
                  std::vector<int64_t>& counts) override;
  void alltoallv(Ctx& c, const void* dsend, const std::vector<int64_t>& scounts,
                 DBuf<uint8_t>& recv, std::vector<int64_t>& rcounts) override;
};

// Returns nullptr (and sets the error) when libnccl cannot be opened.
Comm* make_nccl_comm(const unsigned char id[128], int rank, int size);
bool nccl_unique_id(unsigned char id[128]);

}  // namespace jet
