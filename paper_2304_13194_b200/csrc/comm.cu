// comm.cu — transports of the sharded refinement's exchange step (comm.cuh).
#include "comm.cuh"
#include <dlfcn.h>
#include <algorithm>
#include <numeric>
#include <string>
#include <chrono>

namespace jet {

__global__ void k_sum_slices(const unsigned long long* __restrict__ in, int64_t count, int size,
                             unsigned long long* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long s = 0;
    for (int r = 0; r < size; ++r) s += in[(size_t)r * count + i];
    out[i] = s;
  }
}

void Comm::allreduce_sum(Ctx& c, unsigned long long* d, int64_t count) {
  if (count <= 0) return;
  std::vector<int64_t> counts;
  allgatherv(c, d, count * (int64_t)sizeof(unsigned long long), red_buf, counts);
  k_sum_slices<<<grid_for(c, count, 256), 256, 0, c.stream>>>(
      reinterpret_cast<const unsigned long long*>(red_buf.get()), count, size, d);
  CK(cudaGetLastError());
}

static int64_t comm_reduce(Ctx& c, int64_t v, bool mx) {
  if (!c.comm || c.comm->size == 1) return v;
  DBuf<int64_t> d(1, c.stream);
  h2d(c, d.get(), &v, 1);
  DBuf<uint8_t> recv;
  std::vector<int64_t> counts;
  c.comm->allgatherv(c, d.get(), (int64_t)sizeof(int64_t), recv, counts);
  std::vector<int64_t> all(c.comm->size);
  d2h(c, all.data(), reinterpret_cast<const int64_t*>(recv.get()), c.comm->size);
  c.sync();
  int64_t r = mx ? all[0] : 0;
  for (int64_t x : all) r = mx ? std::max(r, x) : r + x;
  return r;
}
int64_t comm_max(Ctx& c, int64_t v) { return comm_reduce(c, v, true); }
int64_t comm_sum(Ctx& c, int64_t v) { return comm_reduce(c, v, false); }

void LocalGroup::barrier() {
  std::unique_lock<std::mutex> lk(m);
  const int64_t gen = generation;
  if (++arrived == size) {
    arrived = 0;
    ++generation;
    cv.notify_all();
  } else {
    // a rank that failed never arrives: give up instead of hanging the others
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return generation != gen; }))
      throw Error(JET_EINTERNAL, "local group: a rank did not reach the exchange (120 s)");
  }
}

void LocalComm::allgatherv(Ctx& c, const void* dsend, int64_t bytes, DBuf<uint8_t>& recv,
                           std::vector<int64_t>& counts) {
  c.sync();  // the send buffer is complete
  g->ptrs[rank] = dsend;
  g->bytes[rank] = bytes;
  g->barrier();
  counts = g->bytes;
  const int64_t total = std::accumulate(counts.begin(), counts.end(), (int64_t)0);
  recv.ensure((size_t)std::max<int64_t>(total, 1), c.stream);
  int64_t off = 0;
  for (int r = 0; r < size; ++r) {
    if (counts[r])
      CK(cudaMemcpyAsync(recv.get() + off, g->ptrs[r], (size_t)counts[r], cudaMemcpyDeviceToDevice,
                         c.stream));
    off += counts[r];
  }
  c.sync();
  g->barrier();  // no rank reuses its send buffer before every copy is done
}

void LocalComm::alltoallv(Ctx& c, const void* dsend, const std::vector<int64_t>& scounts,
                          DBuf<uint8_t>& recv, std::vector<int64_t>& rcounts) {
  c.sync();  // the send buffer is complete
  g->ptrs[rank] = dsend;
  g->sc[rank] = scounts;
  g->barrier();
  rcounts.assign(size, 0);
  int64_t total = 0;
  for (int s = 0; s < size; ++s) total += (rcounts[s] = g->sc[s][rank]);
  recv.ensure((size_t)std::max<int64_t>(total, 1), c.stream);
  int64_t off = 0;
  for (int s = 0; s < size; ++s) {
    int64_t src = 0;  // rank s's bytes for ranks before this one
    for (int r = 0; r < rank; ++r) src += g->sc[s][r];
    if (rcounts[s])
      CK(cudaMemcpyAsync(recv.get() + off, static_cast<const uint8_t*>(g->ptrs[s]) + src,
                         (size_t)rcounts[s], cudaMemcpyDeviceToDevice, c.stream));
    off += rcounts[s];
  }
  c.sync();
  g->barrier();  // no rank reuses its send buffer before every copy is done
}

// ---- NCCL, opened at run time (no link-time dependency) -------------------
namespace {
typedef struct {
  char internal[128];
} NcclId;
typedef void* NcclComm_t;
typedef int (*PGetUniqueId)(NcclId*);
typedef int (*PCommInitRank)(NcclComm_t*, int, NcclId, int);
typedef int (*PAllGather)(const void*, void*, size_t, int, NcclComm_t, cudaStream_t);
typedef int (*PAllReduce)(const void*, void*, size_t, int, int, NcclComm_t, cudaStream_t);
typedef int (*PCommDestroy)(NcclComm_t);
typedef int (*PSendRecv)(void*, size_t, int, int, NcclComm_t, cudaStream_t);
typedef int (*PGroup)();
typedef const char* (*PGetErrorString)(int);
constexpr int NCCL_INT8 = 0, NCCL_UINT64 = 5, NCCL_SUM = 0;

struct NcclApi {
  void* h = nullptr;
  PGetUniqueId get_id = nullptr;
  PCommInitRank init = nullptr;
  PAllGather allgather = nullptr;
  PAllReduce allreduce = nullptr;
  PSendRecv send = nullptr, recv = nullptr;
  PGroup group_start = nullptr, group_end = nullptr;
  PCommDestroy destroy = nullptr;
  PGetErrorString err = nullptr;
  bool load() {
    if (h) return true;
    for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return false;
    get_id = (PGetUniqueId)dlsym(h, "ncclGetUniqueId");
    init = (PCommInitRank)dlsym(h, "ncclCommInitRank");
    allgather = (PAllGather)dlsym(h, "ncclAllGather");
    allreduce = (PAllReduce)dlsym(h, "ncclAllReduce");
    send = (PSendRecv)dlsym(h, "ncclSend");
    recv = (PSendRecv)dlsym(h, "ncclRecv");
    group_start = (PGroup)dlsym(h, "ncclGroupStart");
    group_end = (PGroup)dlsym(h, "ncclGroupEnd");
    destroy = (PCommDestroy)dlsym(h, "ncclCommDestroy");
    err = (PGetErrorString)dlsym(h, "ncclGetErrorString");
    return get_id && init && allgather && allreduce && send && recv && group_start && group_end &&
           destroy;
  }
};
NcclApi& nccl() {
  static NcclApi a;
  return a;
}

void nck(int rc, const char* what) {
  if (rc != 0)
    throw Error(JET_ECUDA, std::string(what) + ": " + (nccl().err ? nccl().err(rc) : "nccl error"));
}

struct NcclComm : Comm {
  NcclComm_t comm = nullptr;
  DBuf<int64_t> cnt;
  DBuf<uint8_t> stage, padded;
  ~NcclComm() override {
    if (comm) nccl().destroy(comm);
  }
  void alltoallv(Ctx& c, const void* dsend, const std::vector<int64_t>& scounts,
                 DBuf<uint8_t>& recv, std::vector<int64_t>& rcounts) override {
    // counts: all-gather every rank's send-count row, read this rank's column
    cnt.ensure((size_t)size * (size + 1), c.stream);
    h2d(c, cnt.get() + (size_t)size * size, scounts.data(), size);
    nck(nccl().allgather(cnt.get() + (size_t)size * size, cnt.get(), sizeof(int64_t) * size, NCCL_INT8,
                         comm, c.stream),
        "ncclAllGather(counts)");
    std::vector<int64_t> m((size_t)size * size);
    d2h(c, m.data(), cnt.get(), (size_t)size * size);
    c.sync();
    rcounts.assign(size, 0);
    int64_t total = 0;
    for (int s = 0; s < size; ++s) total += (rcounts[s] = m[(size_t)s * size + rank]);
    recv.ensure((size_t)std::max<int64_t>(total, 1), c.stream);
    nck(nccl().group_start(), "ncclGroupStart");
    int64_t so = 0, ro = 0;
    for (int p = 0; p < size; ++p) {
      if (scounts[p])
        nck(nccl().send(const_cast<uint8_t*>(static_cast<const uint8_t*>(dsend)) + so, (size_t)scounts[p],
                        NCCL_INT8, p, comm, c.stream),
            "ncclSend");
      if (rcounts[p])
        nck(nccl().recv(recv.get() + ro, (size_t)rcounts[p], NCCL_INT8, p, comm, c.stream), "ncclRecv");
      so += scounts[p];
      ro += rcounts[p];
    }
    nck(nccl().group_end(), "ncclGroupEnd");
  }
  void allreduce_sum(Ctx& c, unsigned long long* d, int64_t count) override {
    if (count <= 0) return;
    nck(nccl().allreduce(d, d, (size_t)count, NCCL_UINT64, NCCL_SUM, comm, c.stream), "ncclAllReduce");
  }
  void allgatherv(Ctx& c, const void* dsend, int64_t bytes, DBuf<uint8_t>& recv,
                  std::vector<int64_t>& counts) override {
    cnt.ensure((size_t)size + 1, c.stream);
    h2d(c, cnt.get() + size, &bytes, 1);
    nck(nccl().allgather(cnt.get() + size, cnt.get(), sizeof(int64_t), NCCL_INT8, comm, c.stream),
        "ncclAllGather(counts)");
    counts.assign(size, 0);
    d2h(c, counts.data(), cnt.get(), size);
    c.sync();
    const int64_t mx = std::max<int64_t>(1, *std::max_element(counts.begin(), counts.end()));
    stage.ensure((size_t)mx, c.stream);
    padded.ensure((size_t)mx * size, c.stream);
    if (bytes)
      CK(cudaMemcpyAsync(stage.get(), dsend, (size_t)bytes, cudaMemcpyDeviceToDevice, c.stream));
    nck(nccl().allgather(stage.get(), padded.get(), (size_t)mx, NCCL_INT8, comm, c.stream),
        "ncclAllGather");
    const int64_t total = std::accumulate(counts.begin(), counts.end(), (int64_t)0);
    recv.ensure((size_t)std::max<int64_t>(total, 1), c.stream);
    int64_t off = 0;
    for (int r = 0; r < size; ++r) {
      if (counts[r])
        CK(cudaMemcpyAsync(recv.get() + off, padded.get() + (size_t)r * mx, (size_t)counts[r],
                           cudaMemcpyDeviceToDevice, c.stream));
      off += counts[r];
    }
  }
};
}  // namespace

bool nccl_unique_id(unsigned char id[128]) {
  if (!nccl().load()) return false;
  NcclId x;
  if (nccl().get_id(&x) != 0) return false;
  std::copy(x.internal, x.internal + 128, id);
  return true;
}

Comm* make_nccl_comm(const unsigned char id[128], int rank, int size) {
  JET_REQUIRE(nccl().load(), JET_EUNSUPPORTED, "libnccl.so.2 not found");
  NcclId x;
  std::copy(id, id + 128, x.internal);
  auto* c = new NcclComm();
  c->rank = rank;
  c->size = size;
  const int rc = nccl().init(&c->comm, size, x, rank);
  if (rc != 0) {
    delete c;
    nck(rc, "ncclCommInitRank");
  }
  return c;
}

}  // namespace jet
