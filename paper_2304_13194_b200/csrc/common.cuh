// common.cuh — shared infrastructure for the sm_100a Jet partitioner.
//
// Layout in HBM (one CSR level):
//   offs  int64[n+1]   row offsets (int64: R-MAT-27 has > 2^31 entries)
//   adj   int32[nnz]   neighbour ids, rows sorted ascending (graph.py:109)
//   ew    int32[nnz]   edge weights (>= 1)
//   vw    int32[n]     vertex weights (>= 1)
// Sums (conn, gains, part weights, cut) are int64, matching the reference's
// int64 numpy arithmetic (_arrays.py:5).
#pragma once
#include <algorithm>
#include <atomic>
#include <memory>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>
#include <map>
#include <stdexcept>
#include <utility>
#include "../../include/jet.h"

namespace cg = cooperative_groups;

namespace jet {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file,
                             int line);

#define CK(x)                                                     \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) ::jet::throw_cuda(e_, #x, __FILE__, __LINE__); \
  } while (0)

#define JET_REQUIRE(cond, code, msg)          \
  do {                                        \
    if (!(cond)) throw ::jet::Error(code, msg); \
  } while (0)

// Sentinel gain for interior vertices (refine.py:31).
constexpr long long NO_GAIN = -(1LL << 62);
// Part ids are packed in the low bits of 64-bit max keys (refine.py:93-98
// encodes vals*(k+1)+(k-p); we use (conn << KBITS) | (KMASK - p)).
constexpr int KBITS = 21;
constexpr int KMASK = (1 << KBITS) - 1;

// Degree tiers. Tiers 0-3 give each vertex a G-lane group (G = 4,8,16,32)
// that holds the whole row in registers; tier 4 gives a row to one warp with
// a per-warp shared-memory part table; tier 5 gives a row to a whole block.
constexpr int NBINS = 6;
constexpr int BIN_WARP = 4, BIN_BLOCK = 5;
constexpr int64_t WARP_TIER_MAX_DEG = 2048;
// Per-level degree -> tier map. Small levels merge every row of <= 64
// entries into tier 3 (one launch instead of four; launch latency dominates
// there); large levels use the G = 4/8/16/32 split, where the G = 32 tier
// holds rows of 17..64 entries, two per lane.
struct TierMap {
  int lim[4];
  __host__ __device__ __forceinline__ int operator()(int64_t d) const {
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (d <= lim[t]) return t;
    return d <= WARP_TIER_MAX_DEG ? 4 : 5;
  }
};
constexpr int64_t MERGED_TIER_MAX_N = 1 << 18;
inline TierMap tiers_for(int64_t n) {
  return n <= MERGED_TIER_MAX_N ? TierMap{{-1, -1, -1, 64}} : TierMap{{4, 8, 16, 64}};
}
constexpr int TIER_G[4] = {4, 8, 16, 32};

// ---------------------------------------------------------------------------
// Device memory: stream-ordered allocations from the library's private pool
// for the current device (cudaMemPoolCreate; its release threshold keeps
// freed blocks mapped for reuse while contexts live, and the last context on
// a device trims it). The process's default pool is never modified.
cudaMemPool_t current_pool();
void pool_context_opened(int device);
void pool_context_closed(int device);

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = 0;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t st) { alloc(count, st); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; n = o.n; s = o.s;
      o.p = nullptr; o.n = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count, cudaStream_t st) {
    release();
    s = st;
    n = count;
    if (count) {
      cudaError_t e = cudaMallocFromPoolAsync((void**)&p, count * sizeof(T), current_pool(), st);
      if (e != cudaSuccess) {
        p = nullptr;
        n = 0;
        cudaGetLastError();
        throw Error(JET_ENOMEM, "device allocation of " +
                                    std::to_string(count * sizeof(T)) +
                                    " bytes failed: " + cudaGetErrorString(e));
      }
    }
  }
  // Grow to at least `count` elements; contents are not preserved.
  void ensure(size_t count, cudaStream_t st) {
    if (count > n || p == nullptr) alloc(count > 0 ? count : 1, st);
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

// ---------------------------------------------------------------------------
// Device CSR level.
struct DGraph {
  int64_t n = 0, nnz = 0, total_vw = 0;
  int64_t max_deg = 0, max_wdeg = 0, max_ew = 0, max_vw = 0, min_vw = 1;
  bool unit_ew = true;
  TierMap tm{{4, 8, 16, 64}};
  DBuf<int64_t> offs;
  DBuf<int32_t> adj, ew, vw;
  // degree tiers: ascending vertex lists, or identity when one tier holds all
  DBuf<int32_t> bin_store;
  const int32_t* bin_list[NBINS] = {};
  int64_t bin_cnt[NBINS] = {};
  int64_t bin_nnz[NBINS] = {};
  bool identity = false;
  int identity_bin = -1;
  // 1D-distributed level: this rank stores only the rows of
  // [row_lo, row_hi) -- adj/ew hold the entries [offs[row_lo], offs[row_hi]),
  // starting at ent_lo -- while offs and vw are complete (O(n) per rank).
  // row_hi < 0: every row is local. nnz is always the global entry count.
  int64_t row_lo = 0, row_hi = -1, ent_lo = 0;
  bool partial() const { return row_hi >= 0; }
  int64_t local_nnz() const { return partial() ? (int64_t)adj.n : nnz; }
};

struct Ctx;

// Per-launch profiling record (CUDA events on the context stream).
struct ProfRec {
  int cls;
  cudaEvent_t a, b;
  double bytes;
};
struct ProfAgg {
  std::string name;
  int64_t launches = 0;
  double ms = 0, bytes = 0;
};

// Context-owned extension state (defined by the translation unit that uses
// it); released by jet_destroy while the context stream is still alive.
struct CtxExt {
  virtual ~CtxExt() = default;
};

struct Comm;  // comm.cuh: exchange step of the sharded refinement

struct Ctx {
  int device = 0;
  // 1D vertex sharding: with a communicator of size > 1,
  // levels of at least shard_min_n vertices refine with sharded Jetlp
  // sweeps (this rank's vertex block) and exchange the candidates / moves.
  Comm* comm = nullptr;
  int64_t shard_min_n = 1 << 20;
  bool shard_single = false;  // run the sharded path with one rank (transport tests)
  // Graphs and hierarchies allocated on this context's stream hold a
  // reference, so the stream outlives every buffer freed on it whatever
  // order the caller (e.g. interpreter teardown) releases handles in.
  std::atomic<int> refs{1};
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  int max_smem_optin = 0;
  int64_t launches = 0;
  // pinned host mirror for per-iteration scalars
  int64_t* pinned = nullptr;
  size_t pinned_elems = 0;
  uint8_t* pinned_up = nullptr;  // host->device staging (per-pass scalars)
  size_t pinned_up_bytes = 0;
  // scratch for CUB device-wide primitives
  DBuf<uint8_t> cub_tmp;
  // profiling
  bool prof = false;
  std::vector<ProfRec> recs;
  std::vector<cudaEvent_t> event_pool;
  std::vector<ProfAgg> agg;
  std::map<std::string, int> cls_index;
  std::string prof_only;  // empty: record every class
  std::string prof_tag;   // prefix for class names (per-level breakdowns)
  bool prof_by_level = false;
  cudaEvent_t timer_a = nullptr, timer_b = nullptr;
  DBuf<uint8_t> flush_buf;
  int32_t lock_epoch = 0;
  // per-iteration (kind 1/2/3, cut, max part weight, moves) records of
  // jet_refine (refine.py:269-271), filled when set (API entry only)
  std::vector<int64_t>* api_trace = nullptr;
  bool host_levels = false;  // force the host-driven per-pass controller

  cudaEvent_t take_event();
  int prof_class(const char* name);
  void flush_prof();
  void ensure_pinned(size_t elems);
  size_t pool_reserved = 0;
  void reserve_pool(size_t bytes);
  // pinned upload ring (graph upload from pageable host arrays)
  static constexpr int UPLOAD_BUFS = 3;
  static constexpr size_t UPLOAD_CHUNK = (size_t)32 << 20;
  void* up_host[UPLOAD_BUFS] = {};
  cudaEvent_t up_ev[UPLOAD_BUFS] = {};
  DBuf<uint8_t> up_dev;
  void ensure_upload_ring();
  void ensure_pinned_up(size_t bytes);
  long long nsync = 0;  // host waits on the stream (diagnostics: JET_SYNC_STATS)
  void sync() {
    ++nsync;
    CK(cudaStreamSynchronize(stream));
  }
  void* cub_scratch(size_t bytes) {
    cub_tmp.ensure(bytes, stream);
    return cub_tmp.get();
  }
  // Grow-only scratch slots for large per-level temporaries (coarsening):
  // sized once by the finest level, reused by every coarser level and call.
  // Fresh stream-ordered allocations of hundreds of MB occasionally make the
  // pool map new physical memory, which stalls the host for 100s of ms.
  std::unique_ptr<CtxExt> level_ext;  // level.cu: persistent-controller scratch
  static constexpr int NSCRATCH = 28;
  DBuf<uint8_t> scratch_slots[NSCRATCH];
  template <class T>
  T* scratch(int slot, size_t count) {
    DBuf<uint8_t>& b = scratch_slots[slot];
    const size_t bytes = (count > 0 ? count : 1) * sizeof(T);
    if (bytes > b.n) b.alloc(bytes + std::min<size_t>(bytes / 8, (size_t)256 << 20), stream);
    return reinterpret_cast<T*>(b.get());
  }
  // Drop every scratch slot (out-of-memory hierarchies: the contraction
  // temporaries of a 4 G-entry level are ~40 GB).
  void release_scratch() {
    for (auto& s : scratch_slots) s.release();
    cub_tmp.release();
  }
};

// Max / sum of a host scalar over the ranks of c.comm (the value itself
// without a communicator); a device round trip through the transport.
int64_t comm_max(Ctx& c, int64_t v);
int64_t comm_sum(Ctx& c, int64_t v);

void ctx_retain(Ctx* c);
void ctx_release(Ctx* c);  // tears the context down at the last reference

// Launch wrapper: counts the launch, brackets it with events when profiling,
// and checks the launch status. `bytes` = algorithmic bytes of the launch.
template <class F>
inline void launch(Ctx& c, const char* name, double bytes, F&& f) {
  ProfRec r{};
  const bool rec = c.prof && (c.prof_only.empty() || c.prof_only == name);
  if (rec) {
    r.cls = c.prof_by_level ? c.prof_class((c.prof_tag + name).c_str()) : c.prof_class(name);
    r.a = c.take_event();
    r.b = c.take_event();
    r.bytes = bytes;
    CK(cudaEventRecord(r.a, c.stream));
  }
  f();
  CK(cudaGetLastError());
  c.launches++;
  if (rec) {
    CK(cudaEventRecord(r.b, c.stream));
    c.recs.push_back(r);
  }
}

// Grid for a grid-stride kernel: enough blocks for `work_threads`, capped at
// `per_sm` resident blocks on every SM.
inline unsigned grid_for(const Ctx& c, int64_t work_threads, int block,
                         int per_sm = 8) {
  int64_t b = (work_threads + block - 1) / block;
  int64_t cap = (int64_t)c.num_sms * per_sm;
  if (b < 1) b = 1;
  return (unsigned)(b < cap ? b : cap);
}

// Resident blocks per SM of `kern` at this block size (cached per kernel).
int resident_blocks(const void* kern, int block, size_t smem);

// grid_for capped at the blocks that are resident at once: a grid-stride
// kernel whose grid exceeds residency runs a second, partial wave with the
// same per-warp share of the work, so part of the GPU idles at the end.
template <class K>
inline unsigned grid_res(const Ctx& c, K* kern, int64_t work_threads, int block,
                         size_t smem = 0) {
  return grid_for(c, work_threads, block, resident_blocks((const void*)kern, block, smem));
}

template <class T>
inline void h2d(Ctx& c, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, c.stream));
}
template <class T>
inline void d2h(Ctx& c, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToHost, c.stream));
}
template <class T>
inline void d2d(Ctx& c, T* dst, const T* src, size_t count) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyDeviceToDevice, c.stream));
}
template <class T>
inline void dzero(Ctx& c, T* dst, size_t count) {
  if (count) CK(cudaMemsetAsync(dst, 0, count * sizeof(T), c.stream));
}

// ---------------------------------------------------------------------------
// Warp-group helpers (groups of G lanes, G | 32, aligned).
template <int G>
__device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) {
    return 0xffffffffu;
  } else {
    const unsigned lane = threadIdx.x & 31u;
    return ((1u << G) - 1u) << (lane & ~(unsigned)(G - 1));
  }
}
template <int G, class T>
__device__ __forceinline__ T gsum(T x, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) x += __shfl_xor_sync(m, x, o);
  return x;
}
template <int G, class T>
__device__ __forceinline__ T gmax(T x, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    T y = __shfl_xor_sync(m, x, o);
    x = y > x ? y : x;
  }
  return x;
}
template <int G, class T>
__device__ __forceinline__ T gmin(T x, unsigned m) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    T y = __shfl_xor_sync(m, x, o);
    x = y < x ? y : x;
  }
  return x;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned r;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(r));
  return r;
}

// Sum of `w` over the lanes in `peers` (a __match_any_sync group). Narrow
// weights use the single-instruction REDUX; wide ones walk the peer bits.
__device__ __forceinline__ long long peer_sum(unsigned peers, int w, bool wide) {
  if (!wide) return (long long)__reduce_add_sync(peers, (unsigned)w);
  long long s = 0;
  unsigned m = peers;
  while (m) {
    int l = __ffs(m) - 1;
    m &= m - 1;
    s += __shfl_sync(peers, w, l);
  }
  return s;
}

// Sum of x over the lanes of `peers` (a __match_any_sync group the caller is in).
__device__ __forceinline__ long long gsum_peers(unsigned peers, long long x) {
  long long s = 0;
  unsigned m = peers;
  while (m) {
    const int l = __ffs(m) - 1;
    m &= m - 1;
    s += __shfl_sync(peers, x, l);
  }
  return s;
}

// Warp-aggregated append of `v` into list[*cnt] for lanes where `take`.
__device__ __forceinline__ void warp_append(bool take, int32_t v, int32_t* list,
                                            unsigned long long* cnt) {
  const unsigned am = __activemask();
  const unsigned m = __ballot_sync(am, take);
  if (m == 0) return;
  const int leader = __ffs(m) - 1;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == leader) base = atomicAdd(cnt, (unsigned long long)__popc(m));
  base = __shfl_sync(am, base, leader);
  if (take) list[base + __popc(m & lanemask_lt())] = v;
}

// Block-aggregated append: one global atomic per block and call instead of
// one per warp (a hot counter serialises in L2). Every thread of the block
// must call it (block-uniform loop trip counts).
__device__ __forceinline__ void block_append(bool take, int32_t v, int32_t* list,
                                             unsigned long long* cnt) {
  __shared__ unsigned s_wc[32];
  __shared__ unsigned long long s_base;
  const unsigned m = __ballot_sync(0xffffffffu, take);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  if (l == 0) s_wc[w] = __popc(m);
  __syncthreads();
  if (w == 0) {
    const unsigned x = l < nw ? s_wc[l] : 0u;
    unsigned inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (l >= o) inc += y;
    }
    const unsigned tot = __shfl_sync(0xffffffffu, inc, 31);
    if (l < nw) s_wc[l] = inc - x;
    if (l == 0) s_base = tot ? atomicAdd(cnt, (unsigned long long)tot) : 0ull;
  }
  __syncthreads();
  if (take) list[s_base + s_wc[w] + __popc(m & lanemask_lt())] = v;
  __syncthreads();
}

// Block-wide int64 sum returned to every thread (any blockDim <= 1024; all
// threads of the block must call it).
__device__ __forceinline__ long long block_sum_all(long long x) {
  __shared__ long long red_all[33];
  x = gsum<32>(x, 0xffffffffu);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red_all[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = l < nw ? red_all[l] : 0;
    y = gsum<32>(y, 0xffffffffu);
    if (l == 0) red_all[32] = y;
  }
  __syncthreads();
  return red_all[32];
}

// Block-wide int64 sum into *out for any blockDim <= 1024.
__device__ __forceinline__ void block_sum_atomic_any(long long x, unsigned long long* out) {
  __shared__ long long red_any[32];
  x = gsum<32>(x, 0xffffffffu);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) red_any[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = l < nw ? red_any[l] : 0;
    y = gsum<32>(y, 0xffffffffu);
    if (l == 0 && y != 0) atomicAdd(out, (unsigned long long)y);
  }
  __syncthreads();
}

// Block-wide int64 sum into *out (one atomic per block).
template <int BLOCK>
__device__ __forceinline__ void block_sum_atomic(long long x, unsigned long long* out) {
  __shared__ long long red[BLOCK / 32];
  x = gsum<32>(x, 0xffffffffu);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = x;
  __syncthreads();
  if (w == 0) {
    long long y = l < BLOCK / 32 ? red[l] : 0;
    y = gsum<32>(y, 0xffffffffu);
    if (l == 0 && y != 0) atomicAdd(out, (unsigned long long)y);
  }
}

}  // namespace jet
