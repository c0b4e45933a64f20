// graph.cu — device CSR levels: upload + validation, degree tiers, and the
// per-level metrics kernels (cutsize graph.py:215-221, part weights
// graph.py:240-242, projection driver.py:32-45).
#include "common.cuh"
#include "graph.cuh"
#include "small_ops.cuh"
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <algorithm>
#include <cstring>
#include <omp.h>
#include <emmintrin.h>
#include <climits>
#include <cstdlib>

namespace jet {

// host threads for the staging copies (JET_UPLOAD_THREADS, default 16)
static int upload_threads() {
  static const int t = [] {
    const char* e = getenv("JET_UPLOAD_THREADS");
    const int v = e ? atoi(e) : 16;
    return v > 0 ? v : 16;
  }();
  return t;
}

// memcpy split over the host cores (pageable -> pinned staging)
static void parallel_memcpy(void* dst, const void* src, size_t bytes) {
  const size_t piece = (size_t)1 << 21;
  const int64_t np = (int64_t)((bytes + piece - 1) / piece);
  if (np <= 1) {
    memcpy(dst, src, bytes);
    return;
  }
#pragma omp parallel for schedule(static) num_threads(std::min<int>(upload_threads(), omp_get_num_procs()))
  for (int64_t i = 0; i < np; ++i) {
    const size_t o = (size_t)i * piece;
    memcpy((char*)dst + o, (const char*)src + o, std::min(piece, bytes - o));
  }
}

// int64 -> int32 on the host cores while staging into pinned memory, with the
// range check; returns false when a value is outside [lo, hi]. *all_one is
// set when every value equals 1 (unit weights need no transfer at all).
static bool parallel_narrow(int32_t* dst, const int64_t* src, int64_t count, long long lo,
                            long long hi, bool check_ones, bool* all_one) {
  const int64_t piece = (int64_t)1 << 19;
  const int64_t np = (count + piece - 1) / piece;
  int bad = 0, notone = 0;
#pragma omp parallel for schedule(static) num_threads(std::min<int>(upload_threads(), omp_get_num_procs())) \
    reduction(| : bad, notone)
  for (int64_t i = 0; i < np; ++i) {
    const int64_t b = i * piece, e = std::min(count, b + piece);
    long long mn = LLONG_MAX, mx = LLONG_MIN;
    if (check_ones) {
      // pure scan first: a unit-weight chunk is never written
      for (int64_t j = b; j < e; ++j) {
        const long long x = src[j];
        mn = x < mn ? x : mn;
        mx = x > mx ? x : mx;
      }
      if (mn == 1 && mx == 1) continue;
      notone = 1;
      mn = LLONG_MAX;
      mx = LLONG_MIN;
    }
    // non-temporal 16-byte stores into the pinned buffer: no read-for-
    // ownership of the destination lines (the staging is host-memory bound)
    int64_t j = b;
    for (; j < e && ((uintptr_t)(dst + j) & 15); ++j) {
      const long long x = src[j];
      mn = x < mn ? x : mn;
      mx = x > mx ? x : mx;
      dst[j] = (int32_t)x;
    }
    for (; j + 4 <= e; j += 4) {
      const long long x0 = src[j], x1 = src[j + 1], x2 = src[j + 2], x3 = src[j + 3];
      mn = std::min(mn, std::min(std::min(x0, x1), std::min(x2, x3)));
      mx = std::max(mx, std::max(std::max(x0, x1), std::max(x2, x3)));
      _mm_stream_si128(reinterpret_cast<__m128i*>(dst + j),
                       _mm_set_epi32((int)x3, (int)x2, (int)x1, (int)x0));
    }
    for (; j < e; ++j) {
      const long long x = src[j];
      mn = x < mn ? x : mn;
      mx = x > mx ? x : mx;
      dst[j] = (int32_t)x;
    }
    _mm_sfence();
    if (mn < lo || mx > hi) bad = 1;
  }
  if (all_one) *all_one = check_ones && !notone;
  return !bad;
}

__global__ void k_fill_ones(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 1;
}

// ---------------------------------------------------------------------------
// Upload: host arrays (int32 or int64) -> int32 device arrays, with range
// checks the reference performs implicitly through numpy indexing.
enum { BAD_ADJ = 1, BAD_EW = 2, BAD_VW = 4, BAD_OFFS = 8 };

template <class T>
__global__ void k_narrow(const T* __restrict__ in, int32_t* __restrict__ out,
                         int64_t count, long long lo, long long hi, int flag,
                         unsigned* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool b = false;
  for (; i < count; i += stride) {
    long long x = (long long)in[i];
    b |= (x < lo) | (x > hi);
    out[i] = (int32_t)x;
  }
  if (__any_sync(__activemask(), b) && b) atomicOr(bad, (unsigned)flag);
}

__global__ void k_check_offsets(const int64_t* __restrict__ offs, int64_t n,
                                int64_t nnz, unsigned* bad) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool b = false;
  for (; i < n; i += stride) b |= offs[i + 1] < offs[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) b |= (offs[0] != 0) | (offs[n] != nnz);
  if (b) atomicOr(bad, (unsigned)BAD_OFFS);
}

// Per-level statistics: total/max vertex weight, max degree, max edge weight
// and the tier histogram (vertex counts and entry counts per tier).
struct LevelStats {
  unsigned long long total_vw, max_vw, max_deg, max_ew, min_vw;
  unsigned long long bin_cnt[NBINS], bin_nnz[NBINS];
};

__global__ void k_level_stats(const int64_t* __restrict__ offs,
                              const int32_t* __restrict__ vw,
                              const int32_t* __restrict__ ew, int64_t n,
                              int64_t nnz, TierMap tm, LevelStats* st) {
  __shared__ unsigned long long s_cnt[NBINS], s_nnz[NBINS];
  if (threadIdx.x < NBINS) {
    s_cnt[threadIdx.x] = 0;
    s_nnz[threadIdx.x] = 0;
  }
  __syncthreads();
  unsigned long long tv = 0, mv = 0, md = 0, me = 0, mn = ~0ull;
  // tier histogram in registers, reduced per warp (per-vertex shared atomics
  // on six addresses serialised 32-way)
  unsigned long long rc[NBINS], rn[NBINS];
#pragma unroll
  for (int t = 0; t < NBINS; ++t) rc[t] = rn[t] = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    int64_t d = offs[v + 1] - offs[v];
    unsigned long long w = (unsigned long long)vw[v];
    tv += w;
    mv = w > mv ? w : mv;
    mn = w < mn ? w : mn;
    md = (unsigned long long)d > md ? (unsigned long long)d : md;
    const int t = tm(d);
#pragma unroll
    for (int q = 0; q < NBINS; ++q) {
      rc[q] += q == t ? 1ull : 0ull;
      rn[q] += q == t ? (unsigned long long)d : 0ull;
    }
  }
#pragma unroll
  for (int q = 0; q < NBINS; ++q) {
    const unsigned long long c2 = gsum<32>(rc[q], 0xffffffffu);
    const unsigned long long n2 = gsum<32>(rn[q], 0xffffffffu);
    if ((threadIdx.x & 31) == 0 && c2) {
      atomicAdd(&s_cnt[q], c2);
      atomicAdd(&s_nnz[q], n2);
    }
  }
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz; e += stride) {
    unsigned long long w = (unsigned long long)ew[e];
    me = w > me ? w : me;
  }
  tv = gsum<32>(tv, 0xffffffffu);
  mv = gmax<32>(mv, 0xffffffffu);
  md = gmax<32>(md, 0xffffffffu);
  me = gmax<32>(me, 0xffffffffu);
  mn = gmin<32>(mn, 0xffffffffu);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&st->min_vw, mn);
    atomicAdd(&st->total_vw, tv);
    atomicMax(&st->max_vw, mv);
    atomicMax(&st->max_deg, md);
    atomicMax(&st->max_ew, me);
  }
  __syncthreads();
  if (threadIdx.x < NBINS) {
    atomicAdd(&st->bin_cnt[threadIdx.x], s_cnt[threadIdx.x]);
    atomicAdd(&st->bin_nnz[threadIdx.x], s_nnz[threadIdx.x]);
  }
}

struct TierIs {
  const int64_t* offs;
  int t;
  TierMap tm;
  __device__ __forceinline__ bool operator()(const int32_t& v) const {
    return tm(offs[v + 1] - offs[v]) == t;
  }
};

void finalize_graph(Ctx& c, DGraph& g) {
  g.tm = tiers_for(g.n);
  DBuf<LevelStats> st(1, c.stream);
  dzero(c, st.get(), 1);
  CK(cudaMemsetAsync(&st.get()->min_vw, 0xff, sizeof(unsigned long long), c.stream));
  if (g.n > 0) {
    launch(c, "level_stats", 8.0 * g.n + 4.0 * g.n + 4.0 * g.nnz, [&] {
      k_level_stats<<<grid_res(c, k_level_stats, g.n > g.nnz ? g.n : g.nnz, 256), 256, 0, c.stream>>>(
          g.offs.get(), g.vw.get(), g.ew.get(), g.n, g.local_nnz(), g.tm, st.get());
    });
  }
  LevelStats h;
  d2h(c, &h, st.get(), 1);
  c.sync();
  g.total_vw = (int64_t)h.total_vw;
  g.max_vw = (int64_t)h.max_vw;
  g.min_vw = g.n > 0 ? (int64_t)h.min_vw : 1;
  g.max_deg = (int64_t)h.max_deg;
  g.max_ew = (int64_t)h.max_ew;
  if (g.partial()) g.max_ew = comm_max(c, g.max_ew);  // the other ranks' entries
  g.unit_ew = g.nnz == 0 || g.max_ew <= 1;
  g.max_wdeg = g.max_deg * (g.max_ew > 0 ? g.max_ew : 1);  // upper bound
  JET_REQUIRE(g.max_wdeg < (1LL << (63 - KBITS)), JET_EUNSUPPORTED,
              "weighted degree too large for 64-bit gain keys");
  int nonempty = 0, last = -1;
  for (int t = 0; t < NBINS; ++t) {
    g.bin_cnt[t] = (int64_t)h.bin_cnt[t];
    g.bin_nnz[t] = (int64_t)h.bin_nnz[t];
    g.bin_list[t] = nullptr;
    if (g.bin_cnt[t]) {
      nonempty++;
      last = t;
    }
  }
  g.identity = nonempty <= 1;
  g.identity_bin = last;
  if (g.identity) return;
  g.bin_store.alloc((size_t)g.n, c.stream);
  DBuf<int64_t> nsel(1, c.stream);
  int64_t base = 0;
  for (int t = 0; t < NBINS; ++t) {
    if (!g.bin_cnt[t]) continue;
    int32_t* out = g.bin_store.get() + base;
    cub::CountingInputIterator<int32_t> it(0);
    TierIs op{g.offs.get(), t, g.tm};
    if (!small_select(c, "tier_select", op, g.n, out, nsel.get())) {
      size_t tmp = 0;
      CK(cub::DeviceSelect::If(nullptr, tmp, it, out, nsel.get(), (int)g.n, op, c.stream));
      void* p = c.cub_scratch(tmp);
      launch(c, "tier_select", 16.0 * g.n, [&] {
        CK(cub::DeviceSelect::If(p, tmp, it, out, nsel.get(), (int)g.n, op, c.stream));
      });
    }
    g.bin_list[t] = out;
    base += g.bin_cnt[t];
  }
}

// Pipelined host->device copy of `bytes` from pageable `src`; `consume(dptr,
// off, len)` is enqueued on the context stream for every device-side chunk.
template <class F>
static void staged_upload(Ctx& c, const void* src, size_t bytes, F&& consume) {
  c.ensure_upload_ring();
  const size_t CHB = Ctx::UPLOAD_CHUNK;
  const char* s = static_cast<const char*>(src);
  for (size_t off = 0, i = 0; off < bytes; off += CHB, ++i) {
    const size_t len = std::min(CHB, bytes - off);
    const int b = (int)(i % Ctx::UPLOAD_BUFS);
    CK(cudaEventSynchronize(c.up_ev[b]));  // the DMA that last used this buffer
    parallel_memcpy(c.up_host[b], s + off, len);
    uint8_t* d = c.up_dev.get() + (size_t)b * CHB;
    CK(cudaMemcpyAsync(d, c.up_host[b], len, cudaMemcpyHostToDevice, c.stream));
    consume(d, off, len);
    CK(cudaEventRecord(c.up_ev[b], c.stream));
  }
}

std::unique_ptr<DGraph> upload_graph(Ctx& c, int64_t n, const int64_t* offs,
                                     const void* adj, int adt, const void* ew,
                                     int edt, const void* vw, int vdt,
                                     int64_t row_lo, int64_t row_hi) {
  JET_REQUIRE(n >= 1, JET_EINVAL, "graph must have at least one vertex");
  JET_REQUIRE(n < (1LL << 31) - 1, JET_EUNSUPPORTED, "n must be < 2^31");
  JET_REQUIRE(offs, JET_EINVAL, "row_offsets is NULL");
  auto dt_ok = [](int d) { return d == JET_I32 || d == JET_I64; };
  JET_REQUIRE(dt_ok(adt) && dt_ok(edt) && dt_ok(vdt), JET_EINVAL, "bad dtype code");
  const int64_t nnz = offs[n];
  JET_REQUIRE(offs[0] == 0 && nnz >= 0, JET_EINVAL, "row_offsets must start at 0");
  auto g = std::make_unique<DGraph>();
  g->n = n;
  g->nnz = nnz;
  int64_t lnnz = nnz;  // entries stored on this rank
  if (row_hi >= 0) {
    JET_REQUIRE(0 <= row_lo && row_lo <= row_hi && row_hi <= n, JET_EINVAL, "bad row block");
    g->row_lo = row_lo;
    g->row_hi = row_hi;
    g->ent_lo = offs[row_lo];
    lnnz = offs[row_hi] - offs[row_lo];
  }
  g->offs.alloc(n + 1, c.stream);
  g->adj.alloc(lnnz > 0 ? lnnz : 1, c.stream);
  g->ew.alloc(lnnz > 0 ? lnnz : 1, c.stream);
  if (row_hi >= 0) {  // local_nnz() reads the buffer lengths
    g->adj.n = (size_t)lnnz;
    g->ew.n = (size_t)lnnz;
  }
  g->vw.alloc(n, c.stream);
  DBuf<unsigned> bad(1, c.stream);
  dzero(c, bad.get(), 1);
  {
    int64_t* doffs = g->offs.get();
    staged_upload(c, offs, (size_t)(n + 1) * 8, [&](const void* dchunk, size_t off, size_t bytes) {
      CK(cudaMemcpyAsync((char*)doffs + off, dchunk, bytes, cudaMemcpyDeviceToDevice, c.stream));
    });
  }
  launch(c, "check_offsets", 8.0 * (n + 1), [&] {
    k_check_offsets<<<grid_for(c, n, 256), 256, 0, c.stream>>>(g->offs.get(), n, nnz, bad.get());
  });
  // Host arrays stream through a ring of pinned buffers: several host
  // threads copy chunk i+1 into pinned memory while chunk i is DMA'd and
  // narrowed to int32 on the device (pageable cudaMemcpy tops out far below
  // the link rate).
  unsigned host_bad = 0;
  auto put = [&](const void* src, int dt, int32_t* dst, int64_t count, long long lo,
                 long long hi, int flag) {
    if (count == 0) return;
    if (dt == JET_I64) {
      // narrow (and range-check) on the host while staging: half the bytes
      // cross PCIe; all-ones weight chunks are not transferred but filled
      c.ensure_upload_ring();
      const int64_t per = (int64_t)(Ctx::UPLOAD_CHUNK / sizeof(int32_t));
      const int64_t* s64 = static_cast<const int64_t*>(src);
      for (int64_t e0 = 0, i = 0; e0 < count; e0 += per, ++i) {
        const int64_t m = std::min(per, count - e0);
        const int b = (int)(i % Ctx::UPLOAD_BUFS);
        CK(cudaEventSynchronize(c.up_ev[b]));
        bool ones = false;
        int32_t* h32 = static_cast<int32_t*>(c.up_host[b]);
        if (!parallel_narrow(h32, s64 + e0, m, lo, hi, flag != BAD_ADJ, &ones)) host_bad |= flag;
        if (ones) {
          launch(c, "fill_ones", 4.0 * m, [&] {
            k_fill_ones<<<grid_for(c, m, 256), 256, 0, c.stream>>>(dst + e0, m);
          });
        } else {
          CK(cudaMemcpyAsync(dst + e0, h32, (size_t)m * sizeof(int32_t), cudaMemcpyHostToDevice,
                             c.stream));
        }
        CK(cudaEventRecord(c.up_ev[b], c.stream));
      }
      return;
    }
    const size_t esz = dt == JET_I32 ? 4 : 8;
    staged_upload(c, src, (size_t)count * esz, [&](const void* dchunk, size_t off, size_t bytes) {
      const int64_t e0 = (int64_t)(off / esz), m = (int64_t)(bytes / esz);
      if (dt == JET_I32) {
        launch(c, "validate_i32", 8.0 * m, [&] {
          k_narrow<int32_t><<<grid_for(c, m, 256), 256, 0, c.stream>>>(
              (const int32_t*)dchunk, dst + e0, m, lo, hi, flag, bad.get());
        });
      } else {
        launch(c, "narrow_i64", 12.0 * m, [&] {
          k_narrow<int64_t><<<grid_for(c, m, 256), 256, 0, c.stream>>>(
              (const int64_t*)dchunk, dst + e0, m, lo, hi, flag, bad.get());
        });
      }
    });
  };
  const long long I32MAX = 2147483647LL;
  put(adj, adt, g->adj.get(), lnnz, 0, n - 1, BAD_ADJ);
  put(ew, edt, g->ew.get(), lnnz, 1, I32MAX, BAD_EW);
  put(vw, vdt, g->vw.get(), n, 1, I32MAX, BAD_VW);
  unsigned hbad = 0;
  d2h(c, &hbad, bad.get(), 1);
  c.sync();
  hbad |= host_bad;
  JET_REQUIRE(!(hbad & BAD_OFFS), JET_EINVAL, "row_offsets must be non-decreasing from 0 to nnz");
  JET_REQUIRE(!(hbad & BAD_ADJ), JET_EINVAL, "neighbor id out of range");
  JET_REQUIRE(!(hbad & BAD_EW), JET_EINVAL, "edge weights must be in [1, 2^31)");
  JET_REQUIRE(!(hbad & BAD_VW), JET_EINVAL, "vertex weights must be in [1, 2^31)");
  finalize_graph(c, *g);
  return g;
}

// ---------------------------------------------------------------------------
// cutsize: sum over entries with part(u) != part(v), halved (graph.py:215-221)
template <int G, bool UNIT>
__global__ void __launch_bounds__(256) k_cut(GView g, const int32_t* __restrict__ list,
                                             int64_t cnt, const int32_t* __restrict__ parts,
                                             unsigned long long* out) {
  const unsigned gm = group_mask<G>();
  const int gl = threadIdx.x & (G - 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x / G;
  long long acc = 0;
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G; i < cnt; i += stride) {
    const int v = list ? list[i] : (int)i;
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    const int pv = parts[v];
    for (int64_t j = b + gl; j < e; j += G) {
      int u = g.adj[j];
      if (parts[u] != pv) acc += UNIT ? 1 : g.ew[j];
    }
  }
  (void)gm;
  block_sum_atomic<256>(acc, out);
}

int64_t device_cutsize(Ctx& c, const DGraph& g, const int32_t* parts) {
  DBuf<unsigned long long> acc(1, c.stream);
  dzero(c, acc.get(), 1);
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = g.bin_cnt[t];
    if (!cnt) continue;
    const int G = t < 4 ? TIER_G[t] : 32;
    const int32_t* list = tier_list(g, t);
    const unsigned grid = grid_for(c, cnt * G, 256);
    const GView v = view(g);
    launch(c, "cutsize", (g.unit_ew ? 8.0 : 12.0) * g.bin_nnz[t] + 12.0 * cnt, [&] {
      JET_TIER_LAUNCH(k_cut, G, g.unit_ew, grid, 256, 0, c.stream, v, list, cnt, parts, acc.get());
    });
  }
  unsigned long long h = 0;
  d2h(c, &h, acc.get(), 1);
  c.sync();
  return (int64_t)(h / 2);
}

// ---------------------------------------------------------------------------
// part weights: weighted bincount (graph.py:240-242)
__global__ void k_part_weights(const int32_t* __restrict__ parts,
                               const int32_t* __restrict__ vw, int64_t n, int k,
                               unsigned long long* pw) {
  extern __shared__ unsigned long long s_pw[];
  const bool use_smem = k <= 4096;
  if (use_smem)
    for (int i = threadIdx.x; i < k; i += blockDim.x) s_pw[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    int p = parts[v];
    if (use_smem) atomicAdd(&s_pw[p], (unsigned long long)vw[v]);
    else atomicAdd(&pw[p], (unsigned long long)vw[v]);
  }
  __syncthreads();
  if (use_smem)
    for (int i = threadIdx.x; i < k; i += blockDim.x)
      if (s_pw[i]) atomicAdd(&pw[i], s_pw[i]);
}

void device_part_weights(Ctx& c, const DGraph& g, const int32_t* parts, int k,
                         int64_t* d_pw) {
  dzero(c, d_pw, k);
  size_t smem = k <= 4096 ? (size_t)k * 8 : 0;
  launch(c, "part_weights", 8.0 * g.n + 8.0 * k, [&] {
    k_part_weights<<<grid_for(c, g.n, 256, 4), 256, smem, c.stream>>>(
        parts, g.vw.get(), g.n, k, (unsigned long long*)d_pw);
  });
}

// ---------------------------------------------------------------------------
// projection: parts_f[v] = parts_c[vmap[v]]  (driver.py:32-45)
__global__ void k_project(const int32_t* __restrict__ vmap,
                          const int32_t* __restrict__ pc, int32_t* __restrict__ pf,
                          int64_t nf) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < nf; v += stride)
    pf[v] = pc[vmap[v]];
}

void device_project(Ctx& c, const int32_t* vmap, const int32_t* pc, int32_t* pf,
                    int64_t nf) {
  launch(c, "project", 12.0 * nf, [&] {
    k_project<<<grid_for(c, nf, 256), 256, 0, c.stream>>>(vmap, pc, pf, nf);
  });
}

// int64 <-> int32 helpers for the per-kernel entry points

void upload_i64_as_i32(Ctx& c, const int64_t* host, int64_t n, int32_t* dst,
                       long long lo, long long hi, const char* what) {
  if (n <= 0) return;
  DBuf<int64_t> s(n, c.stream);
  DBuf<unsigned> bad(1, c.stream);
  dzero(c, bad.get(), 1);
  h2d(c, s.get(), host, n);
  launch(c, "narrow_i64", 12.0 * n, [&] {
    k_narrow<int64_t><<<grid_for(c, n, 256), 256, 0, c.stream>>>(s.get(), dst, n, lo, hi, 1, bad.get());
  });
  unsigned hb = 0;
  d2h(c, &hb, bad.get(), 1);
  c.sync();
  JET_REQUIRE(!hb, JET_EINVAL, std::string(what) + " out of range");
}

// int32 -> int64 on the host cores, out of pinned memory (the caller's
// pages are first touched here, by all threads)
static void parallel_widen(int64_t* dst, const int32_t* src, int64_t count) {
  const int64_t piece = (int64_t)1 << 18;
  const int64_t np = (count + piece - 1) / piece;
#pragma omp parallel for schedule(static) num_threads(std::min<int>(upload_threads(), omp_get_num_procs()))
  for (int64_t i = 0; i < np; ++i) {
    const int64_t b = i * piece, e = std::min(count, b + piece);
    for (int64_t j = b; j < e; ++j) dst[j] = src[j];
  }
}

// Device int32 -> host int64: the int32 words cross PCIe into the pinned
// ring (half the bytes of a device-side widen, and no pageable staging by the
// driver) and are widened by the host threads, chunk i while chunk i+1 is
// in flight.
void download_i32_as_i64(Ctx& c, const int32_t* dsrc, int64_t n, int64_t* host) {
  if (n <= 0) return;
  c.ensure_upload_ring();
  const int64_t per = (int64_t)(Ctx::UPLOAD_CHUNK / sizeof(int32_t));
  const int64_t nch = (n + per - 1) / per;
  auto enqueue = [&](int64_t i) {
    const int b = (int)(i % Ctx::UPLOAD_BUFS);
    const int64_t len = std::min(per, n - i * per);
    CK(cudaMemcpyAsync(c.up_host[b], dsrc + i * per, (size_t)len * sizeof(int32_t),
                       cudaMemcpyDeviceToHost, c.stream));
    CK(cudaEventRecord(c.up_ev[b], c.stream));
  };
  for (int64_t i = 0; i < std::min<int64_t>(nch, Ctx::UPLOAD_BUFS); ++i) enqueue(i);
  for (int64_t i = 0; i < nch; ++i) {
    const int b = (int)(i % Ctx::UPLOAD_BUFS);
    CK(cudaEventSynchronize(c.up_ev[b]));
    parallel_widen(host + i * per, static_cast<const int32_t*>(c.up_host[b]),
                   std::min(per, n - i * per));
    if (i + Ctx::UPLOAD_BUFS < nch) enqueue(i + Ctx::UPLOAD_BUFS);
  }
}

}  // namespace jet
