// refine.cu — Jetlp gains + gain-ratio filter, afterburner, weak/strong
// rebalancing with bucketed loss selection, and move application.
//
// Reference semantics (all bit-exact):
//   select_destinations  refine.py:78-105   (max conn, ties -> lowest part)
//   gain_ratio_filter    refine.py:108-124  (-F < floor(conn_self * a / b))
//   afterburner          refine.py:127-156  (priority: higher F, then lower id)
//   jetlp_pass           refine.py:159-183
//   _candidate_stats     rebalance.py:91-113
//   loss_slots/bucket_order/select_prefix/_evict  rebalance.py:35-136
//   weak/strong passes   rebalance.py:139-240
//   ConnectivityTable.apply (parts, part weights, exact cut delta) conn.py:215-254
#include "refine.cuh"
#include "rng.h"
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
#include <cmath>

namespace jet {

// ===========================================================================
// Row aggregation framework. For every vertex v of a tier, conn(v, p) is
// aggregated over the row; an Op decides which parts compete for the "best"
// slot, what else is summed, and what to do with the result.
//   tiers 0-3: one G-lane group per row, __match_any_sync groups equal parts
//   tier 4   : one warp per row, per-warp shared-memory table of k entries
//   tier 5   : one block per row, per-block shared-memory table
// ===========================================================================

__device__ __forceinline__ unsigned long long pack_best(long long conn, int p) {
  return ((unsigned long long)conn << KBITS) | (unsigned)(KMASK - p);
}
__device__ __forceinline__ int unpack_part(unsigned long long key) {
  return KMASK - (int)(key & KMASK);
}
__device__ __forceinline__ long long unpack_conn(unsigned long long key) {
  return (long long)(key >> KBITS);
}

// ---- Jetlp gains op --------------------------------------------------------
struct LpOp {
  struct Args {
    const int32_t* parts;
    int32_t* cdest;
    long long* F;
    int32_t* mv;
    const int32_t* lock;
    LpParams p;
    int32_t* out_list;  // candidate list (afterburner on) or move list (off)
    unsigned long long* out_cnt;
    unsigned long long* cut2;
    LpDebug dbg;
  };
  static __device__ __forceinline__ bool skip(const Args&, int, int) { return false; }
  static __device__ __forceinline__ bool competes(const Args&, int p, int own) { return p != own; }
  static __device__ __forceinline__ int extra(const Args&, int, int w) { return w; }
  // self_c = conn(v, own); key = best other part; ex = weighted degree
  static __device__ __forceinline__ void finish(const Args& a, int v, int own,
                                                long long self_c,
                                                unsigned long long key,
                                                long long ex, long long& acc) {
    acc += ex - self_c;
    const bool boundary = key != 0;
    const int dest = boundary ? unpack_part(key) : own;
    const long long F = boundary ? unpack_conn(key) - self_c : NO_GAIN;
    bool cand = false;
    if (boundary && !(a.p.locking && a.lock[v] == a.p.lock_epoch)) {
      if (a.p.afterburner) {
        long long bound = a.p.c_use_float
                              ? (long long)floor(a.p.c_f * (double)self_c)
                              : self_c * a.p.c_num / a.p.c_den;
        cand = -F < bound;
      } else {
        cand = F >= 0;
      }
    }
    if (a.p.afterburner) {
      a.cdest[v] = cand ? dest : -1;
      if (cand) a.F[v] = F;
    } else if (cand) {
      a.mv[v] = dest;
    }
    if (a.dbg.dest) a.dbg.dest[v] = dest;
    if (a.dbg.gain) a.dbg.gain[v] = F;
    if (a.dbg.boundary) a.dbg.boundary[v] = boundary;
    if (a.dbg.conn_self) a.dbg.conn_self[v] = self_c;
    warp_append(cand, v, a.out_list, a.out_cnt);
  }
  static __device__ __forceinline__ void block_done(const Args& a, long long acc) {
    block_sum_atomic<256>(acc, a.cut2);
  }
};

// ---- rebalance candidate stats op (rebalance.py:91-113, 35-51) -------------
struct RbOp {
  struct Args {
    const int32_t* parts;
    const int32_t* vw;
    const int32_t* opidx;   // part -> oversized rank or -1
    const uint8_t* valid;   // part -> valid destination
    const double* hb;       // heavy bound per oversized rank
    int nvalid;
    int strong;
    int rho;
    int slot_min;
    int nb;                 // buckets per oversized part
    int32_t* rkey;
    int32_t* rbest;
    double* rloss;
    int32_t* rcand;
    unsigned long long* rcand_cnt;
    unsigned long long* H;
  };
  static __device__ __forceinline__ bool skip(const Args& a, int, int own) {
    return a.opidx[own] < 0;
  }
  static __device__ __forceinline__ bool competes(const Args& a, int p, int) {
    return a.valid[p] != 0;
  }
  static __device__ __forceinline__ int extra(const Args& a, int p, int w) {
    return a.valid[p] ? w : 0;
  }
  static __device__ __forceinline__ void finish(const Args& a, int v, int own,
                                                long long conn_src,
                                                unsigned long long key,
                                                long long sum_valid, long long&) {
    const int op = a.opidx[own];
    const long long best_conn = key ? unpack_conn(key) : 0;
    const int best_part = key ? unpack_part(key) : -1;
    int slot;
    double loss;
    if (!a.strong) {
      const long long L = conn_src - best_conn;
      loss = (double)L;
      slot = L < 0 ? 0 : L == 0 ? 1 : min(2 + (63 - __clzll(L)), 33);
    } else {
      // numpy: int64 - (int64 / int) -> float64 (rebalance.py:213)
      loss = (double)conn_src - (double)sum_valid / (double)a.nvalid;
      if (loss < 0) slot = 0;
      else if (loss == 0) slot = 1;
      else slot = min(2 + ilogb(loss), 33);
    }
    slot = max(slot, a.slot_min);
    const int w = a.vw[v];
    const bool eligible = (double)w <= a.hb[op];
    bool take = false;
    if (eligible) {
      const int bucket = (slot - a.slot_min) * a.rho + (v % a.rho);
      a.rkey[v] = bucket;
      a.rbest[v] = best_part;
      a.rloss[v] = loss;
      atomicAdd(&a.H[(size_t)op * a.nb + bucket], (unsigned long long)w);
      take = true;
    } else {
      a.rkey[v] = -1;
    }
    warp_append(take, v, a.rcand, a.rcand_cnt);
  }
  static __device__ __forceinline__ void block_done(const Args&, long long) {}
};

// Tiers 0-3. A warp owns 32 consecutive list entries: vertex ids, offsets
// and own parts are loaded once, coalesced. Rows are then swept in G steps
// of 32/G rows (one G-lane group per row); U steps are batched so their
// adjacency loads and neighbour-part gathers are all in flight together
// (the single-row-per-warp form is latency-bound at ~300 GB/s). The result
// of row r is shuffled to lane r, which finishes vertex r.
template <class Op, int G, bool UNIT>
__global__ void __launch_bounds__(256)
    k_agg_small(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
                const int32_t* __restrict__ list, int64_t cnt, bool wide,
                const unsigned long long* __restrict__ dcnt) {
  if (dcnt) cnt = (int64_t)*dcnt;
  constexpr int RPS = 32 / G;         // rows per step
  constexpr int U = G >= 8 ? 8 : G;   // steps per batch (G steps in total)
  const unsigned gm = group_mask<G>();
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long acc = 0;
  for (int64_t base = w0 * 32; base < cnt; base += nw * 32) {
    const int64_t idx = base + lane;
    int v = 0, own = -1, deg = 0;
    int64_t beg = 0;
    if (idx < cnt) {
      v = list ? list[idx] : (int)idx;
      own = parts[v];
      if (Op::skip(a, v, own)) {
        own = -1;
      } else {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
      }
    }
    long long my_self = 0, my_ex = 0;
    unsigned long long my_key = 0;
#pragma unroll
    for (int s0 = 0; s0 < G; s0 += U) {
      int uu[U], ww[U], pp[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int r = (s0 + q) * RPS + grp;
        const int64_t rb = __shfl_sync(0xffffffffu, beg, r);
        const int rd = __shfl_sync(0xffffffffu, deg, r);
        uu[q] = -1;
        ww[q] = 0;
        if (gl < rd) {
          uu[q] = g.adj[rb + gl];
          ww[q] = UNIT ? 1 : g.ew[rb + gl];
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) pp[q] = uu[q] >= 0 ? parts[uu[q]] : -1;
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int st = s0 + q;
        const int rown = __shfl_sync(0xffffffffu, own, st * RPS + grp);
        const int p = pp[q];
        const unsigned peers = __match_any_sync(gm, p);
        const bool comp = p >= 0 && p != rown && Op::competes(a, p, rown);
        const int src = ((lane - st * RPS) & (RPS - 1)) * G;
        if (!wide) {
          // 32-bit sums (weighted degree < 2^31): single-instruction REDUX
          // reductions; best part = max conn, then lowest part id
          const unsigned sm =
              UNIT ? (unsigned)__popc(peers) : __reduce_add_sync(peers, (unsigned)ww[q]);
          const unsigned sc =
              UNIT ? (unsigned)__popc(__ballot_sync(gm, p >= 0 && p == rown))
                   : __reduce_add_sync(gm, (p >= 0 && p == rown) ? (unsigned)ww[q] : 0u);
          const unsigned mx = __reduce_max_sync(gm, comp ? sm : 0u);
          const unsigned pm = __reduce_min_sync(gm, (comp && sm == mx) ? (unsigned)p : 0xffffffffu);
          const unsigned ex = __reduce_add_sync(gm, p >= 0 ? (unsigned)Op::extra(a, p, ww[q]) : 0u);
          const unsigned dsc = __shfl_sync(0xffffffffu, sc, src);
          const unsigned dmx = __shfl_sync(0xffffffffu, mx, src);
          const unsigned dpm = __shfl_sync(0xffffffffu, pm, src);
          const unsigned dex = __shfl_sync(0xffffffffu, ex, src);
          if (lane / RPS == st) {
            my_self = dsc;
            my_key = dmx ? pack_best((long long)dmx, (int)dpm) : 0ull;
            my_ex = dex;
          }
        } else {
          const long long sm = UNIT ? (long long)__popc(peers) : peer_sum(peers, ww[q], wide);
          const bool lead = p >= 0 && (__ffs(peers) - 1) == lane;
          long long sc = (lead && p == rown) ? sm : 0;
          unsigned long long key = (lead && comp) ? pack_best(sm, p) : 0ull;
          long long ex = p >= 0 ? Op::extra(a, p, ww[q]) : 0;
          sc = gsum<G>(sc, gm);
          key = gmax<G>(key, gm);
          ex = gsum<G>(ex, gm);
          sc = __shfl_sync(0xffffffffu, sc, src);
          key = __shfl_sync(0xffffffffu, key, src);
          ex = __shfl_sync(0xffffffffu, ex, src);
          if (lane / RPS == st) {
            my_self = sc;
            my_key = key;
            my_ex = ex;
          }
        }
      }
    }
    if (own >= 0) Op::finish(a, v, own, my_self, my_key, my_ex, acc);
  }
  Op::block_done(a, acc);
}

// Tier 4 (33..2048 entries). A warp owns 32 rows; per-vertex data is loaded
// once, coalesced. Rows are aggregated one after another into a per-warp
// shared-memory part table, but the adjacency of the next chunk batch (of
// this row, or of the next row) is loaded while the current batch's
// neighbour parts are gathered and aggregated, so two batches of loads are
// always in flight. Shared layout per warp: tab[k] (u64), tl[tl_cap] (i32),
// tcnt (i32).
template <class Op, bool UNIT>
__global__ void __launch_bounds__(256)
    k_agg_warp(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
               const int32_t* __restrict__ list, int64_t cnt, bool wide, int k,
               int tl_cap, const unsigned long long* __restrict__ dcnt) {
  if (dcnt) cnt = (int64_t)*dcnt;
  constexpr int U = 2;  // chunks of 32 entries per batch
  extern __shared__ unsigned long long smem[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per = (size_t)k + (size_t)(tl_cap + 3) / 2;
  unsigned long long* tab = smem + wib * per;
  int* tl = reinterpret_cast<int*>(tab + k);
  int* tcnt = tl + tl_cap;
  for (int i = lane; i < k; i += 32) tab[i] = 0;
  if (lane == 0) *tcnt = 0;
  __syncwarp();
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long acc = 0;
  for (int64_t base = w0 * 32; base < cnt; base += nw * 32) {
    const int64_t idx = base + lane;
    int v = 0, own = -1, deg = 0;
    int64_t beg = 0;
    if (idx < cnt) {
      v = list ? list[idx] : (int)idx;
      own = parts[v];
      if (Op::skip(a, v, own)) {
        own = -1;
      } else {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
      }
    }
    long long my_self = 0, my_ex = 0;
    unsigned long long my_key = 0;
    // pipeline state: (row, first chunk) of the batch whose adjacency is loaded
    int r = 0, c0 = 0;
    int64_t rb = __shfl_sync(0xffffffffu, beg, 0);
    int rd = __shfl_sync(0xffffffffu, deg, 0);
    int uu[U], ww[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int j = (c0 + q) * 32 + lane;
      uu[q] = j < rd ? g.adj[rb + j] : -1;
      ww[q] = (j < rd) ? (UNIT ? 1 : g.ew[rb + j]) : 0;
    }
    long long ex = 0;
    while (r < 32) {
      int pp[U];
#pragma unroll
      for (int q = 0; q < U; ++q) pp[q] = uu[q] >= 0 ? parts[uu[q]] : -1;
      // next batch: same row if it has more chunks, else the next row
      const int cur_r = r, cur_d = rd;
      int wv[U];
#pragma unroll
      for (int q = 0; q < U; ++q) wv[q] = ww[q];
      if ((c0 + U) * 32 < rd) {
        c0 += U;
      } else {
        ++r;
        c0 = 0;
        rb = r < 32 ? __shfl_sync(0xffffffffu, beg, r & 31) : 0;
        rd = r < 32 ? __shfl_sync(0xffffffffu, deg, r & 31) : 0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int j = (c0 + q) * 32 + lane;
        uu[q] = (r < 32 && j < rd) ? g.adj[rb + j] : -1;
        ww[q] = (r < 32 && j < rd) ? (UNIT ? 1 : g.ew[rb + j]) : 0;
      }
      // aggregate the current batch
      const int rown = __shfl_sync(0xffffffffu, own, cur_r);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int p = pp[q];
        if (p >= 0) ex += Op::extra(a, p, wv[q]);
        const unsigned peers = __match_any_sync(0xffffffffu, p);
        const long long sm = UNIT ? (long long)__popc(peers) : peer_sum(peers, wv[q], wide);
        if (p >= 0 && (__ffs(peers) - 1) == lane) {
          const unsigned long long old = atomicAdd(&tab[p], (unsigned long long)sm);
          if (old == 0) tl[atomicAdd(tcnt, 1)] = p;
        }
      }
      if (r != cur_r) {  // row cur_r complete: reduce its table
        __syncwarp();
        const int nt = *tcnt;
        long long sc = 0;
        unsigned long long key = 0;
        long long ext;
        if (!wide) {
          // 32-bit sums: REDUX reductions (max conn, then lowest part)
          unsigned usc = 0, bm = 0, bp = 0xffffffffu;
          for (int t = lane; t < nt; t += 32) {
            const int p = tl[t];
            const unsigned cv = (unsigned)tab[p];
            tab[p] = 0;
            if (p == rown) usc = cv;
            else if (Op::competes(a, p, rown) && (cv > bm || (cv == bm && (unsigned)p < bp))) {
              bm = cv;
              bp = (unsigned)p;
            }
          }
          usc = __reduce_add_sync(0xffffffffu, usc);
          const unsigned mx = __reduce_max_sync(0xffffffffu, bm);
          const unsigned pm = __reduce_min_sync(0xffffffffu, bm == mx ? bp : 0xffffffffu);
          sc = usc;
          key = mx ? pack_best((long long)mx, (int)pm) : 0ull;
          ext = __reduce_add_sync(0xffffffffu, (unsigned)ex);
        } else {
          for (int t = lane; t < nt; t += 32) {
            const int p = tl[t];
            const long long cv = (long long)tab[p];
            tab[p] = 0;
            if (p == rown) sc = cv;
            else if (Op::competes(a, p, rown)) {
              const unsigned long long kk = pack_best(cv, p);
              key = kk > key ? kk : key;
            }
          }
          sc = gsum<32>(sc, 0xffffffffu);
          key = gmax<32>(key, 0xffffffffu);
          ext = gsum<32>(ex, 0xffffffffu);
        }
        ex = 0;
        if (lane == cur_r) {
          my_self = sc;
          my_key = key;
          my_ex = ext;
        }
        __syncwarp();
        if (lane == 0) *tcnt = 0;
        __syncwarp();
        (void)cur_d;
      }
    }
    if (own >= 0) Op::finish(a, v, own, my_self, my_key, my_ex, acc);
  }
  Op::block_done(a, acc);
}

// Tier 5: one block (256 threads) per row; block-wide shared part table.
template <class Op, bool UNIT>
__global__ void __launch_bounds__(256)
    k_agg_block(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
                const int32_t* __restrict__ list, int64_t cnt, bool wide, int k,
                const unsigned long long* __restrict__ dcnt) {
  if (dcnt) cnt = (int64_t)*dcnt;
  extern __shared__ unsigned long long smem[];
  unsigned long long* tab = smem;
  int* tl = reinterpret_cast<int*>(tab + k);
  __shared__ int tcnt;
  __shared__ long long r_self[8], r_ex[8];
  __shared__ unsigned long long r_key[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tab[i] = 0;
  if (threadIdx.x == 0) tcnt = 0;
  __syncthreads();
  long long acc = 0;
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int v = list ? list[i] : (int)i;
    const int own = parts[v];
    if (Op::skip(a, v, own)) continue;  // uniform across the block
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    long long ex = 0;
    for (int64_t j0 = b; j0 < e; j0 += blockDim.x) {
      const int64_t j = j0 + threadIdx.x;
      int p = -1, w = 0;
      if (j < e) {
        p = parts[g.adj[j]];
        w = UNIT ? 1 : g.ew[j];
        ex += Op::extra(a, p, w);
      }
      const unsigned peers = __match_any_sync(0xffffffffu, p);
      const long long s = UNIT ? (long long)__popc(peers) : peer_sum(peers, w, wide);
      if (p >= 0 && (__ffs(peers) - 1) == lane) {
        unsigned long long old = atomicAdd(&tab[p], (unsigned long long)s);
        if (old == 0) tl[atomicAdd(&tcnt, 1)] = p;
      }
    }
    __syncthreads();
    const int nt = tcnt;
    long long self_c = 0;
    unsigned long long key = 0;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      const int p = tl[t];
      const long long cv = (long long)tab[p];
      tab[p] = 0;
      if (p == own) self_c = cv;
      else if (Op::competes(a, p, own)) {
        unsigned long long kk = pack_best(cv, p);
        key = kk > key ? kk : key;
      }
    }
    self_c = gsum<32>(self_c, 0xffffffffu);
    key = gmax<32>(key, 0xffffffffu);
    ex = gsum<32>(ex, 0xffffffffu);
    if (lane == 0) {
      r_self[wid] = self_c;
      r_key[wid] = key;
      r_ex[wid] = ex;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int q = 1; q < (int)(blockDim.x >> 5); ++q) {
        self_c += r_self[q];
        key = r_key[q] > key ? r_key[q] : key;
        ex += r_ex[q];
      }
      tcnt = 0;
      Op::finish(a, v, own, self_c, key, ex, acc);
    }
    __syncthreads();
  }
  Op::block_done(a, acc);
}

static int warp_tier_warps(const Ctx& c, int k, int tl_cap, size_t* smem_out) {
  const size_t per = ((size_t)k + (size_t)(tl_cap + 3) / 2) * 8;
  size_t limit = (size_t)c.max_smem_optin;
  int nw = 8;
  while (nw > 1 && per * nw > limit) nw >>= 1;
  JET_REQUIRE(per * nw <= limit, JET_EUNSUPPORTED,
              "k too large for the shared-memory part table (long rows)");
  *smem_out = per * nw;
  return nw;
}

// Launch an aggregation Op over every non-empty tier of g; mk(t) returns the
// Op arguments for tier t (per-tier output lists).
// dlists/dcnts (optional): per-tier vertex lists with device-side lengths
// replace the level's tier lists (the host bound stays g.bin_cnt[t]).
template <class Op, class MakeArgs>
static void run_agg(Ctx& c, const DGraph& g, MakeArgs mk, const int32_t* parts,
                    int k, const char* name, double bytes_per_vertex,
                    int32_t* const* dlists = nullptr,
                    const unsigned long long* dcnts = nullptr) {
  // 32-bit conn sums are exact when every weighted degree is < 2^31
  const bool wide = g.max_wdeg >= (1LL << 31);
  const GView gv = view(g);
  const double bpe = g.unit_ew ? 8.0 : 12.0;  // adj + gathered part (+ weight)
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = g.bin_cnt[t];
    if (!cnt) continue;
    const typename Op::Args a = mk(t);
    const int32_t* list = dlists ? dlists[t] : tier_list(g, t);
    const unsigned long long* dc = dcnts ? dcnts + t : nullptr;
    const double bytes =
        dlists ? 0.0 : bpe * g.bin_nnz[t] + (bytes_per_vertex + (list ? 4.0 : 0.0)) * cnt;
    if (t < 4) {
      const int G = TIER_G[t];
      const unsigned grid = grid_for(c, cnt, 256);
      launch(c, name, bytes, [&] {
#define AGG_K(GG, UU) k_agg_small<Op, GG, UU>
        if (g.unit_ew) {
          switch (G) {
            case 4: AGG_K(4, true)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 8: AGG_K(8, true)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 16: AGG_K(16, true)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            default: AGG_K(32, true)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
          }
        } else {
          switch (G) {
            case 4: AGG_K(4, false)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 8: AGG_K(8, false)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 16: AGG_K(16, false)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            default: AGG_K(32, false)<<<grid, 256, 0, c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
          }
        }
#undef AGG_K
      });
    } else if (t == BIN_WARP) {
      const int tl_cap = (int)std::min<int64_t>(k, WARP_TIER_MAX_DEG);
      size_t smem = 0;
      const int nw = warp_tier_warps(c, k, tl_cap, &smem);
      auto kern = g.unit_ew ? k_agg_warp<Op, true> : k_agg_warp<Op, false>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid = grid_for(c, cnt, nw * 32, 2048 / (nw * 32));
      launch(c, name, bytes, [&] {
        kern<<<grid, nw * 32, smem, c.stream>>>(a, gv, parts, list, cnt, wide, k, tl_cap, dc);
      });
    } else {
      const size_t smem = (size_t)k * 12;
      JET_REQUIRE(smem <= (size_t)c.max_smem_optin, JET_EUNSUPPORTED,
                  "k too large for the block part table (hub rows)");
      auto kern = g.unit_ew ? k_agg_block<Op, true> : k_agg_block<Op, false>;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const unsigned grid = grid_for(c, cnt * 256, 256, 2);
      launch(c, name, bytes, [&] {
        kern<<<grid, 256, smem, c.stream>>>(a, gv, parts, list, cnt, wide, k, dc);
      });
    }
  }
}

// ===========================================================================
// Reduction-only row kernels: afterburner and apply (cut delta, weights).
// Rows of a G-tier list are walked by G-lane groups (G = 32 for tiers 4/5).
// The list length lives on the device (written by the preceding kernel).
// ===========================================================================

struct RbSegsDev {
  int64_t b[NBINS];
};

struct AbArgs {
  const int32_t* parts;
  const int32_t* cdest;
  const long long* F;
  int32_t* mv;
  int32_t* move_list;
  unsigned long long* move_cnt;
  long long* f2_out;  // optional (parity entry point)
};

// Segmented vertex lists (one per tier) with device-side lengths.
struct SegLists {
  const int32_t* list[NBINS];
  const unsigned long long* cnt;  // NBINS consecutive counters
};

// One warp per candidate over all tiers (candidate sets are small).
template <bool UNIT>
__global__ void __launch_bounds__(256)
    k_afterburner(AbArgs a, GView g, SegLists sl, RbSegsDev mseg) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)sl.cnt[t];
    const int32_t* list = sl.list[t];
    for (int64_t i = w0; i < cnt; i += ws) {
      const int v = list[i];
      const int own = a.parts[v];
      const int dv = a.cdest[v];
      const long long Fv = a.F[v];
      const int64_t b = g.offs[v], e = g.offs[v + 1];
      long long f2 = 0;
      for (int64_t j = b + lane; j < e; j += 32) {
        const int u = g.adj[j];
        int eff = a.parts[u];
        const int cu = a.cdest[u];
        if (cu >= 0) {
          const long long Fu = a.F[u];
          if (Fu > Fv || (Fu == Fv && u < v)) eff = cu;
        }
        const int w = UNIT ? 1 : g.ew[j];
        f2 += (eff == dv) ? w : (eff == own) ? -w : 0;
      }
      f2 = gsum<32>(f2, 0xffffffffu);
      if (lane == 0) {
        if (a.f2_out) a.f2_out[v] = f2;
        if (a.move_list && f2 >= 0) {
          a.mv[v] = dv;
          const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
          a.move_list[mseg.b[t] + q] = v;
        }
      }
    }
  }
}

struct ApArgs {
  const int32_t* parts;
  const int32_t* mv;
  unsigned long long* pw;
  unsigned long long* cut2d;
  int k;
};

// Exact cut delta of a move batch (conn.py:231-248): for a moved v and
// neighbour u, c = w([p'(u) != dest] - [p(u) != old]); edges with both ends
// moved appear twice and are halved, so we sum 2c / c and halve at the end.
template <bool UNIT>
__global__ void __launch_bounds__(256) k_apply_delta(ApArgs a, GView g, SegLists sl) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  long long acc = 0;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)sl.cnt[t];
    const int32_t* list = sl.list[t];
    for (int64_t i = w0; i < cnt; i += ws) {
      const int v = list[i];
      const int old = a.parts[v];
      const int dst = a.mv[v];
      const int64_t b = g.offs[v], e = g.offs[v + 1];
      long long d = 0;
      for (int64_t j = b + lane; j < e; j += 32) {
        const int u = g.adj[j];
        const int pu = a.parts[u];
        const int mu = a.mv[u];
        const int nu = mu >= 0 ? mu : pu;
        const long long w = UNIT ? 1 : g.ew[j];
        const long long cc = w * ((long long)(nu != dst) - (long long)(pu != old));
        d += mu >= 0 ? cc : 2 * cc;
      }
      d = gsum<32>(d, 0xffffffffu);
      if (lane == 0) {
        acc += d;
        const unsigned long long wv = (unsigned long long)g.vw[v];
        atomicAdd(&a.pw[dst], wv);
        atomicAdd(&a.pw[old], (unsigned long long)(-(long long)wv));
      }
    }
  }
  block_sum_atomic<256>(acc, a.cut2d);
}

struct CommitArgs {
  int32_t* parts;
  int32_t* mv;
  int32_t* lock;
  int32_t epoch;
  int set_lock;
  const int32_t* lists[NBINS];
  const unsigned long long* cnts;
};

__global__ void k_apply_commit(CommitArgs a) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)a.cnts[t];
    const int32_t* list = a.lists[t];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += stride) {
      const int v = list[i];
      a.parts[v] = a.mv[v];
      a.mv[v] = -1;
      if (a.set_lock) a.lock[v] = a.epoch;
    }
  }
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = val;
}

// ===========================================================================
// Workspace
// ===========================================================================
void Workspace::ensure(Ctx& c, int64_t n, int k) {
  if (n > cap_n) {
    cap_n = n;
    cdest.alloc(n, c.stream);
    mv.alloc(n, c.stream);
    lock.alloc(n, c.stream);
    lists.alloc(2 * n, c.stream);
    rkey.alloc(n, c.stream);
    rbest.alloc(n, c.stream);
    rcand.alloc(n, c.stream);
    evict.alloc(n, c.stream);
    dest_sorted.alloc(n, c.stream);
    F.alloc(n, c.stream);
    rloss.alloc(n, c.stream);
    keys.alloc(n, c.stream);
    keys_alt.alloc(n, c.stream);
    launch(c, "fill", 4.0 * n, [&] {
      k_fill_i32<<<grid_for(c, n, 256), 256, 0, c.stream>>>(mv.get(), n, -1);
    });
    dzero(c, lock.get(), n);
    c.lock_epoch = 0;
  }
  if (k > cap_k || ctr.get() == nullptr) {
    int kk = k > cap_k ? k : cap_k;
    DBuf<unsigned long long> nc(CTR_PW + kk, c.stream);
    dzero(c, nc.get(), CTR_PW + kk);
    if (ctr.get() && cap_k) d2d(c, nc.get() + CTR_PW, ctr.get() + CTR_PW, cap_k);
    ctr = std::move(nc);
    cap_k = kk;
    opidx.alloc(kk, c.stream);
    valid.alloc(kk, c.stream);
    valid_list.alloc(kk, c.stream);
    spare.alloc(kk, c.stream);
    hb.alloc(kk, c.stream);
    deficit.alloc(kk, c.stream);
    required.alloc(kk, c.stream);
    cum_before.alloc(kk, c.stream);
    bstar.alloc(kk, c.stream);
    thr.alloc(kk, c.stream);
  }
  c.ensure_pinned(CTR_PW + (size_t)k + 64);
}

void Workspace::bind_level(const DGraph& g) {
  int64_t b = 0;
  for (int t = 0; t < NBINS; ++t) {
    seg_base[t] = b;
    b += g.bin_cnt[t];
  }
}

// ===========================================================================
// Jetlp pass
// ===========================================================================
static SegLists seg_lists(Workspace& w, bool moves) {
  SegLists sl;
  for (int t = 0; t < NBINS; ++t) sl.list[t] = moves ? w.move_list(t) : w.cand_list(t);
  sl.cnt = w.ctr.get() + (moves ? CTR_MOVE : CTR_CAND);
  return sl;
}

static void launch_rows_reduce_ab(Ctx& c, Workspace& w, const DGraph& g, const AbArgs& a) {
  const GView gv = view(g);
  AbArgs at = a;
  RbSegsDev ms;
  for (int t = 0; t < NBINS; ++t) ms.b[t] = w.seg_base[t];
  if (a.move_list) {
    at.move_list = w.lists.get() + w.cap_n;
    at.move_cnt = w.ctr.get() + CTR_MOVE;
  }
  const SegLists sl = seg_lists(w, false);
  const unsigned grid = grid_for(c, g.n * 32, 256, 4);
  launch(c, "afterburner", 0.0, [&] {
    if (g.unit_ew) k_afterburner<true><<<grid, 256, 0, c.stream>>>(at, gv, sl, ms);
    else k_afterburner<false><<<grid, 256, 0, c.stream>>>(at, gv, sl, ms);
  });
}

void lp_pass(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts, int k,
             const LpParams& p, const LpDebug* dbg) {
  dzero(c, w.ctr.get(), CTR_PW);
  auto mk = [&](int t) {
    LpOp::Args a{};
    a.parts = parts;
    a.cdest = w.cdest.get();
    a.F = w.F.get();
    a.mv = w.mv.get();
    a.lock = w.lock.get();
    a.p = p;
    a.out_list = p.afterburner ? w.cand_list(t) : w.move_list(t);
    a.out_cnt = w.ctr.get() + (p.afterburner ? CTR_CAND : CTR_MOVE) + t;
    a.cut2 = w.ctr.get() + CTR_CUT2;
    if (dbg) a.dbg = *dbg;
    return a;
  };
  // per vertex: 8 offsets + 4 own part + 4 lock + 4 cdest
  run_agg<LpOp>(c, g, mk, parts, k, "lp_gains", 20.0);
  if (p.afterburner) {
    AbArgs ab{};
    ab.parts = parts;
    ab.cdest = w.cdest.get();
    ab.F = w.F.get();
    ab.mv = w.mv.get();
    ab.move_list = w.lists.get();  // non-null: per-tier lists bound below
    ab.f2_out = dbg ? dbg->f2 : nullptr;
    launch_rows_reduce_ab(c, w, g, ab);
  }
}

// Candidate set given explicitly (afterburner parity entry point): cdest and
// F must already hold dests/gains of candidates (-1 elsewhere); this builds
// the per-tier candidate lists.
__global__ void k_distribute(const int32_t* __restrict__ cand, int64_t ncand,
                             const int64_t* __restrict__ offs, TierMap tm, int32_t* lists,
                             RbSegsDev segs, unsigned long long* cnts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lim = (ncand + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lim; i += stride) {
    int v = 0, t = -1;
    if (i < ncand) {
      v = cand[i];
      t = tm(offs[v + 1] - offs[v]);
    }
    for (int tt = 0; tt < NBINS; ++tt)
      warp_append(t == tt, v, lists + segs.b[tt], cnts + tt);
  }
}

void afterburner_only(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts,
                      const int32_t* cand, int64_t ncand, long long* out_f2) {
  dzero(c, w.ctr.get(), CTR_PW);
  RbSegsDev segs;
  for (int t = 0; t < NBINS; ++t) segs.b[t] = w.seg_base[t];
  if (ncand > 0) {
    launch(c, "distribute", 8.0 * ncand, [&] {
      k_distribute<<<grid_for(c, ncand, 256), 256, 0, c.stream>>>(
          cand, ncand, g.offs.get(), g.tm, w.lists.get(), segs, w.ctr.get() + CTR_CAND);
    });
  }
  AbArgs ab{};
  ab.parts = parts;
  ab.cdest = w.cdest.get();
  ab.F = w.F.get();
  ab.mv = w.mv.get();
  ab.move_list = nullptr;
  ab.f2_out = out_f2;
  launch_rows_reduce_ab(c, w, g, ab);
}

// ===========================================================================
// Apply
// ===========================================================================
ApplyResult apply_moves(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts,
                        int k, bool set_lock, int32_t epoch) {
  const GView gv = view(g);
  ApArgs a{parts, w.mv.get(), w.ctr.get() + CTR_PW, w.ctr.get() + CTR_CUT2D, k};
  const SegLists sl = seg_lists(w, true);
  const unsigned grid = grid_for(c, g.n * 32, 256, 4);
  launch(c, "apply_delta", 0.0, [&] {
    if (g.unit_ew) k_apply_delta<true><<<grid, 256, 0, c.stream>>>(a, gv, sl);
    else k_apply_delta<false><<<grid, 256, 0, c.stream>>>(a, gv, sl);
  });
  CommitArgs ca{};
  ca.parts = parts;
  ca.mv = w.mv.get();
  ca.lock = w.lock.get();
  ca.epoch = epoch;
  ca.set_lock = set_lock ? 1 : 0;
  for (int t = 0; t < NBINS; ++t) ca.lists[t] = w.move_list(t);
  ca.cnts = w.ctr.get() + CTR_MOVE;
  launch(c, "apply_commit", 0.0, [&] {
    k_apply_commit<<<grid_for(c, g.n, 256, 2), 256, 0, c.stream>>>(ca);
  });
  int64_t* h = c.pinned;
  d2h(c, h, reinterpret_cast<int64_t*>(w.ctr.get()), CTR_PW + k);
  c.sync();
  ApplyResult r;
  for (int t = 0; t < NBINS; ++t) r.n_moves += h[CTR_MOVE + t];
  const int64_t d2 = h[CTR_CUT2D];
  JET_REQUIRE(d2 % 2 == 0, JET_EINTERNAL, "odd doubled cut delta");
  r.cut_delta = d2 / 2;
  w.h_pw.assign(h + CTR_PW, h + CTR_PW + k);
  return r;
}

// ===========================================================================
// Rebalancing
// ===========================================================================

// First bucket whose cumulative eligible weight reaches the deficit.
template <int BS>
__device__ void rb_scan_op(int op, const unsigned long long* __restrict__ H, int nb,
                           const long long* __restrict__ deficit, int32_t* bstar,
                           long long* cum_before) {
  typedef cub::BlockScan<long long, BS> Scan;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int s_found;
  __shared__ long long s_run, s_cb;
  const unsigned long long* h = H + (size_t)op * nb;
  const long long D = deficit[op];
  if (threadIdx.x == 0) {
    s_found = nb;
    s_run = 0;
    s_cb = 0;
  }
  __syncthreads();
  for (int base = 0; base < nb; base += BS) {
    const int i = base + threadIdx.x;
    const long long x = i < nb ? (long long)h[i] : 0;
    long long incl, total;
    Scan(ts).InclusiveSum(x, incl, total);
    const long long run = s_run;
    const long long cum = run + incl;
    if (i < nb && cum >= D && cum - x < D) {
      s_found = i;
      s_cb = cum - x;
    }
    __syncthreads();
    if (s_found < nb) break;
    if (threadIdx.x == 0) s_run = run + total;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bstar[op] = s_found;
    cum_before[op] = s_found < nb ? s_cb : s_run;
  }
  __syncthreads();
}

// First bucket whose cumulative eligible weight reaches the deficit.
__global__ void k_rb_scan(const unsigned long long* __restrict__ H, int nb,
                          const long long* __restrict__ deficit, int32_t* bstar,
                          long long* cum_before) {
  rb_scan_op<256>(blockIdx.x, H, nb, deficit, bstar, cum_before);
}

struct RbSel {
  const int32_t* parts;
  const int32_t* vw;
  const int32_t* opidx;
  const int32_t* rkey;
  const int32_t* bstar;
  const int32_t* thr;
  int rho;
  int nch;
  unsigned long long* CH;
};

__device__ void rb_chunk(const RbSel& s, const int32_t* __restrict__ rcand,
                         const unsigned long long* __restrict__ cnt_ptr, int64_t t0, int64_t nt) {
  const int64_t cnt = (int64_t)*(const volatile unsigned long long*)cnt_ptr;
  for (int64_t i = t0; i < cnt; i += nt) {
    const int v = rcand[i];
    const int op = s.opidx[s.parts[v]];
    if (s.rkey[v] != s.bstar[op]) continue;
    const int ch = (v / s.rho) >> 5;
    atomicAdd(&s.CH[(size_t)op * s.nch + ch], (unsigned long long)s.vw[v]);
  }
}

__global__ void k_rb_chunk(RbSel s, const int32_t* __restrict__ rcand,
                           const unsigned long long* __restrict__ cnt_ptr) {
  rb_chunk(s, rcand, cnt_ptr, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
           (int64_t)gridDim.x * blockDim.x);
}

// Locate the crossing element of select_prefix (rebalance.py:74-85) inside
// the crossing bucket, then decide whether it is taken:
//   take it iff cum[first] - D <= D - cum[first-1]  or  cum[first-1] < required
// (the min_weight extension of :81-85 always lands on first+1 because
//  deficit >= required). thr = first id NOT selected inside the bucket.
template <int BSZ>
__device__ void rb_find_op(int op, const RbSel& s, const long long* __restrict__ deficit,
                           const long long* __restrict__ required,
                           const long long* __restrict__ cum_before,
                           const int32_t* __restrict__ opart, int64_t n, int nb, int32_t* thr) {
  typedef cub::BlockScan<long long, BSZ> BS;
  __shared__ typename BS::TempStorage ts;
  __shared__ int s_ch;
  __shared__ long long s_run, s_cb;
  const int bs = s.bstar[op];
  if (bs >= nb) {  // shortfall: every eligible candidate leaves
    if (threadIdx.x == 0) thr[op] = 0x7fffffff;
    return;
  }
  const long long D = deficit[op];
  const long long base_cum = cum_before[op];
  const unsigned long long* ch = s.CH + (size_t)op * s.nch;
  if (threadIdx.x == 0) {
    s_ch = -1;
    s_run = base_cum;
    s_cb = 0;
  }
  __syncthreads();
  for (int b0 = 0; b0 < s.nch; b0 += BSZ) {
    const int i = b0 + threadIdx.x;
    const long long x = i < s.nch ? (long long)ch[i] : 0;
    long long incl, total;
    BS(ts).InclusiveSum(x, incl, total);
    const long long run = s_run;
    const long long cum = run + incl;
    if (i < s.nch && cum >= D && cum - x < D) {
      s_ch = i;
      s_cb = cum - x;
    }
    __syncthreads();
    if (s_ch >= 0) break;
    if (threadIdx.x == 0) s_run = run + total;
    __syncthreads();
  }
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int P = opart[op];
    const int sub = bs % s.rho;
    const int64_t j = (int64_t)s_ch * 32 + lane;
    const int64_t v64 = j * s.rho + sub;
    long long w = 0;
    if (s_ch >= 0 && v64 < n) {
      const int v = (int)v64;
      if (s.parts[v] == P && s.rkey[v] == bs) w = s.vw[v];
    }
    long long incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long cum = s_cb + incl;
    const bool hit = w > 0 && cum >= D && cum - w < D;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (m && lane == __ffs(m) - 1) {
      const long long prev = cum - w;
      const long long req = required[op];
      const bool include = (cum - D <= D - prev) || (prev < req);
      thr[op] = (int)v64 + (include ? 1 : 0);
    }
    if (!m && lane == 0) thr[op] = 0x7fffffff;  // unreachable by construction
  }
}

__global__ void k_rb_find(RbSel s, const long long* __restrict__ deficit,
                          const long long* __restrict__ required,
                          const long long* __restrict__ cum_before,
                          const int32_t* __restrict__ opart, int64_t n, int nb, int32_t* thr) {
  rb_find_op<256>(blockIdx.x, s, deficit, required, cum_before, opart, n, nb, thr);
}

// Selected iff (bucket, id) < the part's threshold (select_prefix). Weak
// passes with direct=1 commit vertices that have a valid destination right
// away (their order is unobservable); everything else (weak: vertices that
// need a random destination; strong: all) goes to the evict list.
__device__ void rb_select(const RbSel& s, const int32_t* __restrict__ rcand,
                          const unsigned long long* __restrict__ cnt_ptr,
                          const int32_t* __restrict__ rbest, int strong, int direct,
                          int32_t* evict, unsigned long long* evict_cnt, int32_t* mv,
                          const int64_t* __restrict__ offs, TierMap tm, int32_t* move_lists,
                          RbSegsDev mseg, unsigned long long* move_cnt, int64_t t0, int64_t nt) {
  const int64_t cnt = (int64_t)*(const volatile unsigned long long*)cnt_ptr;
  const int64_t lim = (cnt + 31) / 32 * 32;
  for (int64_t i = t0; i < lim; i += nt) {
    bool sel = false, now = false;
    int v = 0, t = -1;
    if (i < cnt) {
      v = rcand[i];
      const int op = s.opidx[s.parts[v]];
      const int rk = s.rkey[v];
      const int bs = s.bstar[op];
      sel = rk < bs || (rk == bs && v < s.thr[op]);
      if (sel && !strong && direct) {
        const int bp = rbest[v];
        if (bp >= 0) {
          now = true;
          mv[v] = bp;
          t = tm(offs[v + 1] - offs[v]);
        }
      }
    }
    warp_append(sel && !now, v, evict, evict_cnt);
    for (int tt = 0; tt < NBINS; ++tt)
      warp_append(t == tt, v, move_lists + mseg.b[tt], move_cnt + tt);
  }
}

__global__ void k_rb_select(RbSel s, const int32_t* __restrict__ rcand,
                            const unsigned long long* __restrict__ cnt_ptr,
                            const int32_t* __restrict__ rbest, int strong, int direct,
                            int32_t* evict, unsigned long long* evict_cnt, int32_t* mv,
                            const int64_t* __restrict__ offs, TierMap tm, int32_t* move_lists,
                            RbSegsDev mseg, unsigned long long* move_cnt) {
  rb_select(s, rcand, cnt_ptr, rbest, strong, direct, evict, evict_cnt, mv, offs, tm, move_lists,
            mseg, move_cnt, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
            (int64_t)gridDim.x * blockDim.x);
}

// Collect the vertices of oversized parts into per-tier candidate lists.
__global__ void k_rb_collect(const int32_t* __restrict__ parts, const int32_t* __restrict__ opidx,
                             const int64_t* __restrict__ offs, TierMap tm, int64_t n,
                             int32_t* lists, RbSegsDev seg, unsigned long long* cnts) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lim = (n + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < lim; v += stride) {
    int t = -1;
    if (v < n && opidx[parts[v]] >= 0) t = tm(offs[v + 1] - offs[v]);
    if (__ballot_sync(0xffffffffu, t >= 0) == 0) continue;
    for (int tt = 0; tt < NBINS; ++tt) warp_append(t == tt, (int32_t)v, lists + seg.b[tt], cnts + tt);
  }
}

// Single-block tail for small evicted sets (length read on device, bounded
// on the host by sum(deficit) <= cap): bitonic sort of (part, bucket, id)
// keys in shared memory, then weak: valid[draw[i]] in order; strong:
// next-fit (rebalance.py:224-236); then commit the moves.
struct RbTail {
  const int32_t* evict;
  const unsigned long long* evict_cnt;
  const int32_t* parts;
  const int32_t* opidx;
  const int32_t* rkey;
  const int32_t* vw;
  const int64_t* offs;
  TierMap tm;
  const int32_t* valid_list;
  const int32_t* draws;
  const long long* spare;
  int nvalid;
  int nb;
  int strong;
  int32_t* mv;
  int32_t* move_lists;
  RbSegsDev mseg;
  unsigned long long* move_cnt;
};

__device__ void rb_tail(const RbTail& a, unsigned long long* sk) {
  __shared__ long long s_room;
  __shared__ int s_di, s_done;
  __shared__ long long s_wsum[32];
  const int tid = threadIdx.x;
  const int L = (int)*(const volatile unsigned long long*)a.evict_cnt;
  int P2 = 1;
  while (P2 < L) P2 <<= 1;
  for (int i = tid; i < P2; i += blockDim.x) {
    unsigned long long key = ~0ull;
    if (i < L) {
      const int v = a.evict[i];
      const unsigned long long grp =
          (unsigned long long)a.opidx[a.parts[v]] * (unsigned)a.nb + (unsigned)a.rkey[v];
      key = (grp << 32) | (unsigned)v;
    }
    sk[i] = key;
  }
  __syncthreads();
  for (int size = 2; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P2; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool asc = (i & size) == 0;
          const unsigned long long x = sk[i], y = sk[j];
          if ((x > y) == asc) {
            sk[i] = y;
            sk[j] = x;
          }
        }
      }
      __syncthreads();
    }
  }
  if (!a.strong) {
    for (int i = tid; i < L; i += blockDim.x) {
      const int v = (int)(sk[i] & 0xffffffffu);
      a.mv[v] = a.valid_list[a.draws[i]];
      const int t = a.tm(a.offs[v + 1] - a.offs[v]);
      const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
      a.move_lists[a.mseg.b[t] + q] = v;
    }
    return;
  }
  // next-fit; sequential over runs but each run is a parallel prefix test
  if (tid == 0) {
    s_di = 0;
    s_room = a.nvalid > 0 ? a.spare[0] : 0;
    s_done = a.nvalid <= 0;
  }
  __syncthreads();
  for (int base = 0; base < L; base += blockDim.x) {
    const int i = base + tid;
    const long long w = i < L ? (long long)a.vw[(int)(sk[i] & 0xffffffffu)] : 0;
    // block inclusive scan of w
    long long ps = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, ps, o);
      if ((tid & 31) >= o) ps += y;
    }
    if ((tid & 31) == 31) s_wsum[tid >> 5] = ps;
    __syncthreads();
    if (tid < 32) {
      long long x = s_wsum[tid];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, x, o);
        if (tid >= o) x += y;
      }
      s_wsum[tid] = x;
    }
    __syncthreads();
    if (tid >= 32) ps += s_wsum[(tid >> 5) - 1];
    const int lim = L - base < (int)blockDim.x ? L - base : (int)blockDim.x;
    // stash inclusive sums in the (already consumed) key slots' upper half:
    // keep them in a dedicated region after the keys instead
    long long* pbuf = reinterpret_cast<long long*>(sk + P2);
    pbuf[tid] = ps;
    __syncthreads();
    int pos = 0;
    long long before = 0;
    while (true) {
      if (s_done) break;
      const long long room = s_room;
      const bool fits = tid >= pos && tid < lim && ps - before <= room;
      __shared__ int s_first;
      if (tid == 0) s_first = lim;
      __syncthreads();
      if (tid >= pos && tid < lim && !fits) atomicMin(&s_first, tid);
      __syncthreads();
      const int e = s_first;
      if (fits) {
        const int v = (int)(sk[i] & 0xffffffffu);
        a.mv[v] = a.valid_list[s_di];
        const int t = a.tm(a.offs[v + 1] - a.offs[v]);
        const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
        a.move_lists[a.mseg.b[t] + q] = v;
      }
      __syncthreads();
      if (e >= lim) {
        if (tid == 0) s_room = room - (pbuf[lim - 1] - before);
        __syncthreads();
        break;
      }
      if (tid == 0) {
        const long long prev = e > 0 ? pbuf[e - 1] : 0;
        long long r = room - (prev - before);
        const long long we = pbuf[e] - prev;
        int di = s_di;
        while (di < a.nvalid && r < we) {
          di++;
          r = di < a.nvalid ? a.spare[di] : 0;
        }
        s_di = di;
        s_room = r;
        if (di >= a.nvalid) s_done = 1;
      }
      __syncthreads();
      pos = e;
      before = e > 0 ? pbuf[e - 1] : 0;
    }
    __syncthreads();
    if (s_done) break;
  }
}

__global__ void __launch_bounds__(1024) k_rb_tail(RbTail a) {
  extern __shared__ unsigned long long sk_dyn[];
  rb_tail(a, sk_dyn);
}

// The whole selection chain of a rebalancing pass in one cooperative launch:
// bucket scan -> crossing-chunk histogram -> crossing element -> select ->
// (block 0) ordered tail. Replaces five dependent launches.
struct RbCoop {
  RbSel s;
  const unsigned long long* H;
  int nb;
  int nover;
  const long long* deficit;
  const long long* required;
  long long* cum_before;
  const int32_t* opart;
  int64_t n;
  const int32_t* rcand;
  const unsigned long long* rcand_cnt;
  const int32_t* rbest;
  int strong;
  int32_t* evict;
  unsigned long long* evict_cnt;
  const int64_t* offs;
  TierMap tm;
  int32_t* move_lists;
  RbSegsDev mseg;
  unsigned long long* move_cnt;
  RbTail tail;
};

__global__ void __launch_bounds__(1024) k_rb_coop(RbCoop a) {
  extern __shared__ unsigned long long sk_dyn[];
  cg::grid_group grid = cg::this_grid();
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  for (int op = blockIdx.x; op < a.nover; op += gridDim.x)
    rb_scan_op<1024>(op, a.H, a.nb, a.deficit, const_cast<int32_t*>(a.s.bstar), a.cum_before);
  grid.sync();
  rb_chunk(a.s, a.rcand, a.rcand_cnt, t0, nt);
  grid.sync();
  for (int op = blockIdx.x; op < a.nover; op += gridDim.x) {
    rb_find_op<1024>(op, a.s, a.deficit, a.required, a.cum_before, a.opart, a.n, a.nb,
                     const_cast<int32_t*>(a.s.thr));
    __syncthreads();
  }
  grid.sync();
  rb_select(a.s, a.rcand, a.rcand_cnt, a.rbest, a.strong, 1, a.evict, a.evict_cnt, a.tail.mv,
            a.offs, a.tm, a.move_lists, a.mseg, a.move_cnt, t0, nt);
  grid.sync();
  if (blockIdx.x == 0) rb_tail(a.tail, sk_dyn);
}

__global__ void k_rb_keys(const int32_t* __restrict__ evict, int64_t L,
                          const int32_t* __restrict__ parts,
                          const int32_t* __restrict__ opidx,
                          const int32_t* __restrict__ rkey, int nb,
                          unsigned long long* keys) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L; i += stride) {
    const int v = evict[i];
    const unsigned long long grp = (unsigned long long)opidx[parts[v]] * nb + rkey[v];
    keys[i] = (grp << 32) | (unsigned)v;
  }
}

// weak: dest = best valid part, else valid[draw] in eviction order
__global__ void __launch_bounds__(1024)
    k_rb_weak_assign(const unsigned long long* __restrict__ keys, int64_t L,
                     const int32_t* __restrict__ rbest,
                     const int32_t* __restrict__ valid_list,
                     const int32_t* __restrict__ draws, int32_t* dest_sorted) {
  typedef cub::BlockScan<int, 1024> BS;
  __shared__ typename BS::TempStorage ts;
  __shared__ long long s_run;
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (int64_t base = 0; base < L; base += 1024) {
    const int64_t i = base + threadIdx.x;
    int miss = 0, v = 0, bp = -1;
    if (i < L) {
      v = (int)(keys[i] & 0xffffffffu);
      bp = rbest[v];
      miss = bp < 0;
    }
    int excl, total;
    BS(ts).ExclusiveSum(miss, excl, total);
    const long long run = s_run;
    if (i < L) dest_sorted[i] = miss ? valid_list[draws[run + excl]] : bp;
    __syncthreads();
    if (threadIdx.x == 0) s_run = run + total;
    __syncthreads();
  }
}

__global__ void k_rb_count_missing(const unsigned long long* __restrict__ keys, int64_t L,
                                   const int32_t* __restrict__ rbest,
                                   unsigned long long* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  long long m = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L; i += stride)
    m += rbest[(int)(keys[i] & 0xffffffffu)] < 0;
  block_sum_atomic<256>(m, out);
}

// strong: next-fit of the evicted sequence over valid parts ascending with
// spare = sigma - pw (rebalance.py:224-236). One block; each step assigns the
// longest prefix that fits the current room (weights are positive, so the
// fitting elements form a prefix) and then advances past parts whose room is
// below the next weight.
__global__ void __launch_bounds__(1024)
    k_rb_nextfit(const unsigned long long* __restrict__ keys, int64_t L,
                 const int32_t* __restrict__ vw, const int32_t* __restrict__ valid_list,
                 const long long* __restrict__ spare, int nvalid, int32_t* dest_sorted) {
  typedef cub::BlockScan<long long, 1024> BS;
  __shared__ typename BS::TempStorage ts;
  __shared__ long long s_ps[1024];
  __shared__ long long s_room;
  __shared__ int s_di, s_done, s_first;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_di = 0;
    s_room = spare[0];
    s_done = nvalid <= 0;
  }
  __syncthreads();
  for (int64_t base = 0; base < L; base += 1024) {
    const int64_t i = base + tid;
    const long long w = i < L ? (long long)vw[(int)(keys[i] & 0xffffffffu)] : 0;
    long long ps;
    BS(ts).InclusiveSum(w, ps);
    s_ps[tid] = ps;
    __syncthreads();
    const int lim = (int)(L - base < 1024 ? L - base : 1024);
    int pos = 0;
    long long before = 0;
    while (true) {
      if (s_done) {
        if (tid >= pos && tid < lim) dest_sorted[i] = -1;
        break;
      }
      if (tid == 0) s_first = lim;
      __syncthreads();
      const long long room = s_room;
      const bool fits = tid >= pos && tid < lim && ps - before <= room;
      if (tid >= pos && tid < lim && !fits) atomicMin(&s_first, tid);
      __syncthreads();
      const int e = s_first;
      if (fits) dest_sorted[i] = valid_list[s_di];
      __syncthreads();
      if (e >= lim) {
        if (tid == 0) s_room = room - (s_ps[lim - 1] - before);
        __syncthreads();
        break;
      }
      if (tid == 0) {
        const long long prev = e > 0 ? s_ps[e - 1] : 0;
        long long r = room - (prev - before);
        const long long we = s_ps[e] - prev;
        int di = s_di;
        while (di < nvalid && r < we) {
          di++;
          r = di < nvalid ? spare[di] : 0;
        }
        s_di = di;
        s_room = r;
        if (di >= nvalid) s_done = 1;
      }
      __syncthreads();
      pos = e;
      before = e > 0 ? s_ps[e - 1] : 0;
    }
    __syncthreads();
  }
}

struct RbCommit {
  const unsigned long long* keys;
  const int32_t* dest_sorted;
  int32_t* mv;
  const int64_t* offs;
  TierMap tm;
  int32_t* lists;  // move lists base
  int64_t seg_base[NBINS];
  unsigned long long* move_cnt;
  // optional ordered outputs
  int32_t* o_v;
  int32_t* o_dest;
};

__global__ void k_rb_commit(RbCommit a, int64_t L) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lim = (L + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lim; i += stride) {
    int v = 0, d = -1, t = -1;
    if (i < L) {
      v = (int)(a.keys[i] & 0xffffffffu);
      d = a.dest_sorted[i];
      if (d >= 0) {
        a.mv[v] = d;
        t = a.tm(a.offs[v + 1] - a.offs[v]);
      }
      if (a.o_v) {
        a.o_v[i] = v;
        a.o_dest[i] = d;
      }
    }
    for (int tt = 0; tt < NBINS; ++tt)
      warp_append(t == tt, v, a.lists + a.seg_base[tt], a.move_cnt + tt);
  }
}

static int ceil_log2(int64_t x) {
  int r = 0;
  while ((1LL << r) < x) ++r;
  return r;
}

constexpr int TAIL_CAP = 24576;  // evicted vertices ordered by the single-block tail

namespace {
// Packs per-pass host scalars into one pinned buffer for a single H2D copy.
struct Packer {
  std::vector<uint8_t>* host;
  size_t off = 0;
  template <class T>
  size_t put(const T* src, size_t count) {
    off = (off + 15) & ~size_t(15);
    const size_t at = off;
    off += count * sizeof(T);
    if (host->size() < off) host->resize(off);
    if (count) memcpy(host->data() + at, src, count * sizeof(T));
    return at;
  }
};
}  // namespace

bool rebalance_pass(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts,
                    int k, int64_t limit, int64_t sigma, int sub_buckets,
                    bool strong, Pcg64& rng, RebalanceOut* out) {
  const std::vector<int64_t>& pw = w.h_pw;
  std::vector<int32_t> h_opidx(k, -1), h_valid_list, h_opart;
  std::vector<uint8_t> h_valid(k, 0);
  for (int p = 0; p < k; ++p) {
    if (pw[p] > limit) {
      h_opidx[p] = (int32_t)h_opart.size();
      h_opart.push_back(p);
    }
    if (pw[p] < sigma) {
      h_valid[p] = 1;
      h_valid_list.push_back(p);
    }
  }
  dzero(c, w.ctr.get(), CTR_PW);
  if (h_opart.empty()) return true;
  if (h_valid_list.empty()) return false;
  const int nover = (int)h_opart.size();
  const int nvalid = (int)h_valid_list.size();
  // scalars in the reference's own float64 expressions (rebalance.py:127-131)
  const int64_t W = g.total_vw;
  std::vector<double> h_hb(nover);
  std::vector<long long> h_def(nover), h_req(nover), h_spare(nvalid);
  long long sum_def = 0, max_evict = 0;
  for (int i = 0; i < nover; ++i) {
    const int64_t pwp = pw[h_opart[i]];
    h_def[i] = pwp - (sigma + 1);
    h_req[i] = pwp - limit;
    sum_def += h_def[i];
    max_evict += h_def[i] / std::max<int64_t>(g.min_vw, 1) + 1;
    volatile double ideal = (double)W / (double)k;
    volatile double diff = (double)pwp - ideal;
    h_hb[i] = 1.5 * diff;
  }
  for (int i = 0; i < nvalid; ++i) h_spare[i] = sigma - pw[h_valid_list[i]];
  int rho = sub_buckets;
  if ((int64_t)rho >= g.n) rho = 1;  // (slot, v % rho, v) == (slot, v)
  JET_REQUIRE(rho <= 4096, JET_EUNSUPPORTED, "sub_buckets > 4096 is not supported on the GPU path");
  const int slot_min = strong ? 1 - ceil_log2(k) : 0;
  const int ns = 34 - slot_min;
  const int nb = ns * rho;
  const int nch = (int)(((g.n + rho - 1) / rho + 31) / 32);
  // per part at most deficit/min_w + 1 vertices leave (selected prefix < deficit)
  const bool fast = out == nullptr && max_evict <= TAIL_CAP;
  const bool direct = out == nullptr;

  std::vector<uint8_t>& up = w.h_up;
  Packer pk{&up};
  const size_t o_opidx = pk.put(h_opidx.data(), k);
  const size_t o_valid = pk.put(h_valid.data(), k);
  const size_t o_vlist = pk.put(h_valid_list.data(), nvalid);
  const size_t o_opart = pk.put(h_opart.data(), nover);
  const size_t o_hb = pk.put(h_hb.data(), nover);
  const size_t o_def = pk.put(h_def.data(), nover);
  const size_t o_req = pk.put(h_req.data(), nover);
  const size_t o_spare = pk.put(h_spare.data(), nvalid);
  const size_t up_bytes = (pk.off + 15) & ~size_t(15);
  c.ensure_pinned_up(up_bytes + (size_t)std::max<long long>(max_evict, 1) * 4 + 64);
  memcpy(c.pinned_up, up.data(), up_bytes);
  w.up.ensure(up_bytes + 64, c.stream);
  uint8_t* U = w.up.get();
  h2d(c, U, c.pinned_up, up_bytes);
  const int32_t* d_opidx = (const int32_t*)(U + o_opidx);
  const uint8_t* d_valid = U + o_valid;
  const int32_t* d_vlist = (const int32_t*)(U + o_vlist);
  const int32_t* d_opart = (const int32_t*)(U + o_opart);
  const double* d_hb = (const double*)(U + o_hb);
  const long long* d_def = (const long long*)(U + o_def);
  const long long* d_req = (const long long*)(U + o_req);
  const long long* d_spare = (const long long*)(U + o_spare);

  w.H.ensure((size_t)nover * nb, c.stream);
  w.CH.ensure((size_t)nover * nch, c.stream);
  dzero(c, w.H.get(), (size_t)nover * nb);
  dzero(c, w.CH.get(), (size_t)nover * nch);

  RbSegsDev cseg, mseg;
  for (int t = 0; t < NBINS; ++t) {
    cseg.b[t] = w.seg_base[t];
    mseg.b[t] = w.seg_base[t];
  }
  launch(c, "rb_collect", 8.0 * g.n, [&] {
    k_rb_collect<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(parts, d_opidx, g.offs.get(), g.tm, g.n,
                                                             w.lists.get(), cseg,
                                                             w.ctr.get() + CTR_CAND);
  });
  RbOp::Args ra{};
  ra.parts = parts;
  ra.vw = g.vw.get();
  ra.opidx = d_opidx;
  ra.valid = d_valid;
  ra.hb = d_hb;
  ra.nvalid = nvalid;
  ra.strong = strong;
  ra.rho = rho;
  ra.slot_min = slot_min;
  ra.nb = nb;
  ra.rkey = w.rkey.get();
  ra.rbest = w.rbest.get();
  ra.rloss = w.rloss.get();
  ra.rcand = w.rcand.get();
  ra.rcand_cnt = w.ctr.get() + CTR_RCAND;
  ra.H = w.H.get();
  int32_t* clists[NBINS];
  for (int t = 0; t < NBINS; ++t) clists[t] = w.cand_list(t);
  run_agg<RbOp>(c, g, [&](int) { return ra; }, parts, k, "rb_stats", 16.0, clists,
                w.ctr.get() + CTR_CAND);

  int32_t* bstar = w.bstar.get();
  RbSel s{parts, g.vw.get(), d_opidx, w.rkey.get(), bstar, w.thr.get(), rho, nch, w.CH.get()};
  const unsigned long long* rc = w.ctr.get() + CTR_RCAND;
  int32_t* move_base = w.lists.get() + w.cap_n;

  if (fast) {
    RbTail tl{};
    tl.evict = w.evict.get();
    tl.evict_cnt = w.ctr.get() + CTR_EVICT;
    tl.parts = parts;
    tl.opidx = d_opidx;
    tl.rkey = w.rkey.get();
    tl.vw = g.vw.get();
    tl.offs = g.offs.get();
    tl.tm = g.tm;
    tl.valid_list = d_vlist;
    tl.spare = d_spare;
    tl.nvalid = nvalid;
    tl.nb = nb;
    tl.strong = strong;
    tl.mv = w.mv.get();
    tl.move_lists = move_base;
    tl.mseg = mseg;
    tl.move_cnt = w.ctr.get() + CTR_MOVE;
    if (!strong) {
      // draws for the (at most max_evict) vertices without a valid
      // connection, generated on the host while the kernels above run
      const long long D = max_evict;
      int32_t* hd = reinterpret_cast<int32_t*>(c.pinned_up + up_bytes);
      for (long long i = 0; i < D; ++i) hd[i] = (int32_t)rng.bounded((uint64_t)nvalid);
      w.draws.ensure(D > 0 ? D : 1, c.stream);
      h2d(c, w.draws.get(), hd, D);
      tl.draws = w.draws.get();
    }
    RbCoop cp{};
    cp.s = s;
    cp.H = w.H.get();
    cp.nb = nb;
    cp.nover = nover;
    cp.deficit = d_def;
    cp.required = d_req;
    cp.cum_before = w.cum_before.get();
    cp.opart = d_opart;
    cp.n = g.n;
    cp.rcand = w.rcand.get();
    cp.rcand_cnt = rc;
    cp.rbest = w.rbest.get();
    cp.strong = strong;
    cp.evict = w.evict.get();
    cp.evict_cnt = w.ctr.get() + CTR_EVICT;
    cp.offs = g.offs.get();
    cp.tm = g.tm;
    cp.move_lists = move_base;
    cp.mseg = mseg;
    cp.move_cnt = w.ctr.get() + CTR_MOVE;
    cp.tail = tl;
    const size_t smem = (size_t)TAIL_CAP * 8 + 1024 * 8;
    static int coop_grid = 0;
    if (!coop_grid) {
      CK(cudaFuncSetAttribute(k_rb_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rb_coop, 1024, smem));
      JET_REQUIRE(per_sm >= 1, JET_EINTERNAL, "rebalance kernel does not fit on an SM");
      coop_grid = per_sm * c.num_sms;
    }
    void* args[] = {&cp};
    launch(c, "rb_select_coop", 0.0, [&] {
      CK(cudaLaunchCooperativeKernel((const void*)k_rb_coop, dim3(coop_grid), dim3(1024), args,
                                     smem, c.stream));
    });
    return true;
  }

  launch(c, "rb_scan", 8.0 * nover * nb, [&] {
    k_rb_scan<<<nover, 256, 0, c.stream>>>(w.H.get(), nb, d_def, bstar, w.cum_before.get());
  });
  launch(c, "rb_chunk", 0.0, [&] {
    k_rb_chunk<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(s, w.rcand.get(), rc);
  });
  launch(c, "rb_find", 8.0 * nover * nch, [&] {
    k_rb_find<<<nover, 256, 0, c.stream>>>(s, d_def, d_req, w.cum_before.get(), d_opart, g.n, nb,
                                           w.thr.get());
  });
  launch(c, "rb_select", 0.0, [&] {
    k_rb_select<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(
        s, w.rcand.get(), rc, w.rbest.get(), strong, direct ? 1 : 0, w.evict.get(),
        w.ctr.get() + CTR_EVICT, w.mv.get(), g.offs.get(), g.tm, move_base, mseg,
        w.ctr.get() + CTR_MOVE);
  });

  // slow path (large evicted sets, or the parity entry point): order with a
  // device radix sort after reading the evicted count back
  int64_t L = 0;
  d2h(c, &L, reinterpret_cast<int64_t*>(w.ctr.get() + CTR_EVICT), 1);
  c.sync();
  if (L == 0) {
    if (out) {
      out->v->clear();
      out->dest->clear();
      out->gain->clear();
    }
    return true;
  }
  launch(c, "rb_keys", 16.0 * L, [&] {
    k_rb_keys<<<grid_for(c, L, 256), 256, 0, c.stream>>>(w.evict.get(), L, parts, d_opidx,
                                                         w.rkey.get(), nb, w.keys.get());
  });
  const int gbits = ceil_log2((int64_t)nover * nb + 1);
  {
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, w.keys.get(), w.keys_alt.get(), (int)L, 0,
                                      32 + gbits, c.stream));
    void* ptmp = c.cub_scratch(tmp);
    launch(c, "rb_sort", 16.0 * L, [&] {
      CK(cub::DeviceRadixSort::SortKeys(ptmp, tmp, w.keys.get(), w.keys_alt.get(), (int)L, 0,
                                        32 + gbits, c.stream));
    });
  }
  const unsigned long long* sk = w.keys_alt.get();
  if (!strong) {
    int64_t need = L;  // with direct commits every evicted vertex needs a draw
    if (!direct) {
      DBuf<unsigned long long> mc(1, c.stream);
      dzero(c, mc.get(), 1);
      launch(c, "rb_count_missing", 12.0 * L, [&] {
        k_rb_count_missing<<<grid_for(c, L, 256), 256, 0, c.stream>>>(sk, L, w.rbest.get(), mc.get());
      });
      unsigned long long hm = 0;
      d2h(c, &hm, mc.get(), 1);
      c.sync();
      need = (int64_t)hm;
    }
    std::vector<int32_t> h_draws((size_t)need);
    for (int64_t i = 0; i < need; ++i) h_draws[i] = (int32_t)rng.bounded((uint64_t)nvalid);
    w.draws.ensure(need > 0 ? need : 1, c.stream);
    h2d(c, w.draws.get(), h_draws.data(), need);
    c.sync();
    launch(c, "rb_weak_assign", 16.0 * L, [&] {
      k_rb_weak_assign<<<1, 1024, 0, c.stream>>>(sk, L, w.rbest.get(), d_vlist, w.draws.get(),
                                                 w.dest_sorted.get());
    });
  } else {
    launch(c, "rb_nextfit", 16.0 * L, [&] {
      k_rb_nextfit<<<1, 1024, 0, c.stream>>>(sk, L, g.vw.get(), d_vlist, d_spare, nvalid,
                                             w.dest_sorted.get());
    });
  }
  RbCommit rcm{};
  rcm.keys = sk;
  rcm.dest_sorted = w.dest_sorted.get();
  rcm.mv = w.mv.get();
  rcm.offs = g.offs.get();
  rcm.tm = g.tm;
  rcm.lists = move_base;
  for (int t = 0; t < NBINS; ++t) rcm.seg_base[t] = w.seg_base[t];
  rcm.move_cnt = w.ctr.get() + CTR_MOVE;
  DBuf<int32_t> ov, od;
  if (out) {
    ov.alloc(L, c.stream);
    od.alloc(L, c.stream);
    rcm.o_v = ov.get();
    rcm.o_dest = od.get();
  }
  launch(c, "rb_commit", 16.0 * L, [&] {
    k_rb_commit<<<grid_for(c, L, 256), 256, 0, c.stream>>>(rcm, L);
  });
  if (out) {
    std::vector<int32_t> hv(L), hd(L);
    std::vector<double> hl(g.n);
    d2h(c, hv.data(), ov.get(), L);
    d2h(c, hd.data(), od.get(), L);
    d2h(c, hl.data(), w.rloss.get(), g.n);
    c.sync();
    out->v->clear();
    out->dest->clear();
    out->gain->clear();
    for (int64_t i = 0; i < L; ++i) {
      if (hd[i] < 0) continue;
      out->v->push_back(hv[i]);
      out->dest->push_back(hd[i]);
      out->gain->push_back(-hl[hv[i]]);
    }
  }
  return true;
}

}  // namespace jet
