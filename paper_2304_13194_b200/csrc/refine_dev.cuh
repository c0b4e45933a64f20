// refine_dev.cuh — device-side building blocks of the Jet refinement passes,
// shared by the multi-kernel path (refine.cu) and the persistent per-level
// controller kernel (level.cu). Every function takes its work range
// explicitly (warp or thread start + stride) so it runs unchanged as a
// standalone kernel body or as one phase of a cooperative kernel.
#pragma once
#include "refine.cuh"
#include <cub/block/block_scan.cuh>
#include <cub/block/block_radix_sort.cuh>

namespace jet {

// Per-thread visit counters for the roofline accounting ({rows, entries} of
// the stats, afterburner and apply sweeps). Kept in registers for a whole
// level and reduced once at the end: global atomics per warp on two hot
// counters cost more than the sweeps they count.
// lanes per row in the short-row afterburner and apply loops (tiers 0-3)
#ifndef AB_GROUP_LANES
#define AB_GROUP_LANES 8
#endif
#ifndef AP_GROUP_LANES
#define AP_GROUP_LANES 8
#endif

struct WorkAcc {
  // stats rows/entries, afterburner rows/entries, apply rows/entries,
  // boundary-sweep rows/entries
  unsigned long long v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
};

// ===========================================================================
// Row aggregation framework. For every vertex v of a tier, conn(v, p) is
// aggregated over the row; an Op decides which parts compete for the "best"
// slot, what else is summed, and what to do with the result.
//   tiers 0-3: one G-lane group per row, __match_any_sync groups equal parts
//   tier 4   : one warp per row, per-warp shared-memory table of k entries
//   tier 5   : one block per row, per-block shared-memory table
// ===========================================================================

static __device__ __forceinline__ unsigned long long pack_best(long long conn, int p) {
  return ((unsigned long long)conn << KBITS) | (unsigned)(KMASK - p);
}
static __device__ __forceinline__ int unpack_part(unsigned long long key) {
  return KMASK - (int)(key & KMASK);
}
static __device__ __forceinline__ long long unpack_conn(unsigned long long key) {
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
    int32_t* ext;   // optional: weighted external degree of every swept row (< 2^31)
    int32_t* wdeg;  // optional: weighted degree of every swept row (< 2^31)
    LpDebug dbg;
  };
  static __device__ __forceinline__ bool skip(const Args&, int, int) { return false; }
  // Jetlp sweeps only boundary rows already (level kernel): nothing to short-cut
  static __device__ __forceinline__ long long interior_w(const Args&, int, int, bool) { return -1; }
  static __device__ __forceinline__ bool competes(const Args&, int p, int own) { return p != own; }
  static __device__ __forceinline__ int extra(const Args&, int, int w) { return w; }
  // self_c = conn(v, own); key = best other part; ex = weighted degree
  static __device__ __forceinline__ void finish(const Args& a, int v, int own,
                                                long long self_c,
                                                unsigned long long key,
                                                long long ex, long long& acc) {
    acc += ex - self_c;
    if (a.ext) a.ext[v] = (int32_t)(ex - self_c);
    if (a.wdeg) a.wdeg[v] = (int32_t)ex;
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
    block_sum_atomic_any(acc, a.cut2);
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
    unsigned long long* Hs;  // per-slot totals (ns per oversized part)
    const int32_t* ext;      // optional (level kernel): weighted external degrees
    const int32_t* wdeg;     // weighted degrees (weighted levels)
  };
  static __device__ __forceinline__ bool skip(const Args& a, int, int own) {
    return a.opidx[own] < 0;
  }
  // A candidate without neighbours outside its part needs no adjacency: its
  // own-part connectivity is its weighted degree and no part competes.
  // Returns that weight, or -1 when the row has to be swept.
  static __device__ __forceinline__ long long interior_w(const Args& a, int v, int deg, bool unit) {
    if (!a.ext || __ldcg(a.ext + v) != 0) return -1;
    return unit ? (long long)deg : (long long)a.wdeg[v];
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
    const unsigned am = __activemask();
    long long hk = -1, sk = -1;
    if (eligible) {
      const int bucket = (slot - a.slot_min) * a.rho + (v % a.rho);
      a.rkey[v] = bucket;
      a.rbest[v] = best_part;
      a.rloss[v] = loss;
      hk = (long long)op * a.nb + bucket;
      sk = (long long)op * (a.nb / a.rho) + (slot - a.slot_min);
    } else {
      a.rkey[v] = -1;
    }
    // histogram updates aggregated over equal keys of the warp (few slots
    // per oversized part: per-vertex atomics would serialise on them)
    {
      const unsigned peers = __match_any_sync(am, hk);
      const long long s2 = gsum_peers(peers, (long long)w);
      if (hk >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&a.H[hk], (unsigned long long)s2);
    }
    {
      const unsigned peers = __match_any_sync(am, sk);
      const long long s2 = gsum_peers(peers, (long long)w);
      if (sk >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&a.Hs[sk], (unsigned long long)s2);
    }
    warp_append(eligible, v, a.rcand, a.rcand_cnt);
  }
  static __device__ __forceinline__ void block_done(const Args&, long long) {}
};

// ---- asynchronous global->shared copies (LDGSTS) ----------------------------
static __device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
static __device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;\n" ::: "memory");
}

// Entries per lane of short-row tier G: the top short tier (G = 32 lanes)
// holds rows of up to 64 entries, two per lane (TIER_SLOTS in common.cuh).
template <int G>
__host__ __device__ constexpr int tier_e() {
  return G == 32 ? 2 : 1;
}
// Per-warp staging words of the short-row sweep (adjacency, parts, weights).
// (the one-entry-per-lane 32-wide tier pads its rows to 33 words so a lane
// can walk its own row without shared-memory bank conflicts)
template <int G, int RB, bool UNIT, int E = tier_e<G>()>
__host__ __device__ constexpr int stage_words() {
  return RB * (G == 32 && E == 1 ? 33 : G * E) * (UNIT ? 2 : 3);
}

// Tier 3 with rows of <= 32 entries (one entry per lane). Rows are staged as
// in agg_small, but the aggregation is lane-per-row first: each lane walks
// its own staged row (interior test + own-part sum), and only the boundary
// rows -- a minority on refined meshes -- run the warp-cooperative part
// grouping. The former lane-per-entry loop spent ~90 instructions per row,
// most of them per-row broadcasts and reductions that interior rows do not
// need (ncu: the sweep was issue-bound at 60 % issue-active).
template <class Op, bool UNIT, int RB>
static __device__ __forceinline__ void agg_rows32(const typename Op::Args& a, const GView& g,
                                                  const int32_t* __restrict__ parts,
                                                  const int32_t* __restrict__ list, int64_t cnt,
                                                  bool wide,
                                                  const unsigned long long* __restrict__ dcnt,
                                                  int64_t w0, int64_t nw, long long& acc,
                                                  uint32_t* stage) {
  if (dcnt) cnt = (int64_t)*(const volatile unsigned long long*)dcnt;
  constexpr int SP = 33;
  const int lane = threadIdx.x & 31;
  int* s_adj = reinterpret_cast<int*>(stage);
  int* s_p = s_adj + RB * SP;
  int* s_w = s_p + RB * SP;
  const int64_t per_w = (cnt + nw - 1) / nw;
  const int R = per_w >= RB ? RB : (per_w < 1 ? 1 : (int)per_w);
  for (int64_t base = w0 * R; base < cnt; base += nw * R) {
    const int64_t idx = base + lane;
    int v = 0, own = -1, deg = 0;
    int64_t beg = 0;
    long long wself = -1;  // >= 0: interior row, nothing staged
    if (lane < R && idx < cnt) {
      v = list ? list[idx] : (int)idx;
      own = parts[v];
      if (Op::skip(a, v, own)) {
        own = -1;
      } else {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
        wself = Op::interior_w(a, v, deg, UNIT);
        if (wself >= 0) deg = 0;
      }
    }
    for (int r = 0; r < R; ++r) {
      const int64_t rb = __shfl_sync(0xffffffffu, beg, r);
      const int rd = __shfl_sync(0xffffffffu, deg, r);
      if (lane < rd) {
        cp_async4(&s_adj[r * SP + lane], g.adj + rb + lane);
        if (!UNIT) cp_async4(&s_w[r * SP + lane], g.ew + rb + lane);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    for (int r = 0; r < R; ++r) {
      const int rd = __shfl_sync(0xffffffffu, deg, r);
      if (lane < rd) cp_async4(&s_p[r * SP + lane], parts + s_adj[r * SP + lane]);
    }
    cp_async_wait_all();
    __syncwarp();
    // lane r: its own row
    long long my_self = 0, my_ex = 0;
    unsigned long long my_key = 0;
    bool outside = false;
    if (own >= 0) {
      const int* pr = s_p + lane * SP;
      const int* wr = s_w + lane * SP;
      for (int j = 0; j < deg; ++j) {
        const int p = pr[j];
        if (p == own) my_self += UNIT ? 1 : wr[j];
        else outside = true;
      }
      my_ex = Op::extra(a, own, 1) ? my_self : 0;  // extra is linear in w
    }
    // boundary rows: group the parts of the row across the warp
    unsigned bm = __ballot_sync(0xffffffffu, outside);
    while (bm) {
      const int r = __ffs(bm) - 1;
      bm &= bm - 1;
      const int rd = __shfl_sync(0xffffffffu, deg, r);
      const int rown = __shfl_sync(0xffffffffu, own, r);
      int p = -1, w = 0;
      if (lane < rd) {
        p = s_p[r * SP + lane];
        w = UNIT ? 1 : s_w[r * SP + lane];
      }
      const unsigned peers = __match_any_sync(0xffffffffu, p);
      const bool comp = p >= 0 && p != rown && Op::competes(a, p, rown);
      unsigned long long key;
      long long ex;
      if (!wide) {
        const unsigned sm = UNIT ? (unsigned)__popc(peers) : __reduce_add_sync(peers, (unsigned)w);
        const unsigned mx = __reduce_max_sync(0xffffffffu, comp ? sm : 0u);
        const unsigned pm =
            __reduce_min_sync(0xffffffffu, (comp && sm == mx) ? (unsigned)p : 0xffffffffu);
        ex = (long long)__reduce_add_sync(0xffffffffu,
                                          p >= 0 ? (unsigned)Op::extra(a, p, w) : 0u);
        key = mx ? pack_best((long long)mx, (int)pm) : 0ull;
      } else {
        const long long sm = UNIT ? (long long)__popc(peers) : peer_sum(peers, w, wide);
        const bool lead = p >= 0 && (__ffs(peers) - 1) == lane;
        key = (lead && comp) ? pack_best(sm, p) : 0ull;
        key = gmax<32>(key, 0xffffffffu);
        ex = gsum<32>(p >= 0 ? (long long)Op::extra(a, p, w) : 0ll, 0xffffffffu);
      }
      if (lane == r) {
        my_key = key;
        my_ex = ex;
      }
    }
    __syncwarp();  // the next batch reuses the stage
    if (wself >= 0) {
      my_self = wself;
      my_key = 0ull;
      my_ex = Op::extra(a, own, 1) ? wself : 0;  // extra is linear in w
    }
    if (own >= 0) Op::finish(a, v, own, my_self, my_key, my_ex, acc);
  }
}

// Tiers 0-3 (rows of <= G*E entries). A warp owns R <= RB consecutive list
// entries; their ids, offsets and own parts are loaded once, coalesced. The
// rows' adjacency (+weights) is then copied into shared memory with
// fire-and-forget cp.async (one 4-byte copy per entry, all in flight at
// once), and the neighbour parts are gathered the same way, addressed from
// the staged adjacency. Only then are the rows aggregated, G lanes per row,
// from shared memory: three memory round trips per batch of rows instead of
// a dependent load chain per row. Row r's result is shuffled to lane r.
// Rows with no neighbour outside their own part (most rows of a refined
// mesh) take a fast path: conn(v, .) is the own-part sum only. Boundary rows
// group equal parts with __match_any_sync (E = 1) or, two entries per lane
// (E = 2), walk their distinct competing parts in ascending order.
template <class Op, int G, bool UNIT, int RB = 32, int E = tier_e<G>()>
static __device__ __forceinline__ void agg_small(const typename Op::Args& a, const GView& g,
                                                 const int32_t* __restrict__ parts,
                                                 const int32_t* __restrict__ list, int64_t cnt,
                                                 bool wide,
                                                 const unsigned long long* __restrict__ dcnt,
                                                 int64_t w0, int64_t nw, long long& acc,
                                                 uint32_t* stage) {
  if constexpr (G == 32 && E == 1) {
    agg_rows32<Op, UNIT, RB>(a, g, parts, list, cnt, wide, dcnt, w0, nw, acc, stage);
    return;
  }
  if (dcnt) cnt = (int64_t)*(const volatile unsigned long long*)dcnt;
  static_assert(E == 1 || G == 32, "two entries per lane only for one row per step");
  constexpr int S = G * E;     // slots per row
  constexpr int RPS = 32 / G;  // rows per step
  const unsigned gm = group_mask<G>();
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  int* s_adj = reinterpret_cast<int*>(stage);
  int* s_p = s_adj + RB * S;
  int* s_w = s_p + RB * S;
  // rows per batch: RB when there is plenty of work, fewer for small lists
  // so every warp gets rows (latency, not bandwidth, rules there)
  const int64_t per_w = (cnt + nw - 1) / nw;
  const int R = per_w >= RB ? RB : (per_w < 1 ? 1 : (int)per_w);
  for (int64_t base = w0 * R; base < cnt; base += nw * R) {
    const int64_t idx = base + lane;
    int v = 0, own = -1, deg = 0;
    int64_t beg = 0;
    long long wself = -1;  // >= 0: interior row, nothing staged
    if (lane < R && idx < cnt) {
      v = list ? list[idx] : (int)idx;
      own = parts[v];
      if (Op::skip(a, v, own)) {
        own = -1;
      } else {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
        wself = Op::interior_w(a, v, deg, UNIT);
        if (wself >= 0) deg = 0;
      }
    }
    // stage adjacency (+ weights)
    for (int st = 0; st * RPS < R; ++st) {
      const int r = st * RPS + grp;
      const int64_t rb = __shfl_sync(0xffffffffu, beg, r & 31);
      const int rd = __shfl_sync(0xffffffffu, deg, r & 31);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = e * G + gl;
        if (r < R && j < rd) {
          cp_async4(&s_adj[r * S + j], g.adj + rb + j);
          if (!UNIT) cp_async4(&s_w[r * S + j], g.ew + rb + j);
        }
      }
    }
    cp_async_wait_all();
    __syncwarp();
    // gather neighbour parts
    for (int st = 0; st * RPS < R; ++st) {
      const int r = st * RPS + grp;
      const int rd = __shfl_sync(0xffffffffu, deg, r & 31);
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = e * G + gl;
        if (r < R && j < rd) cp_async4(&s_p[r * S + j], parts + s_adj[r * S + j]);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    long long my_self = 0, my_ex = 0;
    unsigned long long my_key = 0;
    for (int st = 0; st * RPS < R; ++st) {
      const int r = st * RPS + grp;
      const int rd = __shfl_sync(0xffffffffu, deg, r & 31);
      const int rown = __shfl_sync(0xffffffffu, own, r & 31);
      int pe[E], we[E];
      bool outside = false;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int j = e * G + gl;
        pe[e] = -1;
        we[e] = 0;
        if (r < R && j < rd) {
          pe[e] = s_p[r * S + j];
          we[e] = UNIT ? 1 : s_w[r * S + j];
        }
        outside |= pe[e] >= 0 && pe[e] != rown;
      }
      const int src = ((lane - st * RPS) & (RPS - 1)) * G;
      // interior fast path (warp-uniform): no row of this step has a
      // neighbour outside its own part
      if (!wide && __ballot_sync(0xffffffffu, outside) == 0) {
        unsigned loc = 0;
#pragma unroll
        for (int e = 0; e < E; ++e) loc += pe[e] >= 0 ? (unsigned)we[e] : 0u;
        const unsigned sc = __reduce_add_sync(gm, loc);
        const unsigned dsc = __shfl_sync(0xffffffffu, sc, src);
        if (lane / RPS == st) {
          my_self = dsc;
          my_key = 0ull;
          my_ex = own >= 0 ? (long long)Op::extra(a, own, (int)dsc) : 0;  // extra is linear in w
        }
        continue;
      }
      if constexpr (E == 1) {
        const int p = pe[0], w = we[0];
        const unsigned peers = __match_any_sync(gm, p);
        const bool comp = p >= 0 && p != rown && Op::competes(a, p, rown);
        if (!wide) {
          // 32-bit sums (weighted degree < 2^31): single-instruction REDUX
          // reductions; best part = max conn, then lowest part id
          const unsigned sm = UNIT ? (unsigned)__popc(peers) : __reduce_add_sync(peers, (unsigned)w);
          const unsigned sc = UNIT ? (unsigned)__popc(__ballot_sync(gm, p >= 0 && p == rown))
                                   : __reduce_add_sync(gm, (p >= 0 && p == rown) ? (unsigned)w : 0u);
          const unsigned mx = __reduce_max_sync(gm, comp ? sm : 0u);
          const unsigned pm = __reduce_min_sync(gm, (comp && sm == mx) ? (unsigned)p : 0xffffffffu);
          const unsigned ex = __reduce_add_sync(gm, p >= 0 ? (unsigned)Op::extra(a, p, w) : 0u);
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
          const long long sm = UNIT ? (long long)__popc(peers) : peer_sum(peers, w, wide);
          const bool lead = p >= 0 && (__ffs(peers) - 1) == lane;
          long long sc = (lead && p == rown) ? sm : 0;
          unsigned long long key = (lead && comp) ? pack_best(sm, p) : 0ull;
          long long ex = p >= 0 ? Op::extra(a, p, w) : 0;
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
      } else {
        // G = 32 (one row per step), E entries per lane: sums over the row,
        // then the distinct competing parts in ascending order (ties on the
        // max therefore keep the lowest part)
        long long lsc = 0, lex = 0;
        bool oth[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int p = pe[e];
          lsc += (p >= 0 && p == rown) ? we[e] : 0;
          lex += p >= 0 ? Op::extra(a, p, we[e]) : 0;
          oth[e] = p >= 0 && p != rown && Op::competes(a, p, rown);
        }
        const long long sc = wide ? gsum<32>(lsc, 0xffffffffu)
                                  : (long long)__reduce_add_sync(0xffffffffu, (unsigned)lsc);
        const long long ex = wide ? gsum<32>(lex, 0xffffffffu)
                                  : (long long)__reduce_add_sync(0xffffffffu, (unsigned)lex);
        long long bm = 0;
        int bp = -1;
        while (true) {
          unsigned c = 0xffffffffu;
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (oth[e]) c = min(c, (unsigned)pe[e]);
          const unsigned cur = __reduce_min_sync(0xffffffffu, c);
          if (cur == 0xffffffffu) break;
          long long lc = 0;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            if (pe[e] == (int)cur) {
              lc += we[e];
              oth[e] = false;
            }
          }
          const long long cc = wide ? gsum<32>(lc, 0xffffffffu)
                                    : (long long)__reduce_add_sync(0xffffffffu, (unsigned)lc);
          if (cc > bm) {
            bm = cc;
            bp = (int)cur;
          }
        }
        if (lane == st) {
          my_self = sc;
          my_key = bm > 0 ? pack_best(bm, bp) : 0ull;
          my_ex = ex;
        }
      }
    }
    __syncwarp();  // the next batch reuses the stage
    if (wself >= 0) {
      my_self = wself;
      my_key = 0ull;
      my_ex = Op::extra(a, own, 1) ? wself : 0;  // extra is linear in w
    }
    if (own >= 0) Op::finish(a, v, own, my_self, my_key, my_ex, acc);
  }
}

// Tier 4 (33..2048 entries). A warp owns 32 rows; per-vertex data is loaded
// once, coalesced. Rows are aggregated one after another into a per-warp
// shared-memory part table, but the adjacency of the next chunk batch (of
// this row, or of the next row) is loaded while the current batch's
// neighbour parts are gathered and aggregated, so two batches of loads are
// always in flight. Shared layout per warp: tab[k] (u64), tl[tl_cap] (i32),
// tcnt (i32).
template <class Op, bool UNIT>
static __device__ void agg_warp(const typename Op::Args& a, const GView& g,
                         const int32_t* __restrict__ parts, const int32_t* __restrict__ list,
                         int64_t cnt, bool wide, int k, int tl_cap,
                         const unsigned long long* __restrict__ dcnt, unsigned long long* smem,
                         int64_t w0, int64_t nw, long long& acc) {
  if (dcnt) cnt = (int64_t)*(const volatile unsigned long long*)dcnt;
  constexpr int U = 2;  // chunks of 32 entries per batch
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per = (size_t)k + (size_t)(tl_cap + 3) / 2;
  unsigned long long* tab = smem + wib * per;
  unsigned* tab32 = reinterpret_cast<unsigned*>(tab);  // narrow weighted sums (lane atomics)
  const bool lane_atomic = !UNIT && !wide;
  int* tl = reinterpret_cast<int*>(tab + k);
  int* tcnt = tl + tl_cap;
  for (int i = lane; i < k; i += 32) tab[i] = 0;
  if (lane == 0) *tcnt = 0;
  __syncwarp();
  const int64_t per_w = (cnt + nw - 1) / nw;
  const int R = per_w >= 32 ? 32 : (per_w < 1 ? 1 : (int)per_w);
  for (int64_t base = w0 * R; base < cnt; base += nw * R) {
    const int64_t idx = base + lane;
    int v = 0, own = -1, deg = 0;
    int64_t beg = 0;
    long long wself = -1;  // >= 0: interior row, nothing staged
    if (lane < R && idx < cnt) {
      v = list ? list[idx] : (int)idx;
      own = parts[v];
      if (Op::skip(a, v, own)) {
        own = -1;
      } else {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
        wself = Op::interior_w(a, v, deg, UNIT);
        if (wself >= 0) deg = 0;
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
    while (r < R) {
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
        rb = __shfl_sync(0xffffffffu, beg, r & 31);
        rd = r < R ? __shfl_sync(0xffffffffu, deg, r & 31) : 0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int j = (c0 + q) * 32 + lane;
        uu[q] = (r < R && j < rd) ? g.adj[rb + j] : -1;
        ww[q] = (r < R && j < rd) ? (UNIT ? 1 : g.ew[rb + j]) : 0;
      }
      // aggregate the current batch
      const int rown = __shfl_sync(0xffffffffu, own, cur_r);
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int p = pp[q];
        if (p >= 0) ex += Op::extra(a, p, wv[q]);
        if (lane_atomic) {
          // weighted, narrow: one 32-bit shared atomic per lane (a REDUX over
          // each match_any group serialises over the groups of the warp)
          if (p >= 0 && atomicAdd(&tab32[p], (unsigned)wv[q]) == 0u) tl[atomicAdd(tcnt, 1)] = p;
        } else {
          const unsigned peers = __match_any_sync(0xffffffffu, p);
          const long long sm = UNIT ? (long long)__popc(peers) : peer_sum(peers, wv[q], wide);
          if (p >= 0 && (__ffs(peers) - 1) == lane) {
            const unsigned long long old = atomicAdd(&tab[p], (unsigned long long)sm);
            if (old == 0) tl[atomicAdd(tcnt, 1)] = p;
          }
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
            unsigned cv;
            if (lane_atomic) {
              cv = tab32[p];
              tab32[p] = 0;
            } else {
              cv = (unsigned)tab[p];
              tab[p] = 0;
            }
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
    if (wself >= 0) {
      my_self = wself;
      my_key = 0ull;
      my_ex = Op::extra(a, own, 1) ? wself : 0;  // extra is linear in w
    }
    if (own >= 0) Op::finish(a, v, own, my_self, my_key, my_ex, acc);
  }
}

// Tier 5: one block (256 threads) per row; block-wide shared part table.
template <class Op, bool UNIT>
static __device__ void agg_block(const typename Op::Args& a, const GView& g,
                          const int32_t* __restrict__ parts, const int32_t* __restrict__ list,
                          int64_t cnt, bool wide, int k, const unsigned long long* __restrict__ dcnt,
                          unsigned long long* smem, long long& acc) {
  if (dcnt) cnt = (int64_t)*(const volatile unsigned long long*)dcnt;
  unsigned long long* tab = smem;
  unsigned* tab32 = reinterpret_cast<unsigned*>(tab);
  const bool lane_atomic = !UNIT && !wide;
  int* tl = reinterpret_cast<int*>(tab + k);
  __shared__ int tcnt;
  __shared__ long long r_self[32], r_ex[32];
  __shared__ unsigned long long r_key[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < k; i += blockDim.x) tab[i] = 0;
  if (threadIdx.x == 0) tcnt = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const int v = list ? list[i] : (int)i;
    const int own = parts[v];
    if (Op::skip(a, v, own)) continue;  // uniform across the block
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    long long ex = 0;
    // four strides of the row in flight per step: hub rows of 10^4-10^5
    // entries were bound by the adjacency -> part gather round trips
    constexpr int U = 4;
    const int64_t step = (int64_t)blockDim.x * U;
    for (int64_t j0 = b; j0 < e; j0 += step) {
      int uu[U], pp[U], ww[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int64_t j = j0 + (int64_t)q * blockDim.x + threadIdx.x;
        uu[q] = j < e ? g.adj[j] : -1;
        ww[q] = j < e ? (UNIT ? 1 : g.ew[j]) : 0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) pp[q] = uu[q] >= 0 ? parts[uu[q]] : -1;
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int p = pp[q], w = ww[q];
        if (p >= 0) ex += Op::extra(a, p, w);
        if (lane_atomic) {  // see agg_warp
          if (p >= 0 && atomicAdd(&tab32[p], (unsigned)w) == 0u) tl[atomicAdd(&tcnt, 1)] = p;
        } else {
          const unsigned peers = __match_any_sync(0xffffffffu, p);
          const long long s = UNIT ? (long long)__popc(peers) : peer_sum(peers, w, wide);
          if (p >= 0 && (__ffs(peers) - 1) == lane) {
            unsigned long long old = atomicAdd(&tab[p], (unsigned long long)s);
            if (old == 0) tl[atomicAdd(&tcnt, 1)] = p;
          }
        }
      }
    }
    __syncthreads();
    const int nt = tcnt;
    long long self_c = 0;
    unsigned long long key = 0;
    for (int t = threadIdx.x; t < nt; t += blockDim.x) {
      const int p = tl[t];
      long long cv;
      if (lane_atomic) {
        cv = (long long)tab32[p];
        tab32[p] = 0;
      } else {
        cv = (long long)tab[p];
        tab[p] = 0;
      }
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

// Afterburner sum of one long row over the entries j = j0, j0 + stride, ...
// (a warp or block per row): RU strides are loaded per step, so each lane
// has RU independent adjacency -> (part, dest) -> F chains in flight
// (one at a time left the dense R-MAT levels latency-bound).
template <bool UNIT, int RU = 4>
static __device__ __forceinline__ long long ab_row_f2(const AbArgs& a, const GView& g, int v, int own,
                                                      int dv, long long Fv, int64_t j0, int64_t e,
                                                      int64_t stride) {
  long long f2 = 0;
  for (; j0 < e; j0 += stride * RU) {
    int uu[RU], ww[RU], pu[RU], cu[RU];
    long long Fu[RU];
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      const int64_t j = j0 + q * stride;
      uu[q] = j < e ? g.adj[j] : -1;
      ww[q] = j < e ? (UNIT ? 1 : g.ew[j]) : 0;
    }
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      pu[q] = uu[q] >= 0 ? a.parts[uu[q]] : -1;
      cu[q] = uu[q] >= 0 ? a.cdest[uu[q]] : -1;
    }
#pragma unroll
    for (int q = 0; q < RU; ++q) Fu[q] = cu[q] >= 0 ? a.F[uu[q]] : 0;
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      int eff = pu[q];
      if (cu[q] >= 0 && (Fu[q] > Fv || (Fu[q] == Fv && uu[q] < v))) eff = cu[q];
      const int w = ww[q];
      f2 += uu[q] < 0 ? 0 : (eff == dv) ? w : (eff == own) ? -w : 0;
    }
  }
  return f2;
}

// Afterburner over the short-row tiers: a G-lane group per row, so a warp
// keeps 32/G rows in flight (a warp per ~10-entry row left the coarse levels
// latency-bound).
template <int G, bool UNIT>
static __device__ __forceinline__ void ab_group_rows(const AbArgs& a, const GView& g,
                                                     const int32_t* __restrict__ list, int64_t cnt,
                                                     int t, const RbSegsDev& mseg, int64_t w0,
                                                     int64_t ws, unsigned long long* wr,
                                                     unsigned long long* we, long long* nmove) {
  constexpr int RPS = 32 / G;
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const unsigned gm = group_mask<G>();
  for (int64_t base = w0 * RPS; base < cnt; base += ws * RPS) {
    const int64_t i = base + grp;
    const bool has = i < cnt;
    int v = 0, own = -1, dv = -1;
    long long Fv = 0;
    int64_t b = 0, e = 0;
    if (has) {
      v = list[i];
      own = a.parts[v];
      dv = a.cdest[v];
      Fv = a.F[v];
      b = g.offs[v];
      e = g.offs[v + 1];
      if (wr && gl == 0) {
        *wr += 1;
        *we += (unsigned long long)(e - b);
      }
    }
    long long f2 = ab_row_f2<UNIT>(a, g, v, own, dv, Fv, b + gl, e, G);
    f2 = gsum<G>(f2, gm);
    if (has && gl == 0) {
      if (a.f2_out) a.f2_out[v] = f2;
      if (f2 >= 0) {
        if (a.move_list) {
          a.mv[v] = dv;
          const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
          a.move_list[mseg.b[t] + q] = v;
        } else if (nmove) {
          a.mv[v] = dv;
          *nmove += 1;
        }
      }
    }
  }
}

// One warp per candidate over all tiers (candidate sets are small).
// With a move list, moves are appended per row (host-driven path); without
// one (level kernel) only mv[v] is set and the moves are counted into
// *nmove, and the apply phase walks the candidate lists skipping unmoved
// rows -- one atomic per row on a hot counter serialises in L2.
// wr/we (optional): += rows / entries visited, for the roofline accounting.
template <bool UNIT>
static __device__ void afterburner_rows(const AbArgs& a, const GView& g, const SegLists& sl,
                                 const RbSegsDev& mseg, int64_t w0, int64_t ws,
                                 unsigned long long* wr = nullptr, unsigned long long* we = nullptr,
                                 long long* nmove = nullptr) {
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)*(const volatile unsigned long long*)(sl.cnt + t);
    const int32_t* list = sl.list[t];
    if (t == BIN_BLOCK) {
      // hub rows (> WARP_TIER_MAX_DEG entries): a block per row
      for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const int v = list[i];
        const int own = a.parts[v];
        const int dv = a.cdest[v];
        const long long Fv = a.F[v];
        const int64_t b = g.offs[v], e = g.offs[v + 1];
        if (wr && threadIdx.x == 0) {
          *wr += 1;
          *we += (unsigned long long)(e - b);
        }
        const long long f2 = block_sum_all(ab_row_f2<UNIT>(a, g, v, own, dv, Fv, b + threadIdx.x, e,
                                                           (int64_t)blockDim.x));
        if (threadIdx.x == 0) {
          if (a.f2_out) a.f2_out[v] = f2;
          if (f2 >= 0) {
            if (a.move_list) {
              a.mv[v] = dv;
              const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
              a.move_list[mseg.b[t] + q] = v;
            } else if (nmove) {
              a.mv[v] = dv;
              *nmove += 1;
            }
          }
        }
      }
      continue;
    }
    if (t < BIN_WARP) {  // short rows: 8-lane groups, four rows per warp step
      ab_group_rows<AB_GROUP_LANES, UNIT>(a, g, list, cnt, t, mseg, w0, ws, wr, we, nmove);
      continue;
    }
    for (int64_t i = w0; i < cnt; i += ws) {
      const int v = list[i];
      const int own = a.parts[v];
      const int dv = a.cdest[v];
      const long long Fv = a.F[v];
      const int64_t b = g.offs[v], e = g.offs[v + 1];
      if (wr && lane == 0) {
        *wr += 1;
        *we += (unsigned long long)(e - b);
      }
      const long long f2 = gsum<32>(ab_row_f2<UNIT>(a, g, v, own, dv, Fv, b + lane, e, 32), 0xffffffffu);
      if (lane == 0) {
        if (a.f2_out) a.f2_out[v] = f2;
        if (f2 >= 0) {
          if (a.move_list) {
            a.mv[v] = dv;
            const unsigned long long q = atomicAdd(a.move_cnt + t, 1ull);
            a.move_list[mseg.b[t] + q] = v;
          } else if (nmove) {
            a.mv[v] = dv;
            *nmove += 1;
          }
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
  int32_t* ext = nullptr;  // optional: weighted external degrees kept current (level kernel, < 2^31)
  // sharded levels: only rows of the owned block [own_lo, own_hi) are walked
  // (their cut / weight deltas are summed over the ranks); own_hi < 0: all
  int64_t own_lo = 0, own_hi = -1;
  __device__ __forceinline__ bool owns(int v) const {
    return own_hi < 0 || ((int64_t)v >= own_lo && (int64_t)v < own_hi);
  }
};

// External-degree upkeep of one entry (v moves old -> dst, neighbour u in pu,
// moving to mu or staying): v's new external degree accumulates in ev; a
// staying neighbour's changes by w([dst != pu] - [old != pu]). A moving
// neighbour recomputes its own, so every counter has one writer kind.
static __device__ __forceinline__ void ext_entry(int32_t* ext, int u, int pu, int mu, int nu,
                                                 int dst, int old, long long w, long long& ev) {
  ev += nu != dst ? w : 0;
  if (mu < 0) {
    const int du = (int)w * ((int)(dst != pu) - (int)(old != pu));
    if (du) atomicAdd(ext + u, du);
  }
}

// Exact cut delta of a move batch (conn.py:231-248): for a moved v and
// neighbour u, c = w([p'(u) != dest] - [p(u) != old]); edges with both ends
// moved appear twice and are halved, so we sum 2c / c and halve at the end.
// Rows whose mv[v] < 0 are skipped (the level kernel applies Jetlp moves
// straight from the candidate lists).
// Cut delta / weight / external-degree upkeep of one long moved row over
// j = j0, j0 + stride, ... with RU strides in flight per step (ab_row_f2).
template <bool UNIT, int RU = 4>
static __device__ __forceinline__ void ap_row(const ApArgs& a, const GView& g, int dst, int old,
                                              int64_t j0, int64_t e, int64_t stride, long long& d,
                                              long long& ev) {
  for (; j0 < e; j0 += stride * RU) {
    int uu[RU], ww[RU], pu[RU], mu[RU];
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      const int64_t j = j0 + q * stride;
      uu[q] = j < e ? g.adj[j] : -1;
      ww[q] = j < e ? (UNIT ? 1 : g.ew[j]) : 0;
    }
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      pu[q] = uu[q] >= 0 ? a.parts[uu[q]] : 0;
      mu[q] = uu[q] >= 0 ? a.mv[uu[q]] : -1;
    }
#pragma unroll
    for (int q = 0; q < RU; ++q) {
      if (uu[q] < 0) continue;
      const int nu = mu[q] >= 0 ? mu[q] : pu[q];
      const long long w = ww[q];
      const long long cc = w * ((long long)(nu != dst) - (long long)(pu[q] != old));
      d += mu[q] >= 0 ? cc : 2 * cc;
      if (a.ext) ext_entry(a.ext, uu[q], pu[q], mu[q], nu, dst, old, w, ev);
    }
  }
}

template <bool UNIT>
static __device__ void apply_delta_rows(const ApArgs& a, const GView& g, const SegLists& sl,
                                 int64_t w0, int64_t ws, long long& acc,
                                 unsigned long long* wr = nullptr, unsigned long long* we = nullptr) {
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)*(const volatile unsigned long long*)(sl.cnt + t);
    const int32_t* list = sl.list[t];
    if (t == BIN_BLOCK) {
      // hub rows: a block per row (block-uniform skip of unmoved rows)
      for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
        const int v = list[i];
        const int dst = a.owns(v) ? a.mv[v] : -1;
        if (dst < 0) continue;
        const int old = a.parts[v];
        const int64_t b = g.offs[v], e = g.offs[v + 1];
        if (wr && threadIdx.x == 0) {
          *wr += 1;
          *we += (unsigned long long)(e - b);
        }
        long long ev = 0;
        ap_row<UNIT>(a, g, dst, old, b + threadIdx.x, e, (int64_t)blockDim.x, acc, ev);
        if (a.ext) {
          ev = block_sum_all(ev);
          if (threadIdx.x == 0) a.ext[v] = (int32_t)ev;
        }
        if (threadIdx.x == 0) {
          const unsigned long long wv = (unsigned long long)g.vw[v];
          atomicAdd(&a.pw[dst], wv);
          atomicAdd(&a.pw[old], (unsigned long long)(-(long long)wv));
        }
      }
      continue;
    }
    if (t < BIN_WARP) {  // short rows: 8-lane groups, four rows per warp step
      constexpr int G = AP_GROUP_LANES, RPS = 32 / G;
      const int gl = lane & (G - 1), grp = lane / G;
      for (int64_t base = w0 * RPS; base < cnt; base += ws * RPS) {
        const int64_t i = base + grp;
        int v = 0, dst = -1, old = 0;
        int64_t b = 0, e = 0;
        if (i < cnt) {
          v = list[i];
          dst = a.owns(v) ? a.mv[v] : -1;
          if (dst >= 0) {
            old = a.parts[v];
            b = g.offs[v];
            e = g.offs[v + 1];
            if (wr && gl == 0) {
              *wr += 1;
              *we += (unsigned long long)(e - b);
            }
          }
        }
        long long d = 0, ev = 0;
        ap_row<UNIT>(a, g, dst, old, b + gl, e, G, d, ev);
        acc += d;
        if (a.ext) {
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) ev += __shfl_xor_sync(0xffffffffu, ev, o);
          if (dst >= 0 && gl == 0) a.ext[v] = (int32_t)ev;
        }
        if (dst >= 0 && gl == 0) {
          const unsigned long long wv = (unsigned long long)g.vw[v];
          atomicAdd(&a.pw[dst], wv);
          atomicAdd(&a.pw[old], (unsigned long long)(-(long long)wv));
        }
      }
      continue;
    }
    for (int64_t i = w0; i < cnt; i += ws) {
      const int v = list[i];
      const int dst = a.owns(v) ? a.mv[v] : -1;
      if (dst < 0) continue;
      const int old = a.parts[v];
      const int64_t b = g.offs[v], e = g.offs[v + 1];
      if (wr && lane == 0) {
        *wr += 1;
        *we += (unsigned long long)(e - b);
      }
      long long d = 0, ev = 0;
      ap_row<UNIT>(a, g, dst, old, b + lane, e, 32, d, ev);
      acc += d;  // per-lane partial sums: the caller reduces over the block
      if (a.ext) {
        ev = gsum<32>(ev, 0xffffffffu);
        if (lane == 0) a.ext[v] = (int32_t)ev;
      }
      if (lane == 0) {
        const unsigned long long wv = (unsigned long long)g.vw[v];
        atomicAdd(&a.pw[dst], wv);
        atomicAdd(&a.pw[old], (unsigned long long)(-(long long)wv));
      }
    }
  }
}

struct CommitArgs {
  int32_t* parts;
  int32_t* mv;
  int32_t* lock;
  int32_t epoch;
  int set_lock;
  const int32_t* lists[NBINS];
  const unsigned long long* cnts;
  int32_t* cdest_reset;  // optional: Jetlp destinations of the listed rows back to -1
};

static __device__ void apply_commit_rows(const CommitArgs& a, int64_t t0, int64_t stride) {
  int64_t cnts[NBINS];
#pragma unroll
  for (int t = 0; t < NBINS; ++t) cnts[t] = (int64_t)__ldcg(a.cnts + t);
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = cnts[t];
    const int32_t* list = a.lists[t];
    for (int64_t i = t0; i < cnt; i += stride) {
      const int v = list[i];
      if (a.cdest_reset) a.cdest_reset[v] = -1;
      const int dst = a.mv[v];
      if (dst < 0) continue;  // unmoved candidate (level kernel, Jetlp pass)
      a.parts[v] = dst;
      a.mv[v] = -1;
      if (a.set_lock) a.lock[v] = a.epoch;
    }
  }
}


template <int BS>
static __device__ void rb_scan_op(int op, const unsigned long long* __restrict__ H, int nb,
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

static __device__ void rb_chunk(const RbSel& s, const int32_t* __restrict__ rcand,
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



// Locate the crossing element of select_prefix (rebalance.py:74-85) inside
// the crossing bucket, then decide whether it is taken:
//   take it iff cum[first] - D <= D - cum[first-1]  or  cum[first-1] < required
// (the min_weight extension of :81-85 always lands on first+1 because
//  deficit >= required). thr = first id NOT selected inside the bucket.
template <int BSZ>
static __device__ void rb_find_op(int op, const RbSel& s, const long long* __restrict__ deficit,
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



// Selected iff (bucket, id) < the part's threshold (select_prefix). Weak
// passes with direct=1 commit vertices that have a valid destination right
// away (their order is unobservable); everything else (weak: vertices that
// need a random destination; strong: all) goes to the evict list.

// ---- warp-level selection helpers: one warp per oversized part, so all
// parts proceed in parallel whatever the grid size (the persistent level
// kernel runs small levels on a handful of blocks).

// First index i of arr[0, len) where run + prefix_sum(arr)[i] >= D; *before =
// run + prefix before i. Returns -1 (and *before = run + total) if never.
static __device__ __forceinline__ int warp_cross_linear(const unsigned long long* __restrict__ arr,
                                                        int len, long long D, long long run,
                                                        long long* before) {
  const int lane = threadIdx.x & 31;
  for (int b0 = 0; b0 < len; b0 += 32) {
    const int i = b0 + lane;
    const long long x = i < len ? (long long)arr[i] : 0;
    long long incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long cum = run + incl;
    const unsigned m = __ballot_sync(0xffffffffu, i < len && cum >= D && cum - x < D);
    if (m) {
      const int l = __ffs(m) - 1;
      *before = __shfl_sync(0xffffffffu, cum - x, l);
      return b0 + l;
    }
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  *before = run;
  return -1;
}

// First index where the running sum (from `run`) of arr reaches D (and was
// below D before it), or -1; *before = running sum before that index (or the
// total). Two levels: every lane sums a contiguous segment with independent
// loads, the warp scans the segment sums, then only the crossing segment is
// walked -- a few memory round trips instead of len/32 dependent ones.
static __device__ __forceinline__ int warp_cross(const unsigned long long* __restrict__ arr, int len,
                                                 long long D, long long run, long long* before) {
  if (len <= 64) return warp_cross_linear(arr, len, D, run, before);
  const int lane = threadIdx.x & 31;
  const int seg = (len + 31) / 32;
  const int b = min(len, lane * seg), e = min(len, b + seg);
  long long sm = 0;
  int i = b;
  for (; i + 8 <= e; i += 8) {  // 8 independent loads in flight per lane
    unsigned long long x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldcg(arr + i + u);
#pragma unroll
    for (int u = 0; u < 8; ++u) sm += (long long)x[u];
  }
  for (; i < e; ++i) sm += (long long)__ldcg(arr + i);
  long long incl = sm;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane >= o) incl += y;
  }
  const long long total = __shfl_sync(0xffffffffu, incl, 31);
  if (run >= D) {  // reached before the first element: no crossing
    *before = run + total;
    return -1;
  }
  const unsigned m = __ballot_sync(0xffffffffu, run + incl >= D);
  if (!m) {
    *before = run + total;
    return -1;
  }
  const int l = __ffs(m) - 1;
  const long long base = run + __shfl_sync(0xffffffffu, incl - sm, l);
  const int lb = min(len, l * seg);
  const int r = warp_cross_linear(arr + lb, min(seg, len - lb), D, base, before);
  return r < 0 ? -1 : lb + r;
}

// bucket crossing (select_prefix on bucket totals): the crossing slot from
// the per-slot totals, then the crossing sub-bucket inside that slot
static __device__ void rb_scan_warp(int op, const unsigned long long* __restrict__ H,
                                    const unsigned long long* __restrict__ Hs, int nb, int rho,
                                    const long long* __restrict__ deficit, int32_t* bstar,
                                    long long* cum_before) {
  const int ns = nb / rho;
  const long long D = deficit[op];
  long long before;
  int b = nb;
  const int sl = warp_cross(Hs + (size_t)op * ns, ns, D, 0, &before);
  if (sl >= 0) {
    long long b2;
    const int sb = warp_cross(H + (size_t)op * nb + (size_t)sl * rho, rho, D, before, &b2);
    b = sl * rho + sb;  // sb >= 0: the slot total crosses, so one of its buckets does
    before = b2;
  }
  if ((threadIdx.x & 31) == 0) {
    bstar[op] = b;
    cum_before[op] = before;
  }
}

// crossing chunk, then the crossing element inside it (see rb_find_op)
static __device__ void rb_find_warp(int op, const RbSel& s, const long long* __restrict__ deficit,
                                    const long long* __restrict__ required,
                                    const long long* __restrict__ cum_before,
                                    const int32_t* __restrict__ opart, int64_t n, int nb,
                                    int32_t* thr) {
  const int lane = threadIdx.x & 31;
  const int bs = s.bstar[op];
  if (bs >= nb) {  // shortfall: every eligible candidate leaves
    if (lane == 0) thr[op] = 0x7fffffff;
    return;
  }
  const long long D = deficit[op];
  long long cb;
  const int ch = warp_cross(s.CH + (size_t)op * s.nch, s.nch, D, cum_before[op], &cb);
  const int P = opart[op];
  const int sub = bs % s.rho;
  const int64_t j = (int64_t)ch * 32 + lane;
  const int64_t v64 = j * s.rho + sub;
  long long w = 0;
  if (ch >= 0 && v64 < n) {
    const int v = (int)v64;
    if (s.parts[v] == P && s.rkey[v] == bs) w = s.vw[v];
  }
  long long incl = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const long long cum = cb + incl;
  const unsigned m = __ballot_sync(0xffffffffu, w > 0 && cum >= D && cum - w < D);
  if (m && lane == __ffs(m) - 1) {
    const long long prev = cum - w;
    const bool include = (cum - D <= D - prev) || (prev < required[op]);
    thr[op] = (int)v64 + (include ? 1 : 0);
  }
  if (!m && lane == 0) thr[op] = 0x7fffffff;  // unreachable by construction
}

// rb_find_warp with a whole block per part (level kernel, grid >= parts):
// every thread sums a contiguous run of chunk totals with independent loads,
// one block scan locates the crossing run, its thread walks it.
template <int BSZ>
static __device__ void rb_find_block(int op, const RbSel& s, const long long* __restrict__ deficit,
                                     const long long* __restrict__ required,
                                     const long long* __restrict__ cum_before,
                                     const int32_t* __restrict__ opart, int64_t n, int nb,
                                     int32_t* thr) {
  typedef cub::BlockScan<long long, BSZ> BS;
  __shared__ typename BS::TempStorage ts;
  __shared__ int s_ch;
  __shared__ long long s_cb;
  const int bs = s.bstar[op];
  if (bs >= nb) {
    if (threadIdx.x == 0) thr[op] = 0x7fffffff;
    return;
  }
  const long long D = deficit[op];
  const long long base = cum_before[op];
  const unsigned long long* chs = s.CH + (size_t)op * s.nch;
  const int per = (s.nch + BSZ - 1) / BSZ;
  const int b = min(s.nch, (int)threadIdx.x * per), e = min(s.nch, b + per);
  long long sm = 0;
  int i = b;
  for (; i + 4 <= e; i += 4) {
    unsigned long long x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = __ldcg(chs + i + u);
#pragma unroll
    for (int u = 0; u < 4; ++u) sm += (long long)x[u];
  }
  for (; i < e; ++i) sm += (long long)__ldcg(chs + i);
  if (threadIdx.x == 0) s_ch = -1;
  long long ex;
  BS(ts).ExclusiveSum(sm, ex);
  __syncthreads();
  long long run = base + ex;
  if (b < e && run < D && run + sm >= D) {  // exactly one thread's run crosses
    for (int j = b; j < e; ++j) {
      const long long x = (long long)__ldcg(chs + j);
      if (run + x >= D) {
        s_ch = j;
        s_cb = run;
        break;
      }
      run += x;
    }
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int ch = s_ch;
    const long long cb = s_cb;
    const int P = opart[op];
    const int sub = bs % s.rho;
    const int64_t v64 = ((int64_t)ch * 32 + lane) * s.rho + sub;
    long long w = 0;
    if (ch >= 0 && v64 < n) {
      const int v = (int)v64;
      if (s.parts[v] == P && s.rkey[v] == bs) w = s.vw[v];
    }
    long long incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const long long cum = cb + incl;
    const unsigned m = __ballot_sync(0xffffffffu, w > 0 && cum >= D && cum - w < D);
    if (m && lane == __ffs(m) - 1) {
      const long long prev = cum - w;
      const bool include = (cum - D <= D - prev) || (prev < required[op]);
      thr[op] = (int)v64 + (include ? 1 : 0);
    }
    if (!m && lane == 0) thr[op] = 0x7fffffff;
  }
  __syncthreads();
}

// Sharded form of rb_find_warp: (a) every rank locates the crossing chunk
// from the all-reduced chunk histogram and contributes the weights of the
// chunk's elements it owns; (b) after the element weights are all-reduced,
// every rank finds the crossing element (same rule as rb_find_warp).
static __device__ void rb_find_a(int op, const RbSel& s, const long long* __restrict__ deficit,
                                 const long long* __restrict__ cum_before,
                                 const int32_t* __restrict__ opart, int64_t n, int nb,
                                 int64_t lo, int64_t hi, int32_t* ch_out, long long* cb_out,
                                 unsigned long long* ew) {
  const int lane = threadIdx.x & 31;
  const int bs = s.bstar[op];
  long long w = 0, cb = 0;
  int ch = -1;
  if (bs < nb) {
    ch = warp_cross(s.CH + (size_t)op * s.nch, s.nch, deficit[op], cum_before[op], &cb);
    const int64_t v64 = ((int64_t)ch * 32 + lane) * s.rho + bs % s.rho;
    if (ch >= 0 && v64 < n && v64 >= lo && v64 < hi) {
      const int v = (int)v64;
      if (s.parts[v] == opart[op] && s.rkey[v] == bs) w = s.vw[v];
    }
  }
  ew[(size_t)op * 32 + lane] = (unsigned long long)w;
  if (lane == 0) {
    ch_out[op] = ch;
    cb_out[op] = cb;
  }
}

static __device__ void rb_find_b(int op, const RbSel& s, const long long* __restrict__ deficit,
                                 const long long* __restrict__ required, int nb,
                                 const int32_t* __restrict__ ch_in,
                                 const long long* __restrict__ cb_in,
                                 const unsigned long long* __restrict__ ew, int32_t* thr) {
  const int lane = threadIdx.x & 31;
  const int bs = s.bstar[op];
  if (bs >= nb) {
    if (lane == 0) thr[op] = 0x7fffffff;
    return;
  }
  const long long D = deficit[op], w = (long long)ew[(size_t)op * 32 + lane];
  const int ch = ch_in[op];
  const int64_t v64 = ((int64_t)ch * 32 + lane) * s.rho + bs % s.rho;
  long long incl = w;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const long long cum = cb_in[op] + incl;
  const unsigned m = __ballot_sync(0xffffffffu, w > 0 && cum >= D && cum - w < D);
  if (m && lane == __ffs(m) - 1) {
    const long long prev = cum - w;
    const bool include = (cum - D <= D - prev) || (prev < required[op]);
    thr[op] = (int)v64 + (include ? 1 : 0);
  }
  if (!m && lane == 0) thr[op] = 0x7fffffff;
}

static __device__ void rb_select(const RbSel& s, const int32_t* __restrict__ rcand,
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
      sel = rk >= 0 && (rk < bs || (rk == bs && v < s.thr[op]));
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



// Collect the vertices of oversized parts into per-tier candidate lists.


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
  int smem_cap;                     // keys that fit the caller's shared buffer
  unsigned long long* gscratch;     // >= 2 * P2 + blockDim words, for larger sets
  int presorted;                    // keys already sorted in gscratch (grid sort)
};

// Warp-aggregated append slot in a shared counter (t < 0: no item).
static __device__ __forceinline__ unsigned smem_warp_slot(unsigned* ctr, int t) {
  const unsigned peers = __match_any_sync(0xffffffffu, t);
  const int lane = threadIdx.x & 31, leader = __ffs(peers) - 1;
  unsigned b = 0;
  if (t >= 0 && lane == leader) b = atomicAdd(&ctr[t], (unsigned)__popc(peers));
  b = __shfl_sync(0xffffffffu, b, leader);
  return b + (unsigned)__popc(peers & ((1u << lane) - 1u));
}

constexpr int RB_RADIX_THREADS = 512, RB_RADIX_ITEMS = 4, RB_RANK_MAX = 512;
#ifndef RB_RADIX_BITS
#define RB_RADIX_BITS 4
#endif
// (a block merge sort measured the same, 6- and 8-bit digits do not fit the
// shared buffer next to the keys)
typedef cub::BlockRadixSort<unsigned long long, RB_RADIX_THREADS, RB_RADIX_ITEMS, cub::NullType,
                           RB_RADIX_BITS>
    RbRadix;

static __device__ void rb_tail(const RbTail& a, unsigned long long* sk_smem) {
  const int tid = threadIdx.x, nth = blockDim.x;
  const int L = (int)*(const volatile unsigned long long*)a.evict_cnt;
  int P2 = 1;
  while (P2 < L) P2 <<= 1;
  constexpr int RCAP = RB_RADIX_THREADS * RB_RADIX_ITEMS;
  constexpr int RTS = (int)((sizeof(typename RbRadix::TempStorage) + 7) / 8);
  unsigned long long* sk;
  if (a.presorted) {
    // ordered by the grid: bring them on chip when they fit (the next-fit
    // walk below makes dependent accesses)
    if (L <= a.smem_cap) {
      for (int i = tid; i < L; i += nth) sk_smem[i] = a.gscratch[i];
      sk = sk_smem;
    } else {
      sk = a.gscratch;
    }
  } else if (L <= nth && L <= RB_RANK_MAX && a.smem_cap >= 2 * RB_RANK_MAX) {
    // small sets: rank = #smaller keys, one key per thread, the others read
    // as shared-memory broadcasts (a sorting network or radix passes cost a
    // fixed 10-30 us here whatever L is)
    unsigned long long* tmp = sk_smem + RB_RANK_MAX;
    unsigned long long key = ~0ull;
    if (tid < L) {
      const int v = a.evict[tid];
      const unsigned long long grp =
          (unsigned long long)a.opidx[a.parts[v]] * (unsigned)a.nb + (unsigned)a.rkey[v];
      key = (grp << 32) | (unsigned)v;
      tmp[tid] = key;
    }
    __syncthreads();
    if (tid < ((L + 31) & ~31)) {
      int r = 0;
#pragma unroll 8
      for (int j = 0; j < L; ++j) r += tmp[j] < key;
      if (tid < L) sk_smem[r] = key;
    }
    sk = sk_smem;
  } else if (nth == RB_RADIX_THREADS && L <= RCAP && a.smem_cap >= RCAP + RTS) {
    // block radix sort of (group, id) over the bits actually used: ~5x
    // faster than the bitonic network below at 2048 keys
    __shared__ unsigned s_gmax, s_vmax;
    if (tid == 0) s_gmax = s_vmax = 0;
    __syncthreads();
    unsigned gg[RB_RADIX_ITEMS], vv[RB_RADIX_ITEMS];
    unsigned gm = 0, vm = 0;
#pragma unroll
    for (int j = 0; j < RB_RADIX_ITEMS; ++j) {
      const int i = tid * RB_RADIX_ITEMS + j;
      gg[j] = vv[j] = 0;
      if (i < L) {
        const int v = a.evict[i];
        vv[j] = (unsigned)v;
        gg[j] = (unsigned)a.opidx[a.parts[v]] * (unsigned)a.nb + (unsigned)a.rkey[v];
        gm = max(gm, gg[j]);
        vm = max(vm, vv[j]);
      }
    }
    gm = __reduce_max_sync(0xffffffffu, gm);
    vm = __reduce_max_sync(0xffffffffu, vm);
    if ((tid & 31) == 0) {
      atomicMax(&s_gmax, gm);
      atomicMax(&s_vmax, vm);
    }
    __syncthreads();
    const int vb = max(1, 32 - __clz((int)s_vmax)), gb = 32 - __clz((int)s_gmax);
    unsigned long long kk[RB_RADIX_ITEMS];
#pragma unroll
    for (int j = 0; j < RB_RADIX_ITEMS; ++j)
      kk[j] = tid * RB_RADIX_ITEMS + j < L ? ((unsigned long long)gg[j] << vb) | vv[j] : ~0ull;
    auto& ts = *reinterpret_cast<typename RbRadix::TempStorage*>(sk_smem + RCAP);
    RbRadix(ts).Sort(kk, 0, vb + gb);
    const unsigned long long vmask = (1ull << vb) - 1;
#pragma unroll
    for (int j = 0; j < RB_RADIX_ITEMS; ++j) sk_smem[tid * RB_RADIX_ITEMS + j] = kk[j] & vmask;
    sk = sk_smem;
    __syncthreads();
  } else {
    sk = (P2 <= a.smem_cap || a.gscratch == nullptr) ? sk_smem : a.gscratch;
    for (int i = tid; i < P2; i += nth) {
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
        for (int i = tid; i < P2; i += nth) {
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
  }
  __syncthreads();
  // from here sk[i] (low 32 bits) = the i-th evicted vertex in key order;
  // each path leaves sk[i] = (dest + 1) << 32 | v for i < s_end (0: no move)
  __shared__ int s_end, s_wide;
  __shared__ unsigned long long s_ws[33];
  if (!a.strong) {
    for (int i = tid; i < L; i += nth) {
      const unsigned v = (unsigned)(sk[i] & 0xffffffffu);
      sk[i] = ((unsigned long long)(unsigned)(a.valid_list[a.draws[i]] + 1) << 32) | v;
    }
    if (tid == 0) s_end = L;
  } else {
    // next-fit (rebalance.py:228-236). The block packs (inclusive prefix of
    // the sorted weights, id) into the keys; one warp then finds each part's
    // segment [start, e) by a 32-ary search for the first prefix above
    // start's prefix + the part's spare, and the next part by a ballot over a
    // register window of spare[] -- a few steps per part switch, nothing per
    // item. (A block-wide round per switch cost 30-40 us per strong pass.)
    for (int i = tid; i < L; i += nth) {
      const unsigned v = (unsigned)(sk[i] & 0xffffffffu);
      sk[i] = ((unsigned long long)(unsigned)a.vw[v] << 32) | v;
    }
    __syncthreads();
    const int ipt = (L + nth - 1) / nth;
    const int lo = min(L, tid * ipt), hi = min(L, lo + ipt);
    unsigned long long run = 0;
    for (int i = lo; i < hi; ++i) run += sk[i] >> 32;
    unsigned long long x = run;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_ws[wid] = x;
    __syncthreads();
    if (tid < 32) {
      unsigned long long t = tid < ((nth + 31) >> 5) ? s_ws[tid] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, t, o);
        if (tid >= o) t += y;
      }
      s_ws[tid] = t;
      if (tid == 31) s_wide = t >= (1ull << 32);
    }
    __syncthreads();
    const bool wide = s_wide;
    if (!wide) {
      unsigned long long pre = x - run + (wid ? s_ws[wid - 1] : 0);
      for (int i = lo; i < hi; ++i) {
        const unsigned long long k = sk[i];
        pre += k >> 32;
        sk[i] = (pre << 32) | (k & 0xffffffffu);
      }
    }
    __syncthreads();
    if (tid < 32) {
      const int nvalid = a.nvalid;
      int wb = 0;  // window of parts [wb, wb + 32) in registers
      long long wsp = lane < nvalid ? a.spare[lane] : 0;
      int wvl = lane < nvalid ? a.valid_list[lane] : -1;
      int di = 0, end = nvalid > 0 ? L : 0;
      // first later part whose whole spare holds weight we (the reference's
      // `while r < w: di += 1; r = spare[di]`); returns false past the last
      auto advance = [&](long long we) {
        ++di;
        while (di < nvalid) {
          if (di >= wb + 32) {
            wb = di;
            wsp = wb + lane < nvalid ? a.spare[wb + lane] : 0;
            wvl = wb + lane < nvalid ? a.valid_list[wb + lane] : -1;
          }
          const unsigned ok =
              __ballot_sync(0xffffffffu, lane >= di - wb && wb + lane < nvalid && wsp >= we);
          if (ok) {
            di = wb + __ffs(ok) - 1;
            return true;
          }
          di = wb + 32;
        }
        return false;
      };
      if (!wide) {
        auto S = [&](int i) -> long long { return (long long)(sk[i] >> 32); };
        int start = 0;
        long long sbase = 0;  // prefix before `start`
        while (nvalid > 0) {
          const int dest = __shfl_sync(0xffffffffu, wvl, di - wb);
          const long long room = __shfl_sync(0xffffffffu, wsp, di - wb);
          // e = first index >= start whose item does not fit: S(e) - sbase > room
          int lo2 = start, hi2 = L;
          while (lo2 < hi2) {
            const int step = (hi2 - lo2 + 31) >> 5;
            const int q = lo2 + lane * step;
            const unsigned bb = __ballot_sync(0xffffffffu, q >= hi2 || S(q) - sbase > room);
            if (!bb) {
              lo2 += 31 * step + 1;
              continue;
            }
            const int j = __ffs(bb) - 1;
            if (j == 0) {
              hi2 = lo2;
            } else {
              hi2 = min(hi2, lo2 + j * step);
              lo2 += (j - 1) * step + 1;
            }
          }
          const int e = lo2;
          const long long prev = e > start ? S(e - 1) : sbase;
          const long long we = e < L ? S(e) - prev : 0;
          __syncwarp();
          for (int i = start + lane; i < e; i += 32)
            sk[i] = ((unsigned long long)(unsigned)(dest + 1) << 32) | (sk[i] & 0xffffffffu);
          if (e >= L) break;
          if (!advance(we)) {
            end = e;
            break;
          }
          start = e;
          sbase = prev;
        }
      } else {
        // totals >= 2^32: walk the weights 32 items at a time
        long long room = nvalid > 0 ? __shfl_sync(0xffffffffu, wsp, 0) : 0;
        bool done = nvalid <= 0;
        for (int base = 0; base < L && !done; base += 32) {
          const int i = base + lane;
          const int lim = L - base < 32 ? L - base : 32;
          const unsigned long long k = i < L ? sk[i] : 0;
          long long incl = (long long)(k >> 32);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const long long y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          int dest = -1, pos = 0;
          long long before = 0;
          while (true) {
            const bool live = lane >= pos && lane < lim;
            const bool fits = live && incl - before <= room;
            const int dv = __shfl_sync(0xffffffffu, wvl, di - wb);
            if (fits) dest = dv;
            const unsigned m = __ballot_sync(0xffffffffu, live && !fits);
            if (!m) {
              room -= __shfl_sync(0xffffffffu, incl, lim - 1) - before;
              break;
            }
            const int e = __ffs(m) - 1;
            const long long prev = e > 0 ? __shfl_sync(0xffffffffu, incl, e - 1) : 0;
            const long long we = __shfl_sync(0xffffffffu, incl, e) - prev;
            if (!advance(we)) {
              done = true;
              end = base + lim;
              break;
            }
            room = __shfl_sync(0xffffffffu, wsp, di - wb);
            pos = e;
            before = prev;
          }
          if (lane < lim)
            sk[i] = (dest >= 0 ? (unsigned long long)(unsigned)(dest + 1) << 32 : 0ull) |
                    (k & 0xffffffffu);
        }
      }
      if (lane == 0) s_end = end;
    }
  }
  // commit: mv[] and the per-tier move lists, one global atomic per tier
  __shared__ unsigned s_tc[NBINS];
  __shared__ unsigned long long s_tb[NBINS];
  if (tid < NBINS) s_tc[tid] = 0;
  __syncthreads();
  const int end = s_end;
  const int lim = (end + 31) & ~31;
  for (int i = tid; i < lim; i += nth) {
    int t = -1;
    if (i < end) {
      const unsigned long long k = sk[i];
      const unsigned v = (unsigned)(k & 0xffffffffu);
      if (k >> 32) {
        a.mv[v] = (int)(k >> 32) - 1;
        t = a.tm(a.offs[v + 1] - a.offs[v]);
        sk[i] = ((unsigned long long)(unsigned)(t + 1) << 32) | v;
      }
    }
    smem_warp_slot(s_tc, t);
  }
  __syncthreads();
  if (tid < NBINS) {
    s_tb[tid] = s_tc[tid] ? atomicAdd(a.move_cnt + tid, (unsigned long long)s_tc[tid]) : 0;
    s_tc[tid] = 0;
  }
  __syncthreads();
  for (int i = tid; i < lim; i += nth) {
    int t = -1;
    unsigned v = 0;
    if (i < end) {
      const unsigned long long k = sk[i];
      v = (unsigned)(k & 0xffffffffu);
      t = (int)(k >> 32) - 1;
    }
    const unsigned pos = smem_warp_slot(s_tc, t);
    if (t >= 0) a.move_lists[a.mseg.b[t] + s_tb[t] + pos] = (int32_t)v;
  }
}




// Candidates of the rebalancing passes: the vertices of oversized parts, by
// degree tier. Blocks take tiles of blockDim * RB_COL_IT consecutive ids
// (coalesced loads, RB_COL_IT independent per thread) and reserve each
// tier's output once per tile -- per-warp appends put tens of thousands of
// same-address atomics on the six counters every pass. Two ids per thread
// measured best (1: 44.98, 2: 44.47, 4: 45.4, 8: 47.5, 16: 51.8 ms of level
// kernels on the headline). All threads of the block must call it.
#ifndef RB_COL_ITEMS
#define RB_COL_ITEMS 2
#endif
constexpr int RB_COL_IT = RB_COL_ITEMS;
template <class Take>
static __device__ void collect_tiled(Take take, const int64_t* __restrict__ offs, TierMap tm,
                                     int64_t n, int32_t* lists, RbSegsDev seg,
                                     unsigned long long* cnts, unsigned long long* pwr,
                                     unsigned long long* pwe) {
  __shared__ unsigned s_wc[NBINS][32];
  __shared__ unsigned long long s_base[NBINS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t tile = (int64_t)blockDim.x * RB_COL_IT;
  unsigned long long wr = 0, we = 0;
  for (int64_t b0 = blockIdx.x * tile; b0 < n; b0 += (int64_t)gridDim.x * tile) {
    const int64_t wbase = b0 + (int64_t)w * 32 * RB_COL_IT;
    int tv[RB_COL_IT];
#pragma unroll
    for (int j = 0; j < RB_COL_IT; ++j) {
      const int64_t v = wbase + j * 32 + lane;
      int t = -1;
      if (v < n && take((int)v)) {
        const int64_t d = offs[v + 1] - offs[v];
        t = tm(d);
        wr += 1;
        we += (unsigned long long)d;
      }
      tv[j] = t;
    }
    unsigned c[NBINS];
#pragma unroll
    for (int tt = 0; tt < NBINS; ++tt) {
      c[tt] = 0;
#pragma unroll
      for (int j = 0; j < RB_COL_IT; ++j) c[tt] += __popc(__ballot_sync(0xffffffffu, tv[j] == tt));
    }
    if (lane == 0)
#pragma unroll
      for (int tt = 0; tt < NBINS; ++tt) s_wc[tt][w] = c[tt];
    __syncthreads();
    if (w < NBINS) {  // warp w: exclusive scan of tier w over the warps, one reservation
      const unsigned x = lane < nw ? s_wc[w][lane] : 0u;
      unsigned inc = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned tot = __shfl_sync(0xffffffffu, inc, 31);
      if (lane < nw) s_wc[w][lane] = inc - x;
      if (lane == 0) s_base[w] = tot ? atomicAdd(cnts + w, (unsigned long long)tot) : 0ull;
    }
    __syncthreads();
    unsigned long long off[NBINS];
#pragma unroll
    for (int tt = 0; tt < NBINS; ++tt) off[tt] = seg.b[tt] + s_base[tt] + s_wc[tt][w];
#pragma unroll
    for (int j = 0; j < RB_COL_IT; ++j) {
      const int t = tv[j];
#pragma unroll
      for (int tt = 0; tt < NBINS; ++tt) {
        const unsigned m = __ballot_sync(0xffffffffu, t == tt);
        if (t == tt) lists[off[tt] + __popc(m & lt)] = (int32_t)(wbase + j * 32 + lane);
        off[tt] += __popc(m);
      }
    }
    __syncthreads();  // s_wc / s_base are rewritten by the next tile
  }
  if (pwr) {  // candidate rows / entries: the stats sweep visits exactly these
    *pwr += wr;
    *pwe += we;
  }
}

static __device__ void rb_collect(const int32_t* __restrict__ parts, const int32_t* __restrict__ opidx,
                           const int64_t* __restrict__ offs, TierMap tm, int64_t n, int32_t* lists,
                           RbSegsDev seg, unsigned long long* cnts, int64_t /*t0*/, int64_t /*stride*/,
                           unsigned long long* pwr = nullptr, unsigned long long* pwe = nullptr) {
  collect_tiled([&](int v) { return opidx[parts[v]] >= 0; }, offs, tm, n, lists, seg, cnts, pwr,
                pwe);
}

}  // namespace jet
