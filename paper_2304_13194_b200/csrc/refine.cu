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
#include "refine_dev.cuh"
#include "comm.cuh"
#include "rng.h"
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
#include <cmath>

namespace jet {

// Kernel wrappers of the aggregation device functions (multi-kernel path).
// E = entries per lane (tier 3 holds rows of up to 64 entries; levels whose
// rows all fit 32 use one entry per lane, as the level kernel does)
template <class Op, int G, bool UNIT, int E = tier_e<G>()>
__global__ void __launch_bounds__(256)
    k_agg_small(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
                const int32_t* __restrict__ list, int64_t cnt, bool wide,
                const unsigned long long* __restrict__ dcnt) {
  extern __shared__ uint32_t agg_stage[];
  long long acc = 0;
  constexpr int RB = G * E == 64 ? 16 : 32;
  agg_small<Op, G, UNIT, RB, E>(a, g, parts, list, cnt, wide, dcnt,
                                (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                                ((int64_t)gridDim.x * blockDim.x) >> 5, acc,
                                agg_stage + (threadIdx.x >> 5) * stage_words<G, RB, UNIT, E>());
  Op::block_done(a, acc);
}

// dynamic shared memory of k_agg_small<Op, G, UNIT, E> (8 warps), set once
template <class Op, int G, bool UNIT, int E = tier_e<G>()>
static size_t agg_small_smem() {
  static const size_t bytes = [] {
    const size_t b = (size_t)8 * stage_words<G, (G * E == 64 ? 16 : 32), UNIT, E>() * 4;
    CK(cudaFuncSetAttribute(k_agg_small<Op, G, UNIT, E>,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)b));
    return b;
  }();
  return bytes;
}

template <class Op, bool UNIT>
__global__ void __launch_bounds__(256)
    k_agg_warp(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
               const int32_t* __restrict__ list, int64_t cnt, bool wide, int k, int tl_cap,
               const unsigned long long* __restrict__ dcnt) {
  extern __shared__ unsigned long long smem[];
  long long acc = 0;
  agg_warp<Op, UNIT>(a, g, parts, list, cnt, wide, k, tl_cap, dcnt, smem,
                     (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                     ((int64_t)gridDim.x * blockDim.x) >> 5, acc);
  Op::block_done(a, acc);
}

template <class Op, bool UNIT>
__global__ void __launch_bounds__(256)
    k_agg_block(typename Op::Args a, GView g, const int32_t* __restrict__ parts,
                const int32_t* __restrict__ list, int64_t cnt, bool wide, int k,
                const unsigned long long* __restrict__ dcnt) {
  extern __shared__ unsigned long long smem[];
  long long acc = 0;
  agg_block<Op, UNIT>(a, g, parts, list, cnt, wide, k, dcnt, smem, acc);
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
            case 4: AGG_K(4, true)<<<grid, 256, agg_small_smem<Op, 4, true>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 8: AGG_K(8, true)<<<grid, 256, agg_small_smem<Op, 8, true>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 16: AGG_K(16, true)<<<grid, 256, agg_small_smem<Op, 16, true>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            default:
              if (g.max_deg <= 32)
                k_agg_small<Op, 32, true, 1><<<grid, 256, agg_small_smem<Op, 32, true, 1>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc);
              else
                AGG_K(32, true)<<<grid, 256, agg_small_smem<Op, 32, true>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc);
              break;
          }
        } else {
          switch (G) {
            case 4: AGG_K(4, false)<<<grid, 256, agg_small_smem<Op, 4, false>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 8: AGG_K(8, false)<<<grid, 256, agg_small_smem<Op, 8, false>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            case 16: AGG_K(16, false)<<<grid, 256, agg_small_smem<Op, 16, false>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc); break;
            default:
              if (g.max_deg <= 32)
                k_agg_small<Op, 32, false, 1><<<grid, 256, agg_small_smem<Op, 32, false, 1>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc);
              else
                AGG_K(32, false)<<<grid, 256, agg_small_smem<Op, 32, false>(), c.stream>>>(a, gv, parts, list, cnt, wide, dc);
              break;
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

template <bool UNIT>
__global__ void __launch_bounds__(256)
    k_afterburner(AbArgs a, GView g, SegLists sl, RbSegsDev mseg) {
  afterburner_rows<UNIT>(a, g, sl, mseg, (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                         ((int64_t)gridDim.x * blockDim.x) >> 5);
}

template <bool UNIT>
__global__ void __launch_bounds__(256) k_apply_delta(ApArgs a, GView g, SegLists sl) {
  long long acc = 0;
  apply_delta_rows<UNIT>(a, g, sl, (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                         ((int64_t)gridDim.x * blockDim.x) >> 5, acc);
  block_sum_atomic<256>(acc, a.cut2d);
}

__global__ void k_apply_commit(CommitArgs a) {
  apply_commit_rows(a, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
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
    opart.alloc(kk, c.stream);
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

// ---------------------------------------------------------------------------
// 1D vertex sharding of the Jetlp pass (comm.cuh for the exchange).
__global__ void k_shard_bounds(const int64_t* __restrict__ offs, int64_t n, int size,
                               int64_t* bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > size) return;
  const int64_t nnz = offs[n];
  const int64_t want = r == size ? nnz + 1 : (nnz * r) / size;
  int64_t lo = 0, hi = n;  // first v with offs[v] >= want (v = n if none)
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (offs[mid] < want) lo = mid + 1;
    else hi = mid;
  }
  bounds[r] = r == 0 ? 0 : (r == size ? n : lo);
}

// [first, last) of the ascending tier list inside [lo, hi)
__global__ void k_sublist(const int32_t* __restrict__ list, int64_t cnt, int64_t lo, int64_t hi,
                          int64_t* out) {
  if (threadIdx.x > 1) return;
  const int64_t key = threadIdx.x == 0 ? lo : hi;
  int64_t a = 0, b = cnt;
  while (a < b) {
    const int64_t mid = (a + b) >> 1;
    if (list[mid] < key) a = mid + 1;
    else b = mid;
  }
  out[threadIdx.x] = a;
}

__global__ void k_iota(int32_t* p, int64_t lo, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (int32_t)(lo + i);
}

void build_shard_lists(Ctx& c, const DGraph& g, int rank, int size, ShardLists& s) {
  s.scratch.ensure((size_t)size + 1 + 2 * NBINS, c.stream);
  if (g.partial()) {  // a distributed level: the block it was given
    s.lo = g.row_lo;
    s.hi = g.row_hi;
  } else {
    k_shard_bounds<<<1, 1024, 0, c.stream>>>(g.offs.get(), g.n, size, s.scratch.get());
    CK(cudaGetLastError());
    std::vector<int64_t> b(size + 1);
    d2h(c, b.data(), s.scratch.get(), size + 1);
    c.sync();
    s.lo = b[rank];
    s.hi = b[rank + 1];
  }
  unsigned long long cnts[NBINS] = {};
  for (int t = 0; t < NBINS; ++t) {
    s.list[t] = nullptr;
    if (!g.bin_cnt[t]) continue;
    const int32_t* full = tier_list(g, t);
    if (!full) {  // identity tier: every vertex
      s.iota.ensure((size_t)std::max<int64_t>(1, s.hi - s.lo), c.stream);
      k_iota<<<grid_for(c, s.hi - s.lo, 256), 256, 0, c.stream>>>(s.iota.get(), s.lo, s.hi - s.lo);
      CK(cudaGetLastError());
      s.list[t] = s.iota.get();
      cnts[t] = (unsigned long long)(s.hi - s.lo);
      continue;
    }
    int64_t* o = s.scratch.get() + size + 1 + 2 * t;
    k_sublist<<<1, 32, 0, c.stream>>>(full, g.bin_cnt[t], s.lo, s.hi, o);
    CK(cudaGetLastError());
    int64_t ab[2];
    d2h(c, ab, o, 2);
    c.sync();
    s.list[t] = const_cast<int32_t*>(full) + ab[0];
    cnts[t] = (unsigned long long)(ab[1] - ab[0]);
  }
  s.dcnt.ensure(NBINS, c.stream);
  h2d(c, s.dcnt.get(), cnts, NBINS);
  c.sync();
}

struct CandRec {
  int32_t v, dest;
  long long F;
};

__global__ void k_pack_cands(SegLists sl, const int32_t* __restrict__ cdest,
                             const long long* __restrict__ F, CandRec* out) {
  int64_t base = 0;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)sl.cnt[t];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int v = sl.list[t][i];
      out[base + i] = CandRec{v, cdest[v], F[v]};
    }
    base += cnt;
  }
}

// remote records only: [0, skip_lo) and [skip_hi, total)
__global__ void k_unpack_cands(const CandRec* __restrict__ in, int64_t total, int64_t skip_lo,
                               int64_t skip_hi, int32_t* cdest, long long* F) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i >= skip_lo && i < skip_hi) continue;
    const CandRec r = in[i];
    cdest[r.v] = r.dest;
    F[r.v] = r.F;
  }
}

__global__ void k_pack_moves(SegLists sl, const int32_t* __restrict__ mv, int2* out) {
  int64_t base = 0;
  for (int t = 0; t < NBINS; ++t) {
    const int64_t cnt = (int64_t)sl.cnt[t];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int v = sl.list[t][i];
      out[base + i] = make_int2(v, mv[v]);
    }
    base += cnt;
  }
}

__global__ void k_unpack_moves(const int2* __restrict__ in, int64_t total, int64_t skip_lo,
                               int64_t skip_hi, int32_t* mv, const int64_t* __restrict__ offs,
                               TierMap tm, int32_t* move_lists, RbSegsDev seg,
                               unsigned long long* move_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (i >= skip_lo && i < skip_hi) continue;
    const int2 r = in[i];
    mv[r.x] = r.y;
    const int t = tm(offs[r.x + 1] - offs[r.x]);
    move_lists[seg.b[t] + atomicAdd(move_cnt + t, 1ull)] = r.x;
  }
}

// candidates of this rank's block [lo, hi) (warp-uniform trip counts)
__global__ void k_rb_collect_range(const int32_t* __restrict__ parts,
                                   const int32_t* __restrict__ opidx,
                                   const int64_t* __restrict__ offs, TierMap tm, int64_t lo,
                                   int64_t hi, int32_t* lists, RbSegsDev seg,
                                   unsigned long long* cnts) {
  const int64_t span = (hi - lo + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < span;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = lo + i;
    int t = -1;
    if (v < hi && opidx[parts[v]] >= 0) t = tm(offs[v + 1] - offs[v]);
    if (__ballot_sync(0xffffffffu, t >= 0) == 0) continue;
    for (int tt = 0; tt < NBINS; ++tt) warp_append(t == tt, (int32_t)v, lists + seg.b[tt], cnts + tt);
  }
}

__global__ void k_rb_find_a(RbSel s, const long long* __restrict__ deficit,
                            const long long* __restrict__ cum_before,
                            const int32_t* __restrict__ opart, int64_t n, int nb, int nover,
                            int64_t lo, int64_t hi, int32_t* ch, long long* cb,
                            unsigned long long* ew) {
  const int op = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (op < nover) rb_find_a(op, s, deficit, cum_before, opart, n, nb, lo, hi, ch, cb, ew);
}

__global__ void k_rb_find_b(RbSel s, const long long* __restrict__ deficit,
                            const long long* __restrict__ required, int nb, int nover,
                            const int32_t* __restrict__ ch, const long long* __restrict__ cb,
                            const unsigned long long* __restrict__ ew, int32_t* thr) {
  const int op = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (op < nover) rb_find_b(op, s, deficit, required, nb, ch, cb, ew, thr);
}

// The pending moves of every rank (this rank's move lists, packed as
// (id, destination)) gathered and appended to every rank's move lists.
void share_moves(Ctx& c, Workspace& w, const DGraph& g, ShardLists& sh) {
  Comm& cm = *c.comm;
  unsigned long long hc[2 * NBINS];
  std::vector<int64_t> counts;
  int64_t total = 0, mine_lo = 0;
  d2h(c, hc, w.ctr.get(), 2 * NBINS);
  c.sync();
  int64_t nm = 0;
  for (int t = 0; t < NBINS; ++t) nm += (int64_t)hc[CTR_MOVE + t];
  sh.send.ensure((size_t)std::max<int64_t>(1, nm) * sizeof(int2), c.stream);
  const SegLists ml = seg_lists(w, true);
  launch(c, "shard_pack", 8.0 * nm, [&] {
    k_pack_moves<<<grid_for(c, nm, 256), 256, 0, c.stream>>>(ml, w.mv.get(), (int2*)sh.send.get());
  });
  cm.allgatherv(c, sh.send.get(), nm * (int64_t)sizeof(int2), sh.recv, counts);
  total = 0;
  for (int r = 0; r < cm.size; ++r) {
    if (r == cm.rank) mine_lo = total;
    total += counts[r];
  }
  total /= (int64_t)sizeof(int2);
  mine_lo /= (int64_t)sizeof(int2);
  RbSegsDev ms;
  for (int t = 0; t < NBINS; ++t) ms.b[t] = w.seg_base[t];
  launch(c, "shard_unpack", 8.0 * total, [&] {
    k_unpack_moves<<<grid_for(c, total, 256), 256, 0, c.stream>>>(
        (const int2*)sh.recv.get(), total, mine_lo, mine_lo + nm, w.mv.get(), g.offs.get(), g.tm,
        w.lists.get() + w.cap_n, ms, w.ctr.get() + CTR_MOVE);
  });
}

void lp_pass_sharded(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts, int k,
                     const LpParams& p, ShardLists& sh) {
  JET_REQUIRE(c.comm && p.afterburner, JET_EUNSUPPORTED,
              "sharded Jetlp needs a communicator and the afterburner");
  Comm& cm = *c.comm;
  dzero(c, w.ctr.get(), CTR_PW);
  launch(c, "shard_fill", 4.0 * g.n, [&] {
    k_fill_i32<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(w.cdest.get(), g.n, -1);
  });
  auto mk = [&](int t) {
    LpOp::Args a{};
    a.parts = parts;
    a.cdest = w.cdest.get();
    a.F = w.F.get();
    a.mv = w.mv.get();
    a.lock = w.lock.get();
    a.p = p;
    a.out_list = w.cand_list(t);
    a.out_cnt = w.ctr.get() + CTR_CAND + t;
    a.cut2 = w.ctr.get() + CTR_CUT2;
    return a;
  };
  run_agg<LpOp>(c, g, mk, parts, k, "lp_gains", 20.0, sh.list, sh.dcnt.get());
  // candidates: (id, destination, gain) of every rank
  unsigned long long hc[2 * NBINS];
  d2h(c, hc, w.ctr.get(), 2 * NBINS);
  c.sync();
  int64_t nc = 0;
  for (int t = 0; t < NBINS; ++t) nc += (int64_t)hc[CTR_CAND + t];
  sh.send.ensure((size_t)std::max<int64_t>(1, nc) * sizeof(CandRec), c.stream);
  const SegLists cl = seg_lists(w, false);
  launch(c, "shard_pack", 16.0 * nc, [&] {
    k_pack_cands<<<grid_for(c, nc, 256), 256, 0, c.stream>>>(cl, w.cdest.get(), w.F.get(),
                                                              (CandRec*)sh.send.get());
  });
  std::vector<int64_t> counts;
  cm.allgatherv(c, sh.send.get(), nc * (int64_t)sizeof(CandRec), sh.recv, counts);
  int64_t total = 0, mine_lo = 0;
  for (int r = 0; r < cm.size; ++r) {
    if (r == cm.rank) mine_lo = total;
    total += counts[r];
  }
  total /= (int64_t)sizeof(CandRec);
  mine_lo /= (int64_t)sizeof(CandRec);
  launch(c, "shard_unpack", 16.0 * total, [&] {
    k_unpack_cands<<<grid_for(c, total, 256), 256, 0, c.stream>>>(
        (const CandRec*)sh.recv.get(), total, mine_lo, mine_lo + nc, w.cdest.get(), w.F.get());
  });
  // afterburner on owned candidates -> owned moves
  AbArgs ab{};
  ab.parts = parts;
  ab.cdest = w.cdest.get();
  ab.F = w.F.get();
  ab.mv = w.mv.get();
  ab.move_list = w.lists.get();
  launch_rows_reduce_ab(c, w, g, ab);
  share_moves(c, w, g, sh);
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
// pw[p] += delta[1 + p]; cut2d = delta[0] (sharded apply, after the all-reduce)
__global__ void k_add_deltas(const unsigned long long* __restrict__ delta, int k,
                             unsigned long long* pw, unsigned long long* cut2d) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < k; p += gridDim.x * blockDim.x)
    pw[p] += delta[1 + p];
  if (blockIdx.x == 0 && threadIdx.x == 0) *cut2d = delta[0];
}

ApplyResult apply_moves(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts,
                        int k, bool set_lock, int32_t epoch, ShardLists* sh) {
  const GView gv = view(g);
  ApArgs a{parts, w.mv.get(), w.ctr.get() + CTR_PW, w.ctr.get() + CTR_CUT2D, k};
  // Sharded level: every rank holds the whole move set (the
  // exchanges gathered it), but walks only the rows it owns; the doubled cut
  // delta and the k part-weight deltas are then summed over the ranks by one
  // all-reduce (k + 1 words) and added to the replicated state.
  const bool shard = sh && c.comm;
  if (shard) {
    sh->delta.ensure((size_t)k + 1, c.stream);
    dzero(c, sh->delta.get(), k + 1);
    a.cut2d = sh->delta.get();
    a.pw = sh->delta.get() + 1;
    a.own_lo = sh->lo;
    a.own_hi = sh->hi;
  }
  const SegLists sl = seg_lists(w, true);
  const unsigned grid = grid_for(c, g.n * 32, 256, 4);
  launch(c, "apply_delta", 0.0, [&] {
    if (g.unit_ew) k_apply_delta<true><<<grid, 256, 0, c.stream>>>(a, gv, sl);
    else k_apply_delta<false><<<grid, 256, 0, c.stream>>>(a, gv, sl);
  });
  if (shard) {
    c.comm->allreduce_sum(c, sh->delta.get(), k + 1);
    launch(c, "apply_add_deltas", 16.0 * k, [&] {
      k_add_deltas<<<grid_for(c, k, 256), 256, 0, c.stream>>>(
          sh->delta.get(), k, w.ctr.get() + CTR_PW, w.ctr.get() + CTR_CUT2D);
    });
  }
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
// First bucket whose cumulative eligible weight reaches the deficit.
__global__ void k_rb_scan(const unsigned long long* __restrict__ H,
                          const unsigned long long* __restrict__ Hs, int nb, int rho, int nover,
                          const long long* __restrict__ deficit, int32_t* bstar,
                          long long* cum_before) {
  const int op = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (op < nover) rb_scan_warp(op, H, Hs, nb, rho, deficit, bstar, cum_before);
}

__global__ void k_rb_chunk(RbSel s, const int32_t* __restrict__ rcand,
                           const unsigned long long* __restrict__ cnt_ptr) {
  rb_chunk(s, rcand, cnt_ptr, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
           (int64_t)gridDim.x * blockDim.x);
}

__global__ void k_rb_find(RbSel s, const long long* __restrict__ deficit,
                          const long long* __restrict__ required,
                          const long long* __restrict__ cum_before,
                          const int32_t* __restrict__ opart, int64_t n, int nb, int nover,
                          int32_t* thr) {
  const int op = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (op < nover) rb_find_warp(op, s, deficit, required, cum_before, opart, n, nb, thr);
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

__global__ void __launch_bounds__(1024) k_rb_tail(RbTail a) {
  extern __shared__ unsigned long long sk_dyn[];
  rb_tail(a, sk_dyn);
}

__global__ void k_rb_collect(const int32_t* __restrict__ parts, const int32_t* __restrict__ opidx,
                             const int64_t* __restrict__ offs, TierMap tm, int64_t n,
                             int32_t* lists, RbSegsDev seg, unsigned long long* cnts) {
  rb_collect(parts, opidx, offs, tm, n, lists, seg, cnts,
             blockIdx.x * (int64_t)blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// The whole selection chain of a rebalancing pass in one cooperative launch:
// bucket scan -> crossing-chunk histogram -> crossing element -> select ->
// (block 0) ordered tail. Replaces five dependent launches.
struct RbCoop {
  RbSel s;
  const unsigned long long* H;
  const unsigned long long* Hs;
  int rho;
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
  for (int64_t op = t0 >> 5; op < a.nover; op += nt >> 5)
    rb_scan_warp((int)op, a.H, a.Hs, a.nb, a.rho, a.deficit, const_cast<int32_t*>(a.s.bstar),
                 a.cum_before);
  grid.sync();
  rb_chunk(a.s, a.rcand, a.rcand_cnt, t0, nt);
  grid.sync();
  for (int64_t op = t0 >> 5; op < a.nover; op += nt >> 5)
    rb_find_warp((int)op, a.s, a.deficit, a.required, a.cum_before, a.opart, a.n, a.nb,
                 const_cast<int32_t*>(a.s.thr));
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

// global evicted ids from the gathered keys; in direct mode every evicted
// vertex lacks a valid connection, so its rbest is -1 (remote vertices' rbest
// entries are stale on this rank and are reset here)
__global__ void k_keys_to_ids(const unsigned long long* __restrict__ keys, int64_t L,
                              int32_t* ids, int32_t* rbest) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = (int)(keys[i] & 0xffffffffu);
    ids[i] = v;
    rbest[v] = -1;
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
                    bool strong, Pcg64& rng, RebalanceOut* out, ShardLists* sh) {
  JET_REQUIRE(!sh || (c.comm && out == nullptr), JET_EINTERNAL, "sharded rebalance misuse");
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
  const bool fast = out == nullptr && max_evict <= TAIL_CAP && sh == nullptr;
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
  w.Hs.ensure((size_t)nover * ns, c.stream);
  dzero(c, w.Hs.get(), (size_t)nover * ns);
  w.CH.ensure((size_t)nover * nch, c.stream);
  dzero(c, w.H.get(), (size_t)nover * nb);
  dzero(c, w.CH.get(), (size_t)nover * nch);

  RbSegsDev cseg, mseg;
  for (int t = 0; t < NBINS; ++t) {
    cseg.b[t] = w.seg_base[t];
    mseg.b[t] = w.seg_base[t];
  }
  if (sh) {  // candidates of this rank's block only
    launch(c, "rb_collect", 8.0 * (sh->hi - sh->lo), [&] {
      k_rb_collect_range<<<grid_for(c, sh->hi - sh->lo, 256), 256, 0, c.stream>>>(
          parts, d_opidx, g.offs.get(), g.tm, sh->lo, sh->hi, w.lists.get(), cseg,
          w.ctr.get() + CTR_CAND);
    });
  } else {
    launch(c, "rb_collect", 8.0 * g.n, [&] {
      k_rb_collect<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(parts, d_opidx, g.offs.get(), g.tm,
                                                               g.n, w.lists.get(), cseg,
                                                               w.ctr.get() + CTR_CAND);
    });
  }
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
  ra.Hs = w.Hs.get();
  int32_t* clists[NBINS];
  for (int t = 0; t < NBINS; ++t) clists[t] = w.cand_list(t);
  run_agg<RbOp>(c, g, [&](int) { return ra; }, parts, k, "rb_stats", 16.0, clists,
                w.ctr.get() + CTR_CAND);
  if (sh) {  // global bucket histograms
    c.comm->allreduce_sum(c, w.H.get(), (int64_t)nover * nb);
    c.comm->allreduce_sum(c, w.Hs.get(), (int64_t)nover * ns);
  }

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
    tl.smem_cap = TAIL_CAP;
    tl.gscratch = nullptr;
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
    cp.Hs = w.Hs.get();
    cp.rho = rho;
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
    k_rb_scan<<<(nover + 7) / 8, 256, 0, c.stream>>>(w.H.get(), w.Hs.get(), nb, rho, nover, d_def,
                                                     bstar, w.cum_before.get());
  });
  launch(c, "rb_chunk", 0.0, [&] {
    k_rb_chunk<<<grid_for(c, g.n, 256), 256, 0, c.stream>>>(s, w.rcand.get(), rc);
  });
  if (sh) {
    // crossing chunk from the global chunk histogram; the chunk's element
    // weights are contributed by their owners and summed
    c.comm->allreduce_sum(c, w.CH.get(), (int64_t)nover * nch);
    DBuf<int32_t> fch(nover, c.stream);
    DBuf<long long> fcb(nover, c.stream);
    DBuf<unsigned long long> few((size_t)nover * 32, c.stream);
    launch(c, "rb_find", 8.0 * nover * nch, [&] {
      k_rb_find_a<<<(nover + 7) / 8, 256, 0, c.stream>>>(s, d_def, w.cum_before.get(), d_opart,
                                                         g.n, nb, nover, sh->lo, sh->hi,
                                                         fch.get(), fcb.get(), few.get());
    });
    c.comm->allreduce_sum(c, few.get(), (int64_t)nover * 32);
    launch(c, "rb_find", 8.0 * nover * 32, [&] {
      k_rb_find_b<<<(nover + 7) / 8, 256, 0, c.stream>>>(s, d_def, d_req, nb, nover, fch.get(),
                                                         fcb.get(), few.get(), w.thr.get());
    });
  } else {
    launch(c, "rb_find", 8.0 * nover * nch, [&] {
      k_rb_find<<<(nover + 7) / 8, 256, 0, c.stream>>>(s, d_def, d_req, w.cum_before.get(),
                                                       d_opart, g.n, nb, nover, w.thr.get());
    });
  }
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
  if (sh) {
    // direct moves (evicted vertices with a valid connection) of every rank
    share_moves(c, w, g, *sh);
    // the evicted sets of every rank, as sort keys
    w.keys.ensure((size_t)g.n + 1, c.stream);
    w.keys_alt.ensure((size_t)g.n + 1, c.stream);
    if (L)
      launch(c, "rb_keys", 16.0 * L, [&] {
        k_rb_keys<<<grid_for(c, L, 256), 256, 0, c.stream>>>(w.evict.get(), L, parts, d_opidx,
                                                             w.rkey.get(), nb, w.keys.get());
      });
    std::vector<int64_t> counts;
    c.comm->allgatherv(c, w.keys.get(), L * 8, sh->recv, counts);
    int64_t tot = 0;
    for (int64_t b : counts) tot += b;
    L = tot / 8;
    if (L)
      CK(cudaMemcpyAsync(w.keys.get(), sh->recv.get(), (size_t)L * 8, cudaMemcpyDeviceToDevice,
                         c.stream));
    if (L == 0) return true;
    launch(c, "rb_evict_ids", 8.0 * L, [&] {
      k_keys_to_ids<<<grid_for(c, L, 256), 256, 0, c.stream>>>(w.keys.get(), L, w.evict.get(),
                                                               w.rbest.get());
    });
  }
  if (L == 0) {
    if (out) {
      out->v->clear();
      out->dest->clear();
      out->gain->clear();
    }
    return true;
  }
  if (!sh)
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
