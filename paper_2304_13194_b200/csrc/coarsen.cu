// coarsen.cu — heavy-edge + two-hop matching and CSR contraction.
//
// match_vertices (coarsen.py:47-107) is sequential in the reference: phase 1
// resolves the proposal snapshot with an ascending-id scan, phase 2 walks
// (centre, vertex) pairs in lexicographic order. Both are reproduced exactly
// by parallel rounds:
//   phase 1: a proposal edge (v -> u) is accepted iff its proposer id v is
//            the minimum over all live proposal edges touching v or u
//            (greedy matching in a fixed priority order == local-minimum
//            rounds);
//   phase 2: a centre is processed once it is the smallest unprocessed centre
//            of every still-unmatched leftover it holds; centres holding at
//            most one unmatched leftover can never pair anything and retire.
// contract (coarsen.py:110-138): coarse ids ascending by lowest member,
// rows merged per coarse vertex, sorted by neighbour and de-duplicated with
// summed weights, self loops dropped.
#include "coarsen.cuh"
#include "small_ops.cuh"
#include "comm.cuh"
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/block/block_radix_sort.cuh>
#include <cub/iterator/counting_input_iterator.cuh>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <climits>

namespace jet {

constexpr int INF32 = 0x7f7f7f7f;  // memset(0x7f) pattern, > any vertex id

__device__ __forceinline__ unsigned long long vload(const unsigned long long* p) {
  return *reinterpret_cast<const volatile unsigned long long*>(p);
}

// grid barrier; a one-block grid needs only __syncthreads (which also
// orders global memory within the block) -- the grid protocol costs ~1.5 us
__device__ __forceinline__ void grid_or_block_sync(cg::grid_group& grid) {
  if (gridDim.x == 1) __syncthreads();
  else grid.sync();
}

static int coop_blocks(Ctx& c, const void* kern, int block) {
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, block, 0));
  JET_REQUIRE(per_sm >= 1, JET_EINTERNAL, "cooperative kernel does not fit on an SM");
  return per_sm * c.num_sms;
}

// ---------------------------------------------------------------------------
// Phase 1: proposals. score = (w, -u) maximised over free neighbours
// (coarsen.py:68-73).
template <int G, bool UNIT>
__global__ void __launch_bounds__(256)
    k_propose(GView g, const int32_t* __restrict__ list, int64_t cnt,
              const int32_t* __restrict__ partner, int32_t* prop, int32_t* elist,
              unsigned long long* ecnt) {
  // same warp-owns-32-rows batching as the refinement sweeps (refine.cu)
  constexpr int RPS = 32 / G;
  constexpr int U = G >= 8 ? 8 : G;
  const unsigned gm = group_mask<G>();
  const int lane = threadIdx.x & 31, gl = lane & (G - 1), grp = lane / G;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = w0 * 32; base < cnt; base += nw * 32) {
    const int64_t idx = base + lane;
    int v = 0, deg = 0;
    bool live = false;
    int64_t beg = 0;
    if (idx < cnt) {
      v = list ? list[idx] : (int)idx;
      live = partner[v] < 0;
      if (live) {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
      }
    }
    unsigned long long mine = 0;
#pragma unroll
    for (int s0 = 0; s0 < G; s0 += U) {
      int uu[U], ww[U], fr[U];
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
      for (int q = 0; q < U; ++q) fr[q] = uu[q] >= 0 ? partner[uu[q]] : 0;
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int st = s0 + q;
        // heaviest free neighbour, ties -> lowest id: two REDUX reductions
        const bool ok = uu[q] >= 0 && fr[q] < 0;
        const unsigned mw = __reduce_max_sync(gm, ok ? (unsigned)ww[q] : 0u);
        const unsigned mu = __reduce_min_sync(gm, (ok && (unsigned)ww[q] == mw) ? (unsigned)uu[q]
                                                                                : 0xffffffffu);
        const int src = ((lane - st * RPS) & (RPS - 1)) * G;
        const unsigned dmw = __shfl_sync(0xffffffffu, mw, src);
        const unsigned dmu = __shfl_sync(0xffffffffu, mu, src);
        if (lane / RPS == st)
          mine = dmw ? (((unsigned long long)dmw << 32) | (0xffffffffu - dmu)) : 0ull;
      }
    }
    int u = -1;
    if (live) {
      u = mine ? (int)(0xffffffffu - (unsigned)(mine & 0xffffffffu)) : -1;
      prop[v] = u;
    }
    warp_append(u >= 0, v, elist, ecnt);
  }
}

// Rows longer than 32 (tiers 4/5): one warp per row, looping over the row.
template <bool UNIT>
__global__ void __launch_bounds__(256)
    k_propose_long(GView g, const int32_t* __restrict__ list, int64_t cnt,
                   const int32_t* __restrict__ partner, int32_t* prop, int32_t* elist,
                   unsigned long long* ecnt) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < cnt; i += nw) {
    const int v = list ? list[i] : (int)i;
    if (partner[v] >= 0) continue;
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    unsigned long long best = 0;
    for (int64_t j = b + lane; j < e; j += 32) {
      const int u = g.adj[j];
      if (partner[u] < 0) {
        const unsigned long long w = UNIT ? 1ull : (unsigned long long)g.ew[j];
        const unsigned long long key = (w << 32) | (unsigned)(0xffffffffu - (unsigned)u);
        best = key > best ? key : best;
      }
    }
    best = gmax<32>(best, 0xffffffffu);
    if (lane == 0) {
      const int u = best ? (int)(0xffffffffu - (unsigned)(best & 0xffffffffu)) : -1;
      prop[v] = u;
      warp_append(u >= 0, v, elist, ecnt);
    }
  }
}

// One resolution round, part A: reset last round's minima, test liveness,
// scatter proposer ids to both endpoints with atomicMin.
__global__ void k_round_a(const int32_t* __restrict__ prop, const int32_t* __restrict__ partner,
                          const int32_t* __restrict__ in, const unsigned long long* __restrict__ in_cnt,
                          int32_t* mn_cur, int32_t* mn_prev, int32_t* out,
                          unsigned long long* out_cnt) {
  const int64_t cnt = (int64_t)*in_cnt;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t lim = (cnt + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lim; i += stride) {
    bool alive = false;
    int v = 0;
    if (i < cnt) {
      v = in[i];
      const int u = prop[v];
      mn_prev[v] = INF32;
      mn_prev[u] = INF32;
      alive = partner[v] < 0 && partner[u] < 0;
      if (alive) {
        atomicMin(&mn_cur[v], v);
        atomicMin(&mn_cur[u], v);
      }
    }
    warp_append(alive, v, out, out_cnt);
  }
}

// Part B: accept edges that are the minimum at both endpoints.
__global__ void k_round_b(const int32_t* __restrict__ prop, int32_t* partner,
                          const int32_t* __restrict__ list,
                          const unsigned long long* __restrict__ cnt_ptr,
                          const int32_t* __restrict__ mn_cur, unsigned long long* reset_cnt) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *reset_cnt = 0;
  const int64_t cnt = (int64_t)*cnt_ptr;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt; i += stride) {
    const int v = list[i];
    const int u = prop[v];
    if (mn_cur[v] == v && mn_cur[u] == v) {
      partner[v] = u;
      partner[u] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// Phase 2 (two-hop): members of each centre are its leftover neighbours in
// ascending id order.
__global__ void k_leftover_deg(const int32_t* __restrict__ left, int64_t nl,
                               const int64_t* __restrict__ offs, int64_t* deg) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl; i += stride) {
    const int v = left[i];
    deg[i] = offs[v + 1] - offs[v];
  }
}

__global__ void k_leftover_pairs(const int32_t* __restrict__ left, int64_t nl,
                                 GView g, const int64_t* __restrict__ poff,
                                 int32_t* keys, int32_t* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nl; i += ws) {
    const int v = left[i];
    const int64_t b = g.offs[v], e = g.offs[v + 1], o = poff[i];
    for (int64_t j = b + lane; j < e; j += 32) {
      keys[o + (j - b)] = g.adj[j];
      vals[o + (j - b)] = v;
    }
  }
}

struct TwoHop {
  int32_t* partner;
  const int32_t* centres;   // centre vertex id per centre index
  const int64_t* coff;      // member offsets per centre index (nc + 1)
  const int32_t* members;   // leftover ids, ascending within each centre
  uint8_t* cact;            // per vertex id: 1 while the centre is active
  uint8_t* ready;           // per centre index
  int32_t* minc;            // per vertex id (leftovers only)
  int64_t nc;
  unsigned long long* stats;  // optional: rounds
};

// Retire centres with <= 1 unmatched member; count the remaining active.
__device__ void th_retire(const TwoHop& t, unsigned long long* active, int64_t w0, int64_t ws) {
  const int lane = threadIdx.x & 31;
  long long act = 0;
  for (int64_t ci = w0; ci < t.nc; ci += ws) {
    const int c = t.centres[ci];
    if (!t.cact[c]) continue;
    const int64_t b = t.coff[ci], e = t.coff[ci + 1];
    int un = 0;
    for (int64_t j0 = b; j0 < e && un < 2; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool u = j < e && t.partner[t.members[j]] < 0;
      un += __popc(__ballot_sync(0xffffffffu, u));
    }
    if (un <= 1) {
      if (lane == 0) t.cact[c] = 0;
    } else if (lane == 0) {
      act++;
    }
  }
  if (lane == 0 && act) atomicAdd(active, (unsigned long long)act);
}

// minc[v] = smallest active centre adjacent to unmatched leftover v.
__device__ void th_minc(const TwoHop& t, const GView& g, const int32_t* __restrict__ left,
                        int64_t nl, int64_t w0, int64_t ws) {
  const int lane = threadIdx.x & 31;
  for (int64_t i = w0; i < nl; i += ws) {
    const int v = left[i];
    if (t.partner[v] >= 0) continue;
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    int m = INF32;
    for (int64_t j = b + lane; j < e; j += 32) {
      const int c = g.adj[j];
      if (t.cact[c] && c < m) m = c;
    }
    m = gmin<32>(m, 0xffffffffu);
    if (lane == 0) t.minc[v] = m;
  }
}

__device__ void th_ready(const TwoHop& t, int64_t w0, int64_t ws) {
  const int lane = threadIdx.x & 31;
  for (int64_t ci = w0; ci < t.nc; ci += ws) {
    const int c = t.centres[ci];
    bool ok = t.cact[c] != 0;
    if (ok) {
      const int64_t b = t.coff[ci], e = t.coff[ci + 1];
      for (int64_t j0 = b; j0 < e && ok; j0 += 32) {
        const int64_t j = j0 + lane;
        bool bad = false;
        if (j < e) {
          const int v = t.members[j];
          bad = t.partner[v] < 0 && t.minc[v] != c;
        }
        ok = !__any_sync(0xffffffffu, bad);
      }
    }
    if (lane == 0) t.ready[ci] = ok;
  }
}

// Ready centres pair their unmatched members consecutively (coarsen.py:95-103).
__device__ void th_pair(const TwoHop& t, int64_t w0, int64_t ws) {
  const int lane = threadIdx.x & 31;
  for (int64_t ci = w0; ci < t.nc; ci += ws) {
    if (!t.ready[ci]) continue;
    const int c = t.centres[ci];
    const int64_t b = t.coff[ci], e = t.coff[ci + 1];
    int pending = -1;
    for (int64_t j0 = b; j0 < e; j0 += 32) {
      const int64_t j = j0 + lane;
      int v = -1;
      bool un = false;
      if (j < e) {
        v = t.members[j];
        un = t.partner[v] < 0;
      }
      const unsigned um = __ballot_sync(0xffffffffu, un);
      const int off = pending >= 0 ? 1 : 0;
      const unsigned below = um & lanemask_lt();
      const int pos = __popc(below) + off;  // position in (pending, unmatched...)
      int mate = -1;
      const int src = below ? 31 - __clz(below) : lane;
      const int vprev = __shfl_sync(0xffffffffu, v, src);
      if (un && (pos & 1)) mate = below ? vprev : pending;
      __syncwarp();
      if (mate >= 0) {
        t.partner[v] = mate;
        t.partner[mate] = v;
      }
      const int total = __popc(um) + off;
      if (total & 1) {
        const int last = um ? 31 - __clz(um) : -1;
        const int lv = __shfl_sync(0xffffffffu, v, last >= 0 ? last : 0);
        pending = last >= 0 ? lv : pending;
      } else {
        pending = -1;
      }
      __syncwarp();
    }
    if (lane == 0) t.cact[c] = 0;
  }
}

// All two-hop rounds in one cooperative launch: retire / minc / ready /
// pair, separated by grid-wide barriers, until no active centre remains.
__global__ void __launch_bounds__(1024)
    k_two_hop(TwoHop t, GView g, const int32_t* __restrict__ left, int64_t nl,
              unsigned long long* active) {
  cg::grid_group grid = cg::this_grid();
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  while (true) {
    if (t.stats && blockIdx.x == 0 && threadIdx.x == 0) t.stats[0] += 1;
    th_retire(t, active, w0, ws);
    grid_or_block_sync(grid);
    if (vload(active) == 0) return;
    th_minc(t, g, left, nl, w0, ws);
    grid_or_block_sync(grid);
    th_ready(t, w0, ws);
    grid_or_block_sync(grid);
    if (w0 == 0 && (threadIdx.x & 31) == 0) *active = 0;
    th_pair(t, w0, ws);
    grid_or_block_sync(grid);
  }
}

// ---------------------------------------------------------------------------
// Two-hop by frontier (same rule, work-efficient). Counters per centre:
// ucnt = unmatched members, good = unmatched members whose smallest active
// centre (minc) is this centre. A centre retires when ucnt <= 1 and is
// processed (pairs its unmatched members consecutively) when good == ucnt.
// Each leftover keeps a cursor into its (sorted) adjacency at its minc. A
// round decides the candidate centres, then updates the counters touched by
// the newly matched members and advances the leftovers whose minc retired;
// only centres whose counters changed are candidates next round.
struct TwoHopF {
  int32_t* partner;
  const int32_t* centres;
  const int64_t* coff;
  const int32_t* members;
  uint8_t* cact;        // per vertex id
  int32_t* cidx;        // vertex id -> centre index
  int32_t* ucnt;        // per centre
  int32_t* good;        // per centre
  int32_t* cflag;       // per centre: round it was queued in
  int32_t* lcur;        // per vertex id (leftovers): offset of minc in its row, or -1
  int32_t* cand;        // 2 x nc
  int32_t* dlist;       // deactivated centres of the round, <= nc
  int32_t* mlist;       // members matched in the round, <= nl
  unsigned long long* cnt;  // [0,1] candidates, [2,3] deactivated, [4,5] matched (by round
                            // parity), [6] rounds
  int64_t nc;
};

__device__ __forceinline__ void thf_queue(const TwoHopF& t, int ci, int round, int32_t* out,
                                          unsigned long long* ocnt) {
  // aggregated over the lanes queueing together (one hot counter)
  warp_append(atomicExch(&t.cflag[ci], round) != round, ci, out, ocnt);
}

__global__ void __launch_bounds__(1024)
    k_two_hop_frontier(TwoHopF t, GView g, const int32_t* __restrict__ left, int64_t nl) {
  cg::grid_group grid = cg::this_grid();
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = t0 >> 5, nw = nt >> 5;
  for (int64_t ci = t0; ci < t.nc; ci += nt) {
    t.ucnt[ci] = (int32_t)(t.coff[ci + 1] - t.coff[ci]);
    t.good[ci] = 0;
    t.cidx[t.centres[ci]] = (int32_t)ci;
  }
  grid_or_block_sync(grid);
  // every neighbour of a leftover is a centre, all active: minc = first entry
  for (int64_t i = t0; i < nl; i += nt) {
    const int v = left[i];
    const int64_t b = g.offs[v];
    if (g.offs[v + 1] > b) {
      t.lcur[v] = 0;
      atomicAdd(&t.good[t.cidx[g.adj[b]]], 1);
    } else {
      t.lcur[v] = -1;
    }
  }
  grid_or_block_sync(grid);
  int cur = 0;
  for (int round = 1;; ++round) {
    const bool all = round == 1;
    const int64_t C = all ? t.nc : (int64_t)vload(t.cnt + cur);
    if (C == 0) break;
    const int32_t* cin = t.cand + (size_t)cur * t.nc;
    int32_t* cout = t.cand + (size_t)(cur ^ 1) * t.nc;
    const int par = round & 1;
    // (1) decide the candidates: retire, or pair (a warp per centre)
    for (int64_t k = w0; k < C; k += nw) {
      const int ci = all ? (int)k : cin[k];
      const int c = t.centres[ci];
      if (!t.cact[c]) continue;
      const int u = t.ucnt[ci];
      if (u <= 1 || t.good[ci] == u) {
        if (u > 1) {
          // pair consecutive unmatched members (coarsen.py:95-103)
          const int64_t b = t.coff[ci], e = t.coff[ci + 1];
          int pending = -1;
          for (int64_t j0 = b; j0 < e; j0 += 32) {
            const int64_t j = j0 + lane;
            int v = -1;
            bool un = false;
            if (j < e) {
              v = t.members[j];
              un = t.partner[v] < 0;
            }
            const unsigned um = __ballot_sync(0xffffffffu, un);
            const int off = pending >= 0 ? 1 : 0;
            const unsigned below = um & lanemask_lt();
            const int pos = __popc(below) + off;
            int mate = -1;
            const int src = below ? 31 - __clz(below) : lane;
            const int vprev = __shfl_sync(0xffffffffu, v, src);
            if (un && (pos & 1)) mate = below ? vprev : pending;
            __syncwarp();
            if (mate >= 0) {
              t.partner[v] = mate;
              t.partner[mate] = v;
            }
            warp_append(mate >= 0, v, t.mlist, t.cnt + 4 + par);
            warp_append(mate >= 0, mate, t.mlist, t.cnt + 4 + par);
            const int total = __popc(um) + off;
            if (total & 1) {
              const int last = um ? 31 - __clz(um) : -1;
              const int lv = __shfl_sync(0xffffffffu, v, last >= 0 ? last : 0);
              pending = last >= 0 ? lv : pending;
            } else {
              pending = -1;
            }
            __syncwarp();
          }
        }
        if (lane == 0) {
          t.cact[c] = 0;
          t.dlist[atomicAdd(t.cnt + 2 + par, 1ull)] = ci;
        }
      }
    }
    if (t0 == 0) {
      t.cnt[cur ^ 1] = 0;
      t.cnt[2 + (par ^ 1)] = 0;  // read by the previous round's phase 2, done
      t.cnt[4 + (par ^ 1)] = 0;
    }
    grid_or_block_sync(grid);
    // (2a) newly matched members leave every active centre's counts
    const int64_t M = (int64_t)vload(t.cnt + 4 + par);
    for (int64_t k = w0; k < M; k += nw) {
      const int v = t.mlist[k];
      const int64_t b = g.offs[v], e = g.offs[v + 1];
      const int mc = t.lcur[v] >= 0 ? g.adj[b + t.lcur[v]] : -1;
      for (int64_t j = b + lane; j < e; j += 32) {
        const int c = g.adj[j];
        if (!t.cact[c]) continue;
        const int ci = t.cidx[c];
        atomicSub(&t.ucnt[ci], 1);
        if (c == mc) atomicSub(&t.good[ci], 1);
        thf_queue(t, ci, round, cout, t.cnt + (cur ^ 1));
      }
    }
    // (2b) unmatched members whose minc just retired move to their next
    // active centre (a warp per retired centre; one thread per member)
    const int64_t D = (int64_t)vload(t.cnt + 2 + par);
    for (int64_t k = w0; k < D; k += nw) {
      const int ci = t.dlist[k];
      const int c = t.centres[ci];
      const int64_t b = t.coff[ci], e = t.coff[ci + 1];
      for (int64_t j = b + lane; j < e; j += 32) {
        const int u = t.members[j];
        if (t.partner[u] >= 0 || t.lcur[u] < 0) continue;
        const int64_t rb = g.offs[u], re = g.offs[u + 1];
        if (g.adj[rb + t.lcur[u]] != c) continue;
        int64_t q = rb + t.lcur[u] + 1;
        while (q < re && !t.cact[g.adj[q]]) ++q;
        if (q < re) {
          t.lcur[u] = (int32_t)(q - rb);
          const int ci2 = t.cidx[g.adj[q]];
          atomicAdd(&t.good[ci2], 1);
          thf_queue(t, ci2, round, cout, t.cnt + (cur ^ 1));
        } else {
          t.lcur[u] = -1;
        }
      }
    }
    if (t0 == 0) t.cnt[6] += 1;
    cur ^= 1;
    grid_or_block_sync(grid);
  }
}

__global__ void k_singletons(int32_t* partner, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (partner[v] < 0) partner[v] = (int32_t)v;
}

__global__ void k_fill(int32_t* p, int64_t n, int32_t val) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) p[i] = val;
}

struct IsFree {
  const int32_t* partner;
  __device__ __forceinline__ bool operator()(const int32_t& v) const { return partner[v] < 0; }
};

__global__ void k_th_mark(const int32_t* __restrict__ cs, int64_t nc, uint8_t* cact) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nc; i += stride) cact[cs[i]] = 1;
}
void th_mark(Ctx& c, const int32_t* cs, int64_t nc, uint8_t* cact) {
  launch(c, "th_mark", 5.0 * nc, [&] {
    k_th_mark<<<grid_for(c, nc, 256), 256, 0, c.stream>>>(cs, nc, cact);
  });
}

static int bits_for(int64_t x) {
  int b = 1;
  while ((1LL << b) <= x) ++b;
  return b;
}

static void two_hop(Ctx& c, const DGraph& g, int32_t* partner) {
  const int64_t n = g.n;
  int32_t* left_p = c.scratch<int32_t>(13, n);
  DBuf<int64_t> nsel(1, c.stream);
  {
    cub::CountingInputIterator<int32_t> it(0);
    IsFree op{partner};
    if (!small_select(c, "th_leftovers", op, n, left_p, nsel.get())) {
      size_t tmp = 0;
      CK(cub::DeviceSelect::If(nullptr, tmp, it, left_p, nsel.get(), (int)n, op, c.stream));
      void* p = c.cub_scratch(tmp);
      launch(c, "th_leftovers", 8.0 * n, [&] {
        CK(cub::DeviceSelect::If(p, tmp, it, left_p, nsel.get(), (int)n, op, c.stream));
      });
    }
  }
  int64_t nl = 0;
  d2h(c, &nl, nsel.get(), 1);
  c.sync();
  if (nl == 0) return;
  DBuf<int64_t> deg(nl + 1, c.stream), poff(nl + 1, c.stream);
  dzero(c, deg.get() + nl, 1);
  launch(c, "th_deg", 20.0 * nl, [&] {
    k_leftover_deg<<<grid_for(c, nl, 256), 256, 0, c.stream>>>(left_p, nl, g.offs.get(), deg.get());
  });
  if (!small_exclusive_sum(c, "th_scan", deg.get(), poff.get(), (int64_t)(nl + 1)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.get(), poff.get(), (int)(nl + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "th_scan", 16.0 * nl, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, deg.get(), poff.get(), (int)(nl + 1), c.stream));
    });
  }
  int64_t np = 0;
  d2h(c, &np, poff.get() + nl, 1);
  c.sync();
  if (np == 0) return;
  const GView gv = view(g);
  int32_t* k0_p = c.scratch<int32_t>(14, np);
  int32_t* v0_p = c.scratch<int32_t>(15, np);
  int32_t* k1_p = c.scratch<int32_t>(16, np);
  int32_t* v1_p = c.scratch<int32_t>(17, np);
  launch(c, "th_pairs", 16.0 * np, [&] {
    k_leftover_pairs<<<grid_for(c, nl * 32, 256), 256, 0, c.stream>>>(left_p, nl, gv, poff.get(),
                                                                     k0_p, v0_p);
  });
  {
    size_t tmp = 0;
    const int eb = bits_for(n);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0_p, k1_p, v0_p, v1_p, (int)np, 0,
                                       eb, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "th_sort", 32.0 * np, [&] {
      CK(cub::DeviceRadixSort::SortPairs(p, tmp, k0_p, k1_p, v0_p, v1_p, (int)np, 0, eb,
                                         c.stream));
    });
  }
  // centres = runs of equal keys
  DBuf<int32_t> centres(np, c.stream);
  DBuf<int64_t> ccnt(np + 1, c.stream), coff(np + 1, c.stream);
  DBuf<int64_t> nruns(1, c.stream);
  {
    size_t tmp = 0;
    CK(cub::DeviceRunLengthEncode::Encode(nullptr, tmp, k1_p, centres.get(), ccnt.get(), nruns.get(),
                                          (int)np, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "th_rle", 12.0 * np, [&] {
      CK(cub::DeviceRunLengthEncode::Encode(p, tmp, k1_p, centres.get(), ccnt.get(), nruns.get(),
                                            (int)np, c.stream));
    });
  }
  int64_t nc = 0;
  d2h(c, &nc, nruns.get(), 1);
  c.sync();
  dzero(c, ccnt.get() + nc, 1);
  if (!small_exclusive_sum(c, "th_scan", ccnt.get(), coff.get(), (int64_t)(nc + 1)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, ccnt.get(), coff.get(), (int)(nc + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "th_scan", 16.0 * nc, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, ccnt.get(), coff.get(), (int)(nc + 1), c.stream));
    });
  }
  uint8_t* cact_p = c.scratch<uint8_t>(18, n);
  uint8_t* ready_p = c.scratch<uint8_t>(19, nc);
  int32_t* minc_p = c.scratch<int32_t>(20, n);
  dzero(c, cact_p, n);
  th_mark(c, centres.get(), nc, cact_p);
  static const bool mstats = getenv("JET_MATCH_STATS") && getenv("JET_MATCH_STATS")[0] == '1';
  static const bool old_th = getenv("JET_TWO_HOP_ROUNDS") && getenv("JET_TWO_HOP_ROUNDS")[0] == '1';
  // few leftovers (meshes): the full-pass rounds are cheaper than the
  // frontier bookkeeping; many (skewed graphs: 10^5-10^6 leftovers under hub
  // centres, hundreds of rounds) -> frontier
  static const int64_t th_frontier_min = [] {
    const char* e = getenv("JET_TH_FRONTIER_MIN");
    return e ? (int64_t)atoll(e) : (int64_t)16384;
  }();
  if (!old_th && nl > th_frontier_min) {
    int32_t* ints = c.scratch<int32_t>(25, 2 * n + 5 * nc + nl + 64);
    unsigned long long* tc = c.scratch<unsigned long long>(26, 8);
    dzero(c, tc, 8);
    int32_t *cidx = ints, *lcur = ints + n, *ucnt = ints + 2 * n, *good = ucnt + nc,
            *cflag = good + nc, *cand = cflag + nc, *dlist = cand + 2 * nc, *mlist = dlist + nc;
    dzero(c, cflag, nc);
    TwoHopF f{partner, centres.get(), coff.get(), v1_p, cact_p, cidx, ucnt, good, cflag, lcur,
              cand, dlist, mlist, tc, nc};
    // a warp per centre in the first round
    const int blocks = std::min<int64_t>(coop_blocks(c, (const void*)k_two_hop_frontier, 1024),
                                         std::max<int64_t>(1, (std::max(nc, nl) + 31) / 32));
    const int32_t* lp = left_p;
    void* args[] = {&f, (void*)&gv, (void*)&lp, (void*)&nl};
    launch(c, "two_hop", 0.0, [&] {
      CK(cudaLaunchCooperativeKernel((const void*)k_two_hop_frontier, dim3(blocks), dim3(1024),
                                     args, 0, c.stream));
    });
    if (mstats) {
      unsigned long long r[8];
      d2h(c, r, tc, 8);
      c.sync();
      fprintf(stderr, "TWOHOPF n=%lld leftovers=%lld centres=%lld blocks=%d rounds=%llu\n",
              (long long)n, (long long)nl, (long long)nc, blocks, r[6]);
    }
    return;
  }
  DBuf<unsigned long long> thst(1, c.stream);
  dzero(c, thst.get(), 1);
  TwoHop t{partner, centres.get(), coff.get(), v1_p, cact_p, ready_p, minc_p, nc,
           mstats ? thst.get() : nullptr};
  DBuf<unsigned long long> act(1, c.stream);
  dzero(c, act.get(), 1);
  const int64_t want = std::max<int64_t>(nc, nl);
  const int blocks = std::min<int64_t>(coop_blocks(c, (const void*)k_two_hop, 1024),
                                       std::max<int64_t>(1, (want * 32 + 1023) / 1024));
  const int32_t* lp = left_p;
  unsigned long long* ap = act.get();
  void* args[] = {&t, (void*)&gv, (void*)&lp, (void*)&nl, (void*)&ap};
  launch(c, "two_hop", 0.0, [&] {
    CK(cudaLaunchCooperativeKernel((const void*)k_two_hop, dim3(blocks), dim3(1024), args, 0,
                                   c.stream));
  });
  if (mstats) {
    unsigned long long r = 0;
    int64_t mx = 0;
    d2h(c, &r, thst.get(), 1);
    c.sync();
    std::vector<int64_t> hc(nc + 1);
    d2h(c, hc.data(), coff.get(), nc + 1);
    c.sync();
    for (int64_t i = 0; i < nc; ++i) mx = std::max(mx, hc[i + 1] - hc[i]);
    fprintf(stderr, "TWOHOP n=%lld leftovers=%lld pairs=%lld centres=%lld max_members=%lld blocks=%d rounds=%llu\n",
            (long long)n, (long long)nl, (long long)np, (long long)nc, (long long)mx, blocks, r);
  }
}

// ---------------------------------------------------------------------------
// All resolution rounds of one proposal snapshot in a single cooperative
// launch: grid-wide rounds while many edges are live, then block 0 finishes
// the long tail of short chains alone (SURVEY §7 hard part 1: up to ~N/2
// rounds on lattices). Lists/counters ping-pong as in the two-kernel form.
struct Resolve {
  const int32_t* prop;
  int32_t* partner;
  int32_t* lists;  // 2 x n
  unsigned long long* cnt;  // 2
  int32_t* mn;     // 2 x n
  int64_t n;
  unsigned long long small;
  unsigned long long* stats;  // optional (JET_MATCH_STATS): rounds, tail edges, tail steps
};

__device__ void resolve_a(const Resolve& R, int in, int out, int64_t t0, int64_t nt) {
  const int64_t cnt = (int64_t)vload(R.cnt + in);
  const int32_t* lin = R.lists + (size_t)in * R.n;
  int32_t* lout = R.lists + (size_t)out * R.n;
  int32_t* mcur = R.mn + (size_t)out * R.n;
  int32_t* mprev = R.mn + (size_t)in * R.n;
  // block-uniform trip count: the surviving edges are appended per block
  const int64_t lim = (cnt + blockDim.x - 1) / blockDim.x * blockDim.x;
  for (int64_t i = t0; i < lim; i += nt) {
    bool alive = false;
    int v = 0;
    if (i < cnt) {
      v = lin[i];
      const int u = R.prop[v];
      mprev[v] = INF32;
      mprev[u] = INF32;
      alive = R.partner[v] < 0 && R.partner[u] < 0;
      if (alive) {
        atomicMin(&mcur[v], v);
        atomicMin(&mcur[u], v);
      }
    }
    block_append(alive, v, lout, R.cnt + out);
  }
}

__device__ void resolve_b(const Resolve& R, int in, int out, int64_t t0, int64_t nt) {
  if (t0 == 0) R.cnt[in] = 0;
  const int64_t cnt = (int64_t)vload(R.cnt + out);
  const int32_t* lst = R.lists + (size_t)out * R.n;
  const int32_t* mcur = R.mn + (size_t)out * R.n;
  for (int64_t i = t0; i < cnt; i += nt) {
    const int v = lst[i];
    const int u = R.prop[v];
    if (mcur[v] == v && mcur[u] == v) {
      R.partner[v] = u;
      R.partner[u] = v;
    }
  }
}

// Shared-memory tail: at most RES_TAIL live edges, their endpoints hashed to
// local slots; the remaining rounds run on chip (one block).
constexpr int RES_TAIL = 2048;
constexpr int RES_HASH = 8192;  // >= 2 endpoints per edge, load <= 1/2
struct ResTailSmem {
  int32_t key[RES_HASH];
  int32_t mn[RES_HASH];
  uint8_t fr[RES_HASH];
  int32_t ev[RES_TAIL], eu[RES_TAIL], evid[RES_TAIL], euid[RES_TAIL];
  int16_t alive[2][RES_TAIL];
  int nalive[2];
};

__device__ __forceinline__ int res_slot(ResTailSmem& S, int v) {
  unsigned h = ((unsigned)v * 2654435761u) & (RES_HASH - 1);
  while (true) {
    const int prev = atomicCAS(&S.key[h], -1, v);
    if (prev == -1 || prev == v) return (int)h;
    h = (h + 1) & (RES_HASH - 1);
  }
}

__device__ void resolve_tail(const Resolve& R, int in, ResTailSmem& S) {
  const long long c0 = clock64();
  int tail_rounds = 0;
  const int L = (int)vload(R.cnt + in);
  const int32_t* lin = R.lists + (size_t)in * R.n;
  // the global minima written for these edges in the previous grid round
  // were already reset by that round's successor; keep the global mn clean
  for (int i = threadIdx.x; i < RES_HASH; i += blockDim.x) {
    S.key[i] = -1;
    S.mn[i] = INF32;
  }
  if (threadIdx.x == 0) S.nalive[0] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int v = lin[i];
    const int u = R.prop[v];
    S.ev[i] = res_slot(S, v);
    S.eu[i] = res_slot(S, u);
    S.evid[i] = v;
    S.euid[i] = u;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < RES_HASH; i += blockDim.x) {
    const int v = S.key[i];
    S.fr[i] = v >= 0 && R.partner[v] < 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    if (S.fr[S.ev[i]] && S.fr[S.eu[i]]) S.alive[0][atomicAdd(&S.nalive[0], 1)] = (int16_t)i;
  }
  __syncthreads();
  int cur = 0;
  while (S.nalive[cur] > 0) {
    const int na = S.nalive[cur];
    for (int q = threadIdx.x; q < na; q += blockDim.x) {
      const int i = S.alive[cur][q];
      atomicMin(&S.mn[S.ev[i]], S.evid[i]);
      atomicMin(&S.mn[S.eu[i]], S.evid[i]);
    }
    if (threadIdx.x == 0) S.nalive[cur ^ 1] = 0;
    __syncthreads();
    for (int q = threadIdx.x; q < na; q += blockDim.x) {
      const int i = S.alive[cur][q];
      const int v = S.evid[i];
      if (S.mn[S.ev[i]] == v && S.mn[S.eu[i]] == v) {
        S.fr[S.ev[i]] = 0;
        S.fr[S.eu[i]] = 0;
        R.partner[v] = S.euid[i];
        R.partner[S.euid[i]] = v;
      }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < na; q += blockDim.x) {
      const int i = S.alive[cur][q];
      S.mn[S.ev[i]] = INF32;
      S.mn[S.eu[i]] = INF32;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < na; q += blockDim.x) {
      const int i = S.alive[cur][q];
      if (S.fr[S.ev[i]] && S.fr[S.eu[i]])
        S.alive[cur ^ 1][atomicAdd(&S.nalive[cur ^ 1], 1)] = (int16_t)i;
    }
    __syncthreads();
    cur ^= 1;
    ++tail_rounds;
  }
  if (threadIdx.x == 0) R.cnt[in] = 0;
  if (R.stats && threadIdx.x == 0) {
    R.stats[2] += (unsigned long long)(clock64() - c0);
    R.stats[3] += (unsigned long long)tail_rounds;
  }
}

__global__ void __launch_bounds__(1024) k_resolve(Resolve R) {
  extern __shared__ unsigned char res_smem[];
  cg::grid_group grid = cg::this_grid();
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  int r = 1;
  while (true) {
    const int in = (r - 1) & 1, out = r & 1;
    const unsigned long long live = vload(R.cnt + in);
    if (live == 0) return;
    if (live <= R.small) break;
    resolve_a(R, in, out, t0, nt);
    grid_or_block_sync(grid);
    resolve_b(R, in, out, t0, nt);
    grid_or_block_sync(grid);
    ++r;
  }
  if (blockIdx.x != 0) return;
  if (R.stats && threadIdx.x == 0) {
    R.stats[0] += (unsigned long long)r;
    R.stats[1] += vload(R.cnt + ((r - 1) & 1));
  }
  // live edges of list `in` were last scattered into mn[in]; that buffer was
  // reset by resolve_a of this round only if the round ran, so clear the
  // entries of the list now (they would otherwise leak into a later call)
  const int in = (r - 1) & 1;
  {
    const int L = (int)vload(R.cnt + in);
    const int32_t* lin = R.lists + (size_t)in * R.n;
    int32_t* mprev = R.mn + (size_t)in * R.n;
    for (int i = threadIdx.x; i < L; i += blockDim.x) {
      const int v = lin[i];
      mprev[v] = INF32;
      mprev[R.prop[v]] = INF32;
    }
  }
  __syncthreads();
  resolve_tail(R, in, *reinterpret_cast<ResTailSmem*>(res_smem));
}

// ---------------------------------------------------------------------------
// Phase-1 resolution by frontier (work-efficient, exact). The ascending-id
// scan accepts the proposal edge e_v = (v, P(v)) iff both endpoints are free
// when v's turn comes. An edge is dead once an endpoint is matched; a live
// edge's turn is decided once every lower-id live edge sharing an endpoint
// is decided, i.e. when it is the lowest live edge at both endpoints -- and
// then it is accepted. Each vertex keeps its incident proposal edges sorted
// by id and a head pointer to its lowest live one. A round (1) accepts the
// frontier (pairwise non-adjacent: no conflicts), (2) refreshes the heads of
// the vertices whose head edge died (neighbours of the newly matched ones),
// (3) queues the refreshed heads that are now lowest at both endpoints.
// Rounds follow the dependency depth, each touching only the frontier.
struct Frontier {
  const int32_t* prop;
  int32_t* partner;
  const unsigned long long* inc;  // sorted (endpoint << 32 | edge id)
  const int32_t* ioff;            // n + 1
  int32_t* head;                  // n (index into inc)
  int32_t* qflag;                 // n: round an edge was queued in
  int32_t* aflag;                 // n: round a vertex was refreshed in
  int32_t* fr;                    // 2 x cap
  int32_t* aff;                   // affected vertices of the round, <= n
  unsigned long long* fcnt;       // [0,1] frontier sizes, [2,3] affected (round parity), [4] rounds
  const int32_t* props;           // proposers
  int64_t ne, cap;
};

__device__ __forceinline__ int fr_other(const Frontier& F, int e, int x) {
  return e == x ? F.prop[e] : e;
}

// edge at x's head, or -1
__device__ __forceinline__ int fr_head_edge(const Frontier& F, int x) {
  const int h = F.head[x];
  return h < F.ioff[x + 1] ? (int)(F.inc[h] & 0xffffffffu) : -1;
}

// lowest live edge at unmatched vertex x, scanning from its (possibly stale,
// never overtaking) head; warp-cooperative, result in every lane
__device__ __forceinline__ int fr_first_live(const Frontier& F, int x, int* pos) {
  const int lane = threadIdx.x & 31;
  const int end = F.ioff[x + 1];
  for (int q = F.head[x]; q < end; q += 32) {
    const int j = q + lane;
    int e = -1;
    bool live = false;
    if (j < end) {
      e = (int)(F.inc[j] & 0xffffffffu);
      live = F.partner[fr_other(F, e, x)] < 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, live);
    if (m) {
      const int l = __ffs(m) - 1;
      *pos = q + l;
      return __shfl_sync(0xffffffffu, e, l);
    }
  }
  *pos = end;
  return -1;
}

// thread-level scan for the lowest live edge at unmatched x, at most `lim`
// entries; returns -2 when the limit is hit (the caller defers x to a warp)
__device__ __forceinline__ int fr_first_live_t(const Frontier& F, int x, int lim, int* pos) {
  const int end = F.ioff[x + 1];
  int q = F.head[x];
  for (int s = 0; q < end; ++q, ++s) {
    if (s == lim) return -2;
    const int e = (int)(F.inc[q] & 0xffffffffu);
    if (F.partner[fr_other(F, e, x)] < 0) {
      *pos = q;
      return e;
    }
  }
  *pos = end;
  return -1;
}

constexpr int FR_SHORT = 64;     // entries a thread scans before deferring to a warp
constexpr int FR_DEFER = 2048;   // deferred entries per block and phase

__global__ void __launch_bounds__(1024) k_resolve_frontier(Frontier F) {
  cg::grid_group grid = cg::this_grid();
  __shared__ int s_def[FR_DEFER];
  __shared__ int s_ndef;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  // initial frontier: edges that are lowest at both endpoints (all live)
  for (int64_t i = t0; i < ((F.ne + 31) & ~31LL); i += nt) {
    bool rd = false;
    int v = 0;
    if (i < F.ne) {
      v = F.props[i];
      rd = fr_head_edge(F, v) == v && fr_head_edge(F, F.prop[v]) == v;
    }
    warp_append(rd, v, F.fr, F.fcnt);
  }
  grid_or_block_sync(grid);
  int cur = 0;
  for (int round = 1;; ++round) {
    const int64_t L = (int64_t)vload(F.fcnt + cur);
    if (L == 0) break;
    const int32_t* fin = F.fr + (size_t)cur * F.cap;
    int32_t* fout = F.fr + (size_t)(cur ^ 1) * F.cap;
    // (1) accept the frontier, and in the same phase (2) collect the
    // unmatched vertices sharing an edge with a newly matched one (their head
    // edge may have died), deduplicated; long incidence lists (hubs) are
    // walked by a warp. A vertex matched in this round may be collected
    // before its partner store is visible; step (3) drops it.
    for (int64_t i = t0; i < L; i += nt) {
      const int v = fin[i], u = F.prop[v];
      F.partner[v] = u;
      F.partner[u] = v;
    }
    const int par = round & 1;
    if (t0 == 0) F.fcnt[cur ^ 1] = 0;
    auto touch = [&](int y) {
      if (F.partner[y] >= 0 || atomicExch(&F.aflag[y], round) == round) return false;
      return true;
    };
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < 2 * L; b0 += nt) {
      if (threadIdx.x == 0) s_ndef = 0;
      __syncthreads();
      const int64_t i = b0 + threadIdx.x;
      int x = -1, beg = 0, len = 0;
      if (i < 2 * L) {
        const int v = fin[i >> 1];
        x = (i & 1) ? F.prop[v] : v;
        beg = F.ioff[x];
        len = F.ioff[x + 1] - beg;
        if (len > FR_SHORT) {
          const int d = atomicAdd(&s_ndef, 1);
          s_def[d] = x;  // d < blockDim <= FR_DEFER
          len = 0;
        }
      }
      // short lists: the warp walks its lanes' lists in step, so each step's
      // appends share one atomic (per-lane appends on the one counter
      // serialised in L2)
      const int maxlen = __reduce_max_sync(0xffffffffu, (unsigned)len);
      for (int j = 0; j < maxlen; ++j) {
        int y = -1;
        if (j < len) {
          y = fr_other(F, (int)(F.inc[beg + j] & 0xffffffffu), x);
          if (!touch(y)) y = -1;
        }
        warp_append(y >= 0, y, F.aff, F.fcnt + 2 + par);
      }
      __syncthreads();
      for (int d = wib; d < s_ndef; d += nwb) {
        const int x = s_def[d];
        const int end = F.ioff[x + 1];
        for (int q0 = F.ioff[x]; q0 < end; q0 += 32) {
          const int q = q0 + lane;
          int y = -1;
          if (q < end) {
            y = fr_other(F, (int)(F.inc[q] & 0xffffffffu), x);
            if (!touch(y)) y = -1;
          }
          warp_append(y >= 0, y, F.aff, F.fcnt + 2 + par);
        }
      }
      __syncthreads();
    }
    grid_or_block_sync(grid);
    // (3) refresh each affected head; queue it if it is also the lowest live
    // edge at its other endpoint
    const int64_t A = (int64_t)vload(F.fcnt + 2 + par);
    if (t0 == 0) F.fcnt[2 + (par ^ 1)] = 0;  // next round's (last read a round ago)
    for (int64_t b0 = (int64_t)blockIdx.x * blockDim.x; b0 < A; b0 += nt) {
      if (threadIdx.x == 0) s_ndef = 0;
      __syncthreads();
      const int64_t i = b0 + threadIdx.x;
      int qh = -1;  // head edge to queue for the next round
      if (i < A && F.partner[F.aff[i]] >= 0) {  // matched this round
        F.head[F.aff[i]] = F.ioff[F.aff[i] + 1];
      } else if (i < A) {
        const int y = F.aff[i];
        int pos, pz;
        const int h = fr_first_live_t(F, y, FR_SHORT, &pos);
        bool defer = h == -2;
        if (!defer) {
          F.head[y] = pos;
          if (h >= 0) {
            const int hz = fr_first_live_t(F, fr_other(F, h, y), FR_SHORT, &pz);
            if (hz == -2) defer = true;
            else if (hz == h && atomicExch(&F.qflag[h], round) != round)
              qh = h;
          }
        }
        if (defer) s_def[atomicAdd(&s_ndef, 1)] = y;
      }
      warp_append(qh >= 0, qh, fout, F.fcnt + (cur ^ 1));
      __syncthreads();
      for (int d = wib; d < s_ndef; d += nwb) {
        const int y = s_def[d];
        int pos, pz;
        const int h = fr_first_live(F, y, &pos);  // (y unmatched: checked above)
        if (lane == 0) F.head[y] = pos;
        if (h < 0) continue;
        const int hz = fr_first_live(F, fr_other(F, h, y), &pz);
        if (lane == 0 && hz == h && atomicExch(&F.qflag[h], round) != round)
          fout[atomicAdd(F.fcnt + (cur ^ 1), 1ull)] = h;
      }
      __syncthreads();
    }
    grid_or_block_sync(grid);
    if (t0 == 0) F.fcnt[4] += 1;
    cur ^= 1;
  }
}

__global__ void k_inc_keys(const int32_t* __restrict__ props, int64_t ne,
                           const int32_t* __restrict__ prop, unsigned long long* keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned v = (unsigned)props[i], u = (unsigned)prop[v];
    keys[2 * i] = ((unsigned long long)v << 32) | v;
    keys[2 * i + 1] = ((unsigned long long)u << 32) | v;
  }
}

// ioff[x] = first incidence of endpoint x (lower bound in the sorted keys)
__global__ void k_inc_offsets(const unsigned long long* __restrict__ keys, int64_t M, int64_t n,
                              int32_t* ioff, int32_t* head, int32_t* aflag) {
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x <= n;
       x += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long key = (unsigned long long)x << 32;
    int64_t lo = 0, hi = M;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    ioff[x] = (int32_t)lo;
    if (x < n) {
      head[x] = (int32_t)lo;
      aflag[x] = 0;
    }
  }
}

static void resolve_frontier(Ctx& c, int64_t n, const int32_t* prop, int32_t* partner,
                             const int32_t* props, int64_t ne) {
  const int64_t M = 2 * ne;
  unsigned long long* keys = c.scratch<unsigned long long>(21, 2 * M);
  int32_t* ints = c.scratch<int32_t>(22, 5 * n + 1);
  int32_t* fr = c.scratch<int32_t>(23, 2 * ne);
  unsigned long long* fcnt = c.scratch<unsigned long long>(24, 8);
  int32_t *ioff = ints, *head = ints + n + 1, *qflag = ints + 2 * n + 1, *aflag = ints + 3 * n + 1,
          *aff = ints + 4 * n + 1;
  dzero(c, fcnt, 8);
  dzero(c, qflag, n);
  launch(c, "match_inc", 16.0 * ne, [&] {
    k_inc_keys<<<grid_for(c, ne, 256), 256, 0, c.stream>>>(props, ne, prop, keys);
  });
  int end_bit = 33;
  while (end_bit < 64 && (1LL << (end_bit - 32)) <= n) ++end_bit;
  size_t tmp = 0;
  CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, keys, keys + M, (int)M, 0, end_bit, c.stream));
  void* p = c.cub_scratch(tmp);
  launch(c, "match_inc_sort", 32.0 * M, [&] {
    CK(cub::DeviceRadixSort::SortKeys(p, tmp, keys, keys + M, (int)M, 0, end_bit, c.stream));
  });
  launch(c, "match_inc", 16.0 * n, [&] {
    k_inc_offsets<<<grid_for(c, n + 1, 256), 256, 0, c.stream>>>(keys + M, M, n, ioff, head,
                                                                 aflag);
  });
  Frontier F{prop, partner, keys + M, ioff, head, qflag, aflag, fr, aff, fcnt, props, ne, ne};
  static int fgrid = 0;
  if (!fgrid) fgrid = coop_blocks(c, (const void*)k_resolve_frontier, 1024);
  const int blocks = (int)std::min<int64_t>(fgrid, std::max<int64_t>(1, (ne + 16383) / 16384));
  void* args[] = {&F};
  launch(c, "match_resolve", 0.0, [&] {
    CK(cudaLaunchCooperativeKernel((const void*)k_resolve_frontier, dim3(blocks), dim3(1024), args,
                                   0, c.stream));
  });
  static const bool mstats = getenv("JET_MATCH_STATS") && getenv("JET_MATCH_STATS")[0] == '1';
  if (mstats) {
    unsigned long long hs[8];
    d2h(c, hs, fcnt, 8);
    c.sync();
    fprintf(stderr, "FRONTIER n=%lld edges=%lld blocks=%d rounds=%llu\n", (long long)n,
            (long long)ne, blocks, hs[4]);
  }
}

void device_match(Ctx& c, const DGraph& g, int32_t* partner) {
  const int64_t n = g.n;
  launch(c, "fill", 4.0 * n, [&] {
    k_fill<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, -1);
  });
  if (g.nnz > 0) {
    int32_t* prop_p = c.scratch<int32_t>(10, n);
    int32_t* lists_p = c.scratch<int32_t>(11, 2 * n);
    int32_t* mn_p = c.scratch<int32_t>(12, 2 * n);
    DBuf<unsigned long long> cnt(2, c.stream);
    CK(cudaMemsetAsync(mn_p, 0x7f, 2 * n * sizeof(int32_t), c.stream));
    const GView gv = view(g);
    while (true) {
      dzero(c, cnt.get(), 2);
      for (int t = 0; t < NBINS; ++t) {
        const int64_t bc = g.bin_cnt[t];
        if (!bc) continue;
        const int G = t < 4 ? TIER_G[t] : 32;
        const int32_t* list = tier_list(g, t);
        // tier 3 holds rows of up to 64 entries: k_propose<32> reads one
        // entry per lane, so such levels propose tier 3 one warp per row
        const bool short_rows = t < 3 || (t == 3 && g.max_deg <= 32);
        const unsigned grid = grid_for(c, short_rows ? bc : bc * 32, 256);
        launch(c, "propose", (g.unit_ew ? 8.0 : 12.0) * g.bin_nnz[t] + 12.0 * bc, [&] {
          if (short_rows)
            JET_TIER_LAUNCH(k_propose, G, g.unit_ew, grid, 256, 0, c.stream, gv, list, bc, partner,
                            prop_p, lists_p, cnt.get());
          else if (g.unit_ew)
            k_propose_long<true><<<grid, 256, 0, c.stream>>>(gv, list, bc, partner, prop_p,
                                                            lists_p, cnt.get());
          else
            k_propose_long<false><<<grid, 256, 0, c.stream>>>(gv, list, bc, partner, prop_p,
                                                             lists_p, cnt.get());
        });
      }
      unsigned long long ne = 0;
      d2h(c, &ne, cnt.get(), 1);
      c.sync();
      if (ne == 0) break;
      static const bool old_rounds = getenv("JET_MATCH_ROUNDS") && getenv("JET_MATCH_ROUNDS")[0] == '1';
      if (!old_rounds) {
        resolve_frontier(c, n, prop_p, partner, lists_p, (int64_t)ne);
        continue;
      }
      // all resolution rounds in one cooperative launch (k_resolve)
      static const bool mstats = getenv("JET_MATCH_STATS") && getenv("JET_MATCH_STATS")[0] == '1';
      static DBuf<unsigned long long>* sbuf = nullptr;
      if (mstats && !sbuf) {
        sbuf = new DBuf<unsigned long long>(4, c.stream);
        dzero(c, sbuf->get(), 4);
      }
      Resolve R{prop_p, partner, lists_p, cnt.get(), mn_p, n,
                (unsigned long long)RES_TAIL, mstats ? sbuf->get() : nullptr};
      const size_t smem = sizeof(ResTailSmem);
      static int res_grid = 0;
      if (!res_grid) {
        CK(cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int per_sm = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_resolve, 1024, smem));
        JET_REQUIRE(per_sm >= 1, JET_EINTERNAL, "k_resolve does not fit on an SM");
        res_grid = per_sm * c.num_sms;
      }
      // fewer, fuller blocks make each grid-wide barrier cheaper
      const int blocks = std::min<int64_t>(res_grid, std::max<int64_t>(8, ((int64_t)ne + 16383) / 16384));
      void* args[] = {&R};
      launch(c, "match_resolve", 0.0, [&] {
        CK(cudaLaunchCooperativeKernel((const void*)k_resolve, dim3(blocks), dim3(1024), args, smem,
                                       c.stream));
      });
      if (mstats) {
        unsigned long long hs[4];
        d2h(c, hs, sbuf->get(), 4);
        c.sync();
        fprintf(stderr, "MATCH n=%lld live=%llu blocks=%d rounds=%llu tail=%llu tail_us=%.1f tail_rounds=%llu\n",
                (long long)n, ne, blocks, hs[0], hs[1], hs[2] / 1965.0, hs[3]);
        dzero(c, sbuf->get(), 4);
      }
    }
    two_hop(c, g, partner);
  }
  launch(c, "singletons", 8.0 * n, [&] {
    k_singletons<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n);
  });
}

// ---------------------------------------------------------------------------
// Throughput-mode matching (jet_config.deterministic == 0). The reference's
// matching is sequential (ascending-id resolution, ordered two-hop walk);
// reproducing it exactly costs many dependent rounds. This mode keeps the
// heavy-edge criterion but breaks weight ties with a symmetric hash of the
// edge, so both endpoints rank their edges alike and every proposal that is
// returned is a locally dominant edge: a few propose/accept rounds match
// most vertices, each a coalesced sweep over the free rows. Leftovers are
// paired under their heaviest neighbour (one centre each, radix-sorted), as
// in mt-Metis leaf matching. Not bit-exact with the reference: the 2 %
// cutsize gate applies (north_star, throughput mode).
__device__ __forceinline__ unsigned edge_hash(int a, int b, unsigned salt) {
  unsigned x = (unsigned)min(a, b) * 0x9E3779B1u ^ ((unsigned)max(a, b) + salt) * 0x85EBCA77u;
  x ^= x >> 15;
  x *= 0x2C1B3C6Du;
  x ^= x >> 12;
  x *= 0x297A2D39u;
  x ^= x >> 15;
  return x | 1u;
}

// Heaviest free neighbour, ties -> highest edge hash, then lowest id. One
// warp per row (rows of any length), 32 rows per warp batch for short rows.
// prev (optional): the previous round's {proposers, pairs}; a round after one
// that matched nothing does nothing (rounds are launched in groups between
// host checks, and must stop exactly where a per-round check would)
__device__ __forceinline__ bool fast_round_dead(const unsigned long long* prev) {
  return prev && (prev[0] == 0 || prev[1] == 0);
}

#ifndef PROPOSE_BATCH
#define PROPOSE_BATCH 4
#endif

template <bool UNIT>
__global__ void __launch_bounds__(256)
    k_propose_fast(GView g, int64_t n, const int32_t* __restrict__ partner, int32_t* prop,
                   int32_t* elist, unsigned long long* ecnt, unsigned salt,
                   const unsigned long long* prev, int64_t v_lo = 0) {
  // vertices [v_lo, n): a distributed level proposes for its own rows only
  if (fast_round_dead(prev)) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t base = v_lo + w0 * 32; base < n; base += nw * 32) {
    const int64_t idx = base + lane;
    int v = (int)idx, deg = 0;
    int64_t beg = 0;
    bool live = false;
    if (idx < n) {
      live = partner[v] < 0;
      if (live) {
        beg = g.offs[v];
        deg = (int)(g.offs[v + 1] - beg);
      }
    }
    // hub rows (> WARP_TIER_MAX_DEG entries) are proposed by k_propose_fast_hub
    const bool hub = deg > WARP_TIER_MAX_DEG;
    unsigned live_m = __ballot_sync(0xffffffffu, live && deg > 0 && !hub);
    int my_u = -1;
    // PB rows per step, their loads interleaved: a row's adjacency load and
    // the dependent partner[] gather are two L2/HBM round trips, and one row
    // at a time left each warp waiting on 2 x 32 of them in sequence
    constexpr int PB = PROPOSE_BATCH;
    while (live_m) {
      int rr[PB], rd[PB];
      int64_t rb[PB];
      int maxd = 0;
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        rr[q] = -1;
        rd[q] = 0;
        rb[q] = 0;
        if (live_m) {
          const int r = __ffs(live_m) - 1;
          live_m &= live_m - 1;
          rr[q] = r;
        }
        const int src = rr[q] < 0 ? 0 : rr[q];
        const int64_t b_ = __shfl_sync(0xffffffffu, beg, src);
        const int d_ = __shfl_sync(0xffffffffu, deg, src);
        if (rr[q] >= 0) {
          rb[q] = b_;
          rd[q] = d_;
          maxd = max(maxd, d_);
        }
      }
      unsigned bw[PB], bh[PB];
      int bu[PB];
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        bw[q] = 0;
        bh[q] = 0;
        bu[q] = -1;
      }
      for (int j = lane; j < maxd; j += 32) {
        int u[PB], pu[PB];
        unsigned w[PB];
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          u[q] = j < rd[q] ? g.adj[rb[q] + j] : -1;
          w[q] = UNIT ? 1u : (j < rd[q] ? (unsigned)g.ew[rb[q] + j] : 0u);
        }
#pragma unroll
        for (int q = 0; q < PB; ++q) pu[q] = u[q] >= 0 ? partner[u[q]] : 0;
#pragma unroll
        for (int q = 0; q < PB; ++q) {
          if (u[q] < 0 || pu[q] >= 0) continue;
          const unsigned h = edge_hash((int)(base + rr[q]), u[q], salt);
          if (w[q] > bw[q] || (w[q] == bw[q] && (h > bh[q] || (h == bh[q] && u[q] < bu[q])))) {
            bw[q] = w[q];
            bh[q] = h;
            bu[q] = u[q];
          }
        }
      }
#pragma unroll
      for (int q = 0; q < PB; ++q) {
        if (rr[q] < 0) break;  // warp-uniform
        const unsigned mw = __reduce_max_sync(0xffffffffu, bw[q]);
        const unsigned mh = __reduce_max_sync(0xffffffffu, bw[q] == mw ? bh[q] : 0u);
        const unsigned mu = __reduce_min_sync(0xffffffffu, (bw[q] == mw && bh[q] == mh && bu[q] >= 0)
                                                                ? (unsigned)bu[q] : 0xffffffffu);
        if (lane == rr[q]) my_u = mw ? (int)mu : -1;
      }
    }
    if (live && !hub) prop[v] = my_u;
    warp_append(live && !hub && my_u >= 0, v, elist, ecnt);
  }
}

// Hub rows: one block per row, same key (weight, edge hash, -id).
template <bool UNIT>
__global__ void __launch_bounds__(256)
    k_propose_fast_hub(GView g, const int32_t* __restrict__ hubs, int64_t nh,
                       const int32_t* __restrict__ partner, int32_t* prop, int32_t* elist,
                       unsigned long long* ecnt, unsigned salt, const unsigned long long* prev) {
  if (fast_round_dead(prev)) return;
  __shared__ unsigned s_w[8], s_h[8], s_u[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t i = blockIdx.x; i < nh; i += gridDim.x) {
    const int v = hubs ? hubs[i] : (int)i;  // identity when every row is a hub
    if (partner[v] >= 0) continue;  // block-uniform
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    unsigned bw = 0, bh = 0, bu = 0xffffffffu;
    for (int64_t j = b + threadIdx.x; j < e; j += blockDim.x) {
      const int u = g.adj[j];
      if (partner[u] >= 0) continue;
      const unsigned ww = UNIT ? 1u : (unsigned)g.ew[j];
      const unsigned h = edge_hash(v, u, salt);
      if (ww > bw || (ww == bw && (h > bh || (h == bh && (unsigned)u < bu)))) {
        bw = ww;
        bh = h;
        bu = (unsigned)u;
      }
    }
    unsigned mw = __reduce_max_sync(0xffffffffu, bw);
    if (lane == 0) s_w[w] = mw;
    __syncthreads();
    mw = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mw = max(mw, s_w[q]);
    unsigned mh = __reduce_max_sync(0xffffffffu, bw == mw ? bh : 0u);
    if (lane == 0) s_h[w] = mh;
    __syncthreads();
    mh = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mh = max(mh, s_h[q]);
    unsigned mu = __reduce_min_sync(0xffffffffu, (bw == mw && bh == mh) ? bu : 0xffffffffu);
    if (lane == 0) s_u[w] = mu;
    __syncthreads();
    if (threadIdx.x == 0) {
      mu = 0xffffffffu;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mu = min(mu, s_u[q]);
      const int pu = mw ? (int)mu : -1;
      prop[v] = pu;
      if (pu >= 0) elist[atomicAdd(ecnt, 1ull)] = v;
    }
    __syncthreads();
  }
}

// Accept mutual proposals (locally dominant edges); count the new pairs.
__global__ void k_accept_mutual(const int32_t* __restrict__ prop, int32_t* partner,
                                const int32_t* __restrict__ elist,
                                const unsigned long long* __restrict__ ecnt,
                                unsigned long long* npairs, const unsigned long long* prev) {
  if (fast_round_dead(prev)) return;
  const int64_t cnt = (int64_t)*ecnt;
  long long mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = elist[i];
    const int u = prop[v];
    if (v < u && prop[u] == v) {
      partner[v] = u;
      partner[u] = v;
      ++mine;
    }
  }
  block_sum_atomic<256>(mine, npairs);
}

// Leftovers: key = (centre, v) packed in 2*vb bits (vb bits hold 0..n),
// centre = heaviest neighbour (ties: lowest id), n for an isolated vertex --
// the radix sort then runs over the bits in use only.
__global__ void k_leaf_keys(GView g, const int32_t* __restrict__ left, int64_t nl, int vb,
                            unsigned long long* keys) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nl; i += nw) {
    const int v = left[i];
    const int64_t b = g.offs[v], e = g.offs[v + 1];
    unsigned long long best = 0;
    for (int64_t j = b + lane; j < e; j += 32) {
      const unsigned long long w = (unsigned long long)g.ew[j];
      const unsigned long long key = (w << 32) | (0xffffffffu - (unsigned)g.adj[j]);
      best = key > best ? key : best;
    }
    best = gmax<32>(best, 0xffffffffu);
    if (lane == 0) {
      const unsigned long long c =
          best ? (0xffffffffu - (best & 0xffffffffu)) : (unsigned long long)g.n;
      keys[i] = (c << vb) | (unsigned)v;
    }
  }
}

// Pair consecutive leftovers under the same centre: (0,1), (2,3), ... of
// each run of the sorted keys.
// One thread per leftover: its rank in its centre's run is found by a binary
// search for the run's first key (a run start walking its run serially took
// 0.5 ms per level on R-MAT, where hub centres collect 10^5 leftovers); even
// ranks pair with the next key of the same run.
__global__ void k_leaf_pair(const unsigned long long* __restrict__ keys, int64_t nl, int vb,
                            int64_t n, int32_t* partner) {
  const unsigned long long vm = (1ull << vb) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nl;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long c = keys[i] >> vb;
    if ((int64_t)c == n) continue;  // isolated vertex
    if (i + 1 >= nl || (keys[i + 1] >> vb) != c) continue;  // last of its run: no successor
    int64_t lo = 0, hi = i;  // first index whose centre is c
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((keys[mid] >> vb) < c) lo = mid + 1;
      else hi = mid;
    }
    if (((i - lo) & 1) == 0) {
      const int a = (int)(keys[i] & vm), b = (int)(keys[i + 1] & vm);
      partner[a] = b;
      partner[b] = a;
    }
  }
}

// throughput-mode matching rounds launched between two host checks
#ifndef MATCH_ROUND_GROUP
#define MATCH_ROUND_GROUP 4
#endif

static void leaf_match(Ctx& c, const DGraph& g, int32_t* partner) {
  const int64_t n = g.n;
  int32_t* left_p = c.scratch<int32_t>(13, n);
  DBuf<int64_t> nsel(1, c.stream);
  {
    cub::CountingInputIterator<int32_t> it(0);
    IsFree op{partner};
    if (!small_select(c, "th_leftovers", op, n, left_p, nsel.get())) {
      size_t tmp = 0;
      CK(cub::DeviceSelect::If(nullptr, tmp, it, left_p, nsel.get(), (int)n, op, c.stream));
      void* p = c.cub_scratch(tmp);
      launch(c, "th_leftovers", 8.0 * n, [&] {
        CK(cub::DeviceSelect::If(p, tmp, it, left_p, nsel.get(), (int)n, op, c.stream));
      });
    }
  }
  int64_t nl = 0;
  d2h(c, &nl, nsel.get(), 1);
  c.sync();
  if (nl < 2) return;
  unsigned long long* k0 = c.scratch<unsigned long long>(14, nl);
  unsigned long long* k1 = c.scratch<unsigned long long>(16, nl);
  const GView gv = view(g);
  int vb = 1;
  while ((1LL << vb) <= n) ++vb;  // vb bits hold 0..n
  launch(c, "leaf_keys", 16.0 * nl, [&] {
    k_leaf_keys<<<grid_for(c, nl * 32, 256), 256, 0, c.stream>>>(gv, left_p, nl, vb, k0);
  });
  if (!small_sort_keys(c, "leaf_sort", k0, k1, nl, 2 * vb)) {
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1, (int)nl, 0, 2 * vb, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "leaf_sort", 32.0 * nl, [&] {
      CK(cub::DeviceRadixSort::SortKeys(p, tmp, k0, k1, (int)nl, 0, 2 * vb, c.stream));
    });
  }
  launch(c, "leaf_pair", 16.0 * nl, [&] {
    k_leaf_pair<<<grid_for(c, nl, 256), 256, 0, c.stream>>>(k1, nl, vb, n, partner);
  });
}

static void device_match_fast(Ctx& c, const DGraph& g, int32_t* partner) {
  const int64_t n = g.n;
  launch(c, "fill", 4.0 * n, [&] {
    k_fill<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, -1);
  });
  if (g.nnz > 0) {
    int32_t* prop_p = c.scratch<int32_t>(10, n);
    int32_t* elist_p = c.scratch<int32_t>(11, n);
    // rounds in groups of RG between host checks: each round has its own
    // {proposers, pairs} counters, and a round after one that matched nothing
    // is a no-op on the device (fast_round_dead), so the result is the same as
    // checking after every round, with a quarter of the host round trips
    constexpr int RG = MATCH_ROUND_GROUP, MAXR = 48;
    static_assert(MAXR % RG == 0, "MATCH_ROUND_GROUP must divide the round cap");
    DBuf<unsigned long long> cnt(2 * MAXR, c.stream);
    dzero(c, cnt.get(), 2 * MAXR);
    const GView gv = view(g);
    int64_t matched = 0;
    int low_rounds = 0;
    static const bool fstats = getenv("JET_MATCH_STATS") && getenv("JET_MATCH_STATS")[0] == '1';
    for (int r0 = 0; r0 < MAXR; r0 += RG) {
      for (int round = r0; round < r0 + RG; ++round) {
        unsigned long long* rc = cnt.get() + 2 * round;
        const unsigned long long* prev = round ? rc - 2 : nullptr;
        const unsigned salt = 0x5bd1e995u * (unsigned)(round + 1);
        launch(c, "propose", (g.unit_ew ? 8.0 : 12.0) * g.nnz + 12.0 * n, [&] {
          if (g.unit_ew)
            k_propose_fast<true><<<grid_res(c, k_propose_fast<true>, n, 256), 256, 0, c.stream>>>(
                gv, n, partner, prop_p, elist_p, rc, salt, prev);
          else
            k_propose_fast<false><<<grid_res(c, k_propose_fast<false>, n, 256), 256, 0, c.stream>>>(
                gv, n, partner, prop_p, elist_p, rc, salt, prev);
        });
        if (g.bin_cnt[BIN_BLOCK]) {
          const int64_t nh = g.bin_cnt[BIN_BLOCK];
          const int32_t* hubs = tier_list(g, BIN_BLOCK);
          const unsigned hg = (unsigned)std::min<int64_t>(nh, 4LL * c.num_sms);
          launch(c, "propose_hub", 0.0, [&] {
            if (g.unit_ew)
              k_propose_fast_hub<true><<<hg, 256, 0, c.stream>>>(gv, hubs, nh, partner, prop_p,
                                                                 elist_p, rc, salt, prev);
            else
              k_propose_fast_hub<false><<<hg, 256, 0, c.stream>>>(gv, hubs, nh, partner, prop_p,
                                                                  elist_p, rc, salt, prev);
          });
        }
        launch(c, "accept", 12.0 * n, [&] {
          k_accept_mutual<<<grid_for(c, n, 256), 256, 0, c.stream>>>(prop_p, partner, elist_p, rc,
                                                                     rc + 1, prev);
        });
      }
      unsigned long long h[2 * RG];
      d2h(c, h, cnt.get() + 2 * r0, 2 * RG);
      c.sync();
      bool done = false;
      for (int q = 0; q < RG && !done; ++q) {
        matched += 2 * (int64_t)h[2 * q + 1];
        if (fstats)
          fprintf(stderr, "FAST n=%lld round=%d proposers=%llu pairs=%llu matched=%lld\n",
                  (long long)n, r0 + q, h[2 * q], h[2 * q + 1], (long long)matched);
        // rounds until no pair is added: stopping at a 1 % yield (of n) left
        // many leftovers to the leaf pairing, whose non-adjacent pairs made
        // the coarse levels refine 2x longer (128^3: 143 -> 72 ms, 3 % lower
        // cut). On dense power-law levels the proposals chain towards the
        // hubs instead, and each round pairs a few hundred of 10^5 proposers
        // for 40+ rounds that each rescan every live row (R-MAT 2^22: 0.3 s
        // of matching): once a round pairs under 0.5 % of its proposers
        // twice in a row, the rest goes to the leaf pairing, which pairs
        // leftovers sharing their heaviest neighbour.
        const bool low = h[2 * q + 1] * 200 < h[2 * q];
        low_rounds = low ? low_rounds + 1 : 0;
        done = h[2 * q] == 0 || h[2 * q + 1] == 0 || low_rounds >= 2;
      }
      if (done) break;
    }
    leaf_match(c, g, partner);
  }
  launch(c, "singletons", 8.0 * n, [&] {
    k_singletons<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n);
  });
}

// ---------------------------------------------------------------------------
// Contraction
__global__ void k_is_rep(const int32_t* __restrict__ partner, int64_t n, int32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    flag[v] = partner[v] >= v ? 1 : 0;
}

// A matching is an involution: partner[partner[v]] == v for every v. The
// contraction sizes its merged-row scratch from that (the member rows of all
// coarse vertices add up to the fine entry count), so the public entry point
// checks it (the internal hierarchy's matchings are involutions by construction).
__global__ void k_check_involution(const int32_t* __restrict__ partner, int64_t n,
                                   unsigned* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride)
    if (partner[partner[v]] != (int32_t)v) atomicOr(bad, 1u);
}

bool device_is_involution(Ctx& c, const int32_t* partner, int64_t n) {
  DBuf<unsigned> bad(1, c.stream);
  dzero(c, bad.get(), 1);
  launch(c, "check_involution", 8.0 * n, [&] {
    k_check_involution<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, bad.get());
  });
  unsigned h = 0;
  d2h(c, &h, bad.get(), 1);
  c.sync();
  return h == 0;
}

struct CoarseMap {
  const int32_t* partner;
  const int32_t* cid;  // exclusive scan of rep flags
  const int64_t* offs;
  const int32_t* vw;
  int32_t* vmap;
  int32_t* cvw;
  int32_t* mem_a;
  int32_t* mem_b;
  int64_t* rowlen;  // deg(a) + deg(b)
  unsigned* overflow;
};

__global__ void k_coarse_map(CoarseMap m, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n; v += stride) {
    const int p = m.partner[v];
    const int rep = p < v ? p : (int)v;
    const int c = m.cid[rep];
    m.vmap[v] = c;
    if (rep == v) {
      long long w = m.vw[v];
      int64_t d = m.offs[v + 1] - m.offs[v];
      if (p != v) {
        w += m.vw[p];
        d += m.offs[p + 1] - m.offs[p];
      }
      if (w > 2147483647LL) atomicOr(m.overflow, 1u);
      m.cvw[c] = (int32_t)w;
      m.mem_a[c] = (int32_t)v;
      m.mem_b[c] = p;
      m.rowlen[c] = d;
    }
  }
}

template <int E>
__device__ __forceinline__ void warp_bitonic(unsigned long long (&x)[E]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int stride = size / 2; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const int rs = stride / 32;
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const int pr = r ^ rs;
          if (pr > r) {
            const bool asc = (((r * 32 + lane) & size) == 0);
            const unsigned long long a = x[r], b = x[pr];
            if ((a > b) == asc) {
              x[r] = b;
              x[pr] = a;
            }
          }
        }
      } else {
#pragma unroll
        for (int r = 0; r < E; ++r) {
          const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[r], stride);
          const bool asc = (((r * 32 + lane) & size) == 0);
          const bool lower = (lane & stride) == 0;
          const unsigned long long lo = x[r] < y ? x[r] : y, hi = x[r] < y ? y : x[r];
          x[r] = (lower == asc) ? lo : hi;
        }
      }
    }
  }
}

struct RowMerge {
  const int64_t* offs;
  const int32_t* adj;
  const int32_t* ew;
  const int32_t* vmap;
  const int32_t* mem_a;
  const int32_t* mem_b;
  const int64_t* toff;  // staging offsets (exclusive scan of rowlen)
  const int64_t* rowlen;
  int32_t* tadj;
  int32_t* tew;
  int64_t* cdeg;
  int32_t* big;  // rows longer than 256 entries
  unsigned long long* big_cnt;
  unsigned* overflow;
  int64_t nc;
  int collect_big;  // append long rows to `big` (0: the list is already built)
  // distributed finest level: coarse rows [c_lo, c_hi) are merged here; fine
  // rows of [row_lo, row_hi) are local (adj/ew from ent_lo), the others come
  // from the import buffer at imp_pos[x]
  int64_t c_lo = 0, c_hi = -1;
  int64_t row_lo = 0, row_hi = INT64_MAX, ent_lo = 0;
  const int64_t* imp_pos = nullptr;
  const int32_t* imp_adj = nullptr;
  const int32_t* imp_ew = nullptr;
};

// gather row entries of member x of coarse vertex c as sort keys
__device__ __forceinline__ unsigned long long merged_key(const RowMerge& m, int c, int64_t idx,
                                                         int a, int b, int64_t da) {
  const int x = idx < da ? a : b;
  const int64_t k = idx < da ? idx : idx - da;
  int u, w;
  if (x >= m.row_lo && x < m.row_hi) {
    const int64_t j = m.offs[x] - m.ent_lo + k;
    u = m.adj[j];
    w = m.ew[j];
  } else {  // a member row owned by another rank (distributed finest level)
    const int64_t j = m.imp_pos[x] + k;
    u = m.imp_adj[j];
    w = m.imp_ew[j];
  }
  const int cv = m.vmap[u];
  if (cv == c) return ~0ull;  // contraction self loop (coarsen.py:133)
  return ((unsigned long long)(unsigned)cv << 32) | (unsigned)w;
}

template <int E>
__device__ void merge_row_warp(const RowMerge& m, int c, unsigned long long* sbuf) {
  const int lane = threadIdx.x & 31;
  const int a = m.mem_a[c], b = m.mem_b[c];
  const int64_t da = m.offs[a + 1] - m.offs[a];
  const int64_t d = m.rowlen[c];
  unsigned long long x[E];
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int64_t idx = r * 32 + lane;
    x[r] = idx < d ? merged_key(m, c, idx, a, b, da) : ~0ull;
  }
  warp_bitonic<E>(x);
#pragma unroll
  for (int r = 0; r < E; ++r) sbuf[r * 32 + lane] = x[r];
  __syncwarp();
  const int64_t base = m.toff[c];
  int outn = 0;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const int i = r * 32 + lane;
    const unsigned long long k = sbuf[i];
    const unsigned cv = (unsigned)(k >> 32);
    const bool head = k != ~0ull && (i == 0 || (unsigned)(sbuf[i - 1] >> 32) != cv);
    long long sum = 0;
    if (head) {
      for (int q = i; q < 32 * E && sbuf[q] != ~0ull && (unsigned)(sbuf[q] >> 32) == cv; ++q)
        sum += (long long)(sbuf[q] & 0xffffffffu);
    }
    const unsigned hm = __ballot_sync(0xffffffffu, head);
    if (head) {
      const int pos = outn + __popc(hm & lanemask_lt());
      if (sum > 2147483647LL) atomicOr(m.overflow, 2u);
      if (m.tadj) {  // nullptr: counting pass of a two-pass contraction
        m.tadj[base + pos] = (int32_t)cv;
        m.tew[base + pos] = (int32_t)sum;
      }
    }
    outn += __popc(hm);
  }
  if (lane == 0) m.cdeg[c] = outn;
  __syncwarp();
}

__global__ void __launch_bounds__(256) k_merge_rows(RowMerge m) {
  __shared__ unsigned long long sbuf[8][256];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t c_hi = m.c_hi < 0 ? m.nc : m.c_hi;
  for (int64_t c = m.c_lo + w0; c < c_hi; c += ws) {
    const int64_t d = m.rowlen[c];
    if (d <= 32) merge_row_warp<1>(m, (int)c, sbuf[wib]);
    else if (d <= 64) merge_row_warp<2>(m, (int)c, sbuf[wib]);
    else if (d <= 128) merge_row_warp<4>(m, (int)c, sbuf[wib]);
    else if (d <= 256) merge_row_warp<8>(m, (int)c, sbuf[wib]);
    else if (m.collect_big) {
      if (lane == 0) {
        const unsigned long long i = atomicAdd(m.big_cnt, 1ull);
        m.big[i] = (int32_t)c;
      }
    }
  }
}

// long rows: gather keys into a segmented buffer for a library segmented sort
__global__ void k_big_gather(RowMerge m, const int32_t* __restrict__ big, int64_t nbig,
                             const int64_t* __restrict__ boff, unsigned long long* keys,
                             int64_t min_len) {
  for (int64_t i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int c = big[i];
    const int64_t d = m.rowlen[c];
    if (d <= min_len) continue;  // sorted on chip by k_big_sort_block
    const int a = m.mem_a[c], b = m.mem_b[c];
    const int64_t da = m.offs[a + 1] - m.offs[a];
    const int64_t o = boff[i];
    for (int64_t idx = threadIdx.x; idx < d; idx += blockDim.x) keys[o + idx] = merged_key(m, c, idx, a, b, da);
  }
}

// Long rows of up to BIG_BLOCK_MAX entries (almost all of them on the dense
// coarse levels of power-law graphs): one block gathers the merged row
// straight from the fine rows into registers, radix-sorts it on chip over
// the coarse-id bits only (+1 bit so contraction self loops, ~0, sort last)
// and writes it sorted: no gather pass and no device-wide segmented sort.
constexpr int BIG_BT = 256, BIG_IPT_S = 4, BIG_IPT_L = 16;
constexpr int64_t BIG_BLOCK_MAX = (int64_t)BIG_BT * BIG_IPT_L;

template <int IPT>
__device__ __forceinline__ void big_sort_row(const RowMerge& m, int c, int64_t d, int64_t o,
                                             int cbits, unsigned long long* out, void* ts_raw) {
  typedef cub::BlockRadixSort<unsigned long long, BIG_BT, IPT> BRS;
  auto& ts = *reinterpret_cast<typename BRS::TempStorage*>(ts_raw);
  const int a = m.mem_a[c], b = m.mem_b[c];
  const int64_t da = m.offs[a + 1] - m.offs[a];
  unsigned long long k[IPT];
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int64_t idx = (int64_t)threadIdx.x * IPT + q;  // blocked arrangement
    k[q] = idx < d ? merged_key(m, c, idx, a, b, da) : ~0ull;
  }
  BRS(ts).Sort(k, 32, 32 + cbits + 1);
#pragma unroll
  for (int q = 0; q < IPT; ++q) {
    const int64_t idx = (int64_t)threadIdx.x * IPT + q;
    if (idx < d) out[o + idx] = k[q];
  }
}

__global__ void __launch_bounds__(BIG_BT)
    k_big_sort_block(RowMerge m, const int32_t* __restrict__ big, int64_t nbig,
                     const int64_t* __restrict__ boff, int cbits, unsigned long long* out) {
  typedef cub::BlockRadixSort<unsigned long long, BIG_BT, BIG_IPT_S> BS;
  typedef cub::BlockRadixSort<unsigned long long, BIG_BT, BIG_IPT_L> BL;
  __shared__ union {
    typename BS::TempStorage s;
    typename BL::TempStorage l;
  } ts;
  for (int64_t i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int c = big[i];
    const int64_t d = m.rowlen[c];  // block-uniform
    if (d > BIG_BLOCK_MAX) continue;
    if (d <= (int64_t)BIG_BT * BIG_IPT_S)
      big_sort_row<BIG_IPT_S>(m, c, d, boff[i], cbits, out, &ts);
    else
      big_sort_row<BIG_IPT_L>(m, c, d, boff[i], cbits, out, &ts);
    __syncthreads();  // the temp storage is reused by the next row
  }
}

// Counting pass of a two-pass contraction, rows of up to BIG_BLOCK_MAX
// entries: the number of distinct coarse neighbours (self loops excluded) by
// one insertion pass into a shared-memory hash set (load factor <= 1/2)
// instead of a radix sort -- the second pass sorts.
constexpr int BIG_HASH_BITS = 13;
constexpr int BIG_HASH = 1 << BIG_HASH_BITS;
static_assert(BIG_HASH >= 2 * BIG_BLOCK_MAX, "hash set load factor");

__global__ void __launch_bounds__(BIG_BT)
    k_big_count_block(RowMerge m, const int32_t* __restrict__ big, int64_t nbig) {
  __shared__ unsigned tab[BIG_HASH];
  __shared__ int s_cnt;
  for (int i = threadIdx.x; i < BIG_HASH; i += BIG_BT) tab[i] = 0xffffffffu;
  for (int64_t i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int c = big[i];
    const int64_t d = m.rowlen[c];  // block-uniform
    if (d > BIG_BLOCK_MAX) continue;
    const int a = m.mem_a[c], b = m.mem_b[c];
    const int64_t da = m.offs[a + 1] - m.offs[a];
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
    int mine = 0;
    for (int64_t idx = threadIdx.x; idx < d; idx += BIG_BT) {
      const unsigned long long k = merged_key(m, c, idx, a, b, da);
      if (k == ~0ull) continue;  // self loop
      const unsigned cv = (unsigned)(k >> 32);
      unsigned h = (cv * 0x9e3779b1u) >> (32 - BIG_HASH_BITS);  // Fibonacci hashing: top bits
      while (true) {
        const unsigned old = atomicCAS(&tab[h], 0xffffffffu, cv);
        if (old == 0xffffffffu) {
          ++mine;
          break;
        }
        if (old == cv) break;
        h = (h + 1) & (BIG_HASH - 1);
      }
    }
    mine = __reduce_add_sync(0xffffffffu, mine);
    if ((threadIdx.x & 31) == 0 && mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) m.cdeg[c] = s_cnt;
    for (int q = threadIdx.x; q < BIG_HASH; q += BIG_BT) tab[q] = 0xffffffffu;
    __syncthreads();
  }
}

// segment ends for the device-wide sort: rows sorted on chip get empty segments
__global__ void k_big_ends(const int32_t* __restrict__ big, int64_t nbig,
                           const int64_t* __restrict__ rowlen, const int64_t* __restrict__ off,
                           int64_t* end) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbig;
       i += (int64_t)gridDim.x * blockDim.x)
    end[i] = rowlen[big[i]] > BIG_BLOCK_MAX ? off[i + 1] : off[i];
}

__global__ void k_big_len(const int32_t* __restrict__ big, int64_t nbig,
                          const int64_t* __restrict__ rowlen, int64_t* len) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nbig; i += stride)
    len[i] = rowlen[big[i]];
}

__global__ void __launch_bounds__(256)
    k_big_dedup(RowMerge m, const int32_t* __restrict__ big, int64_t nbig,
                const int64_t* __restrict__ boff, const unsigned long long* __restrict__ keys,
                int64_t min_len) {
  typedef cub::BlockScan<int, 256> BS;
  __shared__ typename BS::TempStorage ts;
  __shared__ int s_out;
  for (int64_t i = blockIdx.x; i < nbig; i += gridDim.x) {
    const int c = big[i];
    const int64_t o = boff[i], d = m.rowlen[c];
    if (d <= min_len) continue;  // counted by k_big_count_block
    const int64_t base = m.toff[c];
    if (threadIdx.x == 0) s_out = 0;
    __syncthreads();
    for (int64_t j0 = 0; j0 < d; j0 += 256) {
      const int64_t j = j0 + threadIdx.x;
      bool head = false;
      unsigned cv = 0;
      long long sum = 0;
      if (j < d) {
        const unsigned long long k = keys[o + j];
        cv = (unsigned)(k >> 32);
        head = k != ~0ull && (j == 0 || (unsigned)(keys[o + j - 1] >> 32) != cv);
        if (head)
          for (int64_t q = j; q < d && keys[o + q] != ~0ull && (unsigned)(keys[o + q] >> 32) == cv; ++q)
            sum += (long long)(keys[o + q] & 0xffffffffu);
      }
      int rank, total;
      BS(ts).ExclusiveSum(head ? 1 : 0, rank, total);
      const int run = s_out;
      if (head) {
        if (sum > 2147483647LL) atomicOr(m.overflow, 2u);
        if (m.tadj) {
          m.tadj[base + run + rank] = (int32_t)cv;
          m.tew[base + run + rank] = (int32_t)sum;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0) s_out = run + total;
      __syncthreads();
    }
    if (threadIdx.x == 0) m.cdeg[c] = s_out;
    __syncthreads();
  }
}

__global__ void k_rebase(const int64_t* __restrict__ off, int64_t cnt, int64_t base, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = off[i] - base;
}

__global__ void k_copy_rows(const int64_t* __restrict__ toff, const int64_t* __restrict__ coffs,
                            const int32_t* __restrict__ tadj, const int32_t* __restrict__ tew,
                            int32_t* cadj, int32_t* cew, int64_t nc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t ws = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = w0; c < nc; c += ws) {
    const int64_t s = toff[c], o = coffs[c], d = coffs[c + 1] - o;
    for (int64_t j = lane; j < d; j += 32) {
      cadj[o + j] = tadj[s + j];
      cew[o + j] = tew[s + j];
    }
  }
}

static double wall_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
// Long merged rows (> 256 entries): grouped gather / sort / dedup (see
// device_contract). setup() sizes the groups once; run() merges them for a
// RowMerge (counting pass, merging pass, or single pass).
struct LongRows {
  Ctx& c;
  int32_t* big_p;
  int64_t nb;
  const int64_t* rowlen_p;
  int64_t nc;
  struct Grp { int64_t s0, ns, base, cnt; };
  std::vector<Grp> groups;
  DBuf<int64_t> boff, rel, bend;
  DBuf<unsigned long long> bk, bk2;
  int cbits = 1;
  LongRows(Ctx& cc, int32_t* bp, int64_t n_big, const int64_t* rl, int64_t ncoarse)
      : c(cc), big_p(bp), nb(n_big), rowlen_p(rl), nc(ncoarse) {
    // Long rows are gathered, sorted and deduplicated in groups of rows of at
    // most CH entries (one row may exceed it alone): the key buffers stay a
    // few GB however dense the level (the dense coarse levels of R-MAT 2^27
    // route ~4 G entries through here), and CUB's 32-bit item counts hold.
    const int64_t CH = (int64_t)1 << 28;
    while ((1LL << cbits) < nc) ++cbits;
    if (nb <= 0) return;
    DBuf<int64_t> blen(nb + 1, c.stream);
    boff.alloc(nb + 1, c.stream);
    dzero(c, blen.get() + nb, 1);
    launch(c, "big_len", 16.0 * nb, [&] {
      k_big_len<<<grid_for(c, nb, 256), 256, 0, c.stream>>>(big_p, nb, rowlen_p, blen.get());
    });
    {
      size_t tmp = 0;
      CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, blen.get(), boff.get(), (int)(nb + 1), c.stream));
      void* p = c.cub_scratch(tmp);
      launch(c, "big_scan", 16.0 * nb, [&] {
        CK(cub::DeviceScan::ExclusiveSum(p, tmp, blen.get(), boff.get(), (int)(nb + 1), c.stream));
      });
    }
    int64_t BT = 0;
    d2h(c, &BT, boff.get() + nb, 1);
    c.sync();
    if (BT <= CH) {
      groups.push_back({0, nb, 0, BT});
    } else {
      std::vector<int64_t> hb(nb + 1);
      d2h(c, hb.data(), boff.get(), nb + 1);
      c.sync();
      int64_t s0 = 0;
      while (s0 < nb) {
        int64_t s1 = s0 + 1;
        while (s1 < nb && hb[s1 + 1] - hb[s0] <= CH) ++s1;
        groups.push_back({s0, s1 - s0, hb[s0], hb[s1] - hb[s0]});
        s0 = s1;
      }
    }
    int64_t maxcnt = 0;
    for (const Grp& q : groups) maxcnt = std::max(maxcnt, q.cnt);
    bk.alloc(maxcnt, c.stream);
    bk2.alloc(maxcnt, c.stream);
    bend.alloc(nb + 1, c.stream);
    if (groups.size() > 1) rel.alloc(nb + 1, c.stream);
  }
  void run(const RowMerge& r) {
    for (const Grp& q : groups) {
      JET_REQUIRE(q.cnt < (int64_t)INT_MAX, JET_EUNSUPPORTED, "merged coarse row longer than 2^31 entries");
      const int64_t* off = boff.get();
      if (groups.size() > 1) {
        launch(c, "big_rebase", 16.0 * q.ns, [&] {
          k_rebase<<<grid_for(c, q.ns + 1, 256), 256, 0, c.stream>>>(boff.get() + q.s0, q.ns + 1, q.base,
                                                                     rel.get());
        });
        off = rel.get();
      }
      launch(c, "big_gather", 20.0 * q.cnt, [&] {
        k_big_gather<<<grid_for(c, q.ns * 256, 256), 256, 0, c.stream>>>(r, big_p + q.s0, q.ns, off,
                                                                         bk.get(), BIG_BLOCK_MAX);
      });
      launch(c, "big_ends", 16.0 * q.ns, [&] {
        k_big_ends<<<grid_for(c, q.ns, 256), 256, 0, c.stream>>>(big_p + q.s0, q.ns, rowlen_p, off,
                                                                 bend.get());
      });
      size_t tmp = 0;
      CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, bk.get(), bk2.get(), (int)q.cnt, (int)q.ns, off,
                                            bend.get(), c.stream));
      void* p = c.cub_scratch(tmp);
      launch(c, "big_sort", 32.0 * q.cnt, [&] {
        CK(cub::DeviceSegmentedSort::SortKeys(p, tmp, bk.get(), bk2.get(), (int)q.cnt, (int)q.ns, off,
                                              bend.get(), c.stream));
      });
      const bool counting = r.tadj == nullptr;  // first pass of a two-pass contraction
      if (counting) {
        launch(c, "big_count_block", 12.0 * q.cnt, [&] {
          k_big_count_block<<<grid_for(c, q.ns * BIG_BT, BIG_BT), BIG_BT, 0, c.stream>>>(r, big_p + q.s0,
                                                                                        q.ns);
        });
      } else {
        launch(c, "big_sort_block", 20.0 * q.cnt, [&] {
          k_big_sort_block<<<grid_for(c, q.ns * BIG_BT, BIG_BT), BIG_BT, 0, c.stream>>>(
              r, big_p + q.s0, q.ns, off, cbits, bk2.get());
        });
      }
      launch(c, "big_dedup", 16.0 * q.cnt, [&] {
        k_big_dedup<<<grid_for(c, q.ns * 256, 256), 256, 0, c.stream>>>(
            r, big_p + q.s0, q.ns, off, bk2.get(), counting ? BIG_BLOCK_MAX : 0);
      });
    }
  }
};

std::unique_ptr<DGraph> device_contract(Ctx& c, const DGraph& g, const int32_t* partner,
                                        int32_t* vmap, bool two_pass) {
  static const bool dbg = getenv("JET_COARSEN_TIMES") && getenv("JET_COARSEN_TIMES")[0] == '2';
  double tm = dbg ? wall_s() : 0;
  auto mark = [&](const char* what) {
    if (!dbg) return;
    c.sync();
    const double t = wall_s();
    fprintf(stderr, "  contract %s %.2fms\n", what, (t - tm) * 1e3);
    tm = t;
  };
  const int64_t n = g.n;
  int32_t* flag_p = c.scratch<int32_t>(0, n);
  int32_t* cid_p = c.scratch<int32_t>(1, n);
  launch(c, "is_rep", 8.0 * n, [&] {
    k_is_rep<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, flag_p);
  });
  if (!small_exclusive_sum(c, "rep_scan", flag_p, cid_p, (int64_t)(n)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag_p, cid_p, (int)n, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "rep_scan", 8.0 * n, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, flag_p, cid_p, (int)n, c.stream));
    });
  }
  int32_t last[2];
  d2h(c, &last[0], cid_p + n - 1, 1);
  d2h(c, &last[1], flag_p + n - 1, 1);
  c.sync();
  const int64_t nc = (int64_t)last[0] + last[1];
  mark("ids");
  auto cg_ = std::make_unique<DGraph>();
  cg_->n = nc;
  cg_->vw.alloc(nc, c.stream);
  int32_t* mem_a_p = c.scratch<int32_t>(2, nc);
  int32_t* mem_b_p = c.scratch<int32_t>(3, nc);
  int64_t* rowlen_p = c.scratch<int64_t>(4, nc + 1);
  int64_t* toff_p = c.scratch<int64_t>(5, nc + 1);
  int64_t* cdeg_p = c.scratch<int64_t>(6, nc + 1);
  DBuf<unsigned> ovf(1, c.stream);
  dzero(c, ovf.get(), 1);
  CoarseMap cm{partner, cid_p, g.offs.get(), g.vw.get(), vmap, cg_->vw.get(),
               mem_a_p, mem_b_p, rowlen_p, ovf.get()};
  launch(c, "coarse_map", 24.0 * n, [&] {
    k_coarse_map<<<grid_for(c, n, 256), 256, 0, c.stream>>>(cm, n);
  });
  dzero(c, rowlen_p + nc, 1);
  dzero(c, cdeg_p + nc, 1);
  if (!small_exclusive_sum(c, "rowlen_scan", rowlen_p, toff_p, (int64_t)(nc + 1)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, rowlen_p, toff_p, (int)(nc + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "rowlen_scan", 16.0 * nc, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, rowlen_p, toff_p, (int)(nc + 1), c.stream));
    });
  }
  // the merged rows concatenate both members' rows: their lengths sum to the
  // fine graph's entry count (no need to read the scan's total back).
  // Two-pass (memory-tight hierarchies): the first pass only counts each
  // coarse row's distinct entries, the second merges straight into the
  // exact-size coarse arrays -- no fine-sized staging copy (34 GB on R-MAT
  // 2^27) at the price of merging every row twice.
  const int64_t T = g.nnz;
  mark("map+scan");
  int32_t* tadj_p = two_pass ? nullptr : c.scratch<int32_t>(7, T);
  int32_t* tew_p = two_pass ? nullptr : c.scratch<int32_t>(8, T);
  int32_t* big_p = c.scratch<int32_t>(9, nc);
  DBuf<unsigned long long> big_cnt(1, c.stream);
  dzero(c, big_cnt.get(), 1);
  RowMerge rm{g.offs.get(), g.adj.get(), g.ew.get(), vmap, mem_a_p, mem_b_p, toff_p,
              rowlen_p, tadj_p, tew_p, cdeg_p, big_p, big_cnt.get(), ovf.get(), nc, 1};
  launch(c, "contract_rows", 12.0 * g.nnz + 8.0 * T + 16.0 * nc, [&] {
    k_merge_rows<<<grid_for(c, nc * 32, 256), 256, 0, c.stream>>>(rm);
  });
  // final offsets: scanned right away, read back together with the long-row
  // count -- one host wait per level when there are no long rows (meshes);
  // otherwise the long rows are merged and the scan is redone
  cg_->offs.alloc(nc + 1, c.stream);
  auto cdeg_scan = [&] {
    if (small_exclusive_sum(c, "cdeg_scan", cdeg_p, cg_->offs.get(), (int64_t)(nc + 1))) return;
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cdeg_p, cg_->offs.get(), (int)(nc + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "cdeg_scan", 16.0 * nc, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, cdeg_p, cg_->offs.get(), (int)(nc + 1), c.stream));
    });
  };
  cdeg_scan();
  unsigned long long nbig = 0;
  int64_t cnnz = 0;
  unsigned hovf = 0;
  d2h(c, &nbig, big_cnt.get(), 1);
  d2h(c, &cnnz, cg_->offs.get() + nc, 1);
  d2h(c, &hovf, ovf.get(), 1);
  c.sync();
  mark("alloc+rows");
  LongRows longrows(c, big_p, (int64_t)nbig, rowlen_p, nc);
  if (nbig) {
    longrows.run(rm);
    cdeg_scan();
    d2h(c, &cnnz, cg_->offs.get() + nc, 1);
    d2h(c, &hovf, ovf.get(), 1);
    c.sync();
  }
  JET_REQUIRE(!(hovf & 1u), JET_EUNSUPPORTED, "coarse vertex weight exceeds int32");
  JET_REQUIRE(!(hovf & 2u), JET_EUNSUPPORTED, "coarse edge weight exceeds int32");
  cg_->nnz = cnnz;
  cg_->adj.alloc(cnnz > 0 ? cnnz : 1, c.stream);
  cg_->ew.alloc(cnnz > 0 ? cnnz : 1, c.stream);
  mark("big+offs");
  if (two_pass) {
    RowMerge r2 = rm;  // merge again, straight into the coarse arrays
    r2.toff = cg_->offs.get();
    r2.tadj = cg_->adj.get();
    r2.tew = cg_->ew.get();
    r2.collect_big = 0;
    launch(c, "contract_rows", 12.0 * g.nnz + 8.0 * cnnz + 16.0 * nc, [&] {
      k_merge_rows<<<grid_for(c, nc * 32, 256), 256, 0, c.stream>>>(r2);
    });
    longrows.run(r2);
  } else {
    launch(c, "copy_rows", 16.0 * cnnz + 16.0 * nc, [&] {
      k_copy_rows<<<grid_for(c, nc * 32, 256), 256, 0, c.stream>>>(toff_p, cg_->offs.get(), tadj_p,
                                                                  tew_p, cg_->adj.get(), cg_->ew.get(), nc);
    });
  }
  mark("copy");
  finalize_graph(c, *cg_);
  mark("finalize");
  return cg_;
}

// ===========================================================================
// 1D-distributed finest level: every rank holds the rows of
// its block [lo, hi) (DGraph::partial) plus the complete offsets and vertex
// weights. The throughput-mode matching and the contraction run on the owned
// rows with exchanges over the communicator, and produce exactly the
// replicated run's matching and coarse level -- which every rank then holds
// whole (the coarser levels are small enough to replicate, as north_star's
// "coarse levels gathered" allows).
// ===========================================================================
namespace {

__global__ void k_pack_props(const int32_t* __restrict__ elist, const unsigned long long* __restrict__ ecnt,
                             const int32_t* __restrict__ prop, int2* out) {
  const int64_t cnt = (int64_t)*ecnt;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int v = elist[i];
    out[i] = make_int2(v, prop[v]);
  }
}

__global__ void k_unpack_props(const int2* __restrict__ in, int64_t cnt, int32_t* prop) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x)
    prop[in[i].x] = in[i].y;
}

// mutual proposals among this rank's proposers (v < u: the pair's owner)
__global__ void k_accept_pairs(const int32_t* __restrict__ elist, const unsigned long long* __restrict__ ecnt,
                               const int32_t* __restrict__ prop, int2* pairs,
                               unsigned long long* npairs) {
  const int64_t cnt = (int64_t)*ecnt;
  const int64_t lim = (cnt + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < lim;
       i += (int64_t)gridDim.x * blockDim.x) {
    int v = 0, u = 0;
    bool take = false;
    if (i < cnt) {
      v = elist[i];
      u = prop[v];
      take = v < u && prop[u] == v;
    }
    const unsigned m = __ballot_sync(0xffffffffu, take);
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(npairs, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (take) pairs[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = make_int2(v, u);
  }
}

__global__ void k_unpack_pairs(const int2* __restrict__ in, int64_t cnt, int32_t* partner) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    partner[in[i].x] = in[i].y;
    partner[in[i].y] = in[i].x;
  }
}

// [first position >= lo, first position >= hi) of an ascending list
__global__ void k_list_range(const int32_t* __restrict__ list, int64_t cnt, int64_t lo, int64_t hi,
                             int64_t* out) {
  if (threadIdx.x > 1) return;
  const int64_t key = threadIdx.x == 0 ? lo : hi;
  int64_t a = 0, b = cnt;
  while (a < b) {
    const int64_t m = (a + b) / 2;
    if (list[m] < key) a = m + 1;
    else b = m;
  }
  out[threadIdx.x] = a;
}

// this rank's free vertices
__global__ void k_owned_free(const int32_t* __restrict__ partner, int64_t lo, int64_t hi,
                             int32_t* out, unsigned long long* cnt) {
  const int64_t span = (hi - lo + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < span;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = lo + i;
    const bool f = v < hi && partner[v] < 0;
    const unsigned m = __ballot_sync(0xffffffffu, f);
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (f) out[base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u))] = (int32_t)v;
  }
}

// owned rows b whose representative partner[b] < b lives on a lower rank
__global__ void k_export_rows(const int32_t* __restrict__ partner, const int64_t* __restrict__ offs,
                              int64_t lo, int64_t hi, int32_t* ids, int64_t* lens,
                              unsigned long long* cnt) {
  const int64_t span = (hi - lo + 31) / 32 * 32;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < span;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = lo + i;
    bool f = false;
    if (b < hi) {
      const int a = partner[b];
      f = a < b && a < lo;
    }
    const unsigned m = __ballot_sync(0xffffffffu, f);
    unsigned long long base = 0;
    if ((threadIdx.x & 31) == 0 && m) base = atomicAdd(cnt, (unsigned long long)__popc(m));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (f) {
      const unsigned long long q = base + __popc(m & ((1u << (threadIdx.x & 31)) - 1u));
      ids[q] = (int32_t)b;
      lens[q] = offs[b + 1] - offs[b];
    }
  }
}

__global__ void k_gather_rows(const int32_t* __restrict__ ids, const int64_t* __restrict__ eoff,
                              int64_t nr, GView g, int2* out) {
  for (int64_t r = blockIdx.x; r < nr; r += gridDim.x) {
    const int b = ids[r];
    const int64_t s = g.offs[b], d = g.offs[b + 1] - s, o = eoff[r];
    for (int64_t j = threadIdx.x; j < d; j += blockDim.x) out[o + j] = make_int2(g.adj[s + j], g.ew[s + j]);
  }
}

// imported rows: position of each row's entries, split into adj / ew
__global__ void k_import_rows(const int32_t* __restrict__ ids, const int64_t* __restrict__ eoff,
                              int64_t nr, const int2* __restrict__ ent, int64_t ne, int64_t* imp_pos,
                              int32_t* imp_adj, int32_t* imp_ew) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nr; r += stride)
    imp_pos[ids[r]] = eoff[r];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < ne; e += stride) {
    imp_adj[e] = ent[e].x;
    imp_ew[e] = ent[e].y;
  }
}

// owner rank of each export's representative; per-destination counts
__global__ void k_export_dest(const int32_t* __restrict__ ids, int64_t nx,
                              const int32_t* __restrict__ partner, const int64_t* __restrict__ bnd,
                              int size, int32_t* dest, unsigned long long* dcount) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nx;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = partner[ids[i]];
    int lo = 0, hi = size;  // last r with bnd[r] <= a
    while (hi - lo > 1) {
      const int m = (lo + hi) / 2;
      if (bnd[m] <= a) lo = m;
      else hi = m;
    }
    dest[i] = lo;
    atomicAdd(dcount + lo, 1ull);
  }
}

// exports grouped by destination rank (order inside a group is immaterial:
// the receiver indexes rows by id)
__global__ void k_export_group(const int32_t* __restrict__ ids, const int64_t* __restrict__ lens,
                               const int32_t* __restrict__ dest, int64_t nx,
                               const int64_t* __restrict__ doff, unsigned long long* dfill,
                               int32_t* gids, int64_t* glens) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nx;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int d = dest[i];
    const int64_t q = doff[d] + (int64_t)atomicAdd(dfill + d, 1ull);
    gids[q] = ids[i];
    glens[q] = lens[i];
  }
}

// gather `bytes` of every rank, rank-major, into `out` (resized); total bytes
int64_t gather_all(Ctx& c, const void* d, int64_t bytes, DBuf<uint8_t>& out) {
  std::vector<int64_t> counts;
  c.comm->allgatherv(c, d, bytes, out, counts);
  int64_t t = 0;
  for (int64_t x : counts) t += x;
  return t;
}

}  // namespace

// The replicated device_match_fast, round for round, over the owned rows.
static void device_match_fast_dist(Ctx& c, const DGraph& g, int32_t* partner) {
  JET_REQUIRE(c.comm, JET_EINVAL, "a distributed level needs a communicator");
  const int64_t n = g.n, lo = g.row_lo, hi = g.row_hi;
  launch(c, "fill", 4.0 * n, [&] {
    k_fill<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, -1);
  });
  const GView gv = view(g);
  int32_t* prop_p = c.scratch<int32_t>(10, n);
  int32_t* elist_p = c.scratch<int32_t>(11, std::max<int64_t>(1, hi - lo));
  DBuf<unsigned long long> cnt(4, c.stream);
  DBuf<int2> send(std::max<int64_t>(1, hi - lo), c.stream);
  DBuf<uint8_t> recv;
  // this rank's hub rows (the hub tier list restricted to the block)
  const int64_t nh_all = g.bin_cnt[BIN_BLOCK];
  const int32_t* hubs = nullptr;
  int64_t nh = 0;
  if (nh_all) {
    DBuf<int64_t> r(2, c.stream);
    const int32_t* hl = tier_list(g, BIN_BLOCK);
    JET_REQUIRE(hl, JET_EINTERNAL, "identity hub tier on a distributed level");
    k_list_range<<<1, 32, 0, c.stream>>>(hl, nh_all, lo, hi, r.get());
    CK(cudaGetLastError());
    int64_t hr[2];
    d2h(c, hr, r.get(), 2);
    c.sync();
    hubs = hl + hr[0];
    nh = hr[1] - hr[0];
  }
  constexpr int MAXR = 48, RG = 4;
  int low_rounds = 0;
  bool quit = false;
  for (int round = 0; round < MAXR; ++round) {
    dzero(c, cnt.get(), 4);
    const unsigned salt = 0x5bd1e995u * (unsigned)(round + 1);
    launch(c, "propose", (g.unit_ew ? 8.0 : 12.0) * (double)g.local_nnz(), [&] {
      if (g.unit_ew)
        k_propose_fast<true><<<grid_res(c, k_propose_fast<true>, hi - lo, 256), 256, 0, c.stream>>>(
            gv, hi, partner, prop_p, elist_p, cnt.get(), salt, nullptr, lo);
      else
        k_propose_fast<false><<<grid_res(c, k_propose_fast<false>, hi - lo, 256), 256, 0, c.stream>>>(
            gv, hi, partner, prop_p, elist_p, cnt.get(), salt, nullptr, lo);
    });
    if (nh) {
      const unsigned hg = (unsigned)std::min<int64_t>(nh, 4LL * c.num_sms);
      launch(c, "propose_hub", 0.0, [&] {
        if (g.unit_ew)
          k_propose_fast_hub<true><<<hg, 256, 0, c.stream>>>(gv, hubs, nh, partner, prop_p, elist_p,
                                                             cnt.get(), salt, nullptr);
        else
          k_propose_fast_hub<false><<<hg, 256, 0, c.stream>>>(gv, hubs, nh, partner, prop_p, elist_p,
                                                              cnt.get(), salt, nullptr);
      });
    }
    // halo 1: every rank's proposals
    unsigned long long np_local = 0;
    d2h(c, &np_local, cnt.get(), 1);
    c.sync();
    launch(c, "shard_pack", 8.0 * (double)np_local, [&] {
      k_pack_props<<<grid_for(c, (int64_t)np_local, 256), 256, 0, c.stream>>>(elist_p, cnt.get(), prop_p,
                                                                             send.get());
    });
    const int64_t np = gather_all(c, send.get(), (int64_t)np_local * 8, recv) / 8;
    launch(c, "shard_unpack", 8.0 * (double)np, [&] {
      k_unpack_props<<<grid_for(c, np, 256), 256, 0, c.stream>>>((const int2*)recv.get(), np, prop_p);
    });
    // accept the mutual ones this rank owns; halo 2: every rank's pairs
    launch(c, "accept", 12.0 * (double)np_local, [&] {
      k_accept_pairs<<<grid_for(c, (int64_t)np_local, 256), 256, 0, c.stream>>>(
          elist_p, cnt.get(), prop_p, send.get(), cnt.get() + 1);
    });
    unsigned long long pr_local = 0;
    d2h(c, &pr_local, cnt.get() + 1, 1);
    c.sync();
    const int64_t pr = gather_all(c, send.get(), (int64_t)pr_local * 8, recv) / 8;
    launch(c, "shard_unpack", 8.0 * (double)pr, [&] {
      k_unpack_pairs<<<grid_for(c, pr, 256), 256, 0, c.stream>>>((const int2*)recv.get(), pr, partner);
    });
    // the replicated path's stopping rule (device_match_fast), same rounds
    if (np == 0 || pr == 0) break;
    low_rounds = (unsigned long long)pr * 200 < (unsigned long long)np ? low_rounds + 1 : 0;
    quit |= low_rounds >= 2;
    if (quit && round % RG == RG - 1) break;
  }
  // leaf pairing of every rank's leftovers, sorted and paired on every rank
  int32_t* left_p = c.scratch<int32_t>(13, std::max<int64_t>(1, hi - lo));
  dzero(c, cnt.get(), 1);
  launch(c, "th_leftovers", 8.0 * (hi - lo), [&] {
    k_owned_free<<<grid_for(c, hi - lo, 256), 256, 0, c.stream>>>(partner, lo, hi, left_p, cnt.get());
  });
  unsigned long long nl_local = 0;
  d2h(c, &nl_local, cnt.get(), 1);
  c.sync();
  int vb = 1;
  while ((1LL << vb) <= n) ++vb;
  DBuf<unsigned long long> kl(std::max<unsigned long long>(1, nl_local), c.stream);
  if (nl_local)
    launch(c, "leaf_keys", 16.0 * (double)nl_local, [&] {
      k_leaf_keys<<<grid_for(c, (int64_t)nl_local * 32, 256), 256, 0, c.stream>>>(gv, left_p, (int64_t)nl_local,
                                                                                 vb, kl.get());
    });
  const int64_t nl = gather_all(c, kl.get(), (int64_t)nl_local * 8, recv) / 8;
  if (nl >= 2) {
    DBuf<unsigned long long> k1(nl, c.stream);
    const unsigned long long* k0 = (const unsigned long long*)recv.get();
    size_t tmp = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1.get(), (int)nl, 0, 2 * vb, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "leaf_sort", 32.0 * nl, [&] {
      CK(cub::DeviceRadixSort::SortKeys(p, tmp, k0, k1.get(), (int)nl, 0, 2 * vb, c.stream));
    });
    launch(c, "leaf_pair", 16.0 * nl, [&] {
      k_leaf_pair<<<grid_for(c, nl, 256), 256, 0, c.stream>>>(k1.get(), nl, vb, n, partner);
    });
  }
  launch(c, "singletons", 8.0 * n, [&] {
    k_singletons<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n);
  });
}

// The contraction of a distributed level: every rank merges the coarse rows
// whose representative it owns (importing the partner rows that live on
// higher ranks). Coarse ids are ascending in the representative, so the
// ranks' coarse ranges are contiguous and in rank order: a large coarse level
// stays distributed on those ranges (complete offsets and vertex weights,
// own rows), a small one is gathered whole. Either way it equals
// device_contract's result.
static std::unique_ptr<DGraph> device_contract_dist(Ctx& c, const DGraph& g, const int32_t* partner,
                                                    int32_t* vmap) {
  JET_REQUIRE(c.comm, JET_EINVAL, "a distributed level needs a communicator");
  const int64_t n = g.n, lo = g.row_lo, hi = g.row_hi;
  int32_t* flag_p = c.scratch<int32_t>(0, n);
  int32_t* cid_p = c.scratch<int32_t>(1, n);
  launch(c, "is_rep", 8.0 * n, [&] {
    k_is_rep<<<grid_for(c, n, 256), 256, 0, c.stream>>>(partner, n, flag_p);
  });
  if (!small_exclusive_sum(c, "rep_scan", flag_p, cid_p, (int64_t)(n)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag_p, cid_p, (int)n, c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "rep_scan", 8.0 * n, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, flag_p, cid_p, (int)n, c.stream));
    });
  }
  int32_t last[4] = {0, 0, 0, 0};
  d2h(c, &last[0], cid_p + n - 1, 1);
  d2h(c, &last[1], flag_p + n - 1, 1);
  if (lo < n) d2h(c, &last[2], cid_p + lo, 1);
  if (hi < n) d2h(c, &last[3], cid_p + hi, 1);
  c.sync();
  const int64_t nc = (int64_t)last[0] + last[1];
  const int64_t c_lo = lo < n ? last[2] : nc, c_hi = hi < n ? last[3] : nc;
  auto cg_ = std::make_unique<DGraph>();
  cg_->n = nc;
  cg_->vw.alloc(nc, c.stream);
  int32_t* mem_a_p = c.scratch<int32_t>(2, nc);
  int32_t* mem_b_p = c.scratch<int32_t>(3, nc);
  int64_t* rowlen_p = c.scratch<int64_t>(4, nc + 1);
  int64_t* cdeg_p = c.scratch<int64_t>(6, nc + 1);
  DBuf<unsigned> ovf(1, c.stream);
  dzero(c, ovf.get(), 1);
  CoarseMap cm{partner, cid_p, g.offs.get(), g.vw.get(), vmap, cg_->vw.get(),
               mem_a_p, mem_b_p, rowlen_p, ovf.get()};
  launch(c, "coarse_map", 24.0 * n, [&] {
    k_coarse_map<<<grid_for(c, n, 256), 256, 0, c.stream>>>(cm, n);
  });
  // import the partner rows of this rank's representatives
  DBuf<int32_t> xids(std::max<int64_t>(1, hi - lo), c.stream);
  DBuf<int64_t> xlen(std::max<int64_t>(1, hi - lo) + 1, c.stream), xoff(std::max<int64_t>(1, hi - lo) + 1, c.stream);
  DBuf<unsigned long long> xc(1, c.stream);
  dzero(c, xc.get(), 1);
  launch(c, "export_rows", 12.0 * (hi - lo), [&] {
    k_export_rows<<<grid_for(c, hi - lo, 256), 256, 0, c.stream>>>(partner, g.offs.get(), lo, hi, xids.get(),
                                                                   xlen.get(), xc.get());
  });
  unsigned long long nx = 0;
  d2h(c, &nx, xc.get(), 1);
  c.sync();
  // group the exports by the rank that owns their representative and send
  // each rank only its own imports (all-to-all)
  const int size = c.comm->size;
  std::vector<int64_t> bnd(size + 1);
  {
    DBuf<uint8_t> rl;
    DBuf<int64_t> mylo(1, c.stream);
    h2d(c, mylo.get(), &lo, 1);
    gather_all(c, mylo.get(), 8, rl);
    d2h(c, bnd.data(), reinterpret_cast<const int64_t*>(rl.get()), size);
    c.sync();
    bnd[size] = n;
  }
  DBuf<int64_t> bnd_d(size + 1, c.stream), doff_d(size + 1, c.stream);
  h2d(c, bnd_d.get(), bnd.data(), size + 1);
  DBuf<int32_t> xdest(std::max<int64_t>(1, (int64_t)nx), c.stream), gids(std::max<int64_t>(1, (int64_t)nx), c.stream);
  DBuf<int64_t> glens(std::max<int64_t>(1, (int64_t)nx) + 1, c.stream);
  DBuf<unsigned long long> dcnt(2 * size, c.stream);
  dzero(c, dcnt.get(), 2 * size);
  if (nx)
    launch(c, "export_dest", 16.0 * (double)nx, [&] {
      k_export_dest<<<grid_for(c, (int64_t)nx, 256), 256, 0, c.stream>>>(xids.get(), (int64_t)nx, partner,
                                                                        bnd_d.get(), size, xdest.get(),
                                                                        dcnt.get());
    });
  std::vector<unsigned long long> hcnt(size);
  d2h(c, hcnt.data(), dcnt.get(), size);
  c.sync();
  std::vector<int64_t> doff(size + 1, 0), scnt(size);
  for (int r = 0; r < size; ++r) doff[r + 1] = doff[r] + (int64_t)hcnt[r];
  h2d(c, doff_d.get(), doff.data(), size + 1);
  if (nx)
    launch(c, "export_group", 24.0 * (double)nx, [&] {
      k_export_group<<<grid_for(c, (int64_t)nx, 256), 256, 0, c.stream>>>(
          xids.get(), xlen.get(), xdest.get(), (int64_t)nx, doff_d.get(), dcnt.get() + size, gids.get(),
          glens.get());
    });
  int64_t xe = 0;
  {
    dzero(c, glens.get() + nx, 1);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, glens.get(), xoff.get(), (int)(nx + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "export_scan", 16.0 * (double)nx, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, glens.get(), xoff.get(), (int)(nx + 1), c.stream));
    });
  }
  std::vector<int64_t> eb(size + 1);  // entry offsets at the group boundaries
  for (int r = 0; r <= size; ++r) d2h(c, &eb[r], xoff.get() + doff[r], 1);
  c.sync();
  xe = eb[size];
  DBuf<int2> xent(std::max<int64_t>(1, xe), c.stream);
  const GView gv = view(g);
  if (nx)
    launch(c, "export_gather", 16.0 * (double)xe, [&] {
      k_gather_rows<<<grid_for(c, (int64_t)nx * 128, 128), 128, 0, c.stream>>>(gids.get(), xoff.get(),
                                                                             (int64_t)nx, gv, xent.get());
    });
  DBuf<uint8_t> r_ids, r_lens, r_ent;
  std::vector<int64_t> rc;
  for (int r = 0; r < size; ++r) scnt[r] = (doff[r + 1] - doff[r]) * 4;
  c.comm->alltoallv(c, gids.get(), scnt, r_ids, rc);
  int64_t nimp = 0;
  for (int64_t x : rc) nimp += x / 4;
  for (int r = 0; r < size; ++r) scnt[r] = (doff[r + 1] - doff[r]) * 8;
  c.comm->alltoallv(c, glens.get(), scnt, r_lens, rc);
  for (int r = 0; r < size; ++r) scnt[r] = (eb[r + 1] - eb[r]) * 8;
  c.comm->alltoallv(c, xent.get(), scnt, r_ent, rc);
  int64_t ne = 0;
  for (int64_t x : rc) ne += x / 8;
  DBuf<int64_t> ioff(nimp + 1, c.stream);
  DBuf<int64_t> imp_pos(n, c.stream);
  DBuf<int32_t> imp_adj(std::max<int64_t>(1, ne), c.stream), imp_ew(std::max<int64_t>(1, ne), c.stream);
  if (nimp) {
    DBuf<int64_t> l2(nimp + 1, c.stream);
    CK(cudaMemcpyAsync(l2.get(), r_lens.get(), (size_t)nimp * 8, cudaMemcpyDeviceToDevice, c.stream));
    dzero(c, l2.get() + nimp, 1);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, l2.get(), ioff.get(), (int)(nimp + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "import_scan", 16.0 * nimp, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, l2.get(), ioff.get(), (int)(nimp + 1), c.stream));
    });
    launch(c, "import_rows", 16.0 * ne, [&] {
      k_import_rows<<<grid_for(c, std::max(nimp, ne), 256), 256, 0, c.stream>>>(
          (const int32_t*)r_ids.get(), ioff.get(), nimp, (const int2*)r_ent.get(), ne, imp_pos.get(),
          imp_adj.get(), imp_ew.get());
    });
  }
  // merge the owned coarse rows [c_lo, c_hi) into a staging area sized by them
  const int64_t ncl = c_hi - c_lo;
  DBuf<int64_t> toff(ncl + 1, c.stream);
  {
    dzero(c, rowlen_p + nc, 1);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, rowlen_p + c_lo, toff.get(), (int)(ncl + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "rowlen_scan", 16.0 * ncl, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, rowlen_p + c_lo, toff.get(), (int)(ncl + 1), c.stream));
    });
  }
  int64_t T = 0;
  d2h(c, &T, toff.get() + ncl, 1);
  c.sync();
  DBuf<int32_t> tadj(std::max<int64_t>(1, T), c.stream), tew(std::max<int64_t>(1, T), c.stream);
  int32_t* big_p = c.scratch<int32_t>(9, std::max<int64_t>(1, ncl));
  DBuf<unsigned long long> big_cnt(1, c.stream);
  dzero(c, big_cnt.get(), 1);
  dzero(c, cdeg_p, nc + 1);
  RowMerge rm{g.offs.get(), g.adj.get(), g.ew.get(), vmap, mem_a_p, mem_b_p, toff.get() - c_lo,
              rowlen_p, tadj.get(), tew.get(), cdeg_p, big_p, big_cnt.get(), ovf.get(), nc, 1};
  rm.c_lo = c_lo;
  rm.c_hi = c_hi;
  rm.row_lo = lo;
  rm.row_hi = hi;
  rm.ent_lo = g.ent_lo;
  rm.imp_pos = imp_pos.get();
  rm.imp_adj = imp_adj.get();
  rm.imp_ew = imp_ew.get();
  if (ncl > 0)
    launch(c, "contract_rows", 12.0 * T + 8.0 * T, [&] {
      k_merge_rows<<<grid_for(c, ncl * 32, 256), 256, 0, c.stream>>>(rm);
    });
  unsigned long long nbig = 0;
  d2h(c, &nbig, big_cnt.get(), 1);
  c.sync();
  if (nbig) {
    LongRows lr(c, big_p, (int64_t)nbig, rowlen_p, nc);
    lr.run(rm);
  }
  // this rank's coarse rows, compacted, then every rank's
  DBuf<int64_t> loff(ncl + 1, c.stream);
  if (!small_exclusive_sum(c, "cdeg_scan", cdeg_p + c_lo, loff.get(), (int64_t)(ncl + 1)))
  {
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cdeg_p + c_lo, loff.get(), (int)(ncl + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "cdeg_scan", 16.0 * ncl, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, cdeg_p + c_lo, loff.get(), (int)(ncl + 1), c.stream));
    });
  }
  int64_t lnnz = 0;
  d2h(c, &lnnz, loff.get() + ncl, 1);
  c.sync();
  DBuf<int32_t> ladj, lew;
  ladj.alloc(std::max<int64_t>(1, lnnz), c.stream);
  lew.alloc(std::max<int64_t>(1, lnnz), c.stream);
  if (ncl > 0)
    launch(c, "copy_rows", 16.0 * lnnz, [&] {
      k_copy_rows<<<grid_for(c, ncl * 32, 256), 256, 0, c.stream>>>(toff.get(), loff.get(), tadj.get(),
                                                                   tew.get(), ladj.get(), lew.get(), ncl);
    });
  DBuf<uint8_t> gdeg, gadj, gew;
  const int64_t nrow = gather_all(c, cdeg_p + c_lo, ncl * 8, gdeg) / 8;
  JET_REQUIRE(nrow == nc, JET_EINTERNAL, "distributed contraction lost coarse rows");
  const int64_t cnnz_all = comm_sum(c, lnnz);
  // large coarse levels stay distributed (their owned rows only); smaller
  // ones are gathered whole on every rank
  const bool keep = nc > 4096 && (nc >= c.shard_min_n || cnnz_all >= 64 * c.shard_min_n);
  int64_t cnnz = cnnz_all;
  if (!keep) {
    cnnz = gather_all(c, ladj.get(), lnnz * 4, gadj) / 4;
    gather_all(c, lew.get(), lnnz * 4, gew);
  }
  unsigned hovf = 0;
  d2h(c, &hovf, ovf.get(), 1);
  c.sync();
  hovf = (unsigned)comm_max(c, (int64_t)hovf);
  JET_REQUIRE(!(hovf & 1u), JET_EUNSUPPORTED, "coarse vertex weight exceeds int32");
  JET_REQUIRE(!(hovf & 2u), JET_EUNSUPPORTED, "coarse edge weight exceeds int32");
  cg_->offs.alloc(nc + 1, c.stream);
  {
    DBuf<int64_t> d2(nc + 1, c.stream);
    CK(cudaMemcpyAsync(d2.get(), gdeg.get(), (size_t)nc * 8, cudaMemcpyDeviceToDevice, c.stream));
    dzero(c, d2.get() + nc, 1);
    size_t tmp = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d2.get(), cg_->offs.get(), (int)(nc + 1), c.stream));
    void* p = c.cub_scratch(tmp);
    launch(c, "coarse_offs", 16.0 * nc, [&] {
      CK(cub::DeviceScan::ExclusiveSum(p, tmp, d2.get(), cg_->offs.get(), (int)(nc + 1), c.stream));
    });
  }
  cg_->nnz = cnnz;
  if (keep) {  // the coarse rows [c_lo, c_hi): a distributed level again
    int64_t e0 = 0;
    if (c_lo < nc) d2h(c, &e0, cg_->offs.get() + c_lo, 1);
    else e0 = cnnz;
    c.sync();
    cg_->row_lo = c_lo;
    cg_->row_hi = c_hi;
    cg_->ent_lo = e0;
    cg_->adj = std::move(ladj);
    cg_->ew = std::move(lew);
    cg_->adj.n = (size_t)lnnz;
    cg_->ew.n = (size_t)lnnz;
  } else {
    cg_->adj.alloc(cnnz > 0 ? cnnz : 1, c.stream);
    cg_->ew.alloc(cnnz > 0 ? cnnz : 1, c.stream);
    if (cnnz) {
      CK(cudaMemcpyAsync(cg_->adj.get(), gadj.get(), (size_t)cnnz * 4, cudaMemcpyDeviceToDevice, c.stream));
      CK(cudaMemcpyAsync(cg_->ew.get(), gew.get(), (size_t)cnnz * 4, cudaMemcpyDeviceToDevice, c.stream));
    }
  }
  finalize_graph(c, *cg_);
  return cg_;
}

// build_hierarchy (coarsen.py:141-161; MAX_LEVELS 64, stagnation 0.95 twice)
size_t graph_bytes(const DGraph& g) {
  return g.offs.n * sizeof(int64_t) + (g.adj.n + g.ew.n + g.vw.n + g.bin_store.n) * sizeof(int32_t);
}

size_t Hierarchy::resident_bytes() const {
  size_t b = 0;
  for (const auto& o : owned)
    if (o) b += graph_bytes(*o);
  return b;
}

bool Hierarchy::shrink_to(size_t limit, int keep_a, int keep_b) {
  bool any = false;
  for (int i = 1; i < size() && resident_bytes() > limit; ++i) {
    if (i == keep_a || i == keep_b || !owned[i - 1]) continue;
    owned[i - 1].reset();
    ++evictions;
    any = true;
  }
  return any;
}

void Hierarchy::release(int i) {
  if (i >= 1 && i < size()) owned[i - 1].reset();
}

// Contract level i-1 into level i. On a device allocation failure the other
// evictable levels are dropped, the pool's unused memory is returned to the
// driver (freed blocks of other sizes may not fit the request), and the
// contraction is retried once.
static std::unique_ptr<DGraph> contract_level(Ctx& c, Hierarchy& h, int i, const DGraph& fine,
                                              const int32_t* partner, int32_t* vmap) {
  try {
    return device_contract(c, fine, partner, vmap, h.budget != 0);
  } catch (const Error& e) {
    if (e.code != JET_ENOMEM || h.budget == 0) throw;
    c.sync();
    h.shrink_to(0, i - 1, i);
    c.release_scratch();
    CK(cudaStreamSynchronize(c.stream));
    CK(cudaMemPoolTrimTo(current_pool(), 0));
    c.pool_reserved = 0;
    return device_contract(c, fine, partner, vmap, true);
  }
}

// Rebuild chain j -> i (j the highest resident level below i). Uncoarsening
// then needs i-1, i-2, ..., j+1 in turn, so the chain keeps its midpoint as a
// checkpoint when the budget holds it next to level i (recursive halving:
// each later rebuild starts from the nearest checkpoint below it); every other
// intermediate level is dropped as soon as the next one is built.
const DGraph& hier_acquire(Ctx& c, Hierarchy& h, int i) {
  if (h.resident(i)) return h.level(i);
  int j = i - 1;
  while (!h.resident(j)) --j;
  const int mid = (j + i + 1) / 2;
  for (int t = j + 1; t <= i; ++t) {
    JET_REQUIRE(h.partners[t - 1].get() != nullptr, JET_EINTERNAL, "evicted level without its matching");
    // rebuilds overwrite maps[t-1] with identical values
    h.owned[t - 1] = contract_level(c, h, t, h.level(t - 1), h.partners[t - 1].get(),
                                    h.maps[t - 1].get());
    JET_REQUIRE(h.owned[t - 1]->n == h.lv_n[t] && h.owned[t - 1]->nnz == h.lv_nnz[t], JET_EINTERNAL,
                "rebuilt level differs from the original");
    ++h.rebuilds;
    if (t - 1 > j && t - 1 != mid) h.release(t - 1);  // a plain intermediate
    // keep the checkpoint only if it fits next to the target level (level
    // sizes along a chain are close: level t stands in for level i)
    if (t - 1 == mid && h.budget && h.resident_bytes() > h.budget) h.release(t - 1);
  }
  if (h.budget) h.shrink_to(h.budget, i, mid);
  return h.level(i);
}

void device_build_hierarchy(Ctx& c, const DGraph& g0, int64_t target, Hierarchy& h,
                            bool fast, size_t budget) {
  static const bool dbg = getenv("JET_COARSEN_TIMES") && getenv("JET_COARSEN_TIMES")[0] == '1';
  h.base = &g0;
  h.owned.clear();
  h.maps.clear();
  h.partners.clear();
  h.lv_n.assign(1, g0.n);
  h.lv_nnz.assign(1, g0.nnz);
  h.budget = budget;
  h.rebuilds = h.evictions = 0;
  int stagnant = 0;
  const DGraph* fine = &g0;
  DBuf<int32_t> partner;
  while (fine->n > target && (int)h.owned.size() + 1 < 64) {
    if (budget) partner = DBuf<int32_t>();  // a fresh matching per level, kept for rebuilds
    partner.ensure(fine->n, c.stream);
    double t0 = 0, t1 = 0;
    if (dbg) {
      c.sync();
      t0 = wall_s();
    }
    if (fine->partial())  // distributed finest level (throughput mode only)
      device_match_fast_dist(c, *fine, partner.get());
    else if (fast)
      device_match_fast(c, *fine, partner.get());
    else
      device_match(c, *fine, partner.get());
    if (dbg) {
      c.sync();
      t1 = wall_s();
    }
    DBuf<int32_t> vmap(fine->n, c.stream);
    const int lv = h.size();  // the level being built
    auto coarse = fine->partial() ? device_contract_dist(c, *fine, partner.get(), vmap.get())
                                  : contract_level(c, h, lv, *fine, partner.get(), vmap.get());
    if (dbg) {
      c.sync();
      fprintf(stderr, "COARSEN n=%lld match=%.2fms contract=%.2fms resident=%.2fGB\n", (long long)fine->n,
              (t1 - t0) * 1e3, (wall_s() - t1) * 1e3, h.resident_bytes() / 1e9);
    }
    if (coarse->n == fine->n) break;
    const bool stag = (double)coarse->n > 0.95 * (double)fine->n;
    h.maps.push_back(std::move(vmap));
    h.lv_n.push_back(coarse->n);
    h.lv_nnz.push_back(coarse->nnz);
    h.owned.push_back(std::move(coarse));
    if (budget) {
      h.partners.push_back(std::move(partner));
      h.shrink_to(budget, lv, lv);  // the new level stays: it is the next fine one
    }
    fine = h.owned.back().get();
    stagnant = stag ? stagnant + 1 : 0;
    if (stagnant >= 2) break;
  }
}

}  // namespace jet
