// level.cu — one cooperative kernel per refinement level: the whole
// jet_refine loop (refine.py:190-294) runs on the device.
//
// Every iteration is a fixed sequence of grid-wide phases separated by grid
// barriers; block 0 takes the controller decisions between them:
//   decide  : balanced?  -> Jetlp pass | weak | strong | stop  (refine.py:229-263)
//             rebalance scalars (oversized/valid parts, deficits, heavy
//             bounds, spare, the pass's numpy PCG64 stream)      (rebalance.py)
//   pass    : Jetlp: gains+filter sweep, afterburner           (refine.py:78-183)
//             rebalance: collect, stats, bucket scan, crossing chunk,
//             crossing element, select, ordered tail           (rebalance.py:91-240)
//   apply   : exact cut delta + part weights, then commit      (conn.py:215-254)
//   keep    : best / fallback tracking, phi rule               (refine.py:272-286)
// The host launches once per level and reads the counters back once.
#include "refine_dev.cuh"
#include "controller.cuh"
#include "rng_dev.cuh"
#include <cub/block/block_reduce.cuh>
#include <algorithm>
#include <climits>
#include <cstring>
#include <map>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace jet {

#ifndef LV_BLOCK_SIZE
#define LV_BLOCK_SIZE 512
#endif
#ifndef LV_MIN_BLOCKS
#define LV_MIN_BLOCKS 2
#endif
constexpr int LV_BLOCK = LV_BLOCK_SIZE;
#ifndef LV_CLUSTER_N
#define LV_CLUSTER_N 0  // levels up to this many vertices run as one cluster (0: off; measured slower)
#endif
#ifndef LV_CLUSTER_MAX
#define LV_CLUSTER_MAX 16
#endif
constexpr int LV_TAIL_SMEM = 8192;  // evicted keys sorted in shared memory
constexpr int LV_DRAW_SLACK = 64;
constexpr int64_t LV_ROWS_PER_BLOCK = 128;  // measured: 512 -> 128 saves ~2 ms on 128^3
constexpr int64_t LV_ENTRIES_PER_BLOCK = 16384;  // dense coarse levels (R-MAT)
#ifndef LV_RB_ROWS
#define LV_RB_ROWS 8
#endif
constexpr int LV_RB = LV_RB_ROWS;  // rows per warp batch in the staged short-row sweep (8 measured best of 4-32)

struct LevelCtl {
  long long cut, best_cut, keep_cut, keep_worst;
  long long locked, moves, max_evict;
  int has_best, no_improve, rebal_streak, pass_index;
  int epoch, new_epoch;
  int iterations, lp, weak, strong, stuck;
  int kind;  // 0 stop, 1 Jetlp, 2 weak, 3 strong
  int locks_all_clear, stop, copy_keep, abort;
  int nover, nvalid, nb, nch, slot_min, rho;
  int tail_max;  // largest (part, bucket) group of the evicted set
  unsigned long long rejects;
  long long rej_pos[32];  // word positions of Lemire rejections (first 32)
  unsigned long long pcg_state_hi, pcg_state_lo, pcg_inc_hi, pcg_inc_lo;
};

struct LevelArgs {
  GView g;
  int64_t n;
  int k;
  TierMap tm;
  int wide;
  int t3_two;  // tier 3 holds rows of 33..64 entries (two per lane)
  int tail_grid_min;  // evicted sets above this are ranked by the whole grid
  const int32_t* tlist[NBINS];
  int64_t tcnt[NBINS];
  RbSegsDev seg;
  int tl_cap;
  int32_t* parts;
  int32_t* keep;
  int32_t* cdest;
  long long* F;
  int32_t* mv;
  int32_t* lock;
  int32_t* cand_lists;
  int32_t* move_lists;
  unsigned long long* ctr;
  unsigned long long* ctr2;  // second per-pass counter block (CTR_PW words)
  long long* keep_pw;
  int32_t* rkey;
  int32_t* rbest;
  double* rloss;
  int32_t* rcand;
  int32_t* evict;
  unsigned long long* H;
  unsigned long long* Hs;
  unsigned long long* CH;
  int32_t* ext;        // weighted external degree per vertex (boundary iff > 0)
  int bnd_sweeps;      // later Jetlp sweeps visit only the boundary rows (collected first)
  int32_t* blists;     // per-tier boundary rows (segments as cand_lists)
  int32_t* wdeg;       // weighted degrees (written by the first Jetlp sweep; weighted levels)
  int32_t* opidx;
  uint8_t* valid;
  int32_t* valid_list;
  int32_t* opart;
  double* hb;
  long long* deficit;
  long long* required;
  long long* spare;
  long long* cum_before;
  int32_t* bstar;
  int32_t* thr;
  int32_t* draws;
  unsigned long long* gscratch;
  unsigned* tailbuf;  // >= 3 * k * nb_max + 1 + n words (group ranking of the tail)
  long long limit, sigma, W, min_vw;
  long long c_num, c_den;
  double c_f;
  int c_float;
  int afterburner, locking;
  double phi;
  int no_improve_limit;
  int sub_buckets;
  unsigned long long seed;
  int level;
  int64_t H_cap, CH_cap, draws_cap;
  LevelCtl* C;
  long long* trace;  // optional: 6 values per iteration (JET_TRACE)
  int trace_cap;
  unsigned long long* phase_clk;  // optional: clock64 per phase (JET_PHASES)
  unsigned long long* work;       // {stats rows, entries, ab rows, entries, apply rows, entries}
  int cluster_sync;  // the grid is one thread-block cluster: barrier.cluster between phases
};

// All threads of the cluster; release/acquire at cluster scope orders the
// phases' global-memory writes for every CTA (the wait invalidates L1).
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// phase timer for block 0 / thread 0 (diagnostics only)
__device__ __forceinline__ long long dev_clock() {
#ifdef __CUDA_ARCH__
  return clock64();
#else
  return 0;
#endif
}
struct PhaseClock {
  unsigned long long* acc;
  long long t;
  int kind = 0;  // pass kind: phases are accumulated per kind (16 slots each)
  __device__ PhaseClock(unsigned long long* a) : acc(a), t(dev_clock()) {}
  __device__ __forceinline__ void mark(int ph) {
    if (acc && blockIdx.x == 0 && threadIdx.x == 0) {
      const long long now = dev_clock();
      atomicAdd(acc + 24 * kind + ph, (unsigned long long)(now - t));
      t = now;
    }
  }
};

__device__ __forceinline__ long long ldcg64(const long long* p) {
  return (long long)__ldcg(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ int ldv(const int* p) { return *(const volatile int*)p; }

__device__ __forceinline__ int dev_ceil_log2(long long x) {
  int r = 0;
  while ((1LL << r) < x) ++r;
  return r;
}

// Block 0 keeps the controller state in shared memory (bookkeeping and
// decisions are chains of dependent reads on it) and publishes it to global
// memory after each decision; the words from rej_pos on are written by the
// other blocks' draws and are not mirrored.
constexpr int LV_CTL_WORDS = (int)(offsetof(LevelCtl, rej_pos) / 4);
__device__ __forceinline__ void lv_ctl_load(LevelCtl* m, const LevelCtl* g) {
  for (int i = threadIdx.x; i < (int)(sizeof(LevelCtl) / 4); i += blockDim.x)
    reinterpret_cast<unsigned*>(m)[i] = __ldcg(reinterpret_cast<const unsigned*>(g) + i);
  __syncthreads();
}
__device__ __forceinline__ void lv_ctl_publish(LevelCtl* g, const LevelCtl* m) {
  __syncthreads();
  constexpr int WP = (int)(offsetof(LevelCtl, pcg_state_hi) / 4);
  for (int i = threadIdx.x; i < LV_CTL_WORDS + 8; i += blockDim.x) {
    const int w = i < LV_CTL_WORDS ? i : WP + i - LV_CTL_WORDS;
    reinterpret_cast<unsigned*>(g)[w] = reinterpret_cast<const unsigned*>(m)[w];
  }
}

// ---------------------------------------------------------------- decide
// P: the per-pass counter block of the pass being decided (zeroed here)
__device__ void lv_decide(const LevelArgs& A, LevelCtl* C, unsigned long long* P) {
  typedef cub::BlockScan<int, LV_BLOCK> BScan;
  typedef cub::BlockReduce<long long, LV_BLOCK> BRed;
  __shared__ typename BScan::TempStorage ts;
  __shared__ typename BRed::TempStorage tr;
  __shared__ int s_unbal, s_kind, s_no, s_nv;
  const long long* pw = reinterpret_cast<const long long*>(A.ctr + CTR_PW);
  const int tid = threadIdx.x, k = A.k;
  if (tid == 0) s_unbal = 0;
  __syncthreads();
  for (int p = tid; p < k; p += LV_BLOCK)
    if (ldcg64(pw + p) > A.limit) s_unbal = 1;
  __syncthreads();
  if (tid == 0) {
    int kind;
    if (C->stop || C->no_improve >= A.no_improve_limit) {
      kind = 0;
    } else if (!s_unbal) {
      kind = 1;
      C->rebal_streak = 0;
      C->locks_all_clear = !A.locking || C->locked == 0;
      C->new_epoch = A.locking ? C->epoch + 1 : C->epoch;
    } else if (C->rebal_streak >= 2 + k) {
      C->stuck = 1;
      kind = 0;
    } else {
      C->epoch = C->epoch + 1;  // table.reset_locks()
      C->new_epoch = C->epoch;
      C->locked = 0;
      kind = C->rebal_streak < 2 ? 2 : 3;
    }
    s_kind = kind;
    C->kind = kind;
  }
  for (int i = tid; i < CTR_PW; i += LV_BLOCK) P[i] = 0;
  __syncthreads();
  if (s_kind < 2) return;

  // ---- rebalance scalars (rebalance.py:148-156, :127-131, :224)
  const bool strong = s_kind == 3;
  if (tid == 0) {
    s_no = 0;
    s_nv = 0;
  }
  __syncthreads();
  long long my_evict = 0;
  const double ideal = __ddiv_rn((double)A.W, (double)k);
  for (int base = 0; base < k; base += LV_BLOCK) {
    const int p = base + tid;
    long long w = 0;
    int fo = 0, fv = 0;
    if (p < k) {
      w = ldcg64(pw + p);
      fo = w > A.limit;
      fv = w < A.sigma;
    }
    int ro, rv, to, tv;
    BScan(ts).ExclusiveSum(fo, ro, to);
    __syncthreads();
    BScan(ts).ExclusiveSum(fv, rv, tv);
    const int bo = s_no, bv = s_nv;
    if (p < k) {
      A.opidx[p] = fo ? bo + ro : -1;
      A.valid[p] = (uint8_t)fv;
      if (fo) {
        const int i = bo + ro;
        A.opart[i] = p;
        A.deficit[i] = w - (A.sigma + 1);
        A.required[i] = w - A.limit;
        A.hb[i] = __dmul_rn(1.5, __dsub_rn((double)w, ideal));
        my_evict += (w - (A.sigma + 1)) / (A.min_vw > 0 ? A.min_vw : 1) + 1;
      }
      if (fv) {
        A.valid_list[bv + rv] = p;
        A.spare[bv + rv] = A.sigma - w;
      }
    }
    __syncthreads();
    if (tid == 0) {
      s_no = bo + to;
      s_nv = bv + tv;
    }
    __syncthreads();
  }
  const long long tot_evict = BRed(tr).Sum(my_evict);
  if (tid == 0) {
    C->nover = s_no;
    C->nvalid = s_nv;
    // every evicted vertex is a candidate, so at most n leave
    C->max_evict = tot_evict < A.n ? tot_evict : A.n;
    C->rejects = 0;
    if (s_nv == 0) {  // RebalanceInfeasibleError -> rebalance_stuck
      C->stuck = 1;
      C->kind = 0;
    } else {
      const int rho = (int64_t)A.sub_buckets >= A.n ? 1 : A.sub_buckets;
      const int slot_min = strong ? 1 - dev_ceil_log2(k) : 0;
      const int nb = (34 - slot_min) * rho;
      const int nch = (int)(((A.n + rho - 1) / rho + 31) / 32);
      C->rho = rho;
      C->slot_min = slot_min;
      C->nb = nb;
      C->nch = nch;
      if ((int64_t)s_no * nb > A.H_cap || (int64_t)s_no * nch > A.CH_cap ||
          C->max_evict + LV_DRAW_SLACK > A.draws_cap) {
        C->abort = 1;
        C->kind = 0;
      }
      uint64_t sd[3] = {A.seed, (uint64_t)A.level, (uint64_t)C->pass_index};
      DevPcg g;
      if (A.level >= 0) {
        g = dev_seed(sd, 3);
      } else {
        sd[1] = (uint64_t)C->pass_index;
        g = dev_seed(sd, 2);
      }
      C->pcg_state_hi = (unsigned long long)(g.state >> 64);
      C->pcg_state_lo = (unsigned long long)g.state;
      C->pcg_inc_hi = (unsigned long long)(g.inc >> 64);
      C->pcg_inc_lo = (unsigned long long)g.inc;
    }
  }
}

// -------------------------------------------------------------- bookkeep
__device__ void lv_bookkeep(const LevelArgs& A, LevelCtl* C, const unsigned long long* P) {
  typedef cub::BlockReduce<long long, LV_BLOCK> BRed;
  __shared__ typename BRed::TempStorage tr;
  __shared__ int s_copy;
  const long long* pw = reinterpret_cast<const long long*>(A.ctr + CTR_PW);
  const int tid = threadIdx.x, k = A.k;
  long long worst = LLONG_MIN;
  for (int p = tid; p < k; p += LV_BLOCK) worst = max(worst, ldcg64(pw + p));
  worst = BRed(tr).Reduce(worst, cub::Max());
  if (tid == 0) {
    const int kind = C->kind;
    long long nm = 0;
    for (int t = 0; t < NBINS; ++t) nm += (long long)__ldcg(P + CTR_MOVE + t);
    nm += (long long)__ldcg(P + CTR_NMOVE);
    const long long d2 = (long long)__ldcg(P + CTR_CUT2D);
    C->cut += d2 / 2;
    if (kind == 1) {
      C->lp++;
      if (A.locking) {
        C->epoch = C->new_epoch;
        C->locked = nm;
      }
    } else {
      if (kind == 3) C->strong++;
      else C->weak++;
      C->rebal_streak++;
    }
    const bool fixed_point = kind == 1 && nm == 0 && C->locks_all_clear;
    C->pass_index++;
    C->iterations++;
    C->moves += nm;
    C->no_improve++;
    int copy = 0;
    const long long cut = C->cut;
    if (worst <= A.limit) {
      if (!C->has_best || cut < C->best_cut) {
        if (!C->has_best || (double)cut < __dmul_rn(A.phi, (double)C->best_cut)) C->no_improve = 0;
        copy = 1;
        C->best_cut = cut;
        C->keep_cut = cut;
        C->has_best = 1;
      }
    } else if (!C->has_best && worst < C->keep_worst) {
      copy = 1;
      C->keep_worst = worst;
      C->keep_cut = cut;
    }
    if (fixed_point) C->stop = 1;
    C->copy_keep = copy;
    s_copy = copy;
    if (A.trace && C->iterations <= A.trace_cap) {
      long long* t = A.trace + 10 * (C->iterations - 1);
      long long ncand = 0;
      for (int q = 0; q < NBINS; ++q) ncand += (long long)__ldcg(P + CTR_CAND + q);
      t[6] = ncand;
      t[7] = (long long)__ldcg(P + CTR_RCAND);
      t[8] = kind >= 2 ? C->max_evict : 0;
      t[9] = kind >= 2 ? C->nover : 0;
      t[0] = kind;
      t[1] = nm;
      t[2] = cut;
      t[3] = worst;
      t[4] = C->no_improve;
      t[5] = C->has_best;
    }
    // A strong pass that moved nothing left parts, part weights and cut as
    // they were, and strong passes draw no random numbers: every following
    // pass repeats it (still unbalanced, streak >= 2) until no_improve
    // reaches the limit or the stuck guard fires (refine.py:229-263). Book
    // those passes without running them; outputs and stats are unchanged.
    if (kind == 3 && nm == 0 && worst > A.limit && !fixed_point) {
      const int it0 = C->iterations;
      while (C->no_improve < A.no_improve_limit && C->rebal_streak < 2 + k) {
        C->strong++;
        C->rebal_streak++;
        C->pass_index++;
        C->iterations++;
        C->no_improve++;
        if (A.trace && C->iterations <= A.trace_cap && it0 <= A.trace_cap) {
          long long* t = A.trace + 10 * (C->iterations - 1);
          const long long* t0 = A.trace + 10 * (it0 - 1);
          for (int q = 0; q < 10; ++q) t[q] = t0[q];
          t[4] = C->no_improve;
        }
      }
    }
  }
  __syncthreads();
  if (s_copy)
    for (int p = tid; p < k; p += LV_BLOCK) A.keep_pw[p] = ldcg64(pw + p);
}

// ---------------------------------------------------------- rebalancing
__device__ void lv_draws(const LevelArgs& A, const LevelCtl& S, int64_t t0, int64_t nt) {
  LevelCtl* C = A.C;
  const int nvalid = S.nvalid;
  const int64_t D = S.max_evict;
  if (nvalid <= 1) {  // integers(0, 1) returns 0 without drawing
    for (int64_t j = t0; j < D; j += nt) A.draws[j] = 0;
    return;
  }
  DevPcg g;
  g.state = ((du128)S.pcg_state_hi << 64) | S.pcg_state_lo;
  g.inc = ((du128)S.pcg_inc_hi << 64) | S.pcg_inc_lo;
  const uint32_t excl = (uint32_t)nvalid, thr = (0xffffffffu - (uint32_t)(nvalid - 1)) % excl;
  // words [D, D + slack) are only screened: a rejection before D shifts the
  // stream onto them
  for (int64_t j = t0; j < D + LV_DRAW_SLACK; j += nt) {
    const uint64_t m = (uint64_t)pcg_word(g, (uint64_t)j) * excl;
    if ((uint32_t)m < excl && (uint32_t)m < thr) {
      const unsigned long long q = atomicAdd(&C->rejects, 1ull);
      if (q < 32) C->rej_pos[q] = j;
    }
    if (j < D) A.draws[j] = (int32_t)(m >> 32);
  }
}

// Rejected words are skipped by numpy's Lemire loop, so draw j is the word
// at the (j+1)-th accepted position: w = j + #{rejected q <= w} (fixed point,
// at most #rejections + 1 steps). Parallel over the draws.
__device__ void lv_draws_fix_parallel(const LevelArgs& A, const LevelCtl& S, int R, int64_t t0,
                                      int64_t nt) {
  LevelCtl* C = A.C;
  const int64_t D = S.max_evict;
  const int nvalid = S.nvalid;
  DevPcg g;
  g.state = ((du128)S.pcg_state_hi << 64) | S.pcg_state_lo;
  g.inc = ((du128)S.pcg_inc_hi << 64) | S.pcg_inc_lo;
  long long qmin = LLONG_MAX;
  for (int r = 0; r < R; ++r) qmin = min(qmin, *(const volatile long long*)&C->rej_pos[r]);
  for (int64_t j = t0; j < D; j += nt) {
    if (j < qmin) continue;  // before the first rejection nothing moved
    int64_t w = j;
    while (true) {
      int64_t cnt = 0;
      for (int r = 0; r < R; ++r) cnt += *(const volatile long long*)&C->rej_pos[r] <= w;
      if (j + cnt == w) break;
      w = j + cnt;
    }
    const uint64_t m = (uint64_t)pcg_word(g, (uint64_t)w) * (uint32_t)nvalid;
    A.draws[j] = (int32_t)(m >> 32);
  }
}

__device__ void lv_draws_fixup(const LevelArgs& A) {
  // a Lemire rejection shifted the stream: redo the draws sequentially
  LevelCtl* C = A.C;
  DevPcgSeq s;
  s.g.state = ((du128)C->pcg_state_hi << 64) | C->pcg_state_lo;
  s.g.inc = ((du128)C->pcg_inc_hi << 64) | C->pcg_inc_lo;
  const int64_t D = C->max_evict;
  for (int64_t j = 0; j < D; ++j) A.draws[j] = (int32_t)s.below((uint32_t)C->nvalid);
}

__device__ RbSel lv_sel(const LevelArgs& A, const LevelCtl& S) {
  return RbSel{A.parts, A.g.vw, A.opidx, A.rkey, A.bstar, A.thr, S.rho, S.nch, A.CH};
}

// per-warp staging words of the short-row sweeps (largest tier variant)
template <bool UNIT>
__host__ __device__ constexpr int lv_stage_words() {
  return stage_words<32, LV_RB / 2, UNIT, 2>() > stage_words<32, LV_RB, UNIT, 1>()
             ? stage_words<32, LV_RB / 2, UNIT, 2>()
             : stage_words<32, LV_RB, UNIT, 1>();
}

// --------------------------------------------------------- tier sweeps
template <class Op, bool UNIT, class MakeArgs>
__device__ void lv_sweep(const LevelArgs& A, MakeArgs mk, const int32_t* const* lists,
                         const unsigned long long* dcnts, unsigned long long* smem, int64_t w0,
                         int64_t nw, long long& acc) {
  const bool wide = A.wide != 0;
#pragma unroll 1
  for (int t = 0; t < NBINS; ++t) {
    if (A.tcnt[t] == 0) continue;
    // tiers share one shared-memory union (stages / warp tables / block table)
    __syncthreads();
    const typename Op::Args a = mk(t);
    const int32_t* list = lists ? lists[t] : A.tlist[t];
    const unsigned long long* dc = dcnts ? dcnts + t : nullptr;
    const int64_t cnt = A.tcnt[t];
    uint32_t* stg = reinterpret_cast<uint32_t*>(smem) +
                    (threadIdx.x >> 5) * lv_stage_words<UNIT>();
    switch (t) {
      case 0: agg_small<Op, 4, UNIT, LV_RB>(a, A.g, A.parts, list, cnt, wide, dc, w0, nw, acc, stg); break;
      case 1: agg_small<Op, 8, UNIT, LV_RB>(a, A.g, A.parts, list, cnt, wide, dc, w0, nw, acc, stg); break;
      case 2: agg_small<Op, 16, UNIT, LV_RB>(a, A.g, A.parts, list, cnt, wide, dc, w0, nw, acc, stg); break;
      case 3:
        // rows of <= 32 entries on this level: one entry per lane, full batches
        if (A.t3_two)
          agg_small<Op, 32, UNIT, LV_RB / 2, 2>(a, A.g, A.parts, list, cnt, wide, dc, w0, nw, acc, stg);
        else
          agg_small<Op, 32, UNIT, LV_RB, 1>(a, A.g, A.parts, list, cnt, wide, dc, w0, nw, acc, stg);
        break;
      case 4: {
        const size_t per = (size_t)A.k + (size_t)(A.tl_cap + 3) / 2;
        agg_warp<Op, UNIT>(a, A.g, A.parts, list, cnt, wide, A.k, A.tl_cap, dc,
                           smem + 0 * per, w0, nw, acc);
        __syncwarp();
        break;
      }
      default:
        agg_block<Op, UNIT>(a, A.g, A.parts, list, cnt, wide, A.k, dc, smem, acc);
        break;
    }
  }
  __syncthreads();
}

// Grid-wide bitonic sort of the evicted keys (part rank, bucket, id) when
// they outnumber one block's shared memory: chunks of C keys are sorted in
// shared memory, then for every merge size the strides >= C run as global
// compare-exchange passes and the strides < C inside each chunk again.
// A one-block sort of 10^5 keys from global memory took ~0.8 ms per pass.
template <class GSync>
__device__ void lv_grid_sort(const LevelArgs& A, int L, int P2, int nb, unsigned long long* sm,
                             GSync gsync, int64_t t0, int64_t nt) {
  constexpr int C = LV_TAIL_SMEM;
  unsigned long long* keys = A.gscratch;
  for (int64_t i = t0; i < P2; i += nt) {
    unsigned long long key = ~0ull;
    if (i < L) {
      const int v = A.evict[i];
      const unsigned long long grp =
          (unsigned long long)A.opidx[A.parts[v]] * (unsigned)nb + (unsigned)A.rkey[v];
      key = (grp << 32) | (unsigned)v;
    }
    keys[i] = key;
  }
  gsync();
  const int nch = P2 / C;
  auto local = [&](int size_lo, int size_hi, int stride_hi) {
    // sizes [size_lo, size_hi] (doubling); strides from min(size/2, stride_hi) down to 1
    for (int ch = blockIdx.x; ch < nch; ch += gridDim.x) {
      unsigned long long* g = keys + (size_t)ch * C;
      for (int i = threadIdx.x; i < C; i += blockDim.x) sm[i] = g[i];
      __syncthreads();
      for (int size = size_lo; size <= size_hi; size <<= 1) {
        for (int stride = min(size >> 1, stride_hi); stride > 0; stride >>= 1) {
          for (int i = threadIdx.x; i < C; i += blockDim.x) {
            const int j = i ^ stride;
            if (j > i) {
              const bool asc = (((int64_t)ch * C + i) & size) == 0;
              const unsigned long long x = sm[i], y = sm[j];
              if ((x > y) == asc) {
                sm[i] = y;
                sm[j] = x;
              }
            }
          }
          __syncthreads();
        }
      }
      for (int i = threadIdx.x; i < C; i += blockDim.x) g[i] = sm[i];
      __syncthreads();
    }
  };
  local(2, C, C);
  gsync();
  for (int size = 2 * C; size <= P2; size <<= 1) {
    for (int stride = size >> 1; stride >= C; stride >>= 1) {
      for (int64_t i = t0; i < P2; i += nt) {
        const int64_t j = i ^ stride;
        if (j > i) {
          const bool asc = (i & size) == 0;
          const unsigned long long x = keys[i], y = keys[j];
          if ((x > y) == asc) {
            keys[i] = y;
            keys[j] = x;
          }
        }
      }
      gsync();
    }
    local(size, size, C >> 1);
    gsync();
  }
}

// Order of the evicted set without a sort: key (g, v) with group g = (part
// rank, bucket). rank(v) = #evicted in groups < g + #evicted in g with a
// smaller id. Groups are counted, scanned (block 0), the members scattered
// into their group segment, and each member ranks itself inside its
// segment (groups are tiny: bucket = (slot, id mod rho)). Writes the keys in
// sorted order to gscratch. Returns false (uniformly) when a group is too
// large for the quadratic in-segment ranking; the caller then sorts.
constexpr int LV_TAIL_GROUP_MAX = 512;
template <class GSync>
__device__ bool lv_tail_rank(const LevelArgs& A, int L, int nover, int nb, GSync gsync, int64_t t0,
                             int64_t nt) {
  LevelCtl* C = A.C;
  const int G = nover * nb;
  unsigned* hist = A.tailbuf;
  unsigned* base = hist + G;      // per-block exclusive prefix, G
  unsigned* fill = base + G;      // G
  unsigned* bpre = fill + G;      // per-block totals -> exclusive prefix, gridDim.x
  int32_t* seg = reinterpret_cast<int32_t*>(bpre + gridDim.x + 1);
  for (int64_t i = t0; i < G; i += nt) {
    hist[i] = 0;
    fill[i] = 0;
  }
  if (t0 == 0) C->tail_max = 0;
  gsync();
  const int64_t lim = ((int64_t)L + 31) & ~31LL;
  for (int64_t i = t0; i < lim; i += nt) {
    int g = -1;
    if (i < L) {
      const int v = A.evict[i];
      g = A.opidx[A.parts[v]] * nb + A.rkey[v];
    }
    const unsigned peers = __match_any_sync(0xffffffffu, g);
    if (g >= 0 && (int)(threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[g], __popc(peers));
  }
  gsync();
  // scan of the group counts: every block scans its slice of G
  typedef cub::BlockScan<unsigned, LV_BLOCK> BScan;
  typedef cub::BlockReduce<unsigned, LV_BLOCK> BRed;
  __shared__ typename BScan::TempStorage ts;
  __shared__ typename BRed::TempStorage tr;
  __shared__ unsigned s_run;
  const int per = (G + gridDim.x - 1) / gridDim.x;
  const int lo = min(G, (int)blockIdx.x * per), hi = min(G, lo + per);
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  unsigned mx = 0;
  for (int b0 = lo; b0 < hi; b0 += LV_BLOCK) {
    const int i = b0 + threadIdx.x;
    const unsigned x = i < hi ? hist[i] : 0u;
    mx = max(mx, x);
    unsigned ex, tot;
    BScan(ts).ExclusiveSum(x, ex, tot);
    const unsigned run = s_run;
    if (i < hi) base[i] = run + ex;
    __syncthreads();
    if (threadIdx.x == 0) s_run = run + tot;
    __syncthreads();
  }
  mx = BRed(tr).Reduce(mx, cub::Max());
  if (threadIdx.x == 0) {
    bpre[blockIdx.x] = s_run;
    atomicMax(&C->tail_max, (int)mx);
  }
  gsync();
  if (ldv(&C->tail_max) > LV_TAIL_GROUP_MAX) return false;
  if (blockIdx.x == 0) {  // exclusive scan of the block totals (gridDim.x <= 2 * 148)
    unsigned run = 0;
    for (int b0 = 0; b0 < (int)gridDim.x; b0 += LV_BLOCK) {
      const int i = b0 + threadIdx.x;
      const unsigned x = i < (int)gridDim.x ? bpre[i] : 0u;
      unsigned ex, tot;
      BScan(ts).ExclusiveSum(x, ex, tot);
      __syncthreads();
      if (i < (int)gridDim.x) bpre[i] = run + ex;
      run += tot;
    }
  }
  gsync();
  auto gbase = [&](int g) { return base[g] + bpre[g / per]; };
  for (int64_t i = t0; i < L; i += nt) {
    const int v = A.evict[i];
    const int g = A.opidx[A.parts[v]] * nb + A.rkey[v];
    seg[gbase(g) + atomicAdd(&fill[g], 1u)] = v;
  }
  gsync();
  for (int64_t i = t0; i < L; i += nt) {
    const int v = A.evict[i];
    const int g = A.opidx[A.parts[v]] * nb + A.rkey[v];
    const unsigned b = gbase(g), e = b + hist[g];
    unsigned r = 0;
    for (unsigned j = b; j < e; ++j) r += (unsigned)(seg[j] < v);
    A.gscratch[b + r] = ((unsigned long long)g << 32) | (unsigned)v;
  }
  gsync();
  return true;
}

// ---------------------------------------------------------------- kernel
template <bool UNIT>
__global__ void __launch_bounds__(LV_BLOCK, LV_MIN_BLOCKS) k_level(LevelArgs A) {
  extern __shared__ unsigned long long lv_smem[];
  cg::grid_group grid = cg::this_grid();
  // a one-block grid (small levels) synchronises with __syncthreads, which
  // also orders global memory within the block; the grid barrier protocol
  // costs ~1.5 us per phase even for one block
  const bool one_block = gridDim.x == 1;
  const bool clus = A.cluster_sync != 0;
  auto gsync = [&]() {
    if (one_block) __syncthreads();
    else if (clus) cluster_barrier();
    else grid.sync();
  };
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (int64_t)gridDim.x * blockDim.x;
  const int64_t w0 = t0 >> 5, nw = nt >> 5;
  LevelCtl* C = A.C;
  // warp-tier tables: one per warp of the block
  const size_t per = (size_t)A.k + (size_t)(A.tl_cap + 3) / 2;
  unsigned long long* wtab = lv_smem + (threadIdx.x >> 5) * per;
  SegLists cands, moves;
  for (int t = 0; t < NBINS; ++t) {
    cands.list[t] = A.cand_lists + A.seg.b[t];
    moves.list[t] = A.move_lists + A.seg.b[t];
  }
  int32_t* clists[NBINS];
  for (int t = 0; t < NBINS; ++t) clists[t] = A.cand_lists + A.seg.b[t];

  PhaseClock pc(A.phase_clk);
  WorkAcc wk;
  // After the first Jetlp sweep of the level has measured every vertex's
  // external degree, the applied moves keep it current, and later sweeps
  // visit only boundary rows: an interior row has no destination, adds
  // nothing to the cut, and its cdest stays -1 (reset after each pass).
  bool ext_ok = false;
  const int32_t* blp[NBINS];
  for (int t = 0; t < NBINS; ++t) blp[t] = A.blists + A.seg.b[t];
  // Per-pass counters alternate between two blocks by pass parity, so block
  // 0 can book-keep pass i and decide pass i+1 (zeroing the other block)
  // while the other blocks still commit pass i: one grid barrier per pass
  // fewer. The part weights (A.ctr + CTR_PW) are not per pass.
  __shared__ LevelCtl s_mc;  // block 0: controller mirror
  if (blockIdx.x == 0) {
    lv_ctl_load(&s_mc, C);
    lv_decide(A, &s_mc, A.ctr);  // pass_index 0 -> A.ctr
    lv_ctl_publish(C, &s_mc);
  }
  gsync();
  // control words of the pass, read once per block (every warp reading them
  // from L2 puts thousands of requests on one line per phase)
  __shared__ LevelCtl s_ctl;
  __shared__ unsigned long long s_bcast[2];
  const LevelCtl& S = s_ctl;
  while (true) {
    pc.mark(0);
    {
      constexpr int W0 = (int)(offsetof(LevelCtl, rej_pos) / 4);
      constexpr int WP = (int)(offsetof(LevelCtl, pcg_state_hi) / 4);
      static_assert(W0 <= LV_BLOCK && sizeof(LevelCtl) / 4 - WP == 8, "LevelCtl layout");
      const unsigned* src = reinterpret_cast<const unsigned*>(C);
      unsigned* dst = reinterpret_cast<unsigned*>(&s_ctl);
      if ((int)threadIdx.x < W0) dst[threadIdx.x] = __ldcg(src + threadIdx.x);
      else if ((int)threadIdx.x < W0 + 8) dst[WP + threadIdx.x - W0] = __ldcg(src + WP + threadIdx.x - W0);
      __syncthreads();
    }
    const int kind = S.kind;
    pc.kind = kind;
    if (kind == 0) break;
    const int pass = S.pass_index;
    unsigned long long* P = (pass & 1) ? A.ctr2 : A.ctr;
    cands.cnt = P + CTR_CAND;
    moves.cnt = P + CTR_MOVE;
    // the previous pass's state became the kept one: copy it while this
    // pass's first phase runs (only the commit phase writes parts)
    if (S.copy_keep)
      for (int64_t v = t0; v < A.n; v += nt) A.keep[v] = A.parts[v];
    long long acc = 0;
    if (kind == 1) {
      // ---- Jetlp (refine.py:159-183)
      LpParams lp;
      lp.c_num = A.c_num;
      lp.c_den = A.c_den;
      lp.c_f = A.c_f;
      lp.c_use_float = A.c_float;
      lp.afterburner = A.afterburner;
      lp.locking = A.locking;
      lp.lock_epoch = S.epoch;
      auto mk = [&](int t) {
        LpOp::Args a{};
        a.parts = A.parts;
        a.cdest = A.cdest;
        a.F = A.F;
        a.mv = A.mv;
        a.lock = A.lock;
        a.p = lp;
        a.out_list = (A.afterburner ? A.cand_lists : A.move_lists) + A.seg.b[t];
        a.out_cnt = P + (A.afterburner ? CTR_CAND : CTR_MOVE) + t;
        a.cut2 = P + CTR_CUT2;
        a.ext = A.ext;
        a.wdeg = A.ext ? A.wdeg : nullptr;
        return a;
      };
      const bool bnd = ext_ok && A.bnd_sweeps;
      if (bnd) {
        const int32_t* ext = A.ext;
        collect_tiled([&](int v) { return __ldcg(ext + v) != 0; },
                      A.g.offs, A.tm, A.n, A.blists, A.seg, P + CTR_BND, &wk.v[6], &wk.v[7]);
        gsync();
        pc.mark(15);
      }
      // per-warp tables start at lv_smem + warp * per inside agg_warp
      lv_sweep<LpOp, UNIT>(A, mk, bnd ? blp : nullptr, bnd ? P + CTR_BND : nullptr, lv_smem, w0,
                           nw, acc);
      gsync();
      ext_ok = A.ext != nullptr;
      pc.mark(1);
      if (A.afterburner) {
        AbArgs ab{};
        ab.parts = A.parts;
        ab.cdest = A.cdest;
        ab.F = A.F;
        ab.mv = A.mv;
        ab.move_list = nullptr;  // moves flagged in mv[], applied from the candidate lists
        ab.move_cnt = nullptr;
        long long nmv = 0;
        afterburner_rows<UNIT>(ab, A.g, cands, A.seg, w0, nw, &wk.v[2], &wk.v[3], &nmv);
        block_sum_atomic_any(nmv, P + CTR_NMOVE);
        gsync();
        pc.mark(2);
      }
    } else {
      // ---- weak / strong rebalancing (rebalance.py:139-240)
      const int strong = kind == 3;
      const int nover = S.nover, nb = S.nb, nch = S.nch;
      for (int64_t i = t0; i < (int64_t)nover * nb; i += nt) A.H[i] = 0;
      for (int64_t i = t0; i < (int64_t)nover * (nb / S.rho); i += nt) A.Hs[i] = 0;
      for (int64_t i = t0; i < (int64_t)nover * nch; i += nt) A.CH[i] = 0;
      if (!strong) lv_draws(A, S, t0, nt);
      pc.mark(14);
      rb_collect(A.parts, A.opidx, A.g.offs, A.tm, A.n, A.cand_lists, A.seg, P + CTR_CAND, t0, nt,
                 &wk.v[0], &wk.v[1]);
      gsync();
      pc.mark(3);
      RbOp::Args ra{};
      ra.parts = A.parts;
      ra.vw = A.g.vw;
      ra.opidx = A.opidx;
      ra.valid = A.valid;
      ra.hb = A.hb;
      ra.nvalid = S.nvalid;
      ra.strong = strong;
      ra.rho = S.rho;
      ra.slot_min = S.slot_min;
      ra.nb = nb;
      ra.rkey = A.rkey;
      ra.rbest = A.rbest;
      ra.rloss = A.rloss;
      ra.rcand = A.rcand;
      ra.rcand_cnt = P + CTR_RCAND;
      ra.H = A.H;
      ra.Hs = A.Hs;
      ra.ext = ext_ok ? A.ext : nullptr;
      ra.wdeg = A.wdeg;
      lv_sweep<RbOp, UNIT>(A, [&](int) { return ra; }, clists, P + CTR_CAND, lv_smem, w0, nw,
                           acc);
      gsync();
      pc.mark(4);
      const RbSel s = lv_sel(A, S);
      for (int64_t op = w0; op < nover; op += nw)
        rb_scan_warp((int)op, A.H, A.Hs, nb, S.rho, A.deficit, A.bstar, A.cum_before);
      gsync();
      pc.mark(5);
      rb_chunk(s, A.rcand, P + CTR_RCAND, t0, nt);
      gsync();
      pc.mark(6);
      if ((int)gridDim.x >= nover && nch > 512) {  // long chunk rows: a block per part
        if ((int)blockIdx.x < nover)
          rb_find_block<LV_BLOCK>((int)blockIdx.x, s, A.deficit, A.required, A.cum_before, A.opart,
                                  A.n, nb, A.thr);
      } else {
        for (int64_t op = w0; op < nover; op += nw)
          rb_find_warp((int)op, s, A.deficit, A.required, A.cum_before, A.opart, A.n, nb, A.thr);
      }
      gsync();
      pc.mark(7);
      rb_select(s, A.rcand, P + CTR_RCAND, A.rbest, strong, 1, A.evict, P + CTR_EVICT,
                A.mv, A.g.offs, A.tm, A.move_lists, A.seg, P + CTR_MOVE, t0, nt);
      gsync();
      pc.mark(8);
      if (threadIdx.x == 0) {
        s_bcast[0] = __ldcg(P + CTR_EVICT);
        s_bcast[1] = strong ? 0ull : __ldcg(&C->rejects);
      }
      __syncthreads();
      const int Lev = (int)s_bcast[0];
      const unsigned long long rejects = s_bcast[1];
      int P2ev = 1;
      while (P2ev < Lev) P2ev <<= 1;
      if (!strong && rejects) {
        // a Lemire rejection shifted the draw stream: re-derive the draws
        // (in parallel; sequentially only past 32 rejections)
        if (rejects <= 32)
          lv_draws_fix_parallel(A, S, (int)rejects, t0, nt);
        else if (blockIdx.x == 0 && threadIdx.x == 0)
          lv_draws_fixup(A);
        gsync();
      }
      pc.mark(13);
      // large evicted sets: order them with the whole grid, and for weak
      // passes assign the random destinations with the whole grid too
      const bool big_tail = P2ev > A.tail_grid_min;
      if (big_tail && !lv_tail_rank(A, Lev, nover, nb, gsync, t0, nt))
        lv_grid_sort(A, Lev, P2ev, nb, lv_smem, gsync, t0, nt);
      pc.mark(12);
      if (big_tail && !strong) {
        const int nvalid = S.nvalid;
        const int64_t lim = ((int64_t)Lev + 31) & ~31LL;
        for (int64_t i = t0; i < lim; i += nt) {
          int v = 0, t = -1;
          if (i < Lev) {
            v = (int)(A.gscratch[i] & 0xffffffffu);
            A.mv[v] = A.valid_list[nvalid > 1 ? A.draws[i] : 0];
            t = A.tm(A.g.offs[v + 1] - A.g.offs[v]);
          }
          for (int tt = 0; tt < NBINS; ++tt)
            warp_append(t == tt, v, A.move_lists + A.seg.b[tt], P + CTR_MOVE + tt);
        }
      } else if (blockIdx.x == 0) {
        RbTail tl{};
        tl.evict = A.evict;
        tl.evict_cnt = P + CTR_EVICT;
        tl.parts = A.parts;
        tl.opidx = A.opidx;
        tl.rkey = A.rkey;
        tl.vw = A.g.vw;
        tl.offs = A.g.offs;
        tl.tm = A.tm;
        tl.valid_list = A.valid_list;
        tl.draws = A.draws;
        tl.spare = A.spare;
        tl.nvalid = S.nvalid;
        tl.nb = nb;
        tl.strong = strong;
        tl.mv = A.mv;
        tl.move_lists = A.move_lists;
        tl.mseg = A.seg;
        tl.move_cnt = P + CTR_MOVE;
        tl.smem_cap = LV_TAIL_SMEM;
        tl.gscratch = A.gscratch;
        tl.presorted = big_tail;
        rb_tail(tl, lv_smem);
      }
      gsync();
      pc.mark(9);
    }
    // ---- apply (conn.py:215-254)
    {
      ApArgs ap{A.parts, A.mv, A.ctr + CTR_PW, P + CTR_CUT2D, A.k, ext_ok ? A.ext : nullptr};
      long long d = 0;
      apply_delta_rows<UNIT>(ap, A.g, (kind == 1 && A.afterburner) ? cands : moves, w0, nw, d,
                             &wk.v[4], &wk.v[5]);
      block_sum_atomic_any(d, P + CTR_CUT2D);
    }
    gsync();
    pc.mark(10);
    {
      CommitArgs ca{};
      ca.parts = A.parts;
      ca.mv = A.mv;
      ca.lock = A.lock;
      ca.epoch = S.new_epoch;
      ca.set_lock = kind == 1 && A.locking;
      const SegLists& ml = (kind == 1 && A.afterburner) ? cands : moves;
      for (int t = 0; t < NBINS; ++t) ca.lists[t] = ml.list[t];
      ca.cnts = ml.cnt;
      ca.cdest_reset = (kind == 1 && A.afterburner && ext_ok) ? A.cdest : nullptr;
      // block 0 books the pass and decides the next one meanwhile (they read
      // only counters and part weights, final since the apply barrier), so
      // the other blocks commit the moves without it when there are any
      if (gridDim.x == 1)
        apply_commit_rows(ca, t0, nt);
      else if (blockIdx.x > 0)
        apply_commit_rows(ca, t0 - blockDim.x, nt - blockDim.x);
    }
    if (blockIdx.x == 0) {
      pc.mark(16);
      lv_bookkeep(A, &s_mc, P);
      pc.mark(17);
      lv_decide(A, &s_mc, (pass & 1) ? A.ctr : A.ctr2);
      lv_ctl_publish(C, &s_mc);
    }
    gsync();
    pc.mark(11);
    (void)wtab;
  }
  // the returned state is the best balanced one, or the fallback; when the
  // last pass made the kept state, parts already is it
  if (!S.copy_keep)
    for (int64_t v = t0; v < A.n; v += nt) A.parts[v] = A.keep[v];
  for (int i = 0; i < 8; ++i) block_sum_atomic_any((long long)wk.v[i], A.work + i);
}

// ------------------------------------------------------------------ host
// Largest cluster (<= 16 CTAs, non-portable above 8) the level kernel can be
// launched with at this shared-memory size; 0 when clusters are unavailable.
static int level_cluster_max(Ctx& c, const void* kern, size_t smem) {
  static std::map<std::pair<const void*, size_t>, int> cache;
  auto key = std::make_pair(kern, smem);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  int best = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
    (void)cudaGetLastError();
  for (int cs = LV_CLUSTER_MAX; cs >= 2; cs /= 2) {
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(cs);
    lc.blockDim = dim3(LV_BLOCK);
    lc.dynamicSmemBytes = smem;
    lc.stream = c.stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    int nclus = 0;
    if (cudaOccupancyMaxActiveClusters(&nclus, kern, &lc) != cudaSuccess) {
      (void)cudaGetLastError();
      continue;
    }
    if (nclus >= 1) {
      best = cs;
      break;
    }
  }
  cache[key] = best;
  return best;
}

static int ceil_log2_host(int64_t x) {
  int r = 0;
  while ((1LL << r) < x) ++r;
  return r;
}

struct LevelScratch : CtxExt {
  DBuf<LevelCtl> ctl;
  DBuf<long long> keep_pw;
  DBuf<int32_t> backup;
  DBuf<unsigned long long> gscratch;
  DBuf<unsigned> tailbuf;
  DBuf<unsigned long long> work;
  DBuf<unsigned long long> ctr2;
  DBuf<int32_t> ext;
  DBuf<int32_t> blists;
  DBuf<int32_t> wdeg;
};

static LevelScratch& level_scratch(Ctx& c) {
  if (!c.level_ext) c.level_ext.reset(new LevelScratch());
  return *static_cast<LevelScratch*>(c.level_ext.get());
}

bool refine_level_device(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts, int64_t& cut,
                         const jet_config& cfg, bool finest, int level, jet_level_stats& st,
                         DBuf<int32_t>& keep) {
  const int k = cfg.k;
  const int rho = (int64_t)cfg.sub_buckets >= g.n ? 1 : cfg.sub_buckets;
  if (rho > 4096) return false;
  const int tl_cap = (int)std::min<int64_t>(k, WARP_TIER_MAX_DEG);
  const size_t per = ((size_t)k + (size_t)(tl_cap + 3) / 2) * 8;
  size_t smem = (size_t)LV_TAIL_SMEM * 8 + LV_BLOCK * 8;
  smem = std::max(smem, (size_t)(LV_BLOCK / 32) * lv_stage_words<false>() * 4);
  if (g.bin_cnt[BIN_WARP]) smem = std::max(smem, per * (LV_BLOCK / 32));
  if (g.bin_cnt[BIN_BLOCK]) smem = std::max(smem, (size_t)k * 12);
  if (smem > (size_t)c.max_smem_optin) return false;

  w.ensure(c, g.n, k);
  w.bind_level(g);
  LevelScratch& S = level_scratch(c);
  S.ctl.ensure(1, c.stream);
  S.keep_pw.ensure(k, c.stream);
  S.backup.ensure(g.n, c.stream);
  S.gscratch.ensure(4 * (size_t)g.n + 2 * LV_BLOCK + 2 * LV_TAIL_SMEM + 64, c.stream);
  S.work.ensure(8, c.stream);
  dzero(c, S.work.get(), 8);
  keep.ensure(g.n, c.stream);
  const int slot_span = 34 + std::max(0, ceil_log2_host(k) - 1);
  const int64_t nb_max = (int64_t)slot_span * rho;
  const int64_t nch = ((g.n + rho - 1) / rho + 31) / 32;
  w.H.ensure((size_t)k * nb_max, c.stream);
  S.tailbuf.ensure(3 * (size_t)k * nb_max + 2048 + (size_t)g.n, c.stream);
  w.Hs.ensure((size_t)k * slot_span, c.stream);
  w.CH.ensure((size_t)k * nch, c.stream);
  w.draws.ensure(g.n + LV_DRAW_SLACK + 64, c.stream);
  w.hb.ensure(k, c.stream);

  const std::vector<int64_t> pw_in = w.h_pw;
  h2d(c, w.d_pw(), w.h_pw.data(), k);
  h2d(c, S.keep_pw.get(), (const long long*)w.h_pw.data(), k);
  d2d(c, keep.get(), parts, g.n);
  d2d(c, S.backup.get(), parts, g.n);

  LevelCtl h{};
  bool bal = true;
  int64_t worst = 0;
  for (int p = 0; p < k; ++p) {
    bal &= w.h_pw[p] <= cfg.limit;
    worst = std::max<int64_t>(worst, w.h_pw[p]);
  }
  if (getenv("JET_TRACE") && getenv("JET_TRACE")[0] == '1') {
    fprintf(stderr, "LEVEL %d start cut=%lld bal=%d worst=%lld pw=", level, (long long)cut, (int)bal,
            (long long)worst);
    for (int p = 0; p < k && p < 16; ++p) fprintf(stderr, "%lld ", (long long)w.h_pw[p]);
    fprintf(stderr, "\n");
  }
  h.cut = cut;
  h.best_cut = cut;
  h.keep_cut = cut;
  h.keep_worst = worst;
  h.has_best = bal;
  h.epoch = ++c.lock_epoch;
  h.new_epoch = h.epoch;
  h2d(c, S.ctl.get(), &h, 1);

  LevelArgs A{};
  A.g = view(g);
  A.n = g.n;
  A.k = k;
  A.tm = g.tm;
  A.wide = g.max_wdeg >= (1LL << 31);
  A.t3_two = g.max_deg > 32;
  static const int tail_grid_min = [] {
    const char* e = getenv("JET_TAIL_GRID_MIN");
    return e ? atoi(e) : LV_TAIL_SMEM / 4;
  }();
  A.tail_grid_min = tail_grid_min;
  for (int t = 0; t < NBINS; ++t) {
    A.tlist[t] = tier_list(g, t);
    A.tcnt[t] = g.bin_cnt[t];
    A.seg.b[t] = w.seg_base[t];
  }
  A.tl_cap = tl_cap;
  A.parts = parts;
  A.keep = keep.get();
  A.cdest = w.cdest.get();
  A.F = w.F.get();
  A.mv = w.mv.get();
  A.lock = w.lock.get();
  S.ext.ensure(g.n, c.stream);
  S.blists.ensure(w.cap_n, c.stream);
  // (external degrees are int32: levels with weighted degrees >= 2^31 sweep in full)
  A.ext = (getenv("JET_FULL_SWEEPS") || g.max_wdeg >= (1LL << 31)) ? nullptr : S.ext.get();
  static const int64_t bnd_min_n = [] {
    const char* e = getenv("JET_BND_MIN_N");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  A.bnd_sweeps = g.n > bnd_min_n;
  A.blists = S.blists.get();
  S.wdeg.ensure(g.n, c.stream);
  A.wdeg = g.unit_ew ? nullptr : S.wdeg.get();
  A.cand_lists = w.lists.get();
  A.move_lists = w.lists.get() + w.cap_n;
  A.ctr = w.ctr.get();
  S.ctr2.ensure(CTR_PW, c.stream);
  A.ctr2 = S.ctr2.get();
  A.keep_pw = S.keep_pw.get();
  A.rkey = w.rkey.get();
  A.rbest = w.rbest.get();
  A.rloss = w.rloss.get();
  A.rcand = w.rcand.get();
  A.evict = w.evict.get();
  A.H = w.H.get();
  A.Hs = w.Hs.get();
  A.CH = w.CH.get();
  A.opidx = w.opidx.get();
  A.valid = w.valid.get();
  A.valid_list = w.valid_list.get();
  A.opart = w.opart.get();
  A.hb = w.hb.get();
  A.deficit = w.deficit.get();
  A.required = w.required.get();
  A.spare = w.spare.get();
  A.cum_before = w.cum_before.get();
  A.bstar = w.bstar.get();
  A.thr = w.thr.get();
  A.draws = w.draws.get();
  A.gscratch = S.gscratch.get();
  A.tailbuf = S.tailbuf.get();
  A.limit = cfg.limit;
  A.sigma = cfg.sigma;
  A.W = g.total_vw;
  A.min_vw = g.min_vw;
  A.c_num = finest ? cfg.c_finest_num : cfg.c_other_num;
  A.c_den = finest ? cfg.c_finest_den : cfg.c_other_den;
  A.c_f = finest ? cfg.c_finest : cfg.c_other;
  A.c_float = finest ? cfg.c_finest_float : cfg.c_other_float;
  A.afterburner = cfg.afterburner;
  A.locking = cfg.locking;
  A.phi = cfg.phi;
  A.no_improve_limit = level_patience(cfg, level);
  A.sub_buckets = cfg.sub_buckets;
  A.seed = cfg.seed;
  A.level = level;
  A.H_cap = (int64_t)w.H.n;
  A.CH_cap = (int64_t)w.CH.n;
  A.draws_cap = (int64_t)w.draws.n;
  A.C = S.ctl.get();
  A.work = S.work.get();

  static const bool trace_env = getenv("JET_TRACE") && getenv("JET_TRACE")[0] == '1';
  const bool trace_on = trace_env || c.api_trace != nullptr;
  DBuf<long long> trace;
  if (trace_on) {
    trace.alloc(10 * 4096, c.stream);
    A.trace = trace.get();
    A.trace_cap = 4096;
  }
  static const bool phases_on = getenv("JET_PHASES") && getenv("JET_PHASES")[0] == '1';
  DBuf<unsigned long long> pclk;
  if (phases_on) {
    pclk.alloc(96, c.stream);
    dzero(c, pclk.get(), 96);
    A.phase_clk = pclk.get();
  }
  const void* kern = g.unit_ew ? (const void*)k_level<true> : (const void*)k_level<false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, LV_BLOCK, smem));
  if (per_sm < 1) return false;
  // grid barriers dominate small levels: size the cooperative grid to the
  // level (about LV_ROWS_PER_BLOCK vertices per block), capped at residency
  static const int64_t rows_per_block = [] {
    const char* e = getenv("JET_LV_ROWS_PER_BLOCK");
    return e ? std::max<int64_t>(1, atoll(e)) : LV_ROWS_PER_BLOCK;
  }();
  const int64_t want = std::max((g.n + rows_per_block - 1) / rows_per_block,
                                (g.nnz + LV_ENTRIES_PER_BLOCK - 1) / LV_ENTRIES_PER_BLOCK);
  static const int64_t one_block_n = [] {
    const char* e = getenv("JET_LV_ONE_BLOCK_N");
    return e ? (int64_t)atoll(e) : (int64_t)0;
  }();
  int blocks = g.n <= one_block_n
                   ? 1
                   : (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)per_sm * c.num_sms));
  // Small levels: the whole grid is one thread-block cluster of up to 16
  // CTAs synchronised with barrier.cluster (~0.2 us) instead of the
  // cooperative grid barrier (~1.4 us); each pass has ~10-12 barriers.
  static const int64_t cluster_n = [] {
    const char* e = getenv("JET_LV_CLUSTER_N");
    return e ? (int64_t)atoll(e) : (int64_t)LV_CLUSTER_N;
  }();
  int cl = 0;
  if (blocks > 1 && g.n <= cluster_n) {
    cl = std::min(blocks, level_cluster_max(c, kern, smem));
    if (cl < 2) cl = 0;
  }
  A.cluster_sync = cl ? 1 : 0;
  if (cl) blocks = cl;
  void* args[] = {&A};
  launch(c, "refine_level", 0.0, [&] {
    if (cl) {
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(cl);
      lc.blockDim = dim3(LV_BLOCK);
      lc.dynamicSmemBytes = smem;
      lc.stream = c.stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      CK(cudaLaunchKernelExC(&lc, kern, args));
    } else {
      CK(cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(LV_BLOCK), args, smem, c.stream));
    }
  });
  d2h(c, &h, S.ctl.get(), 1);
  unsigned long long wk[8];
  d2h(c, wk, S.work.get(), 8);
  w.h_pw.resize(k);
  d2h(c, w.h_pw.data(), (int64_t*)S.keep_pw.get(), k);
  c.sync();
  if (phases_on) {
    unsigned long long pc[96];
    d2h(c, pc, pclk.get(), 96);
    c.sync();
    static const char* names[24] = {"decide", "lp_sweep", "afterburner", "rb_collect", "rb_stats",
                                    "rb_scan", "rb_chunk", "rb_find", "rb_select", "rb_tail",
                                    "apply_delta", "commit+keep", "tail_sort", "draw_fixup", "rb_prep",
                                    "bnd_collect", "commit_rows", "bookkeep", "", "", "", "", "", ""};
    static const char* kinds[4] = {"stop", "lp", "weak", "strong"};
    const int cnt[4] = {1, h.lp, h.weak, h.strong};
    for (int kd = 1; kd < 4; ++kd) {
      if (!cnt[kd]) continue;
      fprintf(stderr, "PHASES L%d blocks=%d %s x%d (us/pass):", level, blocks, kinds[kd], cnt[kd]);
      for (int i = 0; i < 24; ++i)
        if (pc[24 * kd + i]) fprintf(stderr, " %s=%.1f", names[i], pc[24 * kd + i] / 1965.0 / cnt[kd]);
      fprintf(stderr, "\n");
    }
  }
  if (h.abort) {  // outside the device path's limits: rerun on the host path
    d2d(c, parts, S.backup.get(), g.n);
    w.h_pw = pw_in;
    h2d(c, w.d_pw(), w.h_pw.data(), k);
    c.sync();
    c.lock_epoch = h.epoch + 1;
    return false;
  }
  c.lock_epoch = h.epoch + 1;
  if (c.prof && !c.recs.empty() && c.recs.back().cls == c.prof_class("refine_level")) {
    // algorithmic bytes of the launch (roofline accounting)
    const double ebytes = g.unit_ew ? 8.0 : 12.0;  // adj + neighbour part (+ weight)
    const double list = g.identity ? 0.0 : 4.0;
    const double row_b = 8 + 4 + 4 + 4 + list;  // offsets, own part, lock, cdest (+ list id)
    const double lp_pass = (double)g.n * row_b + (double)g.nnz * ebytes;
    const double reb_pass = (double)g.n * (4 + 8);  // collect: parts + offsets
    // Jetlp: the first sweep of the level visits every row, later ones scan
    // the external degrees and visit the boundary rows (counted on device)
    const int lp_full = A.ext ? std::min(h.lp, 1) : h.lp;
    double b = lp_full * lp_pass + (h.weak + h.strong) * reb_pass;
    b += (double)(h.lp - lp_full) * (double)g.n * 4 + (double)wk[6] * (row_b + 4 + 8) +
         (double)wk[7] * ebytes;
    b += (double)wk[0] * (4 + 8 + 4 + 16) + (double)wk[1] * ebytes;            // rb stats
    b += (double)wk[2] * (4 + 8 + 4 + 4 + 8) + (double)wk[3] * (ebytes + 12);  // afterburner
    b += (double)wk[4] * (4 + 8 + 4 + 4 + 4 + 16) + (double)wk[5] * (ebytes + 4);  // apply
    c.recs.back().bytes = b;
  }
  if (trace_on) {
    std::vector<long long> t(10 * std::min(h.iterations, 4096));
    d2h(c, t.data(), trace.get(), t.size());
    c.sync();
    if (c.api_trace)
      for (size_t i = 0; i < t.size(); i += 10) {
        const int64_t rec[4] = {t[i], t[i + 2], t[i + 3], t[i + 1]};
        c.api_trace->insert(c.api_trace->end(), rec, rec + 4);
      }
    for (size_t i = 0; trace_env && i < t.size(); i += 10)
      fprintf(stderr,
              "TRACE L%d it%zu kind=%lld nm=%lld cut=%lld worst=%lld noimp=%lld best=%lld cand=%lld "
              "rcand=%lld D=%lld nover=%lld\n",
              level, i / 10, t[i], t[i + 1], t[i + 2], t[i + 3], t[i + 4], t[i + 5], t[i + 6], t[i + 7],
              t[i + 8], t[i + 9]);
  }
  cut = h.keep_cut;
  st.iterations += h.iterations;
  st.lp_passes += h.lp;
  st.weak_passes += h.weak;
  st.strong_passes += h.strong;
  st.moves += h.moves;
  st.rebalance_stuck = h.stuck;
  st.balanced = h.has_best;
  return true;
}

}  // namespace jet
