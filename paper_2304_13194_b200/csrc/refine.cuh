// refine.cuh — Jet refinement passes on device (refine.py, rebalance.py,
// conn.py:215-254). The connectivity rows conn(v, p) are never stored: every
// pass rebuilds them on chip from the CSR (register groups for short rows,
// shared-memory part tables for long rows), which is exactly what the
// reference observes of its hash table (only the nonzero contents, SURVEY
// §8(a) A9).
#pragma once
#include "common.cuh"
#include "graph.cuh"
#include <vector>

namespace jet {

// Counter slots in Workspace::ctr (the part weights follow at CTR_PW).
enum {
  CTR_CAND = 0,    // 6 per-tier candidate counts
  CTR_MOVE = 6,    // 6 per-tier move counts
  CTR_CUT2D = 12,  // 2 x cut delta of the applied moves (signed)
  CTR_CUT2 = 13,   // 2 x cut measured by the last gains sweep
  CTR_RCAND = 14,  // rebalance candidates
  CTR_EVICT = 15,  // evicted vertices
  CTR_NMOVE = 16,  // Jetlp moves flagged in place (level kernel)
  CTR_BND = 17,    // 6 per-tier boundary-row counts (level kernel)
  CTR_PW = 32
};

struct LpParams {
  long long c_num = 1, c_den = 4;
  double c_f = 0.25;
  int c_use_float = 0;
  int afterburner = 1;
  int locking = 1;
  int32_t lock_epoch = 0;  // vertices whose lock == epoch are locked
};

// Optional per-vertex outputs of the gains sweep (parity entry points).
struct LpDebug {
  int32_t* dest = nullptr;
  long long* gain = nullptr;
  uint8_t* boundary = nullptr;
  long long* conn_self = nullptr;
  long long* f2 = nullptr;
};

struct Workspace {
  int64_t cap_n = 0;
  int cap_k = 0;
  DBuf<int32_t> cdest, mv, lock, lists, rkey, rbest, rcand, evict, dest_sorted, draws;
  DBuf<long long> F;
  DBuf<double> rloss;
  DBuf<unsigned long long> ctr, H, Hs, CH, keys, keys_alt;
  DBuf<int32_t> opidx, valid_list, bstar, thr, opart;
  DBuf<uint8_t> valid;
  DBuf<double> hb;
  DBuf<long long> deficit, required, spare, cum_before;
  int64_t seg_base[NBINS] = {};
  std::vector<int64_t> h_pw;  // host mirror of the part weights
  std::vector<uint8_t> h_up;  // per-pass host scalars (packed)
  DBuf<uint8_t> up;           // their device copy

  void ensure(Ctx& c, int64_t n, int k);
  void bind_level(const DGraph& g);
  int64_t* d_pw() { return reinterpret_cast<int64_t*>(ctr.get() + CTR_PW); }
  int32_t* cand_list(int t) { return lists.get() + seg_base[t]; }
  int32_t* move_list(int t) { return lists.get() + cap_n + seg_base[t]; }
};

struct ApplyResult {
  int64_t n_moves = 0;
  int64_t cut_delta = 0;
};

// One synchronous Jetlp pass (refine.py:159-183): leaves the move set in the
// workspace move lists and mv[]; nothing is applied.
void lp_pass(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts, int k,
             const LpParams& p, const LpDebug* dbg);

// This rank's vertex block of a level (1D sharding): the
// block [lo, hi) balances entries (row offsets), and every tier list of the
// level -- ascending vertex ids -- restricted to the block is a contiguous
// sub-range, so the sweeps run on sub-lists without copying the graph.
struct ShardLists {
  int64_t lo = 0, hi = 0;
  int32_t* list[NBINS] = {};
  DBuf<int32_t> iota;                // identity tier: explicit [lo, hi)
  DBuf<unsigned long long> dcnt;     // NBINS device counts
  DBuf<int64_t> scratch;
  DBuf<uint8_t> send, recv;          // exchange buffers
  DBuf<unsigned long long> delta;    // sharded apply: {2 x cut delta, k part-weight deltas}
};
void build_shard_lists(Ctx& c, const DGraph& g, int rank, int size, ShardLists& s);

// Jetlp pass on this rank's block: gains/filter sweep over owned vertices,
// all-gather of the candidates (id, destination, gain) so every rank sees
// its neighbours' afterburner inputs, afterburner on owned candidates,
// all-gather of the moves. Every rank then holds the full move set (the
// apply and the rebalancing passes run replicated on identical state).
void lp_pass_sharded(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts, int k,
                     const LpParams& p, ShardLists& sh);
void share_moves(Ctx& c, Workspace& w, const DGraph& g, ShardLists& sh);

// Rebalancing pass (rebalance.py:139-240). Host-side scalars come from the
// part weights in w.h_pw. Returns false when no valid destination exists
// (RebalanceInfeasibleError). `rng` is advanced exactly as numpy's would be.
struct Pcg64;
struct RebalanceOut {
  std::vector<int64_t>* v = nullptr;
  std::vector<int64_t>* dest = nullptr;
  std::vector<double>* gain = nullptr;
  bool exact_rng = false;  // draw exactly #missing values (API mode)
};
// sh != nullptr: sharded (candidates of this rank's block; histograms and
// crossing-chunk element weights all-reduced, direct moves and evicted sets
// all-gathered; the ordered tail runs replicated on the global evicted set).
bool rebalance_pass(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts,
                    int k, int64_t limit, int64_t sigma, int sub_buckets,
                    bool strong, Pcg64& rng, RebalanceOut* out, ShardLists* sh = nullptr);

// Apply the pending moves (conn.py:215-254): parts, part weights, exact cut
// delta, locks. Reads back the part weights into w.h_pw.
ApplyResult apply_moves(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts,
                        int k, bool set_lock, int32_t epoch, ShardLists* sh = nullptr);

// ConnectivityTable surface (conn.cu): nonzero conn(v, p) triples of the
// given rows (all rows when rows == nullptr) sorted by (row, part), and the
// exact-delta apply of a host move list (parts, part weights; returns the cut
// delta).
int64_t conn_triples(Ctx& c, const DGraph& g, const int32_t* parts, int k, const int32_t* rows,
                     int64_t nr, std::vector<int64_t>& row_out, std::vector<int64_t>& part_out,
                     std::vector<int64_t>& w_out);
ApplyResult apply_move_list(Ctx& c, const DGraph& g, int32_t* parts, int k, int64_t* pw,
                            const int2* h_moves, int64_t nm);

// Host helpers for the parity entry points.
void afterburner_only(Ctx& c, Workspace& w, const DGraph& g, const int32_t* parts,
                      const int32_t* cand, int64_t ncand, long long* out_f2);

}  // namespace jet
