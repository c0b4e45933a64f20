// coarsen.cuh — matching, contraction and the level stack.
#pragma once
#include <memory>
#include <vector>
#include "common.cuh"
#include "graph.cuh"

namespace jet {

// levels: 0 = base (not owned), i >= 1 = owned[i-1]; maps[i]: level i -> i+1
//
// Out-of-memory hierarchies (R-MAT 2^27: every level keeps ~m edges, ~10x the
// input CSR in all, more than one B200 holds): with a byte budget set, owned
// levels are evicted lowest-first once the resident ones exceed it, keeping
// only their sizes and the matching that built them (partners[i], n_i words).
// acquire(i) rebuilds an evicted level by re-contracting from the highest
// resident level below it -- contraction is a deterministic function of
// (fine graph, matching), so the rebuilt level is bit-identical.
struct Hierarchy {
  const DGraph* base = nullptr;
  std::vector<std::unique_ptr<DGraph>> owned;  // nullptr: evicted
  std::vector<DBuf<int32_t>> maps;
  std::vector<DBuf<int32_t>> partners;  // partners[i]: the matching of level i (budgeted runs)
  std::vector<int64_t> lv_n, lv_nnz;     // sizes of every level (resident or not)
  size_t budget = 0;                     // bytes of owned levels kept resident (0: unlimited)
  int rebuilds = 0, evictions = 0;
  int size() const { return 1 + (int)owned.size(); }
  bool resident(int i) const { return i == 0 || owned[i - 1] != nullptr; }
  const DGraph& level(int i) const { return i == 0 ? *base : *owned[i - 1]; }
  size_t resident_bytes() const;
  // evict owned levels (lowest first, never `keep_a`/`keep_b`) until the
  // resident ones fit `limit` bytes; false if nothing could be evicted
  bool shrink_to(size_t limit, int keep_a, int keep_b);
  void release(int i);  // drop an owned level for good (uncoarsening is past it)
};
size_t graph_bytes(const DGraph& g);
// The level, rebuilt (and kept within the budget) if it was evicted.
const DGraph& hier_acquire(Ctx& c, Hierarchy& h, int i);

void device_match(Ctx& c, const DGraph& g, int32_t* partner);
// partner[partner[v]] == v for all v (ids already range-checked)
bool device_is_involution(Ctx& c, const int32_t* partner, int64_t n);
// two_pass: count, then merge straight into the exact-size coarse arrays (no
// fine-sized staging buffers; memory-tight hierarchies)
std::unique_ptr<DGraph> device_contract(Ctx& c, const DGraph& g, const int32_t* partner,
                                        int32_t* vmap, bool two_pass = false);
// fast: throughput-mode matching (device_match_fast), else the reference's
// exact matching semantics.
void device_build_hierarchy(Ctx& c, const DGraph& g0, int64_t target, Hierarchy& h,
                            bool fast = false, size_t budget = 0);

}  // namespace jet
