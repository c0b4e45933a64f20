// coarsen.cuh — matching, contraction and the level stack.
#pragma once
#include <memory>
#include <vector>
#include "common.cuh"
#include "graph.cuh"

namespace jet {

// levels: 0 = base (not owned), i >= 1 = owned[i-1]; maps[i]: level i -> i+1
struct Hierarchy {
  const DGraph* base = nullptr;
  std::vector<std::unique_ptr<DGraph>> owned;
  std::vector<DBuf<int32_t>> maps;
  int size() const { return 1 + (int)owned.size(); }
  const DGraph& level(int i) const { return i == 0 ? *base : *owned[i - 1]; }
};

void device_match(Ctx& c, const DGraph& g, int32_t* partner);
// partner[partner[v]] == v for all v (ids already range-checked)
bool device_is_involution(Ctx& c, const int32_t* partner, int64_t n);
std::unique_ptr<DGraph> device_contract(Ctx& c, const DGraph& g, const int32_t* partner,
                                        int32_t* vmap);
// fast: throughput-mode matching (device_match_fast), else the reference's
// exact matching semantics.
void device_build_hierarchy(Ctx& c, const DGraph& g0, int64_t target, Hierarchy& h,
                            bool fast = false);

}  // namespace jet
