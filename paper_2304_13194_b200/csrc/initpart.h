// initpart.h — host initial partitioning (initpart.py:70-94).
#pragma once
#include <cstdint>
#include <vector>

namespace jet {

struct HostGraph {
  int64_t n = 0;
  std::vector<int64_t> offs, adj, ew, vw;
};

std::vector<int32_t> host_initial_partition(const HostGraph& g, int k, int64_t limit,
                                            uint64_t seed, int restarts);

}  // namespace jet
