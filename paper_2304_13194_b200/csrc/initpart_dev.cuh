// initpart_dev.cuh — initial partitioning of the coarsest level on the device.
#pragma once
#include "common.cuh"
#include "graph.cuh"

namespace jet {

// One thread block per restart (initpart_dev.cu); the result equals
// host_initial_partition's (initpart.cpp) and the reference's. Returns false
// (nothing written) when the level is outside this path's limits (n or k >=
// 2^21, total vertex weight >= 2^42, or a k x n table over 2 GB).
bool device_initial_partition(Ctx& c, const DGraph& g, int k, int64_t limit, uint64_t seed,
                              int restarts, int32_t* parts_out);

}  // namespace jet
