// controller.cuh — refinement controller and multilevel driver.
#pragma once
#include <cstring>
#include "common.cuh"
#include "graph.cuh"
#include "refine.cuh"

namespace jet {

void refine_level(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts, int64_t& cut,
                  const jet_config& cfg, bool finest, int level, jet_level_stats& st,
                  DBuf<int32_t>& keep);
// The whole level in one cooperative kernel (level.cu); false when the level
// falls outside its limits (the host-driven refine_level then runs it).
bool refine_level_device(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts, int64_t& cut,
                         const jet_config& cfg, bool finest, int level, jet_level_stats& st,
                         DBuf<int32_t>& keep);
void check_partition_args(const DGraph& g, const jet_config& cfg);
// no_improve_limit of a level (shortened on coarse levels in throughput mode)
int level_patience(const jet_config& cfg, int level);
void run_partition(Ctx& c, const DGraph& g0, const jet_config& cfg, int32_t* parts_out,
                   int64_t* pw_out, jet_run_stats* st);

}  // namespace jet
