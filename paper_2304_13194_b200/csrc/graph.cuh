// graph.cuh — device CSR views and the graph-level entry points.
#pragma once
#include <memory>
#include "common.cuh"

namespace jet {

// POD view of a level passed by value to kernels.
struct GView {
  const int64_t* __restrict__ offs;
  const int32_t* __restrict__ adj;
  const int32_t* __restrict__ ew;
  const int32_t* __restrict__ vw;
  int64_t n;
};
// A partial (distributed) level's adj/ew are shifted so global entry indices
// offs[v] .. offs[v+1] address the local rows; only local rows may be read.
inline GView view(const DGraph& g) {
  return GView{g.offs.get(), g.adj.get() - g.ent_lo, g.ew.get() - g.ent_lo, g.vw.get(), g.n};
}

// Launch KERNEL<G, UNIT> for a runtime tier width G in {4,8,16,32}.
#define JET_TIER_LAUNCH(KERNEL, G, UNIT, GRID, BLOCK, SMEM, STREAM, ...)             \
  do {                                                                              \
    if (UNIT) {                                                                     \
      switch (G) {                                                                  \
        case 4: KERNEL<4, true><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;  \
        case 8: KERNEL<8, true><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;  \
        case 16: KERNEL<16, true><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break; \
        default: KERNEL<32, true><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break; \
      }                                                                             \
    } else {                                                                        \
      switch (G) {                                                                  \
        case 4: KERNEL<4, false><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;  \
        case 8: KERNEL<8, false><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break;  \
        case 16: KERNEL<16, false><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break; \
        default: KERNEL<32, false><<<GRID, BLOCK, SMEM, STREAM>>>(__VA_ARGS__); break; \
      }                                                                             \
    }                                                                               \
  } while (0)

inline const int32_t* tier_list(const DGraph& g, int t) {
  return g.identity ? nullptr : g.bin_list[t];
}

void finalize_graph(Ctx& c, DGraph& g);
// row_hi >= 0: a 1D-distributed level -- adj/ew hold only the entries of
// rows [row_lo, row_hi) (the caller passes that slice); offs and vw complete.
std::unique_ptr<DGraph> upload_graph(Ctx& c, int64_t n, const int64_t* offs,
                                     const void* adj, int adt, const void* ew,
                                     int edt, const void* vw, int vdt,
                                     int64_t row_lo = 0, int64_t row_hi = -1);
int64_t device_cutsize(Ctx& c, const DGraph& g, const int32_t* parts);
void device_part_weights(Ctx& c, const DGraph& g, const int32_t* parts, int k,
                         int64_t* d_pw);
void device_project(Ctx& c, const int32_t* vmap, const int32_t* pc, int32_t* pf,
                    int64_t nf);
void upload_i64_as_i32(Ctx& c, const int64_t* host, int64_t n, int32_t* dst,
                       long long lo, long long hi, const char* what);
void download_i32_as_i64(Ctx& c, const int32_t* dsrc, int64_t n, int64_t* host);
void set_last_error(const std::string& s);
// gen.cu: the reference's generators + preprocess, on the device
std::unique_ptr<DGraph> device_rmat(Ctx& c, int scale, int edge_factor, uint64_t seed,
                                    const double probs[4]);
std::unique_ptr<DGraph> device_rgg(Ctx& c, int64_t n, double radius, uint64_t seed);

}  // namespace jet
