// conn.cu — the reference's ConnectivityTable surface (conn.py:29-272) on the
// device, for callers outside the refinement loop.
//
// The refinement kernels never store conn(v, p): they rebuild the rows on chip
// in every pass (refine_dev.cuh). What the reference exposes of its table is
// the set of nonzero (row, part, weight) triples (`get_many`, `row_items`,
// `nonzero_triples`, conn.py:70-123) and the exact-delta `apply`
// (conn.py:215-254). Both are provided here:
//   conn_triples : nonzero conn(v, p) of a set of rows, sorted by (row, part)
//                  (radix sort + reduce-by-key of (row, neighbour part) keys)
//   apply_move_list : parts, part weights and the exact cut delta of a move
//                  list, by the same apply kernels the refinement uses.
#include "common.cuh"
#include "graph.cuh"
#include "refine.cuh"
#include "refine_dev.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <vector>

namespace jet {

__global__ void k_row_degrees(const int64_t* __restrict__ offs, const int32_t* __restrict__ rows,
                              int64_t nr, int64_t n, int64_t* deg) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = rows ? rows[i] : i;
    deg[i] = offs[v + 1] - offs[v];
  }
  (void)n;
}

// one warp per selected row: key = row index * k + part of the neighbour
__global__ void k_conn_keys(GView g, const int32_t* __restrict__ rows, int64_t nr,
                            const int32_t* __restrict__ parts, int k,
                            const int64_t* __restrict__ out_off, unsigned long long* keys,
                            long long* vals) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < nr; i += nw) {
    const int64_t v = rows ? rows[i] : i;
    const int64_t lo = g.offs[v], hi = g.offs[v + 1], o = out_off[i];
    for (int64_t e = lo + lane; e < hi; e += 32) {
      keys[o + e - lo] = (unsigned long long)i * (unsigned long long)k +
                         (unsigned long long)parts[g.adj[e]];
      vals[o + e - lo] = g.ew ? (long long)g.ew[e] : 1LL;
    }
  }
}

int64_t conn_triples(Ctx& c, const DGraph& g, const int32_t* parts, int k, const int32_t* rows,
                     int64_t nr, std::vector<int64_t>& row_out, std::vector<int64_t>& part_out,
                     std::vector<int64_t>& w_out) {
  row_out.clear();
  part_out.clear();
  w_out.clear();
  if (nr == 0) return 0;
  DBuf<int64_t> deg(nr + 1, c.stream), off(nr + 1, c.stream);
  launch(c, "conn_degrees", 16.0 * nr, [&] {
    k_row_degrees<<<grid_for(c, nr, 256), 256, 0, c.stream>>>(g.offs.get(), rows, nr, g.n,
                                                                deg.get());
  });
  dzero(c, deg.get() + nr, 1);
  size_t tmp = 0;
  CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg.get(), off.get(), nr + 1, c.stream));
  CK(cub::DeviceScan::ExclusiveSum(c.cub_scratch(tmp), tmp, deg.get(), off.get(), nr + 1,
                                   c.stream));
  int64_t total = 0;
  d2h(c, &total, off.get() + nr, 1);
  c.sync();
  if (total == 0) return 0;
  DBuf<unsigned long long> ka(total, c.stream), kb(total, c.stream), ku(total, c.stream);
  DBuf<long long> va(total, c.stream), vb(total, c.stream), vs(total, c.stream);
  DBuf<int64_t> nuniq(1, c.stream);
  const GView gv = view(g);
  launch(c, "conn_keys", 16.0 * total, [&] {
    k_conn_keys<<<grid_for(c, nr * 32, 256), 256, 0, c.stream>>>(gv, rows, nr, parts, k,
                                                                  off.get(), ka.get(), va.get());
  });
  int bits = 1;
  while (bits < 64 && ((unsigned long long)nr * (unsigned long long)k) >> bits) ++bits;
  tmp = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, ka.get(), kb.get(), va.get(), vb.get(), total,
                                     0, bits, c.stream));
  CK(cub::DeviceRadixSort::SortPairs(c.cub_scratch(tmp), tmp, ka.get(), kb.get(), va.get(),
                                     vb.get(), total, 0, bits, c.stream));
  tmp = 0;
  CK(cub::DeviceReduce::ReduceByKey(nullptr, tmp, kb.get(), ku.get(), vb.get(), vs.get(),
                                    nuniq.get(), cub::Sum(), total, c.stream));
  CK(cub::DeviceReduce::ReduceByKey(c.cub_scratch(tmp), tmp, kb.get(), ku.get(), vb.get(),
                                    vs.get(), nuniq.get(), cub::Sum(), total, c.stream));
  int64_t nu = 0;
  d2h(c, &nu, nuniq.get(), 1);
  c.sync();
  std::vector<unsigned long long> hk(nu);
  std::vector<long long> hv(nu);
  std::vector<int32_t> hr;
  d2h(c, hk.data(), ku.get(), nu);
  d2h(c, hv.data(), vs.get(), nu);
  if (rows) {
    hr.resize(nr);
    d2h(c, hr.data(), rows, nr);
  }
  c.sync();
  for (int64_t i = 0; i < nu; ++i) {
    if (hv[i] <= 0) continue;  // conn rows hold positive weights only
    const int64_t ri = (int64_t)(hk[i] / (unsigned long long)k);
    row_out.push_back(rows ? hr[ri] : ri);
    part_out.push_back((int64_t)(hk[i] % (unsigned long long)k));
    w_out.push_back(hv[i]);
  }
  return (int64_t)row_out.size();
}

__global__ void k_scatter_moves(const int2* __restrict__ in, int64_t total, int32_t* mv,
                                const int64_t* __restrict__ offs, TierMap tm,
                                int32_t* move_lists, RbSegsDev seg,
                                unsigned long long* move_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int2 r = in[i];
    mv[r.x] = r.y;
    const int t = tm(offs[r.x + 1] - offs[r.x]);
    move_lists[seg.b[t] + atomicAdd(move_cnt + t, 1ull)] = r.x;
  }
}

ApplyResult apply_move_list(Ctx& c, const DGraph& g, int32_t* parts, int k, int64_t* pw,
                            const int2* h_moves, int64_t nm) {
  Workspace w;
  w.ensure(c, g.n, k);
  w.bind_level(g);
  dzero(c, w.ctr.get(), CTR_PW);
  h2d(c, w.d_pw(), pw, k);
  ApplyResult r;
  if (nm > 0) {
    DBuf<int2> dm(nm, c.stream);
    h2d(c, dm.get(), h_moves, nm);
    RbSegsDev ms;
    for (int t = 0; t < NBINS; ++t) ms.b[t] = w.seg_base[t];
    launch(c, "apply_scatter", 8.0 * nm, [&] {
      k_scatter_moves<<<grid_for(c, nm, 256), 256, 0, c.stream>>>(
          dm.get(), nm, w.mv.get(), g.offs.get(), g.tm, w.lists.get() + w.cap_n, ms,
          w.ctr.get() + CTR_MOVE);
    });
    r = apply_moves(c, w, g, parts, k, false, 0);
  } else {
    c.sync();
    w.h_pw.assign(pw, pw + k);
  }
  for (int p = 0; p < k; ++p) pw[p] = w.h_pw[p];
  return r;
}

}  // namespace jet
