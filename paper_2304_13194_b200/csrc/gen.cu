// gen.cu — on-device benchmark inputs: the reference's
// rmat_graph and geometric_graph (generators.py:32-97) and its preprocess
// (graph.py:132-200), reproduced exactly so a device-generated graph equals
// the reference's graph for the same arguments, at sizes the host
// generator cannot reach (R-MAT scale 22: 153 s on the host; scale 27 does
// not fit).
//
// Random numbers: numpy's default_rng(words) PCG64 stream. Generator.random
// takes the i-th 64-bit output as (x >> 11) * 2^-53; PCG64 is an LCG, so
// output i is reached directly by jump-ahead (rng_dev.cuh) and the R-MAT
// rounds (one random() call of E draws each) are stride-E LCG steps.
//
// Preprocess: drop self loops, symmetrise, sort + unique (unit weights: the
// max-merge keeps 1), then the largest connected component (ties: the one
// holding the smallest vertex id) renumbered in ascending id order. The
// components come from a lock-free union-find whose roots are component
// minima (a root is only ever hooked under a smaller root).
#include "graph.cuh"
#include "rng_dev.cuh"
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include "../../include/jet.h"
#include <cstdlib>
#include <cstdio>
#include <vector>

namespace jet {

namespace {

typedef unsigned __int128 hu128;

struct Lcg {
  du128 mul, add;  // state -> mul * state + add
};

// host: coefficients of `delta` PCG64 steps (same recurrence as pcg_advance)
Lcg host_stride(uint64_t inc_hi, uint64_t inc_lo, uint64_t delta) {
  const hu128 mult = ((hu128)0x2360ED051FC65DA4ULL << 64) | (hu128)0x4385DF649FCCF645ULL;
  hu128 am = 1, ap = 0, cm = mult, cp = ((hu128)inc_hi << 64) | inc_lo;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  return Lcg{(du128)am, (du128)ap};
}

__device__ __forceinline__ double next_double(du128 s) {
  return (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_seed(const uint64_t* words, int nw, DevPcg* out) {
  uint64_t w[4];
  for (int i = 0; i < nw; ++i) w[i] = words[i];
  *out = dev_seed(w, nw);
}

// R-MAT edge i over all rounds -> two directed codes (u*n+v, v*n+u), or two
// sentinels (n*n) for a self loop (preprocess drops those).
__global__ void k_rmat(const DevPcg* g0, int64_t E, int scale, Lcg st, double a, double ab,
                       double abc, uint64_t n, uint64_t* codes) {
  const DevPcg g = *g0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E;
       i += (int64_t)gridDim.x * blockDim.x) {
    du128 s = pcg_advance(g.state, g.inc, (uint64_t)i + 1);
    uint64_t u = 0, v = 0;
    for (int r = 0; r < scale; ++r) {
      if (r) s = st.mul * s + st.add;
      const double d = next_double(s);
      const uint64_t down = d >= ab;
      const uint64_t right = (d >= a && d < ab) || d >= abc;
      u = (u << 1) | down;
      v = (v << 1) | right;
    }
    const uint64_t sent = n * n;
    codes[2 * i] = u == v ? sent : u * n + v;
    codes[2 * i + 1] = u == v ? sent : v * n + u;
  }
}

// rows from sorted unique codes: adj = code % n, offs[u] = first entry of row u
__global__ void k_codes_to_csr(const uint64_t* codes, int64_t M, uint64_t n, int64_t* offs,
                               int32_t* adj) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= M;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t u = e < M ? (int64_t)(codes[e] / n) : (int64_t)n;
    const int64_t pu = e > 0 ? (int64_t)(codes[e - 1] / n) : -1;
    for (int64_t r = pu + 1; r <= u; ++r) offs[r] = e;
    if (e < M) adj[e] = (int32_t)(codes[e] % n);
  }
}

// ---- random geometric graph ---------------------------------------------
__global__ void k_rgg_points(const DevPcg* g0, int64_t n, int64_t cells, double* pts,
                             int32_t* cell) {
  const DevPcg g = *g0;
  const double cf = (double)cells;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const du128 s = pcg_advance(g.state, g.inc, (uint64_t)(2 * i) + 1);
    const du128 s2 = pcg_advance(s, g.inc, 1);
    const double x = next_double(s), y = next_double(s2);
    pts[2 * i] = x;
    pts[2 * i + 1] = y;
    const int64_t cx = min((int64_t)__dmul_rn(x, cf), cells - 1);
    const int64_t cy = min((int64_t)__dmul_rn(y, cf), cells - 1);
    cell[i] = (int32_t)(cx * cells + cy);
  }
}

__global__ void k_count_cells(const int32_t* cell, int64_t n, int32_t* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[cell[i]], 1);
}

__global__ void k_scatter_cells(const int32_t* cell, int64_t n, const int64_t* cstart,
                                int32_t* fill, int32_t* order) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = cell[i];
    order[cstart[c] + atomicAdd(&fill[c], 1)] = (int32_t)i;
  }
}

// neighbours of point i in the 3x3 cell block with (xi-xj)^2 + (yi-yj)^2 <=
// r^2, evaluated as numpy does (separate multiply and add, no fma)
template <bool FILL>
__global__ void k_rgg_rows(const double* pts, const int32_t* cell, int64_t n, int64_t cells,
                           const int64_t* cstart, const int32_t* order, double r2, int64_t* deg,
                           const int64_t* offs, int32_t* adj) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double xi = pts[2 * i], yi = pts[2 * i + 1];
    const int64_t c = cell[i], cx = c / cells, cy = c % cells;
    int64_t k = 0, base = FILL ? offs[i] : 0;
    for (int64_t ox = cx - 1; ox <= cx + 1; ++ox) {
      if (ox < 0 || ox >= cells) continue;
      for (int64_t oy = cy - 1; oy <= cy + 1; ++oy) {
        if (oy < 0 || oy >= cells) continue;
        const int64_t cc = ox * cells + oy;
        for (int64_t q = cstart[cc]; q < cstart[cc + 1]; ++q) {
          const int j = order[q];
          if (j == i) continue;
          const double dx = __dsub_rn(xi, pts[2 * (int64_t)j]);
          const double dy = __dsub_rn(yi, pts[2 * (int64_t)j + 1]);
          if (__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)) <= r2) {
            if (FILL) adj[base + k] = j;
            ++k;
          }
        }
      }
    }
    if (!FILL) deg[i] = k;
  }
}

// ---- largest connected component + renumbering ----------------------------
__device__ __forceinline__ int uf_find(int32_t* parent, int x) {
  while (true) {
    const int p = parent[x];
    if (p == x) return x;
    const int gp = parent[p];
    if (gp != p) parent[x] = gp;  // path halving (benign race)
    x = gp;
  }
}

__global__ void k_uf_init(int32_t* parent, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = (int32_t)i;
}

// one warp per row; each undirected edge is hooked from its lower endpoint
__global__ void k_uf_hook(const int64_t* offs, const int32_t* adj, int64_t n, int32_t* parent) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    for (int64_t j = offs[u] + lane; j < offs[u + 1]; j += 32) {
      const int w = adj[j];
      if (w <= u) continue;
      int a = uf_find(parent, (int)u), b = uf_find(parent, w);
      while (a != b) {
        const int hi = max(a, b), lo = min(a, b);
        const int prev = atomicCAS(&parent[hi], hi, lo);
        if (prev == hi) break;
        a = uf_find(parent, prev);
        b = uf_find(parent, lo);
      }
    }
  }
}

// read-only chase: a path-halving write racing with another thread's
// flattening store could re-point an already flattened vertex at a non-root
__global__ void k_uf_flatten(int32_t* parent, int64_t n, unsigned long long* size) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int r = (int)i;
    while (true) {
      const int p = *(volatile int32_t*)&parent[r];
      if (p == r) break;
      r = p;
    }
    parent[i] = r;
    atomicAdd(&size[r], 1ull);
  }
}

// key = (size, -root) maximised: largest component, ties -> smallest id
__global__ void k_best_comp(const unsigned long long* size, int64_t n, unsigned long long* best) {
  unsigned long long mine = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (size[i]) mine = max(mine, (size[i] << 32) | (0xffffffffull - (unsigned long long)i));
  for (int o = 16; o; o >>= 1) mine = max(mine, __shfl_xor_sync(0xffffffffu, mine, o));
  if ((threadIdx.x & 31) == 0 && mine) atomicMax(best, mine);
}

__global__ void k_keep_deg(const int32_t* parent, const int64_t* offs, int64_t n,
                           const unsigned long long* best, int32_t* keep, int64_t* kdeg) {
  const int root = (int)(0xffffffffull - (*best & 0xffffffffull));
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool k = parent[i] == root;
    keep[i] = k;
    kdeg[i] = k ? offs[i + 1] - offs[i] : 0;
  }
}

// new ids = exclusive scan of keep; rows of kept vertices copied in order
// (their neighbours are in the same component, the map is monotone, so rows
// stay sorted)
__global__ void k_renumber(const int64_t* offs, const int32_t* adj, int64_t n, const int32_t* keep,
                           const int32_t* newid, const int64_t* noffs, int64_t* out_offs,
                           int32_t* out_adj) {
  const int lane = threadIdx.x & 31;
  for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n;
       u += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    if (!keep[u]) continue;
    const int64_t b = offs[u], e = offs[u + 1], o = noffs[u];
    for (int64_t j = b + lane; j < e; j += 32) out_adj[o + (j - b)] = newid[adj[j]];
    if (lane == 0) out_offs[newid[u]] = o;
  }
}

__global__ void k_fill1(int32_t* p, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 1;
}

template <class F>
void cub_call(Ctx& c, const char* name, F&& f) {
  size_t tmp = 0;
  CK(f(nullptr, tmp));
  void* p = c.cub_scratch(tmp);
  launch(c, name, 0.0, [&] { CK(f(p, tmp)); });
}

// Largest component of the CSR (offs, adj) over n vertices -> finalized graph.
std::unique_ptr<DGraph> lcc_graph(Ctx& c, int64_t n, DBuf<int64_t>& offs, DBuf<int32_t>& adj) {
  const int64_t nnz = n ? [&] {
    int64_t x = 0;
    d2h(c, &x, offs.get() + n, 1);
    c.sync();
    return x;
  }() : 0;
  JET_REQUIRE(nnz > 0, JET_EINVAL, "no edges remain after cleaning");
  DBuf<int32_t> parent(n, c.stream), keep(n, c.stream), newid(n + 1, c.stream);
  DBuf<unsigned long long> size(n, c.stream), best(1, c.stream);
  DBuf<int64_t> kdeg(n + 1, c.stream), noffs(n + 1, c.stream);
  dzero(c, size.get(), n);
  dzero(c, best.get(), 1);
  launch(c, "gen_uf", 0.0, [&] {
    k_uf_init<<<grid_for(c, n, 256), 256, 0, c.stream>>>(parent.get(), n);
    k_uf_hook<<<grid_for(c, n * 32, 256), 256, 0, c.stream>>>(offs.get(), adj.get(), n,
                                                              parent.get());
    k_uf_flatten<<<grid_for(c, n, 256), 256, 0, c.stream>>>(parent.get(), n, size.get());
    k_best_comp<<<grid_for(c, n, 256), 256, 0, c.stream>>>(size.get(), n, best.get());
    k_keep_deg<<<grid_for(c, n, 256), 256, 0, c.stream>>>(parent.get(), offs.get(), n,
                                                          best.get(), keep.get(), kdeg.get());
  });
  dzero(c, kdeg.get() + n, 1);
  cub_call(c, "gen_scan", [&](void* p, size_t& t) {
    return cub::DeviceScan::ExclusiveSum(p, t, kdeg.get(), noffs.get(), (int)(n + 1), c.stream);
  });
  cub_call(c, "gen_scan", [&](void* p, size_t& t) {
    return cub::DeviceScan::ExclusiveSum(p, t, keep.get(), newid.get(), (int)n, c.stream);
  });
  unsigned long long hb = 0;
  int64_t nk_nnz = 0;
  d2h(c, &hb, best.get(), 1);
  d2h(c, &nk_nnz, noffs.get() + n, 1);
  c.sync();
  const int64_t nk = (int64_t)(hb >> 32);
  if (getenv("JET_GEN_DEBUG") && getenv("JET_GEN_DEBUG")[0] == '1') {
    std::vector<int32_t> hp(n), hk(n), hn(n);
    std::vector<unsigned long long> hs(n);
    d2h(c, hp.data(), parent.get(), n);
    d2h(c, hk.data(), keep.get(), n);
    d2h(c, hn.data(), newid.get(), n);
    d2h(c, hs.data(), size.get(), n);
    c.sync();
    const int root = (int)(0xffffffffull - (hb & 0xffffffffull));
    int64_t roots = 0, eq = 0, kk = 0, bad = 0;
    for (int64_t i = 0; i < n; ++i) {
      roots += hp[i] == i;
      eq += hp[i] == root;
      kk += hk[i];
      if (hp[hp[i]] != hp[i]) ++bad;
    }
    fprintf(stderr, "LCC n=%lld root=%d nk=%lld size[root]=%llu roots=%lld parent==root %lld keep %lld "
            "non-flat %lld newid[n-1]=%d\n", (long long)n, root, (long long)nk, hs[root],
            (long long)roots, (long long)eq, (long long)kk, (long long)bad, hn[n - 1]);
  }
  auto g = std::make_unique<DGraph>();
  g->n = nk;
  g->nnz = nk_nnz;
  g->offs.alloc(nk + 1, c.stream);
  g->adj.alloc(nk_nnz, c.stream);
  g->ew.alloc(nk_nnz, c.stream);
  g->vw.alloc(nk, c.stream);
  launch(c, "gen_renumber", 0.0, [&] {
    k_renumber<<<grid_for(c, n * 32, 256), 256, 0, c.stream>>>(
        offs.get(), adj.get(), n, keep.get(), newid.get(), noffs.get(), g->offs.get(),
        g->adj.get());
    k_fill1<<<grid_for(c, nk_nnz, 256), 256, 0, c.stream>>>(g->ew.get(), nk_nnz);
    k_fill1<<<grid_for(c, nk, 256), 256, 0, c.stream>>>(g->vw.get(), nk);
  });
  h2d(c, g->offs.get() + nk, &nk_nnz, 1);
  c.sync();
  finalize_graph(c, *g);
  return g;
}

DBuf<DevPcg> seed_rng(Ctx& c, const std::vector<uint64_t>& words) {
  DBuf<uint64_t> w(words.size(), c.stream);
  h2d(c, w.get(), words.data(), words.size());
  DBuf<DevPcg> g(1, c.stream);
  k_seed<<<1, 1, 0, c.stream>>>(w.get(), (int)words.size(), g.get());
  CK(cudaGetLastError());
  c.sync();
  return g;
}

}  // namespace

std::unique_ptr<DGraph> device_rmat(Ctx& c, int scale, int edge_factor, uint64_t seed,
                                    const double probs[4]) {
  JET_REQUIRE(scale >= 1 && scale <= 30 && edge_factor >= 1, JET_EINVAL, "bad R-MAT size");
  const uint64_t n = 1ULL << scale;
  const int64_t E = (int64_t)n * edge_factor;
  // two 8-byte codes per edge, sorted with a double buffer (2 x 16 B per edge
  // at the peak), then a 4-byte adjacency and the largest component's CSR
  {
    size_t fr = 0, tot = 0;
    CK(cudaMemGetInfo(&fr, &tot));
    const double need = 32.0 * (double)E + 8.0 * (double)n;
    JET_REQUIRE(need < 0.9 * (double)(fr + c.pool_reserved), JET_ENOMEM,
                "R-MAT edge list does not fit in device memory");
  }
  DBuf<DevPcg> g0 = seed_rng(c, {seed, (uint64_t)scale, (uint64_t)edge_factor});
  DevPcg hg;
  d2h(c, &hg, g0.get(), 1);
  c.sync();
  const Lcg st = host_stride((uint64_t)(hg.inc >> 64), (uint64_t)hg.inc, (uint64_t)E);
  // thresholds exactly as numpy evaluates a + b and a + b + c
  const double a = probs[0], ab = probs[0] + probs[1], abc = (probs[0] + probs[1]) + probs[2];
  DBuf<uint64_t> codes(2 * E, c.stream), sorted(2 * E, c.stream);
  launch(c, "gen_rmat", 0.0, [&] {
    k_rmat<<<grid_for(c, E, 256), 256, 0, c.stream>>>(g0.get(), E, scale, st, a, ab, abc, n,
                                                      codes.get());
  });
  int end_bit = 1;
  while (end_bit < 64 && (1ULL << end_bit) <= n * n) ++end_bit;
  // 64-bit item counts (2E reaches 2^32 at scale 27, edge factor 16); the
  // double-buffer form needs no third copy of the keys
  const int64_t ne = 2 * E;
  cub::DoubleBuffer<uint64_t> db(codes.get(), sorted.get());
  cub_call(c, "gen_sort", [&](void* p, size_t& t) {
    return cub::DeviceRadixSort::SortKeys(p, t, db, ne, 0, end_bit, c.stream);
  });
  uint64_t* srt = db.Current();
  uint64_t* uni = db.Alternate();
  DBuf<int64_t> nu(1, c.stream);
  cub_call(c, "gen_unique", [&](void* p, size_t& t) {
    return cub::DeviceSelect::Unique(p, t, srt, uni, nu.get(), ne, c.stream);
  });
  int64_t M = 0;
  d2h(c, &M, nu.get(), 1);
  c.sync();
  uint64_t last = 0;
  if (M) {
    d2h(c, &last, uni + M - 1, 1);
    c.sync();
    if (last == n * n) --M;  // the self-loop sentinel
  }
  DBuf<int64_t> offs(n + 1, c.stream);
  DBuf<int32_t> adj(M > 0 ? M : 1, c.stream);
  launch(c, "gen_csr", 0.0, [&] {
    k_codes_to_csr<<<grid_for(c, M + 1, 256), 256, 0, c.stream>>>(uni, M, n, offs.get(),
                                                                   adj.get());
  });
  c.cub_tmp.release();
  codes.release();
  sorted.release();
  return lcc_graph(c, (int64_t)n, offs, adj);
}

std::unique_ptr<DGraph> device_rgg(Ctx& c, int64_t n, double radius, uint64_t seed) {
  JET_REQUIRE(n >= 1 && n < (1LL << 31) && radius > 0, JET_EINVAL, "bad geometric graph size");
  const int64_t cells = std::max<int64_t>(1, (int64_t)(1.0 / radius));
  JET_REQUIRE(cells * cells < (1LL << 31), JET_EUNSUPPORTED, "too many cells");
  DBuf<DevPcg> g0 = seed_rng(c, {seed, (uint64_t)n});
  DBuf<double> pts(2 * n, c.stream);
  DBuf<int32_t> cell(n, c.stream), ccnt(cells * cells + 1, c.stream), fill(cells * cells, c.stream),
      order(n, c.stream);
  DBuf<int64_t> cstart(cells * cells + 1, c.stream), deg(n + 1, c.stream), offs(n + 1, c.stream);
  dzero(c, ccnt.get(), cells * cells + 1);
  dzero(c, fill.get(), cells * cells);
  launch(c, "gen_rgg_points", 0.0, [&] {
    k_rgg_points<<<grid_for(c, n, 256), 256, 0, c.stream>>>(g0.get(), n, cells, pts.get(),
                                                            cell.get());
    k_count_cells<<<grid_for(c, n, 256), 256, 0, c.stream>>>(cell.get(), n, ccnt.get());
  });
  cub_call(c, "gen_scan", [&](void* p, size_t& t) {
    return cub::DeviceScan::ExclusiveSum(p, t, ccnt.get(), cstart.get(), (int)(cells * cells + 1),
                                         c.stream);
  });
  const double r2 = radius * radius;
  launch(c, "gen_rgg_rows", 0.0, [&] {
    k_scatter_cells<<<grid_for(c, n, 256), 256, 0, c.stream>>>(cell.get(), n, cstart.get(),
                                                               fill.get(), order.get());
    k_rgg_rows<false><<<grid_for(c, n, 128), 128, 0, c.stream>>>(
        pts.get(), cell.get(), n, cells, cstart.get(), order.get(), r2, deg.get(), nullptr,
        nullptr);
  });
  dzero(c, deg.get() + n, 1);
  cub_call(c, "gen_scan", [&](void* p, size_t& t) {
    return cub::DeviceScan::ExclusiveSum(p, t, deg.get(), offs.get(), (int)(n + 1), c.stream);
  });
  int64_t nnz = 0;
  d2h(c, &nnz, offs.get() + n, 1);
  c.sync();
  JET_REQUIRE(nnz > 0, JET_EINVAL, "radius too small: no edges generated");
  JET_REQUIRE(nnz < (1LL << 31), JET_EUNSUPPORTED, "geometric graph above 2^31 entries");
  DBuf<int32_t> adj(nnz, c.stream), adj_sorted(nnz, c.stream);
  launch(c, "gen_rgg_rows", 0.0, [&] {
    k_rgg_rows<true><<<grid_for(c, n, 128), 128, 0, c.stream>>>(
        pts.get(), cell.get(), n, cells, cstart.get(), order.get(), r2, nullptr, offs.get(),
        adj.get());
  });
  cub_call(c, "gen_sort", [&](void* p, size_t& t) {
    return cub::DeviceSegmentedSort::SortKeys(p, t, adj.get(), adj_sorted.get(), (int)nnz, (int)n,
                                              offs.get(), offs.get() + 1, c.stream);
  });
  if (getenv("JET_GEN_NO_LCC") && getenv("JET_GEN_NO_LCC")[0] == '1') {  // diagnostics
    auto g = std::make_unique<DGraph>();
    g->n = n;
    g->nnz = nnz;
    g->offs = std::move(offs);
    g->adj = std::move(adj_sorted);
    g->ew.alloc(nnz, c.stream);
    g->vw.alloc(n, c.stream);
    k_fill1<<<grid_for(c, nnz, 256), 256, 0, c.stream>>>(g->ew.get(), nnz);
    k_fill1<<<grid_for(c, n, 256), 256, 0, c.stream>>>(g->vw.get(), n);
    finalize_graph(c, *g);
    return g;
  }
  return lcc_graph(c, n, offs, adj_sorted);
}

}  // namespace jet
