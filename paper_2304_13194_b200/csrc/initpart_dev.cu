// initpart_dev.cu — initial partitioning of the coarsest level on the device
// (initpart.py:30-94), one thread block per restart; the same semantics as
// the host restatement (initpart.cpp) and the reference:
//   seeds   : first = default_rng([seed, restart]).integers(n); the others
//             farthest-first by BFS hops (np.argmax: first maximum), a
//             pruned BFS per new seed (only its new Voronoi cell changes);
//   growing : the lightest part with an unassigned neighbour (ties: lowest
//             id) takes its best-connected unassigned vertex (ties: lowest
//             id); no frontier left: the lightest part takes the lowest
//             unassigned id;
//   choice  : key (unbalanced, cut), first restart on ties (host side).
// Every step is a block-wide reduction over packed (value, index) keys;
// the per-part connectivity to unassigned vertices is a dense k x n table
// per restart (the coarsest graph has ~max(200, 2k) vertices).
#include "initpart_dev.cuh"
#include "rng_dev.cuh"
#include <cub/block/block_reduce.cuh>
#include <climits>
#include <vector>

namespace jet {

namespace {

constexpr int IP_BT = 1024;
typedef cub::BlockReduce<unsigned long long, IP_BT> IpReduce;

struct IpArgs {
  GView g;
  int64_t n;
  int k;
  int64_t limit;
  uint64_t seed;
  int64_t* dist;     // restarts x n
  int32_t* fr;       // restarts x 2n
  int32_t* parts;    // restarts x n
  long long* wts;    // restarts x k
  long long* conn;   // restarts x k x n
  int32_t* fcnt;     // restarts x k
  long long* score;  // restarts x 2: {unbalanced, cut}
};

__device__ unsigned long long block_max(unsigned long long x, IpReduce::TempStorage& ts,
                                        unsigned long long* s_out) {
  const unsigned long long r = IpReduce(ts).Reduce(x, cub::Max());
  if (threadIdx.x == 0) *s_out = r;
  __syncthreads();
  return *s_out;
}

// min_dist <- min(min_dist, hops(src, .)); pruned level-synchronous BFS
// (full = true: the first seed, every vertex starts unreached)
__device__ void ip_bfs(const IpArgs& A, int64_t* dist, int32_t* fr, int src, bool full,
                       int* s_cnt) {
  const int64_t n = A.n;
  if (full) {
    for (int64_t v = threadIdx.x; v < n; v += IP_BT) dist[v] = LLONG_MAX;
    __syncthreads();
  } else if (dist[src] == 0) {
    return;
  }
  int32_t* cur = fr;
  int32_t* nxt = fr + n;
  if (threadIdx.x == 0) {
    dist[src] = 0;
    cur[0] = src;
    s_cnt[0] = 1;
  }
  __syncthreads();
  int len = s_cnt[0];
  long long d = 0;
  while (len > 0) {
    if (threadIdx.x == 0) s_cnt[1] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < len; i += IP_BT) {
      const int v = cur[i];
      for (int64_t j = A.g.offs[v]; j < A.g.offs[v + 1]; ++j) {
        const int u = A.g.adj[j];
        // atomicMin returns the old value: exactly one improver enqueues u
        const unsigned long long old =
            atomicMin(reinterpret_cast<unsigned long long*>(dist + u), (unsigned long long)(d + 1));
        if ((long long)old > d + 1) nxt[atomicAdd(&s_cnt[1], 1)] = u;
      }
    }
    __syncthreads();
    len = s_cnt[1];
    int32_t* t = cur;
    cur = nxt;
    nxt = t;
    ++d;
    __syncthreads();
  }
  if (full) {
    for (int64_t v = threadIdx.x; v < n; v += IP_BT)
      if (dist[v] == LLONG_MAX) dist[v] = n + 1;  // unreachable: infinitely far
    __syncthreads();
  }
}

__global__ void __launch_bounds__(IP_BT) k_initpart(IpArgs A) {
  __shared__ IpReduce::TempStorage ts;
  __shared__ unsigned long long s_red;
  __shared__ int s_cnt[2];
  const int r = blockIdx.x;
  const int64_t n = A.n;
  const int k = A.k;
  int64_t* dist = A.dist + (size_t)r * n;
  int32_t* fr = A.fr + (size_t)r * 2 * n;
  int32_t* parts = A.parts + (size_t)r * n;
  long long* wts = A.wts + (size_t)r * k;
  long long* conn = A.conn + (size_t)r * k * n;
  int32_t* fcnt = A.fcnt + (size_t)r * k;

  // ---- farthest-first seeds (initpart.py:33-40)
  __shared__ int s_seed;
  if (threadIdx.x == 0) {
    const uint64_t sd[2] = {A.seed, (uint64_t)r};
    DevPcgSeq s;
    s.g = dev_seed(sd, 2);
    s_seed = n > 1 ? (int)s.below((uint32_t)n) : 0;
  }
  __syncthreads();
  ip_bfs(A, dist, fr, s_seed, true, s_cnt);
  for (int64_t v = threadIdx.x; v < n; v += IP_BT) parts[v] = -1;
  for (int p = threadIdx.x; p < k; p += IP_BT) {
    wts[p] = 0;
    fcnt[p] = 0;
  }
  for (int64_t i = threadIdx.x; i < (int64_t)k * n; i += IP_BT) conn[i] = 0;
  __syncthreads();
  // seeds are assigned in order after all are chosen; keep them in fr's
  // second half (the BFS frontiers use [0, 2n) only while seeding)
  __shared__ int s_first;
  if (threadIdx.x == 0) s_first = s_seed;
  __syncthreads();
  int32_t* seeds = parts;  // parts are all -1 until growing: reuse as the seed list
  // (seeds must be recorded before parts is initialised for growing)
  if (threadIdx.x == 0) seeds[0] = s_first;
  __syncthreads();
  for (int j = 1; j < k; ++j) {
    unsigned long long best = 0;
    for (int64_t v = threadIdx.x; v < n; v += IP_BT) {
      const unsigned long long key = ((unsigned long long)dist[v] << 32) | (0xffffffffu - (unsigned)v);
      best = key > best ? key : best;
    }
    best = block_max(best, ts, &s_red);
    const int nxt = (int)(0xffffffffu - (unsigned)(best & 0xffffffffu));
    if (threadIdx.x == 0) seeds[j] = nxt;
    __syncthreads();
    ip_bfs(A, dist, fr, nxt, false, s_cnt);
  }
  // move the seeds aside (fr is free now) and reset parts
  for (int j = threadIdx.x; j < k; j += IP_BT) fr[j] = seeds[j];
  __syncthreads();
  for (int64_t v = threadIdx.x; v < n; v += IP_BT) parts[v] = -1;
  __syncthreads();

  // ---- greedy growing (initpart.py:42-66)
  auto assign = [&](int v, int p) {
    // v leaves the unassigned set: every part it counted towards loses it
    for (int q = threadIdx.x; q < k; q += IP_BT)
      if (conn[(size_t)q * n + v] > 0) fcnt[q]--;
    __syncthreads();
    if (threadIdx.x == 0) {
      parts[v] = p;
      wts[p] += A.g.vw[v];
    }
    __syncthreads();
    for (int64_t j = A.g.offs[v] + threadIdx.x; j < A.g.offs[v + 1]; j += IP_BT) {
      const int u = A.g.adj[j];
      if (parts[u] >= 0) continue;  // only unassigned connectivity is ever read
      const long long old = atomicAdd(reinterpret_cast<unsigned long long*>(conn + (size_t)p * n + u),
                                      (unsigned long long)A.g.ew[j]);
      if (old == 0) atomicAdd(&fcnt[p], 1);
    }
    __syncthreads();
  };
  for (int p = 0; p < k; ++p) assign(fr[p], p);
  for (int64_t left = n - k; left > 0; --left) {
    // lightest part with a frontier (ties: lowest id); key fits 64 bits for
    // part weights < 2^42 and k < 2^21 (checked by the host)
    unsigned long long pk = 0;
    for (int p = threadIdx.x; p < k; p += IP_BT)
      if (fcnt[p] > 0) {
        const unsigned long long key = ~(((unsigned long long)wts[p] << 21) | (unsigned)p);
        pk = key > pk ? key : pk;
      }
    pk = block_max(pk, ts, &s_red);
    int p, v;
    if (pk) {
      p = (int)((~pk) & ((1u << 21) - 1));
      // its best-connected unassigned vertex (ties: lowest id)
      const long long* row = conn + (size_t)p * n;
      unsigned long long vk = 0;
      for (int64_t u = threadIdx.x; u < n; u += IP_BT)
        if (parts[u] < 0 && row[u] > 0) {
          const unsigned long long key = ((unsigned long long)row[u] << 21) | (((1u << 21) - 1) - (unsigned)u);
          vk = key > vk ? key : vk;
        }
      vk = block_max(vk, ts, &s_red);
      v = (int)(((1u << 21) - 1) - (unsigned)(vk & ((1u << 21) - 1)));
    } else {
      // disconnected remainder: the lightest part takes the lowest free id
      unsigned long long wk = 0;
      for (int q = threadIdx.x; q < k; q += IP_BT) {
        const unsigned long long key = ~(((unsigned long long)wts[q] << 21) | (unsigned)q);
        wk = key > wk ? key : wk;
      }
      wk = block_max(wk, ts, &s_red);
      p = (int)((~wk) & ((1u << 21) - 1));
      unsigned long long fk = 0;
      for (int64_t u = threadIdx.x; u < n; u += IP_BT)
        if (parts[u] < 0) fk = max(fk, (unsigned long long)(0xffffffffu - (unsigned)u));
      fk = block_max(fk, ts, &s_red);
      v = (int)(0xffffffffu - (unsigned)fk);
    }
    assign(v, p);
  }
  // ---- score: (unbalanced, cut)
  unsigned long long cut2 = 0;
  for (int64_t v = threadIdx.x; v < n; v += IP_BT)
    for (int64_t j = A.g.offs[v]; j < A.g.offs[v + 1]; ++j)
      if (parts[A.g.adj[j]] != parts[v]) cut2 += (unsigned long long)A.g.ew[j];
  const unsigned long long tot = IpReduce(ts).Sum(cut2);
  __syncthreads();
  unsigned long long unb = 0;
  for (int q = threadIdx.x; q < k; q += IP_BT) unb |= wts[q] > A.limit ? 1ull : 0ull;
  unb = block_max(unb, ts, &s_red);
  if (threadIdx.x == 0) {
    A.score[2 * r] = (long long)unb;
    A.score[2 * r + 1] = (long long)(tot / 2);
  }
}

}  // namespace

bool device_initial_partition(Ctx& c, const DGraph& g, int k, int64_t limit, uint64_t seed,
                              int restarts, int32_t* parts_out) {
  const int64_t n = g.n;
  if (g.partial() || n >= (1LL << 21) || k >= (1 << 21) || g.total_vw >= (1LL << 42) ||
      (double)k * (double)n * 8.0 * restarts > 2e9)
    return false;  // outside the packed keys / table size of this path
  if (k == 1) {
    dzero(c, parts_out, n);
    return true;
  }
  DBuf<int64_t> dist((size_t)restarts * n, c.stream);
  DBuf<int32_t> fr((size_t)restarts * 2 * n, c.stream), parts((size_t)restarts * n, c.stream),
      fcnt((size_t)restarts * k, c.stream);
  DBuf<long long> wts((size_t)restarts * k, c.stream), conn((size_t)restarts * k * n, c.stream),
      score((size_t)restarts * 2, c.stream);
  IpArgs A{view(g), n, k, limit, seed, dist.get(), fr.get(), parts.get(), wts.get(), conn.get(),
           fcnt.get(), score.get()};
  launch(c, "initpart", 0.0, [&] { k_initpart<<<restarts, IP_BT, 0, c.stream>>>(A); });
  std::vector<long long> sc((size_t)restarts * 2);
  d2h(c, sc.data(), score.get(), sc.size());
  c.sync();
  int best = 0;
  for (int r = 1; r < restarts; ++r)
    if (sc[2 * r] < sc[2 * best] || (sc[2 * r] == sc[2 * best] && sc[2 * r + 1] < sc[2 * best + 1]))
      best = r;
  d2d(c, parts_out, parts.get() + (size_t)best * n, n);
  return true;
}

}  // namespace jet
