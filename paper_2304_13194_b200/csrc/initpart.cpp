// initpart.cpp — initial partitioning of the coarsest level on the host.
//
// Restates initpart.py:11-94 (greedy graph growing from farthest-first BFS
// seeds, `restarts` seeded attempts, key = (unbalanced, cut)). The coarsest
// graph has at most max(200, 2k) vertices in the normal case, so this runs
// on the host like the reference does (SURVEY §8(f) row 1 lists the GPU port
// as the next step). Instead of the reference's dense k x n scans per step
// it keeps per-part frontier counts and lazy max-heaps, which select exactly
// the same (part, vertex) pair at every step:
//   part   = lightest part with an unassigned neighbour (ties -> lowest id)
//   vertex = argmax conn[part][u] over unassigned u (ties -> lowest id)
// Restarts run on separate host threads.
#include <algorithm>
#include <cstdint>
#include <queue>
#include <thread>
#include <vector>
#include "rng.h"
#include "initpart.h"

namespace jet {

namespace {

struct Entry {
  int64_t conn;
  int32_t u;
  bool operator<(const Entry& o) const {  // max-heap: larger conn, then smaller id
    if (conn != o.conn) return conn < o.conn;
    return u > o.u;
  }
};

void bfs_hops(const HostGraph& g, int32_t src, std::vector<int64_t>& dist,
              std::vector<int32_t>& queue) {
  const int64_t n = g.n;
  std::fill(dist.begin(), dist.end(), -1);
  dist[src] = 0;
  queue.clear();
  queue.push_back(src);
  for (size_t h = 0; h < queue.size(); ++h) {
    const int32_t v = queue[h];
    for (int64_t j = g.offs[v]; j < g.offs[v + 1]; ++j) {
      const int32_t u = (int32_t)g.adj[j];
      if (dist[u] < 0) {
        dist[u] = dist[v] + 1;
        queue.push_back(u);
      }
    }
  }
  for (int64_t v = 0; v < n; ++v)
    if (dist[v] < 0) dist[v] = n + 1;  // unreachable counts as infinitely far
}

// min_dist[v] = min(min_dist[v], hops(src, v)) without a full BFS: a vertex
// is expanded only when src improves its distance. If hops(src, u) >=
// min_dist[u] = hops(s', u) for an earlier seed s', no vertex behind u can
// be closer to src than to s', so the pruned search yields exactly the
// reference's np.minimum(min_dist, _bfs_hops(graph, src)) (initpart.py:38-40)
// while visiting only src's new Voronoi cell.
void bfs_improve(const HostGraph& g, int32_t src, std::vector<int64_t>& min_dist,
                 std::vector<int32_t>& queue) {
  queue.clear();
  if (min_dist[src] == 0) return;
  min_dist[src] = 0;
  queue.push_back(src);
  for (size_t h = 0; h < queue.size(); ++h) {
    const int32_t v = queue[h];
    const int64_t dv = min_dist[v] + 1;
    for (int64_t j = g.offs[v]; j < g.offs[v + 1]; ++j) {
      const int32_t u = (int32_t)g.adj[j];
      if (dv < min_dist[u]) {
        min_dist[u] = dv;
        queue.push_back(u);
      }
    }
  }
}

std::vector<int32_t> grow_single(const HostGraph& g, int k, Pcg64 rng) {
  const int64_t n = g.n;
  std::vector<int32_t> seeds;
  seeds.push_back((int32_t)rng.bounded((uint64_t)n));
  std::vector<int64_t> min_dist(n), d(n);
  std::vector<int32_t> queue;
  queue.reserve(n);
  bfs_hops(g, seeds[0], min_dist, queue);
  for (int j = 1; j < k; ++j) {
    int32_t nxt = (int32_t)(std::max_element(min_dist.begin(), min_dist.end()) - min_dist.begin());
    seeds.push_back(nxt);
    bfs_improve(g, nxt, min_dist, queue);
  }
  (void)d;

  std::vector<int32_t> parts(n, -1);
  std::vector<int64_t> weights(k, 0);
  std::vector<int64_t> fcnt(k, 0);  // unassigned vertices with conn[p][u] > 0
  std::vector<std::vector<std::pair<int32_t, int64_t>>> vconn(n);  // u -> (p, conn)
  std::vector<std::priority_queue<Entry>> heap(k);
  int64_t unassigned = n;
  int64_t first_free = 0;

  auto conn_add = [&](int32_t u, int32_t p, int64_t w) -> int64_t {
    for (auto& e : vconn[u])
      if (e.first == p) return e.second += w;
    vconn[u].push_back({p, w});
    fcnt[p]++;
    return w;
  };
  auto assign = [&](int32_t v, int32_t p) {
    parts[v] = p;
    weights[p] += g.vw[v];
    unassigned--;
    for (auto& e : vconn[v]) fcnt[e.first]--;
    for (int64_t j = g.offs[v]; j < g.offs[v + 1]; ++j) {
      const int32_t u = (int32_t)g.adj[j];
      if (parts[u] >= 0) continue;  // only unassigned connectivity is ever read
      const int64_t c = conn_add(u, p, g.ew[j]);
      heap[p].push(Entry{c, u});
    }
  };
  auto conn_of = [&](int32_t u, int32_t p) -> int64_t {
    for (auto& e : vconn[u])
      if (e.first == p) return e.second;
    return 0;
  };

  for (int p = 0; p < k; ++p) assign(seeds[p], p);
  while (unassigned > 0) {
    int best = -1;
    for (int p = 0; p < k; ++p)
      if (fcnt[p] > 0 && (best < 0 || weights[p] < weights[best])) best = p;
    int32_t v;
    if (best >= 0) {
      auto& h = heap[best];
      while (true) {
        Entry e = h.top();
        if (parts[e.u] < 0 && conn_of(e.u, best) == e.conn) {
          v = e.u;
          break;
        }
        h.pop();
      }
    } else {
      // disconnected remainder: seed the lightest part afresh
      best = (int)(std::min_element(weights.begin(), weights.end()) - weights.begin());
      while (parts[first_free] >= 0) first_free++;
      v = (int32_t)first_free;
    }
    assign(v, best);
  }
  return parts;
}

}  // namespace

std::vector<int32_t> host_initial_partition(const HostGraph& g, int k, int64_t limit,
                                            uint64_t seed, int restarts) {
  const int64_t n = g.n;
  if (k == 1) return std::vector<int32_t>(n, 0);
  std::vector<std::vector<int32_t>> res(restarts);
  std::vector<std::thread> th;
  for (int r = 0; r < restarts; ++r)
    th.emplace_back([&, r] { res[r] = grow_single(g, k, default_rng({seed, (uint64_t)r})); });
  for (auto& t : th) t.join();
  int best = -1;
  bool best_unbal = true;
  int64_t best_cut = 0;
  for (int r = 0; r < restarts; ++r) {
    std::vector<int64_t> w(k, 0);
    for (int64_t v = 0; v < n; ++v) w[res[r][v]] += g.vw[v];
    bool unbal = false;
    for (int p = 0; p < k; ++p) unbal |= w[p] > limit;
    int64_t cut2 = 0;
    for (int64_t v = 0; v < n; ++v)
      for (int64_t j = g.offs[v]; j < g.offs[v + 1]; ++j)
        if (res[r][v] != res[r][g.adj[j]]) cut2 += g.ew[j];
    const int64_t cut = cut2 / 2;
    if (best < 0 || (unbal < best_unbal) || (unbal == best_unbal && cut < best_cut)) {
      best = r;
      best_unbal = unbal;
      best_cut = cut;
    }
  }
  return res[best];
}

}  // namespace jet
