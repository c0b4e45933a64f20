// controller.cu — the Jet refinement controller (refine.py:190-294) and the
// multilevel driver (driver.py:48-126) as native host code driving the
// device passes. Per iteration the only device->host traffic is the counter
// block (move counts, doubled cut delta) plus the k part weights.
#include "controller.cuh"
#include "comm.cuh"
#include "coarsen.cuh"
#include "initpart.h"
#include "initpart_dev.cuh"
#include "rng.h"
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace jet {

// Jet loop patience of a level: the reference's no_improve_limit, shortened
// in throughput mode (jet_config.throughput_patience).
int level_patience(const jet_config& cfg, int level) {
  if (cfg.deterministic || cfg.throughput_patience <= 0 || level < cfg.patience_from_level ||
      cfg.k < cfg.patience_min_k)
    return cfg.no_improve_limit;
  return std::min(cfg.throughput_patience, cfg.no_improve_limit);
}

static double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

void refine_level(Ctx& c, Workspace& w, const DGraph& g, int32_t* parts, int64_t& cut,
                  const jet_config& cfg, bool finest, int level, jet_level_stats& st,
                  DBuf<int32_t>& keep) {
  // sharded levels run the host-driven passes: the exchange
  // steps are collectives between ranks, outside any kernel
  // a distributed level (DGraph::partial) holds only its own rows: sharded
  const bool sharded = g.partial() || (c.comm && (c.comm->size > 1 || c.shard_single) &&
                                       g.n >= c.shard_min_n && cfg.afterburner != 0);
  JET_REQUIRE(!g.partial() || (c.comm && cfg.afterburner != 0), JET_EUNSUPPORTED,
              "a distributed level needs a communicator and the afterburner");
  if (!sharded && !c.host_levels &&
      refine_level_device(c, w, g, parts, cut, cfg, finest, level, st, keep))
    return;
  const int k = cfg.k;
  const int64_t limit = cfg.limit, sigma = cfg.sigma;
  w.ensure(c, g.n, k);
  w.bind_level(g);
  h2d(c, w.d_pw(), w.h_pw.data(), k);
  keep.ensure(g.n, c.stream);
  ShardLists sh;
  if (sharded) build_shard_lists(c, g, c.comm->rank, c.comm->size, sh);

  LpParams lp;
  lp.c_num = finest ? cfg.c_finest_num : cfg.c_other_num;
  lp.c_den = finest ? cfg.c_finest_den : cfg.c_other_den;
  lp.c_f = finest ? cfg.c_finest : cfg.c_other;
  lp.c_use_float = finest ? cfg.c_finest_float : cfg.c_other_float;
  lp.afterburner = cfg.afterburner;
  lp.locking = cfg.locking;

  auto balanced = [&] {
    for (int p = 0; p < k; ++p)
      if (w.h_pw[p] > limit) return false;
    return true;
  };
  auto worst = [&] { return *std::max_element(w.h_pw.begin(), w.h_pw.end()); };

  // `keep` holds the best balanced state, or while none exists the least
  // imbalanced fallback (refine.py:212-214, 274-283)
  bool has_best = balanced();
  int64_t best_cut = cut, keep_worst = worst();
  std::vector<int64_t> keep_pw = w.h_pw;
  int64_t keep_cut = cut;
  d2d(c, keep.get(), parts, g.n);

  int no_improve = 0, rebal_streak = 0, pass_index = 0;
  int64_t locked = 0;
  int32_t epoch = ++c.lock_epoch;  // fresh table: no vertex locked
  const int patience = level_patience(cfg, level);
  while (no_improve < patience) {
    bool is_lp = false, locks_all_clear = false, strong_pass = false;
    if (balanced()) {
      rebal_streak = 0;
      locks_all_clear = !cfg.locking || locked == 0;
      lp.lock_epoch = epoch;
      if (sharded) lp_pass_sharded(c, w, g, parts, k, lp, sh);
      else lp_pass(c, w, g, parts, k, lp, nullptr);
      is_lp = true;
      st.lp_passes++;
    } else {
      if (rebal_streak >= 2 + k) {
        st.rebalance_stuck = 1;
        break;
      }
      epoch = ++c.lock_epoch;  // table.reset_locks()
      locked = 0;
      // default_rng([seed, *seed_path, pass_index]); level < 0 = empty path
      Pcg64 rng = level >= 0 ? default_rng({cfg.seed, (uint64_t)level, (uint64_t)pass_index})
                             : default_rng({cfg.seed, (uint64_t)pass_index});
      const bool strong = rebal_streak >= 2;
      strong_pass = strong;
      if (!rebalance_pass(c, w, g, parts, k, limit, sigma, cfg.sub_buckets, strong, rng, nullptr,
                          sharded ? &sh : nullptr)) {
        st.rebalance_stuck = 1;
        break;
      }
      if (strong) st.strong_passes++;
      else st.weak_passes++;
      rebal_streak++;
    }
    const bool set_lock = is_lp && cfg.locking;
    const int32_t new_epoch = set_lock ? ++c.lock_epoch : epoch;
    const ApplyResult ar = apply_moves(c, w, g, parts, k, set_lock, new_epoch, sharded ? &sh : nullptr);
    if (set_lock) {
      epoch = new_epoch;
      locked = ar.n_moves;
    }
    const bool fixed_point = is_lp && ar.n_moves == 0 && locks_all_clear;
    cut += ar.cut_delta;
    pass_index++;
    st.iterations++;
    st.moves += ar.n_moves;
    no_improve++;
    if (balanced()) {
      if (!has_best || cut < best_cut) {
        if (!has_best || (double)cut < cfg.phi * (double)best_cut) no_improve = 0;
        d2d(c, keep.get(), parts, g.n);
        best_cut = cut;
        keep_cut = cut;
        keep_pw = w.h_pw;
        has_best = true;
      }
    } else if (!has_best) {
      const int64_t wv = worst();
      if (wv < keep_worst) {
        d2d(c, keep.get(), parts, g.n);
        keep_worst = wv;
        keep_cut = cut;
        keep_pw = w.h_pw;
      }
    }
    if (c.api_trace) {
      const int64_t rec[4] = {is_lp ? 1 : (strong_pass ? 3 : 2), cut, worst(), ar.n_moves};
      c.api_trace->insert(c.api_trace->end(), rec, rec + 4);
    }
    static const bool trace_on = getenv("JET_TRACE") && getenv("JET_TRACE")[0] == '1';
    if (trace_on)
      fprintf(stderr, "TRACE L%d it%d kind=%d nm=%lld cut=%lld worst=%lld noimp=%d best=%d\n", level,
              st.iterations - 1, is_lp ? 1 : (rebal_streak <= 2 ? 2 : 3), (long long)ar.n_moves,
              (long long)cut, (long long)worst(), no_improve, has_best ? 1 : 0);
    if (fixed_point) break;
    // a strong pass that moved nothing repeats identically (no RNG, same
    // state) until the loop ends: book those passes (level.cu lv_bookkeep)
    if (strong_pass && ar.n_moves == 0 && !balanced()) {
      while (no_improve < patience && rebal_streak < 2 + k) {
        st.strong_passes++;
        rebal_streak++;
        pass_index++;
        st.iterations++;
        no_improve++;
        if (c.api_trace) {
          const int64_t rec[4] = {3, cut, worst(), 0};
          c.api_trace->insert(c.api_trace->end(), rec, rec + 4);
        }
      }
    }
  }
  d2d(c, parts, keep.get(), g.n);
  cut = keep_cut;
  w.h_pw = keep_pw;
  st.balanced = has_best ? 1 : 0;
}

static void download_host_graph(Ctx& c, const DGraph& g, HostGraph& h) {
  h.n = g.n;
  h.offs.resize(g.n + 1);
  std::vector<int32_t> a(g.nnz), e(g.nnz), v(g.n);
  d2h(c, h.offs.data(), g.offs.get(), g.n + 1);
  d2h(c, a.data(), g.adj.get(), g.nnz);
  d2h(c, e.data(), g.ew.get(), g.nnz);
  d2h(c, v.data(), g.vw.get(), g.n);
  c.sync();
  h.adj.assign(a.begin(), a.end());
  h.ew.assign(e.begin(), e.end());
  h.vw.assign(v.begin(), v.end());
}

void check_partition_args(const DGraph& g, const jet_config& cfg) {
  JET_REQUIRE(cfg.k >= 1, JET_EINVAL, "k must be >= 1");
  JET_REQUIRE(cfg.k <= g.n, JET_EINVAL,
              "k=" + std::to_string(cfg.k) + " exceeds vertex count " + std::to_string(g.n));
  JET_REQUIRE(cfg.k <= KMASK, JET_EUNSUPPORTED, "k too large");
  JET_REQUIRE(g.max_vw <= cfg.limit, JET_EBALANCE,
              "vertex weight " + std::to_string(g.max_vw) + " exceeds the part weight limit " +
                  std::to_string(cfg.limit));
  JET_REQUIRE((double)cfg.k * (double)cfg.limit >= (double)g.total_vw, JET_EBALANCE,
              "k * limit cannot hold the total vertex weight");
  JET_REQUIRE(cfg.no_improve_limit >= 1 && cfg.sub_buckets >= 1 && cfg.restarts >= 1, JET_EINVAL,
              "invalid refiner configuration");
}

void run_partition(Ctx& c, const DGraph& g0, const jet_config& cfg, int32_t* parts_out,
                   int64_t* pw_out, jet_run_stats* st) {
  check_partition_args(g0, cfg);
  JET_REQUIRE(!g0.partial() || !cfg.deterministic, JET_EUNSUPPORTED,
              "a distributed graph partitions in throughput mode (the deterministic matching "
              "follows the reference's sequential scan)");
  const int k = cfg.k;
  const double t0 = now_s();
  const long long nsync0 = c.nsync;
  jet_run_stats local{};
  jet_run_stats& S = st ? *st : local;
  const double t_up = S.t_upload;
  memset(&S, 0, sizeof(S));
  S.t_upload = t_up;
  if (k == 1) {
    dzero(c, parts_out, g0.n);
    c.sync();
    S.t_total = now_s() - t0;
    S.n_levels = 1;
    S.cutsize = 0;
    S.balanced = 1;
    S.max_part_weight = g0.total_vw;
    if (pw_out) pw_out[0] = g0.total_vw;
    return;
  }
  const int64_t target = std::max<int64_t>(std::max<int64_t>(cfg.coarse_target, 2LL * k), 32);
  // a partition needs ~12x the level-0 CSR (hierarchy, workspaces, sort
  // temporaries); reserve it in the pool before starting, so no allocation
  // inside the pipeline has to map new memory (100s of ms stalls measured on
  // dense coarse levels of R-MAT 2^25), capped at 60 % of free memory
  // (cudaMemGetInfo only when the pool has to grow: the query itself stalled
  // the host for 50-90 ms in ~1 of 8 calls).
  // When the whole hierarchy cannot fit (R-MAT 2^26+: every level keeps ~m
  // edges), the owned levels get a byte budget: what is left after the input,
  // the contraction's working set (two-pass: the coarse level being built +
  // the long-row sort groups, ~1.3x the input CSR) and the refinement
  // workspace; evicted levels are rebuilt on demand (coarsen.cuh Hierarchy).
  size_t budget = 0;
  {
    const size_t csr = graph_bytes(g0);
    const char* eb = getenv("JET_HIER_BUDGET_MB");
    if (eb && atoll(eb) > 0) {
      budget = (size_t)atoll(eb) << 20;
    } else if (12 * csr > c.pool_reserved) {
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      size_t used = 0, resv = 0;
      cudaMemPool_t pool = current_pool();
      CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &resv));
      CK(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
      const size_t avail = fr + (resv > used ? resv - used : 0);
      const size_t work = (size_t)(1.3 * (double)csr) + (size_t)g0.n * 96 + ((size_t)3 << 30);
      if (12 * csr > avail) {  // the hierarchy may not fit: budgeted
        budget = avail > work + csr ? avail - work : csr;
        c.reserve_pool(std::min<size_t>(avail / 20 * 19, c.pool_reserved + fr / 20 * 19));
      } else {
        c.reserve_pool(std::min<size_t>(12 * csr, c.pool_reserved + fr / 10 * 6));
      }
    }
  }
  const double t_res = now_s();
  Hierarchy h;
  c.prof_tag = "coarsen:";
  device_build_hierarchy(c, g0, target, h, cfg.deterministic == 0, budget);
  if (budget) c.release_scratch();
  c.prof_tag.clear();
  const double t_hier = now_s();
  c.sync();
  const double t1 = now_s();
  if (getenv("JET_SYNC_STATS") || getenv("JET_HIER_STATS"))
    fprintf(stderr, "COARSEN_SPLIT pre %.2f ms hierarchy %.2f ms final sync %.2f ms budget %.2f GB "
            "resident %.2f GB evictions %d\n",
            (t_res - t0) * 1e3, (t_hier - t_res) * 1e3, (t1 - t_hier) * 1e3, budget / 1e9,
            h.resident_bytes() / 1e9, h.evictions);
  S.t_coarsen = t1 - t0;

  const int top = h.size() - 1;
  const DGraph& gc = h.level(top);
  Workspace w;
  w.ensure(c, g0.n, k);
  w.h_pw.assign(k, 0);
  int64_t cut = 0;
  DBuf<int32_t> pa(g0.n, c.stream), pb(g0.n, c.stream), keep(g0.n, c.stream);
  // initial partition: one block per restart on the device (initpart_dev.cu)
  // when asked for and within its limits, else the host restatement
  // (initpart.cpp); both reproduce initpart.py:30-94 exactly
  if (cfg.initpart_device && device_initial_partition(c, gc, k, cfg.limit, cfg.seed, cfg.restarts,
                                                      pa.get())) {
    device_part_weights(c, gc, pa.get(), k, w.d_pw());
    d2h(c, w.h_pw.data(), w.d_pw(), k);
    cut = device_cutsize(c, gc, pa.get());  // synchronises
  } else {
    HostGraph hg;
    download_host_graph(c, gc, hg);
    std::vector<int32_t> ip = host_initial_partition(hg, k, cfg.limit, cfg.seed, cfg.restarts);
    int64_t cut2 = 0;
    for (int64_t v = 0; v < hg.n; ++v) {
      w.h_pw[ip[v]] += hg.vw[v];
      for (int64_t j = hg.offs[v]; j < hg.offs[v + 1]; ++j)
        if (ip[v] != ip[hg.adj[j]]) cut2 += hg.ew[j];
    }
    cut = cut2 / 2;
    h2d(c, pa.get(), ip.data(), hg.n);
  }
  const double t2 = now_s();
  S.t_initial = t2 - t1;

  int32_t* cur = pa.get();
  int32_t* nxt = pb.get();
  int li = 0;
  for (int level = top; level >= 0; --level) {
    if (level != top) h.release(level + 1);  // projected from: no longer needed
    const int rb0 = h.rebuilds;
    const double tr = now_s();
    const DGraph& g = hier_acquire(c, h, level);
    if (h.rebuilds != rb0) {
      c.release_scratch();
      if (getenv("JET_HIER_STATS")) {
        c.sync();
        fprintf(stderr, "HIER rebuilt L%d (%d contractions, %.2f s) resident %.2f GB\n", level,
                h.rebuilds - rb0, now_s() - tr, h.resident_bytes() / 1e9);
      }
    }
    if (level != top) {
      device_project(c, h.maps[level].get(), cur, nxt, g.n);
      std::swap(cur, nxt);
    }
    jet_level_stats& L = S.levels[li++];
    memset(&L, 0, sizeof(L));
    L.level = level;
    L.distributed = g.partial() ? 1 : 0;
    L.n = g.n;
    L.m = g.nnz / 2;
    L.cut_in = cut;
    L.balanced_in = *std::max_element(w.h_pw.begin(), w.h_pw.end()) <= cfg.limit;
    const double tl = now_s();
    c.prof_tag = "L" + std::to_string(level) + ":";
    refine_level(c, w, g, cur, cut, cfg, level == 0, level, L, keep);
    c.prof_tag.clear();
    c.sync();
    L.seconds = now_s() - tl;
    L.cut_out = cut;
    L.balanced = *std::max_element(w.h_pw.begin(), w.h_pw.end()) <= cfg.limit;
  }
  d2d(c, parts_out, cur, g0.n);
  c.sync();
  const double t3 = now_s();
  S.t_uncoarsen = t3 - t2;
  S.t_total = t3 - t0;
  S.n_levels = h.size();
  S.cutsize = cut;
  S.max_part_weight = *std::max_element(w.h_pw.begin(), w.h_pw.end());
  S.balanced = S.max_part_weight <= cfg.limit;
  if (pw_out) std::copy(w.h_pw.begin(), w.h_pw.end(), pw_out);
  if (getenv("JET_SYNC_STATS"))
    fprintf(stderr, "SYNC_STATS host waits=%lld (coarsen %.3f s, uncoarsen %.3f s)\n", c.nsync - nsync0,
            S.t_coarsen, S.t_uncoarsen);
}

}  // namespace jet
