// capi.cu — extern "C" surface declared in include/jet.h. Every function
// converts C++ exceptions into jet_status codes + jet_last_error().
#include "common.cuh"
#include "graph.cuh"
#include "coarsen.cuh"
#include "comm.cuh"
#include "refine.cuh"
#include "controller.cuh"
#include "initpart.h"
#include "rng.h"
#include <chrono>
#include <cstring>
#include <cstdlib>

struct jet_graph {
  std::unique_ptr<jet::DGraph> g;
  int device = 0;
  jet::Ctx* ctx = nullptr;  // owning handles keep their context (stream) alive
};
struct jet_hierarchy {
  jet::Hierarchy h;
  std::vector<jet_graph> views;  // non-owning wrappers around h's levels
  int device = 0;
  jet::Ctx* ctx = nullptr;
};

using namespace jet;

#define API_BEGIN try {
#define API_END                              \
  }                                          \
  catch (const Error& e) {                   \
    set_last_error(e.what());                \
    return e.code;                           \
  }                                          \
  catch (const std::exception& e) {          \
    set_last_error(e.what());                \
    return JET_EINTERNAL;                    \
  }                                          \
  return JET_OK;

static Ctx& C(jet_ctx* c) {
  JET_REQUIRE(c, JET_EINVAL, "context is NULL");
  Ctx* x = reinterpret_cast<Ctx*>(c);
  CK(cudaSetDevice(x->device));
  return *x;
}
static const DGraph& G(const jet_graph* g) {
  JET_REQUIRE(g && g->g, JET_EINVAL, "graph is NULL");
  return *g->g;
}

static DBuf<int32_t> upload_parts(Ctx& c, const int64_t* parts, int64_t n, int64_t k) {
  DBuf<int32_t> d(n, c.stream);
  upload_i64_as_i32(c, parts, n, d.get(), 0, k - 1, "part id");
  return d;
}

static Pcg64 from_c(const jet_pcg64& s) {
  Pcg64 g;
  g.state = ((u128)s.state_hi << 64) | s.state_lo;
  g.inc = ((u128)s.inc_hi << 64) | s.inc_lo;
  g.has_uint32 = s.has_uint32 != 0;
  g.uinteger = s.uinteger;
  return g;
}
static void to_c(const Pcg64& g, jet_pcg64& s) {
  s.state_hi = (uint64_t)(g.state >> 64);
  s.state_lo = (uint64_t)g.state;
  s.inc_hi = (uint64_t)(g.inc >> 64);
  s.inc_lo = (uint64_t)g.inc;
  s.has_uint32 = g.has_uint32 ? 1 : 0;
  s.uinteger = g.uinteger;
}

extern "C" {

int jet_graph_upload(jet_ctx* ctx, int64_t n, const int64_t* row_offsets, const void* adjacency,
                     int adj_dtype, const void* edge_weights, int ew_dtype,
                     const void* vertex_weights, int vw_dtype, jet_graph** out) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(out, JET_EINVAL, "out is NULL");
  auto g = upload_graph(c, n, row_offsets, adjacency, adj_dtype, edge_weights, ew_dtype,
                        vertex_weights, vw_dtype);
  jet_graph* jg = new jet_graph();
  jg->g = std::move(g);
  jg->device = c.device;
  jg->ctx = &c;
  ctx_retain(&c);
  *out = jg;
  API_END
}

int jet_graph_upload_block(jet_ctx* ctx, int64_t n, const int64_t* row_offsets,
                           const void* adjacency_block, int adj_dtype,
                           const void* edge_weights_block, int ew_dtype,
                           const void* vertex_weights, int vw_dtype, int64_t row_lo,
                           int64_t row_hi, jet_graph** out) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(out, JET_EINVAL, "out is NULL");
  JET_REQUIRE(row_hi >= 0, JET_EINVAL, "row_hi must be >= 0");
  auto g = upload_graph(c, n, row_offsets, adjacency_block, adj_dtype, edge_weights_block, ew_dtype,
                        vertex_weights, vw_dtype, row_lo, row_hi);
  jet_graph* jg = new jet_graph();
  jg->g = std::move(g);
  jg->device = c.device;
  jg->ctx = &c;
  ctx_retain(&c);
  *out = jg;
  API_END
}

int jet_graph_block(const jet_graph* g, int64_t* row_lo, int64_t* row_hi,
                    int64_t* local_entries) {
  API_BEGIN
  JET_REQUIRE(g && g->g, JET_EINVAL, "graph is NULL");
  const DGraph& d = *g->g;
  if (row_lo) *row_lo = d.partial() ? d.row_lo : 0;
  if (row_hi) *row_hi = d.partial() ? d.row_hi : d.n;
  if (local_entries) *local_entries = d.local_nnz();
  API_END
}

struct jet_group {
  jet::LocalGroup g;
  explicit jet_group(int n) : g(n) {}
};

int jet_comm_nccl_id(uint8_t* id128) {
  API_BEGIN
  JET_REQUIRE(id128, JET_EINVAL, "id is NULL");
  JET_REQUIRE(nccl_unique_id(id128), JET_EUNSUPPORTED, "ncclGetUniqueId failed (libnccl.so.2)");
  API_END
}

int jet_comm_attach_nccl(jet_ctx* ctx, const uint8_t* id128, int32_t rank, int32_t size) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(id128 && size >= 1 && rank >= 0 && rank < size, JET_EINVAL, "bad rank/size");
  Comm* m = make_nccl_comm(id128, rank, size);
  delete c.comm;
  c.comm = m;
  API_END
}

int jet_comm_local_group(int32_t size, jet_group** out) {
  API_BEGIN
  JET_REQUIRE(out && size >= 1, JET_EINVAL, "bad group size");
  *out = new jet_group(size);
  API_END
}

void jet_comm_local_group_free(jet_group* g) { delete g; }

int jet_comm_attach_local(jet_ctx* ctx, jet_group* g, int32_t rank) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(g && rank >= 0 && rank < g->g.size, JET_EINVAL, "bad rank");
  delete c.comm;
  c.comm = new LocalComm(&g->g, rank);
  API_END
}

int jet_comm_detach(jet_ctx* ctx) {
  API_BEGIN
  Ctx& c = C(ctx);
  delete c.comm;
  c.comm = nullptr;
  API_END
}

int jet_set_shard_min_vertices(jet_ctx* ctx, int64_t n) {
  API_BEGIN
  JET_REQUIRE(n >= 1, JET_EINVAL, "shard_min_vertices must be >= 1");
  C(ctx).shard_min_n = n;
  const char* e = getenv("JET_SHARD_SINGLE");
  C(ctx).shard_single = e && e[0] == '1';
  API_END
}

int jet_generate_rmat(jet_ctx* ctx, int32_t scale, int32_t edge_factor, uint64_t seed,
                      const double* probs4, jet_graph** out) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(out, JET_EINVAL, "out is NULL");
  const double def[4] = {0.57, 0.19, 0.19, 0.05};
  auto g = device_rmat(c, scale, edge_factor, seed, probs4 ? probs4 : def);
  jet_graph* jg = new jet_graph();
  jg->g = std::move(g);
  jg->device = c.device;
  jg->ctx = &c;
  ctx_retain(&c);
  *out = jg;
  API_END
}

int jet_generate_geometric(jet_ctx* ctx, int64_t n, double radius, uint64_t seed,
                           jet_graph** out) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(out, JET_EINVAL, "out is NULL");
  auto g = device_rgg(c, n, radius, seed);
  jet_graph* jg = new jet_graph();
  jg->g = std::move(g);
  jg->device = c.device;
  jg->ctx = &c;
  ctx_retain(&c);
  *out = jg;
  API_END
}

int jet_graph_info(const jet_graph* g, int64_t* n, int64_t* nnz, int64_t* total_vertex_weight) {
  API_BEGIN
  const DGraph& d = G(g);
  if (n) *n = d.n;
  if (nnz) *nnz = d.nnz;
  if (total_vertex_weight) *total_vertex_weight = d.total_vw;
  API_END
}

int jet_graph_download(jet_ctx* ctx, const jet_graph* g, int64_t* row_offsets, int64_t* adjacency,
                       int64_t* edge_weights, int64_t* vertex_weights) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  if (row_offsets) {
    d2h(c, row_offsets, d.offs.get(), d.n + 1);
    c.sync();
  }
  if (adjacency) download_i32_as_i64(c, d.adj.get(), d.nnz, adjacency);
  if (edge_weights) download_i32_as_i64(c, d.ew.get(), d.nnz, edge_weights);
  if (vertex_weights) download_i32_as_i64(c, d.vw.get(), d.n, vertex_weights);
  API_END
}

void jet_graph_free(jet_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  Ctx* c = g->ctx;
  delete g;
  ctx_release(c);
}

int jet_cutsize(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int64_t* cut_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  auto p = upload_parts(c, parts, d.n, 1LL << 31);
  *cut_out = device_cutsize(c, d, p.get());
  API_END
}

int jet_conn_triples(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int32_t k,
                     const int64_t* rows, int64_t n_rows, int64_t* row_out, int64_t* part_out,
                     int64_t* weight_out, int64_t cap, int64_t* count) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  JET_REQUIRE(count && n_rows >= 0, JET_EINVAL, "bad arguments");
  auto p = upload_parts(c, parts, d.n, k);
  DBuf<int32_t> dr;
  if (rows) {
    dr.alloc(std::max<int64_t>(n_rows, 1), c.stream);
    upload_i64_as_i32(c, rows, n_rows, dr.get(), 0, d.n - 1, "row id");
  }
  std::vector<int64_t> r, q, w;
  const int64_t nt = conn_triples(c, d, p.get(), k, rows ? dr.get() : nullptr,
                                  rows ? n_rows : d.n, r, q, w);
  *count = nt;
  if (row_out || part_out || weight_out) {
    JET_REQUIRE(cap >= nt, JET_EINVAL, "output capacity too small");
    for (int64_t i = 0; i < nt; ++i) {
      if (row_out) row_out[i] = r[i];
      if (part_out) part_out[i] = q[i];
      if (weight_out) weight_out[i] = w[i];
    }
  }
  API_END
}

int jet_apply_moves(jet_ctx* ctx, const jet_graph* g, int64_t* parts, int32_t k,
                    int64_t* part_weights, int64_t* cut, const int64_t* move_vertices,
                    const int64_t* move_dests, int64_t n_moves) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  JET_REQUIRE(parts && part_weights && cut && n_moves >= 0, JET_EINVAL, "bad arguments");
  std::vector<int2> mv((size_t)std::max<int64_t>(n_moves, 1));
  std::vector<uint8_t> seen;
  if (n_moves) seen.assign((size_t)d.n, 0);
  for (int64_t i = 0; i < n_moves; ++i) {
    const int64_t v = move_vertices[i], t = move_dests[i];
    JET_REQUIRE(v >= 0 && v < d.n, JET_EINVAL, "move vertex out of range");
    JET_REQUIRE(t >= 0 && t < k, JET_EINVAL, "move destination out of range");
    JET_REQUIRE(!seen[v], JET_EINVAL, "duplicate vertex in move list");
    JET_REQUIRE(parts[v] != t, JET_EASSERT, "move to current part");
    seen[v] = 1;
    mv[i] = make_int2((int)v, (int)t);
  }
  auto p = upload_parts(c, parts, d.n, k);
  const ApplyResult r = apply_move_list(c, d, p.get(), k, part_weights, mv.data(), n_moves);
  *cut += r.cut_delta;
  download_i32_as_i64(c, p.get(), d.n, parts);
  API_END
}

int jet_part_weights(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int32_t k,
                     int64_t* pw_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1, JET_EINVAL, "k must be >= 1");
  auto p = upload_parts(c, parts, d.n, k);
  DBuf<int64_t> pw(k, c.stream);
  device_part_weights(c, d, p.get(), k, pw.get());
  d2h(c, pw_out, pw.get(), k);
  c.sync();
  API_END
}

int jet_match(jet_ctx* ctx, const jet_graph* g, int64_t* partner_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  DBuf<int32_t> partner(d.n, c.stream);
  device_match(c, d, partner.get());
  download_i32_as_i64(c, partner.get(), d.n, partner_out);
  API_END
}

int jet_contract(jet_ctx* ctx, const jet_graph* g, const int64_t* partner, jet_graph** coarse_out,
                 int64_t* vmap_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  DBuf<int32_t> pd(d.n, c.stream), vmap(d.n, c.stream);
  upload_i64_as_i32(c, partner, d.n, pd.get(), 0, d.n - 1, "partner");
  JET_REQUIRE(device_is_involution(c, pd.get(), d.n), JET_EINVAL,
              "partner is not a matching (partner[partner[v]] != v)");
  auto cg_ = device_contract(c, d, pd.get(), vmap.get());
  if (vmap_out) download_i32_as_i64(c, vmap.get(), d.n, vmap_out);
  jet_graph* jg = new jet_graph();
  jg->g = std::move(cg_);
  jg->device = c.device;
  jg->ctx = &c;
  ctx_retain(&c);
  *coarse_out = jg;
  API_END
}

int jet_hierarchy_build(jet_ctx* ctx, const jet_graph* g, int64_t target, jet_hierarchy** out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  jet_hierarchy* h = new jet_hierarchy();
  h->device = c.device;
  try {
    device_build_hierarchy(c, d, target, h->h);
    c.sync();
  } catch (...) {
    delete h;
    throw;
  }
  h->ctx = &c;
  ctx_retain(&c);
  *out = h;
  API_END
}

int jet_hierarchy_levels(const jet_hierarchy* h) { return h ? h->h.size() : 0; }

const jet_graph* jet_hierarchy_level(const jet_hierarchy* h, int i) {
  if (!h || i < 0 || i >= h->h.size()) return nullptr;
  // wrap without taking ownership: release() is never called on these
  auto* self = const_cast<jet_hierarchy*>(h);
  if (self->views.empty()) {
    self->views.resize(h->h.size());
  }
  jet_graph& v = self->views[i];
  if (!v.g) v.g.reset(const_cast<DGraph*>(&h->h.level(i)));
  return &v;
}

int jet_hierarchy_map(jet_ctx* ctx, const jet_hierarchy* h, int i, int64_t* vmap_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(h && i >= 0 && i + 1 < h->h.size(), JET_EINVAL, "map index out of range");
  download_i32_as_i64(c, h->h.maps[i].get(), h->h.level(i).n, vmap_out);
  API_END
}

void jet_hierarchy_free(jet_hierarchy* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (auto& v : h->views) v.g.release();  // non-owning
  Ctx* c = h->ctx;
  delete h;
  ctx_release(c);
}

int jet_project(jet_ctx* ctx, int64_t n_coarse, const int64_t* coarse_parts, int64_t n_fine,
                const int64_t* vmap, int64_t* fine_parts_out) {
  API_BEGIN
  Ctx& c = C(ctx);
  DBuf<int32_t> pc(n_coarse, c.stream), vm(n_fine, c.stream), pf(n_fine, c.stream);
  upload_i64_as_i32(c, coarse_parts, n_coarse, pc.get(), 0, (1LL << 31) - 1, "part id");
  upload_i64_as_i32(c, vmap, n_fine, vm.get(), 0, n_coarse - 1, "vmap");
  device_project(c, vm.get(), pc.get(), pf.get(), n_fine);
  download_i32_as_i64(c, pf.get(), n_fine, fine_parts_out);
  API_END
}

int jet_select_destinations(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int32_t k,
                            int64_t* dest, int64_t* gain, uint8_t* is_boundary, int64_t* conn_self) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  auto p = upload_parts(c, parts, d.n, k);
  Workspace w;
  w.ensure(c, d.n, k);
  w.bind_level(d);
  DBuf<int32_t> od(d.n, c.stream);
  DBuf<long long> og(d.n, c.stream), oc(d.n, c.stream);
  DBuf<uint8_t> ob(d.n, c.stream);
  LpDebug dbg;
  dbg.dest = od.get();
  dbg.gain = og.get();
  dbg.boundary = ob.get();
  dbg.conn_self = oc.get();
  LpParams lp;
  lp.afterburner = 1;
  lp.locking = 0;
  lp_pass(c, w, d, p.get(), k, lp, &dbg);
  if (dest) download_i32_as_i64(c, od.get(), d.n, dest);
  if (gain) d2h(c, gain, (int64_t*)og.get(), d.n);
  if (is_boundary) d2h(c, is_boundary, ob.get(), d.n);
  if (conn_self) d2h(c, conn_self, (int64_t*)oc.get(), d.n);
  c.sync();
  API_END
}

int jet_afterburner(jet_ctx* ctx, const jet_graph* g, const int64_t* cand, int64_t n_cand,
                    const int64_t* parts, const int64_t* dests, const int64_t* gains, int64_t* out) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  auto p = upload_parts(c, parts, d.n, KMASK);
  Workspace w;
  w.ensure(c, d.n, 1);
  w.bind_level(d);
  std::vector<int32_t> cd(d.n, -1), cl(n_cand > 0 ? n_cand : 1);
  std::vector<long long> F(d.n, 0);
  for (int64_t i = 0; i < n_cand; ++i) {
    const int64_t v = cand[i];
    JET_REQUIRE(v >= 0 && v < d.n, JET_EINVAL, "candidate id out of range");
    JET_REQUIRE(dests[v] >= 0 && dests[v] < KMASK, JET_EINVAL, "destination out of range");
    cd[v] = (int32_t)dests[v];
    F[v] = gains[v];
    cl[i] = (int32_t)v;
  }
  h2d(c, w.cdest.get(), cd.data(), d.n);
  h2d(c, w.F.get(), F.data(), d.n);
  DBuf<int32_t> dcl(cl.size(), c.stream);
  h2d(c, dcl.get(), cl.data(), n_cand);
  DBuf<long long> f2(d.n, c.stream);
  afterburner_only(c, w, d, p.get(), dcl.get(), n_cand, f2.get());
  std::vector<long long> hf(d.n);
  d2h(c, hf.data(), f2.get(), d.n);
  c.sync();
  for (int64_t i = 0; i < n_cand; ++i) out[i] = hf[cand[i]];
  API_END
}

int jet_jetlp_pass(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int32_t k,
                   uint8_t* locks, int64_t c_num, int64_t c_den, double c_float,
                   int32_t c_use_float, int32_t afterburner, int32_t locking,
                   int64_t* move_vertices, int64_t* move_dests, int64_t* move_gains,
                   int64_t* n_moves) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  JET_REQUIRE(c_den >= 1, JET_EINVAL, "bad ratio");
  auto p = upload_parts(c, parts, d.n, k);
  Workspace w;
  w.ensure(c, d.n, k);
  w.bind_level(d);
  LpParams lp;
  lp.c_num = c_num;
  lp.c_den = c_den;
  lp.c_f = c_float;
  lp.c_use_float = c_use_float;
  lp.afterburner = afterburner;
  lp.locking = locking;
  lp.lock_epoch = ++c.lock_epoch;
  if (locking && locks) {
    std::vector<int32_t> lk(d.n);
    for (int64_t v = 0; v < d.n; ++v) lk[v] = locks[v] ? lp.lock_epoch : 0;
    h2d(c, w.lock.get(), lk.data(), d.n);
  }
  DBuf<long long> f2(d.n, c.stream), gn(d.n, c.stream);
  LpDebug dbg;
  dbg.f2 = f2.get();
  dbg.gain = gn.get();
  lp_pass(c, w, d, p.get(), k, lp, &dbg);
  std::vector<int32_t> mv(d.n);
  std::vector<long long> hf2(d.n), hg(d.n);
  d2h(c, mv.data(), w.mv.get(), d.n);
  d2h(c, hf2.data(), f2.get(), d.n);
  d2h(c, hg.data(), gn.get(), d.n);
  c.sync();
  int64_t m = 0;
  for (int64_t v = 0; v < d.n; ++v) {
    if (mv[v] < 0) continue;
    move_vertices[m] = v;
    move_dests[m] = mv[v];
    move_gains[m] = afterburner ? hf2[v] : hg[v];
    m++;
  }
  *n_moves = m;
  if (locking && locks)
    for (int64_t v = 0; v < d.n; ++v) locks[v] = mv[v] >= 0;
  API_END
}

int jet_rebalance_pass(jet_ctx* ctx, const jet_graph* g, const int64_t* parts, int32_t k,
                       const int64_t* part_weights, int64_t limit, int64_t sigma,
                       int32_t sub_buckets, int32_t strong, jet_pcg64* rng,
                       int64_t* move_vertices, int64_t* move_dests, double* move_gains,
                       int64_t* n_moves) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  JET_REQUIRE(sub_buckets >= 1, JET_EINVAL, "sub_buckets must be >= 1");
  auto p = upload_parts(c, parts, d.n, k);
  Workspace w;
  w.ensure(c, d.n, k);
  w.bind_level(d);
  w.h_pw.assign(part_weights, part_weights + k);
  Pcg64 r = from_c(*rng);
  std::vector<int64_t> vv, dd;
  std::vector<double> gg;
  RebalanceOut out;
  out.v = &vv;
  out.dest = &dd;
  out.gain = &gg;
  out.exact_rng = true;
  const bool ok = rebalance_pass(c, w, d, p.get(), k, limit, sigma, sub_buckets, strong != 0, r, &out);
  JET_REQUIRE(ok, JET_EREBALANCE, "no part below the destination threshold " + std::to_string(sigma));
  to_c(r, *rng);
  for (size_t i = 0; i < vv.size(); ++i) {
    move_vertices[i] = vv[i];
    move_dests[i] = dd[i];
    move_gains[i] = gg[i];
  }
  *n_moves = (int64_t)vv.size();
  API_END
}

static int refine_impl(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in,
                       const jet_config* cfg, int32_t finest, int32_t level, int64_t* parts_out,
                       int64_t* pw_out, int64_t* cut_out, jet_level_stats* stats);

int jet_refine_trace(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in,
                     const jet_config* cfg, int32_t finest, int32_t level, int64_t* parts_out,
                     int64_t* pw_out, int64_t* cut_out, jet_level_stats* stats,
                     int64_t* trace_out, int64_t trace_cap, int64_t* trace_len) {
  std::vector<int64_t> tr;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (c) c->api_trace = &tr;
  const int rc = refine_impl(ctx, g, parts_in, cfg, finest, level, parts_out, pw_out, cut_out,
                             stats);
  if (c) c->api_trace = nullptr;
  if (rc != JET_OK) return rc;
  const int64_t nrec = (int64_t)tr.size() / 4;
  if (trace_len) *trace_len = nrec;
  if (trace_out)
    for (int64_t i = 0; i < 4 * std::min(nrec, trace_cap); ++i) trace_out[i] = tr[i];
  return JET_OK;
}

int jet_refine(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in, const jet_config* cfg,
               int32_t finest, int32_t level, int64_t* parts_out, int64_t* pw_out, int64_t* cut_out,
               jet_level_stats* stats) {
  return refine_impl(ctx, g, parts_in, cfg, finest, level, parts_out, pw_out, cut_out, stats);
}

static int refine_impl(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in,
                       const jet_config* cfg, int32_t finest, int32_t level, int64_t* parts_out,
                       int64_t* pw_out, int64_t* cut_out, jet_level_stats* stats) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(cfg, JET_EINVAL, "config is NULL");
  const int k = cfg->k;
  JET_REQUIRE(k >= 1 && k <= KMASK, JET_EINVAL, "bad k");
  auto p = upload_parts(c, parts_in, d.n, k);
  Workspace w;
  w.ensure(c, d.n, k);
  DBuf<int64_t> pw(k, c.stream);
  device_part_weights(c, d, p.get(), k, pw.get());
  w.h_pw.resize(k);
  d2h(c, w.h_pw.data(), pw.get(), k);
  c.sync();
  int64_t cut = device_cutsize(c, d, p.get());
  jet_level_stats st{};
  st.level = level;
  st.n = d.n;
  st.m = d.nnz / 2;
  st.cut_in = cut;
  DBuf<int32_t> keep;
  const auto t0 = std::chrono::steady_clock::now();
  refine_level(c, w, d, p.get(), cut, *cfg, finest != 0, level, st, keep);
  c.sync();
  st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  st.cut_out = cut;
  if (parts_out) download_i32_as_i64(c, p.get(), d.n, parts_out);
  if (pw_out) memcpy(pw_out, w.h_pw.data(), sizeof(int64_t) * k);
  if (cut_out) *cut_out = cut;
  if (stats) *stats = st;
  API_END
}

int jet_initial_partition(int64_t n, const int64_t* row_offsets, const int64_t* adjacency,
                          const int64_t* edge_weights, const int64_t* vertex_weights, int32_t k,
                          int64_t limit, uint64_t seed, int32_t restarts, int64_t* parts_out) {
  API_BEGIN
  JET_REQUIRE(k >= 1, JET_EINVAL, "k must be >= 1");
  JET_REQUIRE(k <= n, JET_EINVAL, "k exceeds vertex count");
  JET_REQUIRE(restarts >= 1, JET_EINVAL, "restarts must be >= 1");
  HostGraph h;
  h.n = n;
  h.offs.assign(row_offsets, row_offsets + n + 1);
  h.adj.assign(adjacency, adjacency + row_offsets[n]);
  h.ew.assign(edge_weights, edge_weights + row_offsets[n]);
  h.vw.assign(vertex_weights, vertex_weights + n);
  auto parts = host_initial_partition(h, k, limit, seed, restarts);
  for (int64_t v = 0; v < n; ++v) parts_out[v] = parts[v];
  API_END
}

int jet_partition_graph(jet_ctx* ctx, const jet_graph* g, const jet_config* cfg, int64_t* parts_out,
                        int64_t* part_weights_out, jet_run_stats* stats) {
  API_BEGIN
  Ctx& c = C(ctx);
  const DGraph& d = G(g);
  JET_REQUIRE(cfg, JET_EINVAL, "config is NULL");
  const int64_t l0 = c.launches;
  DBuf<int32_t> parts(d.n, c.stream);
  run_partition(c, d, *cfg, parts.get(), part_weights_out, stats);
  if (parts_out) download_i32_as_i64(c, parts.get(), d.n, parts_out);
  if (stats) stats->kernel_launches = c.launches - l0;
  API_END
}

int jet_partition(jet_ctx* ctx, int64_t n, const int64_t* row_offsets, const void* adjacency,
                  int adj_dtype, const void* edge_weights, int ew_dtype, const void* vertex_weights,
                  int vw_dtype, const jet_config* cfg, int64_t* parts_out, int64_t* part_weights_out,
                  jet_run_stats* stats) {
  API_BEGIN
  Ctx& c = C(ctx);
  JET_REQUIRE(cfg, JET_EINVAL, "config is NULL");
  const int64_t l0 = c.launches;
  const auto t0 = std::chrono::steady_clock::now();
  auto g = upload_graph(c, n, row_offsets, adjacency, adj_dtype, edge_weights, ew_dtype,
                        vertex_weights, vw_dtype);
  const double t_up = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  DBuf<int32_t> parts(g->n, c.stream);
  jet_run_stats local{};
  jet_run_stats* S = stats ? stats : &local;
  S->t_upload = t_up;
  run_partition(c, *g, *cfg, parts.get(), part_weights_out, S);
  const auto t1 = std::chrono::steady_clock::now();
  download_i32_as_i64(c, parts.get(), g->n, parts_out);
  S->t_download = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
  S->kernel_launches = c.launches - l0;
  API_END
}

int jet_rng_seed(const uint32_t* words, int32_t n_words, jet_pcg64* out) {
  API_BEGIN
  std::vector<uint32_t> w(words, words + n_words);
  to_c(seed_pcg64(w), *out);
  API_END
}

int jet_rng_integers(jet_pcg64* rng, int64_t high, int64_t count, int64_t* out) {
  API_BEGIN
  JET_REQUIRE(high >= 1, JET_EINVAL, "high <= low");
  Pcg64 g = from_c(*rng);
  for (int64_t i = 0; i < count; ++i) out[i] = (int64_t)g.bounded((uint64_t)high);
  to_c(g, *rng);
  API_END
}

}  // extern "C"
