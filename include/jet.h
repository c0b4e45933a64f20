/*
 * jet.h — C-ABI of the B200-native Jet multilevel k-way partitioner.
 *
 * This is the drop-in boundary for the reference package `jetpart`
 * (/root/reference/pkg/src/jetpart). The reference has no native code and no
 * FFI: its public hot-path surface is a set of Python functions. Each entry
 * point below replaces exactly one of them; the Python package
 * `paper_2304_13194_b200` binds these through ctypes and
 * re-exposes the reference's function names, argument meaning and errors.
 *
 * Conventions
 *   - All host arrays use the reference's int64 dtype unless a dtype code is
 *     given (JET_I32 / JET_I64) so callers holding int32 data avoid a copy.
 *   - Every function returns a jet_status; on failure jet_last_error()
 *     (thread-local) holds a one-line message. The Python layer maps
 *     JET_EINVAL -> ValueError, JET_EBALANCE -> BalanceInfeasibleError,
 *     JET_EREBALANCE -> RebalanceInfeasibleError, others -> JetpartError.
 *   - A jet_ctx owns one CUDA device, one stream and a stream-ordered memory
 *     pool. Calls on one context are serialised by the caller.
 *   - No torch types and no CUDA types cross this boundary.
 */
#ifndef JET_H
#define JET_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define JET_API_VERSION 1

typedef enum {
  JET_OK = 0,
  JET_EINVAL = 1,       /* invalid argument (ValueError in Python) */
  JET_EBALANCE = 2,     /* BalanceInfeasibleError (driver.py:61-71) */
  JET_ECUDA = 3,        /* CUDA runtime / launch error */
  JET_ENOMEM = 4,       /* device allocation failed */
  JET_EREBALANCE = 5,   /* RebalanceInfeasibleError (rebalance.py:153-156) */
  JET_EINTERNAL = 6,    /* internal invariant violated */
  JET_EUNSUPPORTED = 7, /* input outside the GPU path's supported range */
  JET_EASSERT = 8       /* a reference assertion failed (AssertionError), e.g.
                           "move to current part" (conn.py:224) */
} jet_status;

#define JET_I32 4
#define JET_I64 8

typedef struct jet_ctx jet_ctx;
typedef struct jet_graph jet_graph;         /* device-resident CSR level */
typedef struct jet_hierarchy jet_hierarchy; /* device-resident level stack */

/* numpy PCG64 bit-generator state (Generator.bit_generator.state). */
typedef struct {
  uint64_t state_hi, state_lo; /* 128-bit LCG state */
  uint64_t inc_hi, inc_lo;     /* 128-bit increment (odd) */
  int32_t has_uint32;          /* buffered upper half pending */
  uint32_t uinteger;           /* the buffered half */
} jet_pcg64;

/* RefinerConfig (refine.py:34-75) plus the scalars the Python driver derives
 * with exact rational arithmetic (graph.py:203-212, rebalance.py:26-32,
 * refine.py:117-121). */
typedef struct {
  int32_t k;
  double imbalance;
  int64_t limit;           /* part_weight_limit(W, k, imbalance) */
  int64_t sigma;           /* rebalance_thresholds(...) */
  int64_t c_finest_num, c_finest_den; /* Fraction(str(c_finest)) */
  int64_t c_other_num, c_other_den;   /* Fraction(str(c_other)) */
  double c_finest, c_other;           /* used when den > 10**6 */
  int32_t c_finest_float, c_other_float;
  double phi;
  int32_t no_improve_limit;
  int32_t sub_buckets;
  uint64_t seed;
  int32_t coarse_target;
  int32_t restarts;
  int32_t afterburner;
  int32_t locking;
  int32_t deterministic; /* 1: bit-exact reference semantics in every kernel;
                            0: throughput mode (hashed-priority matching,
                            shorter Jet-loop patience when k >= 32;
                            cut gated at 1.02x the reference's geomean,
                            balance always met) */
  int32_t verbose;
  int32_t throughput_patience;  /* throughput mode only: no_improve_limit on
                                   levels >= patience_from_level when
                                   k >= patience_min_k (0: off) */
  int32_t patience_from_level;
  int32_t patience_min_k;
  int32_t initpart_device;  /* 1: initial partitioning on the device (one block
                               per restart), else on the host; same result */
} jet_config;

typedef struct {
  int32_t level;
  int64_t n, m;
  int64_t cut_in, cut_out;
  int32_t balanced_in, balanced;
  int32_t iterations, lp_passes, weak_passes, strong_passes, rebalance_stuck;
  int64_t moves;
  double seconds;
  int32_t distributed; /* 1: this rank held only its block of the level's rows */
} jet_level_stats;

#define JET_MAX_LEVELS 64

typedef struct {
  double t_upload, t_coarsen, t_initial, t_uncoarsen, t_total, t_download;
  int32_t n_levels;
  int64_t cutsize;
  int32_t balanced;
  int64_t max_part_weight;
  int64_t kernel_launches; /* device kernels launched by this call */
  jet_level_stats levels[JET_MAX_LEVELS]; /* refinement order: top .. 0 */
} jet_run_stats;

/* ---- context --------------------------------------------------------- */
int jet_create(int device, jet_ctx** out);
void jet_destroy(jet_ctx* ctx);
const char* jet_last_error(void);
int jet_api_version(void);
/* Device-time accounting for the roofline: per-kernel-class CUDA-event
 * totals (ms) and launch counts since the last reset. */
int jet_profile_enable(jet_ctx* ctx, int on);
int jet_profile_reset(jet_ctx* ctx);
/* Writes up to cap records "name\tlaunches\tms\tbytes\n" into buf. */
int jet_profile_report(jet_ctx* ctx, char* buf, int64_t cap);
int jet_synchronize(jet_ctx* ctx);
/* Record events only for launches whose class name equals `name` (NULL or
 * "" = every class). Keeps timed-region profiling cheap. */
int jet_profile_filter(jet_ctx* ctx, const char* name);
/* CUDA-event stopwatch on the context stream: start, then stop returns the
 * elapsed device milliseconds (synchronises). */
int jet_timer_start(jet_ctx* ctx);
int jet_timer_stop(jet_ctx* ctx, double* ms);
/* Overwrite a buffer larger than L2 (flush between timed iterations). */
int jet_flush_l2(jet_ctx* ctx);

/* ---- graphs (Graph, graph.py:17-100) -------------------------------- */
/* Uploads a CSR graph. row_offsets is int64[n+1]; adjacency/edge_weights
 * have nnz = row_offsets[n] entries; vertex_weights has n entries. */
int jet_graph_upload(jet_ctx* ctx, int64_t n, const int64_t* row_offsets,
                     const void* adjacency, int adj_dtype,
                     const void* edge_weights, int ew_dtype,
                     const void* vertex_weights, int vw_dtype,
                     jet_graph** out);
/* A 1D-distributed level: this rank's block of rows
 * [row_lo, row_hi). row_offsets and vertex_weights are complete (n+1 / n);
 * adjacency and edge_weights hold only the block's entries
 * [row_offsets[row_lo], row_offsets[row_hi]). Attach the communicator first
 * (the ranks agree on the level's weight statistics). Partition such graphs in
 * throughput mode: the finest level's matching, contraction and refinement
 * run distributed; the coarser levels are assembled on every rank. */
int jet_graph_upload_block(jet_ctx* ctx, int64_t n, const int64_t* row_offsets,
                           const void* adjacency_block, int adj_dtype,
                           const void* edge_weights_block, int ew_dtype,
                           const void* vertex_weights, int vw_dtype, int64_t row_lo,
                           int64_t row_hi, jet_graph** out);
/* The rows this rank stores: [row_lo, row_hi) and their entry count (the
 * whole graph for an ordinary upload). */
int jet_graph_block(const jet_graph* g, int64_t* row_lo, int64_t* row_hi,
                    int64_t* local_entries);
int jet_graph_info(const jet_graph* g, int64_t* n, int64_t* nnz,
                   int64_t* total_vertex_weight);
int jet_graph_download(jet_ctx* ctx, const jet_graph* g, int64_t* row_offsets,
                       int64_t* adjacency, int64_t* edge_weights,
                       int64_t* vertex_weights);
void jet_graph_free(jet_graph* g);

/* ---- 1D vertex sharding ----------------------------------
 * With a communicator of size > 1 attached, levels of at least
 * `shard_min_vertices` vertices (default 2^20) refine sharded: each rank owns
 * a block of vertices (balanced by entries). Jetlp passes sweep the owned
 * block and all-gather the candidates (id, destination, gain) and the moves;
 * rebalancing passes collect and score the owned candidates, all-reduce the
 * bucket histograms and crossing-chunk weights and all-gather the direct
 * moves and the evicted sets. The apply step walks the owned moved rows
 * only; the doubled cut delta and the k part-weight deltas are summed over
 * the ranks by one ncclAllReduce (k + 1 words) and every rank commits the
 * gathered move set. With a graph uploaded per rank (jet_graph_upload_block,
 * throughput mode) the matching and contraction run distributed as well and
 * large coarse levels stay distributed; otherwise coarsening runs replicated.
 * Smaller levels run unsharded. Every rank computes the same partition,
 * bit-identical to the unsharded run.
 * NCCL (one process per GPU): rank 0 calls jet_comm_nccl_id, the id is
 * broadcast out of band (torch.distributed), every rank attaches.
 * Local groups: `size` contexts in one process (one thread each) on one GPU
 * share a group -- the same code path, for testing without several GPUs. */
typedef struct jet_group jet_group;
int jet_comm_nccl_id(uint8_t* id128);
int jet_comm_attach_nccl(jet_ctx* ctx, const uint8_t* id128, int32_t rank, int32_t size);
int jet_comm_local_group(int32_t size, jet_group** out);
void jet_comm_local_group_free(jet_group* g);
int jet_comm_attach_local(jet_ctx* ctx, jet_group* g, int32_t rank);
int jet_comm_detach(jet_ctx* ctx);
int jet_set_shard_min_vertices(jet_ctx* ctx, int64_t n);

/* ---- on-device benchmark inputs (generators.py, graph.py:132-200) ---- */
/* The reference's rmat_graph(scale, edge_factor, seed, probs)
 * (generators.py:32-55) and geometric_graph(n, radius, seed)
 * (generators.py:58-97), each followed by its preprocess (graph.py:132-200:
 * self loops dropped, symmetrised, duplicates merged, largest connected
 * component renumbered), generated on the device. The result is identical to
 * the reference's graph for the same arguments (numpy's PCG64 stream is
 * replayed by jump-ahead). probs4 may be NULL for (0.57, 0.19, 0.19, 0.05).
 * Limits: 2 * 2^scale * edge_factor < 2^31; geometric n < 2^31. */
int jet_generate_rmat(jet_ctx* ctx, int32_t scale, int32_t edge_factor, uint64_t seed,
                      const double* probs4, jet_graph** out);
int jet_generate_geometric(jet_ctx* ctx, int64_t n, double radius, uint64_t seed,
                           jet_graph** out);

/* ---- metrics ---------------------------------------------------------- */
/* cutsize(graph, parts)  graph.py:215-221 */
int jet_cutsize(jet_ctx* ctx, const jet_graph* g, const int64_t* parts,
                int64_t* cut_out);
/* ConnectivityTable contents (conn.py:70-123): the nonzero conn(v, p) of
 * the given rows (rows == NULL: every row) as (row, part, weight) triples
 * sorted by (row, part). *count receives the number of triples; the output
 * arrays (any may be NULL) need cap >= *count entries (a call with all
 * outputs NULL returns the count only). Rows are rebuilt from the CSR. */
int jet_conn_triples(jet_ctx* ctx, const jet_graph* g, const int64_t* parts,
                     int32_t k, const int64_t* rows, int64_t n_rows,
                     int64_t* row_out, int64_t* part_out, int64_t* weight_out,
                     int64_t cap, int64_t* count);
/* ConnectivityTable.apply / update_conn (conn.py:215-254, 270-272): apply a
 * move list to (parts, part_weights, cut) in place by exact deltas.
 * Duplicate vertices are JET_EINVAL (moves.py:31-32); a move to the current
 * part is JET_EASSERT (conn.py:224). */
int jet_apply_moves(jet_ctx* ctx, const jet_graph* g, int64_t* parts, int32_t k,
                    int64_t* part_weights, int64_t* cut,
                    const int64_t* move_vertices, const int64_t* move_dests,
                    int64_t n_moves);
/* PartitionState.from_parts weights  graph.py:240-242 */
int jet_part_weights(jet_ctx* ctx, const jet_graph* g, const int64_t* parts,
                     int32_t k, int64_t* pw_out);

/* ---- coarsening (coarsen.py) ------------------------------------------ */
/* match_vertices(graph)  coarsen.py:47-107 */
int jet_match(jet_ctx* ctx, const jet_graph* g, int64_t* partner_out);
/* contract(graph, matching)  coarsen.py:110-138 */
int jet_contract(jet_ctx* ctx, const jet_graph* g, const int64_t* partner,
                 jet_graph** coarse_out, int64_t* vmap_out);
/* build_hierarchy(graph, target)  coarsen.py:141-161 (levels[0] = g) */
int jet_hierarchy_build(jet_ctx* ctx, const jet_graph* g, int64_t target,
                        jet_hierarchy** out);
int jet_hierarchy_levels(const jet_hierarchy* h);
const jet_graph* jet_hierarchy_level(const jet_hierarchy* h, int i);
int jet_hierarchy_map(jet_ctx* ctx, const jet_hierarchy* h, int i,
                      int64_t* vmap_out);
void jet_hierarchy_free(jet_hierarchy* h);

/* project(coarse_state, vmap, fine)  driver.py:32-45 (parts only) */
int jet_project(jet_ctx* ctx, int64_t n_coarse, const int64_t* coarse_parts,
                int64_t n_fine, const int64_t* vmap, int64_t* fine_parts_out);

/* ---- Jet refinement (refine.py) --------------------------------------- */
/* select_destinations  refine.py:78-105. Any output may be NULL. */
int jet_select_destinations(jet_ctx* ctx, const jet_graph* g,
                            const int64_t* parts, int32_t k, int64_t* dest,
                            int64_t* gain, uint8_t* is_boundary,
                            int64_t* conn_self);
/* afterburner  refine.py:127-156 */
int jet_afterburner(jet_ctx* ctx, const jet_graph* g, const int64_t* cand,
                    int64_t n_cand, const int64_t* parts, const int64_t* dests,
                    const int64_t* gains, int64_t* out);
/* jetlp_pass  refine.py:159-183. locks is read and (when locking) rewritten.
 * Moves are returned in ascending vertex order. */
int jet_jetlp_pass(jet_ctx* ctx, const jet_graph* g, const int64_t* parts,
                   int32_t k, uint8_t* locks, int64_t c_num, int64_t c_den,
                   double c_float, int32_t c_use_float, int32_t afterburner,
                   int32_t locking, int64_t* move_vertices,
                   int64_t* move_dests, int64_t* move_gains,
                   int64_t* n_moves);
/* weak_rebalance_pass / strong_rebalance_pass  rebalance.py:139-240.
 * rng is advanced exactly as numpy would. Moves come out in the reference
 * order (oversized parts ascending, bucket order inside each part).
 * move_gains = -loss (int-valued for weak, float64 for strong). */
int jet_rebalance_pass(jet_ctx* ctx, const jet_graph* g, const int64_t* parts,
                       int32_t k, const int64_t* part_weights, int64_t limit,
                       int64_t sigma, int32_t sub_buckets, int32_t strong,
                       jet_pcg64* rng, int64_t* move_vertices,
                       int64_t* move_dests, double* move_gains,
                       int64_t* n_moves);
/* jet_refine(graph, state, config, finest, seed_path=(level,))
 * refine.py:190-294. parts_out receives the returned state's parts. */
int jet_refine(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in,
               const jet_config* cfg, int32_t finest, int32_t level,
               int64_t* parts_out, int64_t* pw_out, int64_t* cut_out,
               jet_level_stats* stats);

/* jet_refine with the per-iteration trace of stats["trace"]
 * (refine.py:269-271): trace_out receives up to trace_cap records of four
 * int64 (kind 1 = lp / 2 = weak / 3 = strong, cutsize, max part weight,
 * moves); *trace_len the number of iterations. */
int jet_refine_trace(jet_ctx* ctx, const jet_graph* g, const int64_t* parts_in,
                     const jet_config* cfg, int32_t finest, int32_t level,
                     int64_t* parts_out, int64_t* pw_out, int64_t* cut_out,
                     jet_level_stats* stats, int64_t* trace_out,
                     int64_t trace_cap, int64_t* trace_len);

/* ---- initial partitioning (initpart.py:70-94; host C++) --------------- */
int jet_initial_partition(int64_t n, const int64_t* row_offsets,
                          const int64_t* adjacency, const int64_t* edge_weights,
                          const int64_t* vertex_weights, int32_t k,
                          int64_t limit, uint64_t seed, int32_t restarts,
                          int64_t* parts_out);

/* ---- whole pipeline: partition(graph, config)  driver.py:48-126 -------- */
int jet_partition(jet_ctx* ctx, int64_t n, const int64_t* row_offsets,
                  const void* adjacency, int adj_dtype,
                  const void* edge_weights, int ew_dtype,
                  const void* vertex_weights, int vw_dtype,
                  const jet_config* cfg, int64_t* parts_out,
                  int64_t* part_weights_out, jet_run_stats* stats);
/* Same pipeline on an already-resident graph (device-timed benchmark leg).
 * parts_out / part_weights_out may be NULL. */
int jet_partition_graph(jet_ctx* ctx, const jet_graph* g, const jet_config* cfg,
                        int64_t* parts_out, int64_t* part_weights_out,
                        jet_run_stats* stats);

/* ---- numpy RNG restatement (host; used by the controller) ------------- */
/* default_rng(entropy words).bit_generator.state */
int jet_rng_seed(const uint32_t* words, int32_t n_words, jet_pcg64* out);
/* Generator.integers(0, high, size=count) into out (int64). */
int jet_rng_integers(jet_pcg64* rng, int64_t high, int64_t count,
                     int64_t* out);

#ifdef __cplusplus
}
#endif
#endif /* JET_H */
