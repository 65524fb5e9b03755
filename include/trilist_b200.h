/*
 * trilist_b200.h -- C-ABI of the B200-native AOT triangle-listing path.
 *
 * Drop-in boundary for the hot path of the reference C++ library `trilist`
 * (/root/reference/proj).  Every entry point lists the reference interface it
 * replaces.  All pointers are plain host pointers unless a parameter name
 * starts with `d_` (device pointer).  Functions return TL_OK (0) or a TL_E*
 * code; tl_last_error() returns the thread-local message of the last failure.
 * The error codes map onto the reference's exception types:
 *   TL_EINVAL -> std::invalid_argument   TL_ERANGE -> std::out_of_range
 *   TL_ELOGIC -> std::logic_error        TL_ECUDA/TL_ENOMEM -> std::runtime_error
 *
 * There is no CPU fallback: every compute step below runs as a CUDA kernel for
 * sm_100a; without a usable CUDA device the calls fail with TL_ENODEV.
 */
#ifndef TRILIST_B200_H
#define TRILIST_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TL_OK 0
#define TL_EINVAL 1
#define TL_ERANGE 2
#define TL_ELOGIC 3
#define TL_ECUDA 4
#define TL_ENOMEM 5
#define TL_ECAPACITY 6
#define TL_ENODEV 7
#define TL_EPARSE 8   /* ParseError (graph.hpp:89-96): the message starts with "line N: " */
#define TL_ELENGTH 9  /* std::length_error                                            */
#define TL_EIO 10     /* std::runtime_error (cannot open / read a file)              */
#define TL_ECANCELED 11 /* a batch callback returned non-zero: the run stopped        */

#define TL_API __attribute__((visibility("default")))

typedef struct tl_graph tl_graph;       /* device-resident Graph (graph.hpp:31-73)            */
typedef struct tl_oriented tl_oriented; /* device-resident OrientedGraph (ordering.hpp:62-108) */

/* The reference's kernels (Algorithm, engine.hpp:18; names engine.cpp:7-15). */
#define TL_ALGO_AOT 0      /* "aot"     aot_pivot      engine.hpp:238-276 */
#define TL_ALGO_CF_MERGE 1 /* "cf"      cf_merge_pivot engine.hpp:164-184 */
#define TL_ALGO_CF_HASH 2  /* "cf-hash" cf_hash_pivot  engine.hpp:186-215 */
#define TL_ALGO_KCLIST3 3  /* "kclist"  kclist3_pivot  engine.hpp:217-236 */

/* RunStats (engine.hpp:28-54) plus device-side extras.  The six reference
 * counters are exactly what the reference kernel of the run's algorithm keeps. */
typedef struct tl_stats {
  uint64_t triangles;
  uint64_t probes;            /* aot, cf-hash: sum of min(deg+) (aot_cost); kclist: kclist_cost; cf: 0 */
  uint64_t merge_comparisons; /* cf only: iterations of the merge loops                                */
  uint64_t table_builds;      /* aot, kclist: m; cf-hash: probe-set insertions; cf: 0                 */
  uint64_t positive_triangles;
  uint64_t negative_triangles;
  uint64_t probes_executed;   /* probes left after rank-window early exit                          */
  uint64_t hash_sum;          /* order-independent triangle hash (hash mode): with Z(v) = fmix64(v +  */
  uint64_t hash_xor;          /* 0x9E3779B97F4A7C15) of the original ids, sum of Z(a)Z(b)Z(c) mod 2^64  */
                              /* and xor of Z(a)&Z(b)&Z(c) over the emitted triangles                  */
  uint64_t tasks;             /* work items scheduled                                              */
  double list_ms;             /* device time of the listing kernels (CUDA events)                  */
  double prep_ms;             /* device time of per-run task construction                          */
  uint64_t kernel_launches;   /* device kernels this call launched (task building + listing)       */
} tl_stats;

/* RunOptions (engine.hpp:56-60) + ParallelConfig-equivalent partitioning. */
typedef struct tl_run_options {
  uint32_t skip_negative_phase; /* RunOptions::aot_skip_negative_phase (fault injection)           */
  uint32_t check_hygiene;       /* RunOptions::check_bitmap_between_pivots: accepted, no-op         */
  uint32_t part;                /* this device's share of the cost-balanced edge partition          */
  uint32_t nparts;              /* number of shares (GPUs); 0 or 1 = whole graph                    */
  void* stream;                 /* cudaStream_t to run on; NULL = the handle's own stream           */
  uint32_t algorithm;           /* TL_ALGO_* for tl_run_*; 0 (aot) when zero-initialised            */
  uint32_t cf_hash_reuse_last_table; /* RunOptions::cf_hash_reuse_last_table (engine.hpp:58)      */
} tl_run_options;

/* ---------------------------------------------------------------- runtime */
TL_API const char* tl_last_error(void);
TL_API int tl_device_count(int* count);
TL_API const char* tl_version(void);

/* ------------------------------------------------- synthetic generators */
/* Seeded generators of the BASELINE configs; written on device,
 * bit-identical to oracle/trilist_oracle.c.  d_pairs holds 2*npairs uint32. */
TL_API int tl_gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint32_t* d_pairs, void* stream);
TL_API int tl_gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint32_t* d_pairs, void* stream);
/* Chung-Lu: prefix is the host-computed fixed-point weight prefix (n+1). */
TL_API int tl_chung_lu_prefix(uint64_t seed, uint32_t n, double avg, double gamma, uint64_t* prefix);
TL_API int tl_gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs,
                           uint32_t* d_pairs, void* stream);

/* -------------------------------------------------------- L0 graph core */
/* Graph::from_edges(min_vertices, span<pair>) -- graph.hpp:38-41, graph.cpp:189-206
 * (self-loops dropped, duplicates collapsed, n = max(min_vertices, max id + 1)).
 * `pairs` holds 2*npairs uint32 (u0,v0,u1,v1,...) in host memory, or in device
 * memory of `device` when pairs_on_device != 0. */
TL_API int tl_graph_from_pairs(const uint32_t* pairs, uint64_t npairs, uint32_t min_vertices,
                               int device, int pairs_on_device, void* stream, tl_graph** out);
TL_API int tl_graph_free(tl_graph* g);
/* num_vertices()/num_edges() (graph.hpp:43-44) + load diagnostics (graph.hpp:81-86). */
TL_API int tl_graph_info(const tl_graph* g, uint32_t* n, uint64_t* m, uint64_t* duplicates,
                         uint64_t* self_loops);
/* degree(u) for all u (graph.hpp:50-51). */
TL_API int tl_graph_degrees(tl_graph* g, uint32_t* degrees);
/* offsets() (n+1) / adjacency() (2m): symmetric ascending CSR (graph.hpp:56-57). */
TL_API int tl_graph_csr(tl_graph* g, uint64_t* offsets, uint32_t* adjacency);

/* Edge-list ingestion -- load_edge_list_text / load_edge_list / load_edge_list_file
 * (graph.hpp:99-108, graph.cpp:40-146, :240-275): whitespace-separated id pairs,
 * lines starting with a comment prefix skipped, parsed on the device, then
 * Graph::from_edges on the device.  On a ParseError the call returns TL_EPARSE
 * and *error_line holds the 1-based line (the first bad line, as the
 * reference reports it). */
#define TL_LOAD_ONE_INDEXED 1u /* LoadOptions::one_indexed */
#define TL_LOAD_COMPACT_IDS 2u /* LoadOptions::compact_ids */
typedef struct tl_load_diag {  /* LoadDiagnostics (graph.hpp:81-86) */
  uint64_t lines_read;
  uint64_t edges_parsed;
  uint64_t self_loops_dropped;
  uint64_t duplicates_dropped;
} tl_load_diag;
TL_API int tl_graph_from_text(const char* text, uint64_t len, uint32_t flags, const char* comment_prefixes,
                              int device, tl_graph** out, tl_load_diag* diag, uint64_t* error_line);
/* gzip-transparent; path "-" reads stdin. */
TL_API int tl_graph_from_file(const char* path, uint32_t flags, const char* comment_prefixes, int device,
                              tl_graph** out, tl_load_diag* diag, uint64_t* error_line);

/* ---------------------------------------------------------- L1 ordering */
/* degree_order(const Graph&) -- ordering.hpp:24, ordering.cpp:69-84: rank[u] by
 * ascending (degree, id).  rank has n entries. */
TL_API int tl_degree_order(tl_graph* g, uint32_t* rank);
/* orient(const Graph&, const VertexOrder&) -- ordering.hpp:112, ordering.cpp:185-227.
 * rank == NULL orients by the device-computed degree order.  Throws-equivalent
 * TL_EINVAL unless rank is a permutation of 0..n-1 (ordering.cpp:187-188). */
TL_API int tl_orient(tl_graph* g, const uint32_t* rank, tl_oriented** out);
/* Upload of a host OrientedGraph in the reference layout (out-lists of original
 * ids, rank-ascending; ordering.hpp:102-105) -- the drop-in path for callers
 * that already hold an oriented graph. */
TL_API int tl_oriented_from_csr(uint32_t n, uint64_t m, const uint64_t* out_offsets,
                                const uint32_t* out, const uint32_t* rank, int device, void* stream,
                                tl_oriented** out_graph);
TL_API int tl_oriented_free(tl_oriented* og);
/* num_vertices/num_edges/max_out_degree -- ordering.hpp:67-68, :99. */
TL_API int tl_oriented_info(const tl_oriented* og, uint32_t* n, uint64_t* m, uint32_t* max_out_degree);
/* Reference layout download: out/in CSR of original ids (rank-ascending lists)
 * and rank[] (ordering.hpp:69-80).  Any pointer may be NULL. */
TL_API int tl_oriented_csr(tl_oriented* og, uint64_t* out_offsets, uint32_t* out,
                           uint64_t* in_offsets, uint32_t* in, uint32_t* rank);
/* cost_model(const OrientedGraph&) -- engine.hpp:338-344, engine.cpp:37-49:
 * costs[0]=cf_cost, costs[1]=kclist_cost, costs[2]=aot_cost. */
TL_API int tl_cost_model(tl_oriented* og, uint64_t* costs);

/* ------------------------------------------------------ L2/L3 AOT listing */
/* run_parallel_count(Algorithm::aot, g, cfg, opt) -- parallel.hpp:81-82, parallel.cpp:5-8
 * (the per-pivot kernel aot_pivot, engine.hpp:238-276, as sm_100a kernels). */
TL_API int tl_aot_count(tl_oriented* og, const tl_run_options* opt, tl_stats* stats);
/* Count + order-independent hash of the canonical triangle set (no emission
 * buffer; hash_sum/hash_xor filled). */
TL_API int tl_aot_hash(tl_oriented* og, const tl_run_options* opt, tl_stats* stats);
/* run_parallel_collecting / run_collecting -- parallel.hpp:85-88, engine.cpp:31-35.
 * Writes the emissions of this part as uint32 triples: raw role order
 * (pivot, neighbor, witness) of engine.hpp:256/:269 when canonical == 0, or the
 * sorted canonical (a<b<c) set (canonicalize_emissions, engine.cpp:51-57) when
 * canonical != 0.  triples == NULL only counts (one counting pass, whose
 * emission count is cached on the handle to size the listing call); otherwise
 * one listing pass runs (plus a counting pass when no count is cached) and cap
 * must be at least the emission count (TL_ECAPACITY otherwise). */
TL_API int tl_aot_list(tl_oriented* og, const tl_run_options* opt, uint32_t* triples, uint64_t cap,
                       int canonical, tl_stats* stats);

/* --------------------------------------------- L2/L3 any kernel by name */
/* run_counting / run_collecting / run_parallel_count / run_parallel_collecting
 * for Algorithm = opt->algorithm (engine.hpp:324-329, parallel.hpp:81-88).
 * Same contracts as tl_aot_count / tl_aot_hash / tl_aot_list; emission role
 * order is the kernel's own (pivot, neighbor, witness): kclist and cf emit
 * (u, v, w) for the edge u->v, cf-hash (u, v, w) for the edge u->v whichever
 * side it hashed (engine.hpp:212).  tl_aot_* ignore opt->algorithm. */
TL_API int tl_run_count(tl_oriented* og, const tl_run_options* opt, tl_stats* stats);
TL_API int tl_run_hash(tl_oriented* og, const tl_run_options* opt, tl_stats* stats);
TL_API int tl_run_list(tl_oriented* og, const tl_run_options* opt, uint32_t* triples, uint64_t cap,
                       int canonical, tl_stats* stats);

/* run_parallel(algo, g, cfg, SinkFactory) / run_algorithm(algo, g, sink) with an
 * arbitrary sink (parallel.hpp:25-78, engine.hpp:125-134, :294-304) in
 * bounded host memory.  The emissions of the run (raw role order, as
 * tl_run_list with canonical == 0) are produced in batches of at most
 * batch_triples triples (0 = 2^24): the claim-cost cut splits the run into
 * consecutive claim ranges, each listed on the device into a batch buffer
 * (a range that overflows is split in two and listed again), copied to one of
 * host_buffers (0 = 3, at least 2) pinned host buffers, and handed to
 * fn(user, triples, count) on the CALLING thread, in order, while the device
 * already lists the following ranges.  `triples` is valid only during the
 * call.  fn returning non-zero stops the run (TL_ECANCELED).  Host memory:
 * host_buffers x 12 x batch_triples bytes; device memory: 2 batch buffers.
 * opt->part/nparts selects every nparts-th top-level range (multi-GPU: each
 * rank streams its own share).  stats = the counters summed over the ranges
 * (identical to tl_run_count's). */
typedef int (*tl_batch_fn)(void* user, const uint32_t* triples, uint64_t count);
TL_API int tl_run_list_batches(tl_oriented* og, const tl_run_options* opt, uint64_t batch_triples,
                               uint32_t host_buffers, tl_batch_fn fn, void* user, tl_stats* stats);

/* The same listing into DEVICE memory of the handle's device (d_triples holds
 * cap triples): one listing pass, no counting pass and no host copy -- the
 * emissions stay resident for a device consumer.  Returns TL_ECAPACITY (stats
 * filled, stats->triangles = the emission count) when cap is too small. */
TL_API int tl_run_list_device(tl_oriented* og, const tl_run_options* opt, uint32_t* d_triples, uint64_t cap,
                              int canonical, tl_stats* stats);

/* verify_equivalence's comparison (engine.cpp:82-130) for one orientation,
 * on the device: every algorithm in `algorithms` (TL_ALGO_*) lists its
 * emissions, which are canonicalised, sorted and de-duplicated on the device
 * and compared with the baseline by device set differences -- the oracle's
 * triples `reference` (host, any order, sorted and de-duplicated here) when
 * have_reference != 0, else the first algorithm's set.  opt carries the
 * RunOptions (skip_negative_phase, cf_hash_reuse_last_table, stream);
 * opt->algorithm is ignored.  results[nalgos]; reference_count = size of the
 * baseline set.  Only counters and the first TL_VERIFY_SAMPLES differences of
 * each side leave the device. */
#define TL_VERIFY_SAMPLES 32 /* VerifyReport::kMaxSamples (engine.hpp:362) */
typedef struct tl_verify_result {
  uint32_t algorithm; /* TL_ALGO_* */
  uint32_t pass;
  uint64_t unique_triangles;
  uint64_t duplicate_emissions;
  uint64_t missing_count; /* in the baseline, not emitted */
  uint64_t extra_count;   /* emitted, not in the baseline */
  uint32_t n_missing_samples;
  uint32_t n_extra_samples;
  uint32_t missing_samples[3 * TL_VERIFY_SAMPLES]; /* sorted canonical triples */
  uint32_t extra_samples[3 * TL_VERIFY_SAMPLES];
  tl_stats stats;
} tl_verify_result;
TL_API int tl_verify(tl_oriented* og, const uint32_t* algorithms, uint32_t nalgos, const tl_run_options* opt,
                     const uint32_t* reference, uint64_t nreference, int have_reference,
                     tl_verify_result* results, uint64_t* reference_count);

/* ------------------------------------------- several GPUs, one process */
/* run_parallel_* over a device list (parallel.hpp:25-88; ParallelConfig,
 * parallel.hpp:14-17, is the reference's only knob).  tl_multi_create
 * replicates the oriented graph on devs[0..ndev) (device-to-device copies of
 * the resident CSR + claims; a device equal to og's own uses og itself,
 * borrowed: og must outlive the tl_multi) and creates one NCCL communicator
 * per device (ncclCommInitAll; NCCL is loaded at run time).  A run splits the
 * directed edges into ndev cost-balanced parts (part d on devs[d], one host
 * thread per device, no exchange during compute); the counters and the hash
 * sum are combined by ncclAllReduce(sum), the hash xors and the per-device
 * emission counts by ncclAllGather, folded as tl_fold_parts does.  Results are
 * identical to the single-device calls for any ndev.  opt->part/nparts must
 * be 0/1 and opt->stream NULL.  tl_multi_list writes part d's raw emissions at
 * its gathered offset (triples == NULL only counts). */
typedef struct tl_multi tl_multi;
TL_API int tl_multi_create(tl_oriented* og, const int* devs, int ndev, tl_multi** out);
TL_API int tl_multi_free(tl_multi* mg);
TL_API int tl_multi_count(tl_multi* mg, const tl_run_options* opt, tl_stats* stats);
TL_API int tl_multi_hash(tl_multi* mg, const tl_run_options* opt, tl_stats* stats);
TL_API int tl_multi_list(tl_multi* mg, const tl_run_options* opt, uint32_t* triples, uint64_t cap, tl_stats* stats);
/* Host fold of per-part stats (any multi-GPU caller, e.g. torch.distributed
 * ranks that gathered their tl_stats): counters and hash_sum summed mod 2^64,
 * hash_xor xor-ed, list_ms / prep_ms = the slowest part's, offsets[d] (may be
 * NULL) = exclusive scan of the parts' triangle counts (listing offsets). */
TL_API int tl_fold_parts(const tl_stats* parts, uint32_t nparts, tl_stats* total, uint64_t* offsets);

/* degeneracy_order / random_order -- ordering.cpp:86-120.  The degeneracy
 * order removes, one vertex at a time, the vertex of least (current degree,
 * id) -- an inherently sequential chain -- and random_order is a Fisher-Yates
 * chain of n dependent swaps; both run on the host (O(m log n) / O(n)) over
 * the graph's CSR and return rank[n] for tl_orient.  Not on the AOT path,
 * which uses the device degree order. */
TL_API int tl_degeneracy_order(tl_graph* g, uint32_t* rank);
TL_API int tl_random_order(uint32_t n, uint64_t seed, uint32_t* rank);

/* brute_force_triangles(const Graph&, OracleOptions) -- oracle.hpp:18, oracle.cpp:8-25,
 * as a device kernel: sorted canonical set.  TL_EINVAL if n > max_vertices. */
TL_API int tl_brute_force(tl_graph* g, uint32_t max_vertices, uint32_t* triples, uint64_t cap,
                          uint64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* TRILIST_B200_H */
