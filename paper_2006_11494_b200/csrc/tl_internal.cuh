// tl_internal.cuh -- device-resident graph handles and pipeline entry points.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <array>
#include <map>
#include <memory>
#include <tuple>

#include "tl_common.cuh"

namespace tlb {
struct AotPlan;  // a run's work records and tasks (tl_aot.cu), cached per handle
}

// Opaque C-ABI handles (trilist_b200.h).
struct tl_graph {
  int device = 0;
  cudaStream_t stream = nullptr;  // own stream (non-blocking)
  uint32_t n = 0;
  uint32_t nb = 0;  // id bits: every id < 2^nb
  uint64_t m = 0;
  uint64_t duplicates = 0;
  uint64_t self_loops = 0;
  uint32_t max_deg = 0;
  tlb::DBuf<uint64_t> keys;  // m sorted unique (lo << nb | hi), lo < hi
  tlb::DBuf<uint32_t> deg;   // n undirected degrees
  ~tl_graph();
};

// OrientedGraph in rank space: vertex r is the vertex of rank r; every
// out-list is ascending (= rank-ascending, the orient() layout, which AOT's
// early exit relies on).  Claims group the directed edges by the pivot that
// processes them (aot_pivot's two phases, engine.hpp:247-272):
//   edge t->h with h < t in (deg+, id) order: pivot t, traverse N+(h) from 0
//                                            (positive phase)
//   otherwise:                               pivot h, traverse N+(t) after h
//                                            (negative phase)
struct tl_oriented {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t aux = nullptr;  // side stream for work overlapped with a run (created on first use)
  uint32_t n = 0;
  uint32_t nb = 0;
  uint64_t m = 0;
  uint32_t max_out_degree = 0;
  uint64_t cost[3] = {0, 0, 0};  // cf, kclist, aot
  tlb::DBuf<uint64_t> off;        // n+1
  tlb::DBuf<uint32_t> col;        // m rank ids
  tlb::DBuf<uint32_t> orig;       // n: rank -> original id
  tlb::DBuf<uint32_t> rank;       // n: original id -> rank
  tlb::DBuf<uint64_t> claim_off;  // n+1, by pivot
  tlb::DBuf<uint64_t> win;        // m claim windows {begin:40 | len:23 | neg:1} into col
  tlb::DBuf<uint32_t> claim_s;    // m traversed vertex ids s | neg << 31
  tlb::DBuf<uint64_t> vword;      // n: rank -> vertex_word(original id), the hash sink's table (built on first use)
  // forward claims (kclist3 / cf merge: pivot t traverses N+(h) for every
  // edge t->h; grouped by t = the out-CSR itself), built on first use
  tlb::DBuf<uint64_t> fwd_win;    // m windows {off[h] | deg+(h) << 40}
  // claim-cost prefix (m+1) of the last claim set used (aot_run), key =
  // forward << 1 | skip_negative
  tlb::DBuf<uint64_t> cp;
  uint32_t cp_key = ~0u;
  uint64_t cp_total = 0;  // CP[m]
  // emission count per (algorithm, skip_negative, part, nparts): sizes listing buffers
  std::map<std::tuple<uint32_t, uint32_t, uint32_t, uint32_t>, uint64_t> tri_cache;
  // Work construction cached per handle (the graph is immutable): the cost
  // cut of a part per (claim set, part, nparts, range) -- {cb, ce, pb, pe, vb,
  // ve, table_builds, logical, has_logical} -- and the work records + tasks per
  // (claim set, claim range, task size).  A step of a partitioned run then
  // rebuilds nothing.
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, std::array<uint64_t, 9>> cuts;
  std::map<std::tuple<uint32_t, uint64_t, uint64_t, uint64_t>, std::shared_ptr<tlb::AotPlan>> plans;
  ~tl_oriented();
};

namespace tlb {

constexpr uint32_t kNegBit = 0x80000000u;
constexpr uint32_t kWinLenShift = 40;
constexpr uint64_t kWinBeginMask = (1ull << kWinLenShift) - 1;
constexpr uint64_t kWinLenMask = (1ull << 23) - 1;

struct DeviceGuard {
  int prev = 0;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) TL_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = 0;
    cudaGetDevice(&cur);
    if (cur != prev) cudaSetDevice(prev);
  }
};

// TL_DEBUG_PREP=1: host-side phase timeline (synchronises the stream at
// every mark, so only for diagnosis).
struct PhaseClock {
  const char* tag;
  cudaStream_t s;
  bool on = getenv("TL_DEBUG_PREP") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  PhaseClock(const char* tag_, cudaStream_t s_) : tag(tag_), s(s_) {}
  void mark(const char* what) const {
    if (!on) return;
    cudaStreamSynchronize(s);
    fprintf(stderr, "[tl %s] %-14s %9.3f ms\n", tag, what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

// ---- tl_build.cu ----
void gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint32_t* d_pairs, cudaStream_t s);
void gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint32_t* d_pairs, cudaStream_t s);
void gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs,
                  uint32_t* d_pairs, cudaStream_t s);
void chung_lu_prefix_host(uint64_t seed, uint32_t n, double avg, double gamma, uint64_t* prefix);

void graph_from_pairs(tl_graph& g, const uint32_t* d_pairs, uint64_t npairs, uint32_t min_vertices);

// ---- tl_parse.cu ----
struct ParseFailure : TlError {
  uint64_t line;
  ParseFailure(uint64_t line_no, const std::string& msg);
};
void graph_from_text(tl_graph& g, const char* text, uint64_t len, uint32_t flags, const char* comment_prefixes,
                     tl_load_diag* diag);
std::string read_text_file(const std::string& path);
void graph_csr(tl_graph& g, DBuf<uint64_t>& off, DBuf<uint32_t>& adj);
void degree_order(tl_graph& g, DBuf<uint32_t>& rank);  // device rank[n]
void orient(tl_graph& g, const uint32_t* d_rank, tl_oriented& og);
void oriented_from_csr(tl_oriented& og, uint32_t n, uint64_t m, const uint64_t* d_out_off,
                       const uint32_t* d_out, const uint32_t* d_rank);
void oriented_from_host_csr(tl_oriented& og, uint32_t n, uint64_t m, const uint64_t* h_off, const uint32_t* h_out,
                            const uint32_t* h_rank);
void oriented_download(tl_oriented& og, uint64_t* out_off, uint32_t* out, uint64_t* in_off,
                       uint32_t* in, uint32_t* rank);
bool is_permutation(const uint32_t* d_rank, uint32_t n, cudaStream_t s);

// Lexicographic sort of uint32 triples (n_items x 3) in place.
void sort_triples(uint32_t* d_triples, uint64_t count, uint32_t nb, cudaStream_t s);
void canonicalize_triples(uint32_t* d_triples, uint64_t count, cudaStream_t s);
uint64_t brute_force(tl_graph& g, DBuf<uint32_t>& out);

// ---- tl_orders.cu (host: sequential by definition) ----
void degeneracy_order_host(uint32_t n, const uint64_t* off, const uint32_t* adj, uint32_t* rank);
void random_order_host(uint32_t n, uint64_t seed, uint32_t* rank);

// ---- tl_aot.cu ----
enum class AotMode { count = 0, hash = 1, list = 2 };
// The reference's four kernels (engine.hpp:18), numbered as TL_ALGO_*.
enum class Algo : uint32_t { aot = 0, cf_merge = 1, cf_hash = 2, kclist3 = 3 };
struct AotResult {
  uint64_t positive = 0, negative = 0, executed = 0, logical = 0, windowed = 0;
  uint64_t hash_sum = 0, hash_xor = 0, emitted = 0, tasks = 0, table_builds = 0, launches = 0;
  // RunStats as the reference reports them for the algorithm (engine.hpp:28-36)
  uint64_t triangles = 0, probes = 0, merge_comparisons = 0, report_positive = 0, report_negative = 0;
  float list_ms = 0.f, prep_ms = 0.f;
};
struct RunSpec {
  Algo algo = Algo::aot;
  AotMode mode = AotMode::count;
  bool skip_negative = false;  // RunOptions::aot_skip_negative_phase (aot only)
  bool reuse = false;          // RunOptions::cf_hash_reuse_last_table (cf-hash only)
  uint32_t part = 0, nparts = 1;
  bool range = false;          // run the cost cut's own claim range (no interleaving): batched listing
};
// out/out_cap only for AotMode::list (device buffer of 3*out_cap uint32).
AotResult aot_run(tl_oriented& og, const RunSpec& spec, cudaStream_t s, uint32_t* d_out, uint64_t out_cap);
void fill_stats_from(const AotResult& r, tl_stats* st);  // tl_capi.cu
void ensure_device_setup(int device);                     // tl_capi.cu
void set_last_error(const std::string& msg);              // tl_capi.cu: the thread's tl_last_error()

// ---- tl_stream.cu ----
// Batched listing (tl_run_list_batches): emissions of `spec` in batches of at
// most batch_triples, handed in order to fn on the calling thread while an
// internal thread keeps the device listing ahead into a ring of pinned host
// buffers.  Returns the summed run counters.
AotResult list_batches(tl_oriented& og, const RunSpec& spec, cudaStream_t s, uint64_t batch_triples,
                       uint32_t host_buffers, tl_batch_fn fn, void* user);

// ---- tl_verify.cu ----
void verify_algorithms(tl_oriented& og, const uint32_t* algos, uint32_t nalgos, const RunSpec& base,
                       const uint32_t* h_reference, uint64_t nreference, bool have_reference, cudaStream_t s,
                       tl_verify_result* results, uint64_t* reference_count);

}  // namespace tlb
