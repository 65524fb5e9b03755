// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj
// sources, compiled by oracle/Makefile into oracle/_ref/libtrilist_ref.so).
// It calls only the reference's public API:
//   Graph::from_edges        graph.hpp:38-41
//   make_order / degree_order ordering.hpp:24, :38
//   orient                   ordering.hpp:112
//   run_parallel(_count)     parallel.hpp:25-88
//   cost_model               engine.hpp:344
//   brute_force_triangles    oracle.hpp:18
// Used by tests/ (as the parity anchor) and by bench.py's cpu_baseline and
// --impl reference legs (as the CPU baseline).  Never linked by the product.
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <sstream>
#include <string_view>
#include <thread>
#include <vector>

#include "trilist/engine.hpp"
#include "trilist/graph.hpp"
#include "trilist/oracle.hpp"
#include "trilist/ordering.hpp"
#include "trilist/parallel.hpp"

using namespace trilist;

namespace {
thread_local std::string g_err;

struct Handle {
  Graph g;
  OrientedGraph og;
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void fill_stats(const RunStats& s, std::uint64_t* out) {
  if (!out) return;
  out[0] = s.triangles;
  out[1] = s.probes;
  out[2] = s.merge_comparisons;
  out[3] = s.table_builds;
  out[4] = s.positive_triangles;
  out[5] = s.negative_triangles;
}

std::uint64_t fmix64(std::uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Order-independent hash sink, one per worker.
struct HashSink {
  std::uint64_t* acc;  // [count, sum, xor]
  void operator()(VertexId a, VertexId b, VertexId c) const {
    // Z(v) = fmix64(v + golden); sum of Z(a) Z(b) Z(c), xor of Z(a) & Z(b) & Z(c)
    const std::uint64_t za = fmix64(a + 0x9E3779B97F4A7C15ull), zb = fmix64(b + 0x9E3779B97F4A7C15ull),
                        zc = fmix64(c + 0x9E3779B97F4A7C15ull);
    acc[0] += 1;
    acc[1] += za * zb * zc;
    acc[2] ^= za & zb & zc;
  }
};

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

unsigned ref_hardware_threads() { return std::max(1u, std::thread::hardware_concurrency()); }

// order: "degree" | "id" | "degeneracy" | "random:SEED"; local: "rank-asc" | ...
// times[3] = from_edges, make_order, orient (+local order) seconds.
int ref_prepare(const std::uint32_t* pairs, std::uint64_t npairs, std::uint32_t min_vertices,
                const char* order, const char* local, void** out, double* times) {
  return guarded([&] {
    auto* h = new Handle;
    double t0 = now_s();
    auto ps = reinterpret_cast<const std::pair<VertexId, VertexId>*>(pairs);
    h->g = Graph::from_edges(min_vertices, std::span<const std::pair<VertexId, VertexId>>(ps, npairs));
    double t1 = now_s();
    VertexOrder vo = make_order(h->g, parse_order_spec(order));
    double t2 = now_s();
    h->og = orient(h->g, vo);
    LocalOrder lo = parse_local_order(local);
    if (lo.policy != LocalOrderPolicy::rank_asc) h->og = apply_local_order(h->og, lo);
    double t3 = now_s();
    if (times) {
      times[0] = t1 - t0;
      times[1] = t2 - t1;
      times[2] = t3 - t2;
    }
    *out = h;
  });
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

std::uint32_t ref_n(void* h) { return static_cast<Handle*>(h)->og.num_vertices(); }
std::uint64_t ref_m(void* h) { return static_cast<Handle*>(h)->og.num_edges(); }
std::uint32_t ref_max_out_degree(void* h) { return static_cast<Handle*>(h)->og.max_out_degree(); }

int ref_count(void* hp, unsigned threads, unsigned chunk, int skip_negative, std::uint64_t* stats,
              double* wall) {
  return guarded([&] {
    auto* h = static_cast<Handle*>(hp);
    RunOptions opt;
    opt.aot_skip_negative_phase = skip_negative != 0;
    RunStats s = run_parallel_count(Algorithm::aot, h->og, ParallelConfig{threads, chunk}, opt);
    fill_stats(s, stats);
    if (wall) *wall = s.wall_time_s;
  });
}

// hash[3] = count, sum, xor over canonical original-id triples.
int ref_hash(void* hp, unsigned threads, unsigned chunk, std::uint64_t* hash, std::uint64_t* stats,
             double* wall) {
  return guarded([&] {
    auto* h = static_cast<Handle*>(hp);
    std::vector<std::array<std::uint64_t, 8>> accs(threads);  // padded per worker
    for (auto& a : accs) a.fill(0);
    RunStats s = run_parallel(Algorithm::aot, h->og, ParallelConfig{threads, chunk},
                              [&](unsigned w) { return HashSink{accs[w].data()}; });
    std::uint64_t c = 0, sum = 0, x = 0;
    for (auto& a : accs) {
      c += a[0];
      sum += a[1];
      x ^= a[2];
    }
    hash[0] = c;
    hash[1] = sum;
    hash[2] = x;
    fill_stats(s, stats);
    if (wall) *wall = s.wall_time_s;
  });
}

// Raw role-ordered emissions (pivot, neighbor, witness), worker buffers
// concatenated.  Writes min(count, cap) triples; *count gets the total.
int ref_collect(void* hp, unsigned threads, unsigned chunk, int skip_negative, std::uint32_t* out,
                std::uint64_t cap, std::uint64_t* count, std::uint64_t* stats, double* wall) {
  return guarded([&] {
    auto* h = static_cast<Handle*>(hp);
    RunOptions opt;
    opt.aot_skip_negative_phase = skip_negative != 0;
    std::vector<std::vector<std::array<VertexId, 3>>> bufs;
    RunStats s = run_parallel_collecting(Algorithm::aot, h->og, ParallelConfig{threads, chunk}, bufs, opt);
    std::uint64_t k = 0;
    for (auto& b : bufs)
      for (auto& t : b) {
        if (out && k < cap) std::memcpy(out + 3 * k, t.data(), 12);
        ++k;
      }
    *count = k;
    fill_stats(s, stats);
    if (wall) *wall = s.wall_time_s;
  });
}

// Any kernel by name ("cf" | "cf-hash" | "kclist" | "aot", engine.cpp:17-24).
// flags: bit0 = aot_skip_negative_phase, bit1 = cf_hash_reuse_last_table.
// hash (nullable) = count, sum, xor through a per-worker hash sink.
int ref_run(void* hp, const char* algo, unsigned threads, unsigned chunk, int flags, std::uint64_t* hash,
            std::uint64_t* stats, double* wall) {
  return guarded([&] {
    auto* h = static_cast<Handle*>(hp);
    RunOptions opt;
    opt.aot_skip_negative_phase = (flags & 1) != 0;
    opt.cf_hash_reuse_last_table = (flags & 2) != 0;
    Algorithm a = parse_algorithm(algo);
    RunStats s;
    if (hash) {
      std::vector<std::array<std::uint64_t, 8>> accs(threads);
      for (auto& x : accs) x.fill(0);
      s = run_parallel(a, h->og, ParallelConfig{threads, chunk}, [&](unsigned w) { return HashSink{accs[w].data()}; },
                       opt);
      hash[0] = hash[1] = hash[2] = 0;
      for (auto& x : accs) {
        hash[0] += x[0];
        hash[1] += x[1];
        hash[2] ^= x[2];
      }
    } else {
      s = run_parallel_count(a, h->og, ParallelConfig{threads, chunk}, opt);
    }
    fill_stats(s, stats);
    if (wall) *wall = s.wall_time_s;
  });
}

// Raw emissions of any kernel (run_parallel_collecting), as ref_collect.
int ref_collect_algo(void* hp, const char* algo, unsigned threads, unsigned chunk, int flags, std::uint32_t* out,
                     std::uint64_t cap, std::uint64_t* count, std::uint64_t* stats, double* wall) {
  return guarded([&] {
    auto* h = static_cast<Handle*>(hp);
    RunOptions opt;
    opt.aot_skip_negative_phase = (flags & 1) != 0;
    opt.cf_hash_reuse_last_table = (flags & 2) != 0;
    std::vector<std::vector<std::array<VertexId, 3>>> bufs;
    RunStats s = run_parallel_collecting(parse_algorithm(algo), h->og, ParallelConfig{threads, chunk}, bufs, opt);
    std::uint64_t k = 0;
    for (auto& b : bufs)
      for (auto& t : b) {
        if (out && k < cap) std::memcpy(out + 3 * k, t.data(), 12);
        ++k;
      }
    *count = k;
    fill_stats(s, stats);
    if (wall) *wall = s.wall_time_s;
  });
}

int ref_cost_model(void* hp, std::uint64_t* out) {
  return guarded([&] {
    CostModel cm = cost_model(static_cast<Handle*>(hp)->og);
    out[0] = cm.cf_cost;
    out[1] = cm.kclist_cost;
    out[2] = cm.aot_cost;
  });
}

// Sorted canonical set from brute_force_triangles (oracle.cpp:8-25).
int ref_brute_force(void* hp, std::uint32_t max_vertices, std::uint32_t* out, std::uint64_t cap,
                    std::uint64_t* count) {
  return guarded([&] {
    auto tris = brute_force_triangles(static_cast<Handle*>(hp)->g, OracleOptions{max_vertices});
    std::uint64_t k = 0;
    for (const Triangle& t : tris) {
      if (out && k < cap) {
        out[3 * k] = t.a;
        out[3 * k + 1] = t.b;
        out[3 * k + 2] = t.c;
      }
      ++k;
    }
    *count = k;
  });
}

// Reference OrientedGraph layout (original ids, rank-sorted lists).
int ref_download_oriented(void* hp, std::uint64_t* out_off, std::uint32_t* out, std::uint64_t* in_off,
                          std::uint32_t* in, std::uint32_t* rank) {
  return guarded([&] {
    const OrientedGraph& og = static_cast<Handle*>(hp)->og;
    std::uint64_t pos_out = 0, pos_in = 0;
    for (VertexId u = 0; u < og.num_vertices(); ++u) {
      if (out_off) out_off[u] = pos_out;
      if (in_off) in_off[u] = pos_in;
      for (VertexId v : og.out_neighbors(u)) {
        if (out) out[pos_out] = v;
        ++pos_out;
      }
      for (VertexId v : og.in_neighbors(u)) {
        if (in) in[pos_in] = v;
        ++pos_in;
      }
      if (rank) rank[u] = og.rank(u);
    }
    if (out_off) out_off[og.num_vertices()] = pos_out;
    if (in_off) in_off[og.num_vertices()] = pos_in;
  });
}

// load_edge_list_text (graph.cpp:240-248) then degree order + orient.
// Returns 0, 1 (other error) or 2 (ParseError; *err_line set).
// diag[4] = lines_read, edges_parsed, self_loops_dropped, duplicates_dropped.
int ref_load_text(const char* text, std::uint64_t len, int one_indexed, int compact, const char* comments,
                  void** out, std::uint64_t* diag, std::uint64_t* err_line) {
  try {
    LoadOptions opt;
    opt.one_indexed = one_indexed != 0;
    opt.compact_ids = compact != 0;
    if (comments) opt.comment_prefixes = comments;
    LoadResult r = load_edge_list_text(std::string_view(text, len), opt);
    auto* h = new Handle;
    h->g = std::move(r.graph);
    h->og = orient(h->g, degree_order(h->g));
    diag[0] = r.diagnostics.lines_read;
    diag[1] = r.diagnostics.edges_parsed;
    diag[2] = r.diagnostics.self_loops_dropped;
    diag[3] = r.diagnostics.duplicates_dropped;
    *out = h;
    return 0;
  } catch (const ParseError& e) {
    g_err = e.what();
    *err_line = e.line();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// write_edge_list (graph.cpp:277-281) into a caller buffer; returns the size.
std::uint64_t ref_write_edge_list(void* hp, char* buf, std::uint64_t cap) {
  std::ostringstream os;
  write_edge_list(static_cast<Handle*>(hp)->g, os);
  std::string s = os.str();
  if (buf) std::memcpy(buf, s.data(), std::min<std::uint64_t>(cap, s.size()));
  return s.size();
}

int ref_download_graph(void* hp, std::uint64_t* off, std::uint32_t* adj) {
  return guarded([&] {
    const Graph& g = static_cast<Handle*>(hp)->g;
    std::memcpy(off, g.offsets().data(), sizeof(std::uint64_t) * g.offsets().size());
    std::memcpy(adj, g.adjacency().data(), sizeof(std::uint32_t) * g.adjacency().size());
  });
}

}  // extern "C"
