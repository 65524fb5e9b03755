// trilist.hpp -- C++ facade of the reference `trilist` API over the B200 C-ABI.
//
// Same names, argument meaning and exception types as the reference headers
// (graph.hpp, ordering.hpp, engine.hpp, parallel.hpp, oracle.hpp under
// /root/reference/proj/include/trilist); every computation runs through
// include/trilist_b200.h on a CUDA device.  Differences, all documented in
// INTEGRATION.md:
//   * all four kernels (aot, cf, cf-hash, kclist) run on the device with the
//     reference's exact counters; the device keeps rank-ascending lists, and
//     other local orders are host-side views (counters are layout-invariant,
//     test_engine.cpp:172-185; cf still rejects non-rank-ascending layouts).
//   * the degeneracy and random orders are sequential chains by definition
//     and are computed on the host (tl_degeneracy_order / tl_random_order);
//     the degree order and everything after it run on the device.
//   * ParallelConfig is validated exactly like the reference (workers >= 1,
//     chunk >= 1) but no longer partitions work: the GPU schedules its own
//     cost-balanced tasks.
#pragma once

#include <array>
#include <compare>
#include <condition_variable>
#include <cstdint>
#include <exception>
#include <initializer_list>
#include <iosfwd>
#include <string_view>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <utility>
#include <vector>

#include "trilist_b200.h"

namespace trilist {

using VertexId = std::uint32_t;
using EdgeCount = std::uint64_t;

// ------------------------------------------------------------- graph.hpp
struct Triangle {
  VertexId a = 0;
  VertexId b = 0;
  VertexId c = 0;
  friend auto operator<=>(const Triangle&, const Triangle&) = default;
};

Triangle canonical_triangle(VertexId x, VertexId y, VertexId z);

/// Rethrows a C-ABI failure as the reference's exception type.
[[noreturn]] void throw_status(int code, const std::string& context);
inline void check(int code, const char* context) {
  if (code != TL_OK) throw_status(code, context);
}

/// Undirected simple graph (graph.hpp:31-73).  The CSR lives on the device;
/// host accessors download it lazily.
class Graph {
 public:
  Graph() = default;

  static Graph from_edges(VertexId min_vertices, std::span<const std::pair<VertexId, VertexId>> edges);
  static Graph from_edges(VertexId min_vertices, std::initializer_list<std::pair<VertexId, VertexId>> edges);
  /// Extension: pairs already resident in device memory (2*npairs uint32).
  static Graph from_device_pairs(VertexId min_vertices, const std::uint32_t* d_pairs, std::uint64_t npairs,
                                 int device = 0, void* stream = nullptr);

  VertexId num_vertices() const { return n_; }
  EdgeCount num_edges() const { return m_; }

  std::span<const VertexId> neighbors(VertexId u) const;
  VertexId degree(VertexId u) const;  // std::out_of_range if u >= n
  bool has_edge(VertexId u, VertexId v) const;
  const std::vector<EdgeCount>& offsets() const;
  const std::vector<VertexId>& adjacency() const;
  bool validate(std::string* why = nullptr) const;

  std::uint64_t duplicates_dropped() const { return dups_; }
  std::uint64_t self_loops_dropped() const { return loops_; }
  tl_graph* handle() const { return h_.get(); }
  int device() const { return device_; }
  static Graph adopt(tl_graph* h, int device) { return wrap(h, device); }  // takes ownership

 private:
  struct HostCsr {
    std::vector<EdgeCount> offsets;
    std::vector<VertexId> adjacency;
  };
  static Graph wrap(tl_graph* h, int device);
  const HostCsr& csr() const;

  std::shared_ptr<tl_graph> h_;
  int device_ = 0;
  VertexId n_ = 0;
  EdgeCount m_ = 0;
  std::uint64_t dups_ = 0, loops_ = 0;
  mutable std::shared_ptr<HostCsr> csr_;
};

// --------------------------------------------------- graph.hpp: loading
struct LoadOptions {
  std::string comment_prefixes = "#%";  // line-leading chars that mark comments
  bool one_indexed = false;             // input numbers vertices from 1
  bool compact_ids = false;             // remap ids to 0..n-1 by first appearance
};

struct LoadDiagnostics {
  std::uint64_t lines_read = 0;
  std::uint64_t edges_parsed = 0;  // pairs seen, before normalization
  std::uint64_t self_loops_dropped = 0;
  std::uint64_t duplicates_dropped = 0;
};

struct LoadResult {
  Graph graph;
  LoadDiagnostics diagnostics;
};

/// Input rejection with the 1-based line it occurred on (graph.hpp:89-96).
class ParseError : public std::runtime_error {
 public:
  ParseError(const std::string& what, std::uint64_t line) : std::runtime_error(what), line_(line) {}
  std::uint64_t line() const { return line_; }

 private:
  std::uint64_t line_;
};

/// Parsed on the device (tl_graph_from_text / tl_graph_from_file).
LoadResult load_edge_list(std::istream& in, const LoadOptions& options = {});
LoadResult load_edge_list_text(std::string_view text, const LoadOptions& options = {});
/// gzip-transparent; "-" reads stdin.
LoadResult load_edge_list_file(const std::string& path, const LoadOptions& options = {});
/// Writes each undirected edge once, smaller endpoint first, ascending.
void write_edge_list(const Graph& g, std::ostream& out);

// ---------------------------------------------------------- ordering.hpp
struct VertexOrder {
  std::vector<VertexId> rank;
  bool is_permutation() const;
  std::vector<VertexId> vertices_by_rank() const;
};

VertexOrder id_order(const Graph& g);
VertexOrder degree_order(const Graph& g);  // device counting order, ordering.cpp:69-84
VertexOrder degeneracy_order(const Graph& g);  // sequential chain: host (tl_degeneracy_order), ordering.cpp:86-114
VertexOrder random_order(const Graph& g, std::uint64_t seed);  // Fisher-Yates chain: host (tl_random_order)

enum class OrderKind { id, degree, degeneracy, random };
struct OrderSpec {
  OrderKind kind = OrderKind::degree;
  std::uint64_t seed = 0;
};
VertexOrder make_order(const Graph& g, const OrderSpec& spec);
OrderSpec parse_order_spec(const std::string& text);
std::string to_string(const OrderSpec& spec);

enum class LocalOrderPolicy { rank_asc, degree_desc, random };
struct LocalOrder {
  LocalOrderPolicy policy = LocalOrderPolicy::rank_asc;
  std::uint64_t seed = 0;
};
LocalOrder parse_local_order(const std::string& text);
std::string to_string(const LocalOrder& local);

/// Degree-oriented DAG (ordering.hpp:62-108).  The device copy is always
/// rank-ascending (AOT's early exit needs it); the host accessor lists follow
/// local_order() exactly like the reference's.
class OrientedGraph {
 public:
  OrientedGraph() = default;

  /// Extension: upload a host OrientedGraph in the reference layout.
  static OrientedGraph from_csr(VertexId n, std::span<const EdgeCount> out_offsets, std::span<const VertexId> out,
                                std::span<const VertexId> rank, int device = 0);

  VertexId num_vertices() const { return n_; }
  EdgeCount num_edges() const { return m_; }
  std::span<const VertexId> out_neighbors(VertexId u) const;
  std::span<const VertexId> in_neighbors(VertexId u) const;
  VertexId out_degree(VertexId u) const;
  VertexId in_degree(VertexId u) const;
  VertexId undirected_degree(VertexId u) const { return out_degree(u) + in_degree(u); }
  VertexId rank(VertexId u) const { return order().rank[u]; }
  const VertexOrder& order() const;
  const LocalOrder& local_order() const { return local_; }
  bool out_degree_before(VertexId a, VertexId b) const {
    VertexId da = out_degree(a), db = out_degree(b);
    return da != db ? da < db : a < b;
  }
  bool out_lists_rank_sorted() const;
  VertexId max_out_degree() const { return max_out_; }

  tl_oriented* handle() const { return h_.get(); }
  int device() const { return device_; }
  /// Extension: this graph replicated on `devices` (created on first use and
  /// kept; tl_multi_create), for runs split over several GPUs.
  tl_multi* multi(const std::vector<int>& devices) const;

 private:
  friend OrientedGraph orient(const Graph&, const VertexOrder&);
  friend OrientedGraph apply_local_order(OrientedGraph g, const LocalOrder& local);
  struct HostLayout {
    std::vector<EdgeCount> out_offsets, in_offsets;
    std::vector<VertexId> out, in;
    VertexOrder order;
  };
  static OrientedGraph wrap(tl_oriented* h, int device);
  static void rewrite_lists(HostLayout& L, const LocalOrder& local);
  const HostLayout& host() const;

  std::shared_ptr<tl_oriented> h_;
  int device_ = 0;
  VertexId n_ = 0;
  EdgeCount m_ = 0;
  VertexId max_out_ = 0;
  LocalOrder local_;
  mutable std::shared_ptr<HostLayout> host_;
  mutable std::shared_ptr<tl_multi> multi_;
  mutable std::vector<int> multi_devices_;
};

OrientedGraph orient(const Graph& g, const VertexOrder& order);
OrientedGraph apply_local_order(OrientedGraph g, const LocalOrder& local);

enum class EdgePolarity { positive, negative };
EdgePolarity edge_polarity(const OrientedGraph& g, VertexId u, VertexId v);

// ------------------------------------------------------------ engine.hpp
enum class Algorithm { cf_merge, cf_hash, kclist3, aot };
inline constexpr std::array<Algorithm, 4> kAllAlgorithms = {Algorithm::cf_merge, Algorithm::cf_hash,
                                                            Algorithm::kclist3, Algorithm::aot};
/// Algorithms with a B200 implementation (all of them).
inline constexpr std::array<Algorithm, 4> kDeviceAlgorithms = kAllAlgorithms;
const char* to_string(Algorithm a);
Algorithm parse_algorithm(const std::string& name);

struct RunStats {
  std::uint64_t triangles = 0;
  std::uint64_t probes = 0;
  std::uint64_t merge_comparisons = 0;
  std::uint64_t table_builds = 0;
  std::uint64_t positive_triangles = 0;
  std::uint64_t negative_triangles = 0;
  double wall_time_s = 0.0;  // listing kernels only (CUDA events), like the reference's
  // device extras
  std::uint64_t probes_executed = 0;
  std::uint64_t hash_sum = 0;
  std::uint64_t hash_xor = 0;

  void add_counters(const RunStats& o) {
    triangles += o.triangles;
    probes += o.probes;
    merge_comparisons += o.merge_comparisons;
    table_builds += o.table_builds;
    positive_triangles += o.positive_triangles;
    negative_triangles += o.negative_triangles;
  }
  bool counters_equal(const RunStats& o) const {
    return triangles == o.triangles && probes == o.probes && merge_comparisons == o.merge_comparisons &&
           table_builds == o.table_builds && positive_triangles == o.positive_triangles &&
           negative_triangles == o.negative_triangles;
  }
};

struct RunOptions {
  bool check_bitmap_between_pivots = false;  // accepted; the device tables are per work item
  bool cf_hash_reuse_last_table = false;     // skip rebuild if same owner, pivot-scoped
  bool aot_skip_negative_phase = false;      // fault injection hook for the verifier
};

struct NullSink {
  void operator()(VertexId, VertexId, VertexId) const noexcept {}
};
struct CollectingSink {
  std::vector<std::array<VertexId, 3>>* out;
  void operator()(VertexId a, VertexId b, VertexId c) const { out->push_back({a, b, c}); }
};

namespace detail {
void require_device_algorithm(Algorithm a);
std::uint32_t algorithm_code(Algorithm a);                    // TL_ALGO_*
void assert_layout(Algorithm a, const OrientedGraph& g);      // cf: rank-ascending lists (engine.hpp:143-149)
RunStats device_count(Algorithm algo, const OrientedGraph& g, const RunOptions& opt, int mode /*0 count, 1 hash*/);
RunStats device_list(Algorithm algo, const OrientedGraph& g, const RunOptions& opt,
                     std::vector<std::array<VertexId, 3>>& raw);
}  // namespace detail

namespace detail {
/// Batched listing (tl_run_list_batches): the run's emissions, raw role order,
/// handed to fn(user, triples, count) in batches of at most batch_triples
/// (0: TRILIST_BATCH_TRIPLES or 2^24) on the calling thread while the device
/// lists ahead; bounded host memory.  *canceled is set when fn stopped the run.
using BatchFn = int (*)(void* user, const std::uint32_t* triples, std::uint64_t count);
RunStats device_batches(Algorithm algo, const OrientedGraph& g, const RunOptions& opt, BatchFn fn, void* user,
                        bool* canceled);

/// Replays each batch into `workers` sinks: slice w of a batch goes to sink w,
/// on worker thread w (the calling thread is worker 0) -- run_parallel's one
/// sink per worker (parallel.hpp:32-35, :55-72).  The first exception a sink
/// throws stops the run and is rethrown by the caller.
template <typename Sink>
class BatchReplayer {
 public:
  explicit BatchReplayer(std::vector<Sink>& sinks) : sinks_(sinks), workers_(unsigned(sinks.size())) {
    for (unsigned w = 1; w < workers_; ++w) threads_.emplace_back([this, w] { loop(w); });
  }
  ~BatchReplayer() {
    {
      std::lock_guard<std::mutex> lock(mu_);
      stop_ = true;
    }
    start_.notify_all();
    for (auto& t : threads_) t.join();
  }
  static int call(void* self, const std::uint32_t* t, std::uint64_t count) {
    return static_cast<BatchReplayer*>(self)->replay(t, count);
  }
  std::exception_ptr error() const { return error_; }

 private:
  int replay(const std::uint32_t* t, std::uint64_t count) {
    {
      std::lock_guard<std::mutex> lock(mu_);
      batch_ = t;
      count_ = count;
      pending_ = workers_ - 1;
      ++generation_;
    }
    start_.notify_all();
    slice(0);
    std::unique_lock<std::mutex> lock(mu_);
    done_.wait(lock, [this] { return pending_ == 0; });
    return error_ ? 1 : 0;
  }
  void slice(unsigned w) {
    try {
      const std::uint64_t b = count_ * w / workers_, e = count_ * (w + 1) / workers_;
      Sink& sink = sinks_[w];
      for (std::uint64_t i = b; i < e; ++i) sink(batch_[3 * i], batch_[3 * i + 1], batch_[3 * i + 2]);
    } catch (...) {
      std::lock_guard<std::mutex> lock(mu_);
      if (!error_) error_ = std::current_exception();
    }
  }
  void loop(unsigned w) {
    std::uint64_t seen = 0;
    while (true) {
      {
        std::unique_lock<std::mutex> lock(mu_);
        start_.wait(lock, [&] { return stop_ || generation_ != seen; });
        if (stop_) return;
        seen = generation_;
      }
      slice(w);
      {
        std::lock_guard<std::mutex> lock(mu_);
        --pending_;
      }
      done_.notify_all();
    }
  }
  std::vector<Sink>& sinks_;
  unsigned workers_;
  std::vector<std::thread> threads_;
  std::mutex mu_;
  std::condition_variable start_, done_;
  const std::uint32_t* batch_ = nullptr;
  std::uint64_t count_ = 0, generation_ = 0;
  unsigned pending_ = 0;
  bool stop_ = false;
  std::exception_ptr error_;
};

template <typename Sink>
RunStats replay_batches(Algorithm algo, const OrientedGraph& g, std::vector<Sink>& sinks, const RunOptions& opt) {
  BatchReplayer<Sink> rep(sinks);
  bool canceled = false;
  RunStats s = device_batches(algo, g, opt, &BatchReplayer<Sink>::call, &rep, &canceled);
  if (rep.error()) std::rethrow_exception(rep.error());
  return s;
}
}  // namespace detail

/// run_algorithm (engine.hpp:294-304): NullSink counts; CollectingSink appends
/// the device list in one copy; any other sink gets every emission (role order
/// pivot, neighbor, witness) replayed from bounded host batches.
template <typename Sink>
RunStats run_algorithm(Algorithm algo, const OrientedGraph& g, Sink&& sink, const RunOptions& opt = {}) {
  using S = std::decay_t<Sink>;
  if constexpr (std::is_same_v<S, NullSink>) {
    return detail::device_count(algo, g, opt, 0);
  } else if constexpr (std::is_same_v<S, CollectingSink>) {
    return detail::device_list(algo, g, opt, *sink.out);
  } else {
    struct Ref {  // the caller's sink, by reference
      std::remove_reference_t<Sink>* p;
      void operator()(VertexId a, VertexId b, VertexId c) { (*p)(a, b, c); }
    };
    std::vector<Ref> one{Ref{&sink}};
    return detail::replay_batches(algo, g, one, opt);
  }
}

template <typename Sink>
RunStats cf_merge(const OrientedGraph& g, Sink&& sink, const RunOptions& opt = {}) {
  return run_algorithm(Algorithm::cf_merge, g, sink, opt);
}
template <typename Sink>
RunStats cf_hash(const OrientedGraph& g, Sink&& sink, const RunOptions& opt = {}) {
  return run_algorithm(Algorithm::cf_hash, g, sink, opt);
}
template <typename Sink>
RunStats kclist3(const OrientedGraph& g, Sink&& sink, const RunOptions& opt = {}) {
  return run_algorithm(Algorithm::kclist3, g, sink, opt);
}
template <typename Sink>
RunStats aot(const OrientedGraph& g, Sink&& sink, const RunOptions& opt = {}) {
  return run_algorithm(Algorithm::aot, g, sink, opt);
}

RunStats run_counting(Algorithm algo, const OrientedGraph& g, const RunOptions& opt = {});
RunStats run_collecting(Algorithm algo, const OrientedGraph& g, std::vector<std::array<VertexId, 3>>& out,
                        const RunOptions& opt = {});
/// Extension: count + order-independent hash of the canonical triangle set.
RunStats run_hashing(Algorithm algo, const OrientedGraph& g, const RunOptions& opt = {});

struct CostModel {
  std::uint64_t cf_cost = 0;
  std::uint64_t kclist_cost = 0;
  std::uint64_t aot_cost = 0;
};
CostModel cost_model(const OrientedGraph& g);

std::vector<Triangle> canonicalize_emissions(std::span<const std::array<VertexId, 3>> raw);

struct VerifyAlgorithmResult {
  Algorithm algorithm = Algorithm::aot;
  RunStats stats;
  std::uint64_t unique_triangles = 0;
  std::uint64_t duplicate_emissions = 0;
  std::uint64_t missing_count = 0;
  std::uint64_t extra_count = 0;
  std::vector<Triangle> missing_samples;
  std::vector<Triangle> extra_samples;
  bool pass = true;
};

struct VerifyReport {
  static constexpr std::size_t kMaxSamples = 32;
  bool pass = true;
  std::string reference;
  std::uint64_t reference_count = 0;
  std::vector<VerifyAlgorithmResult> results;
};

VerifyReport verify_equivalence(const Graph& g, std::span<const Algorithm> algorithms, const VertexOrder& order,
                                const LocalOrder& local = {}, const std::vector<Triangle>* reference = nullptr,
                                const RunOptions& opt = {});

// ---------------------------------------------------------- parallel.hpp
struct ParallelConfig {
  unsigned workers = 1;
  VertexId chunk = 64;
  /// Extension: the CUDA devices run_parallel_count / run_parallel_hashing
  /// split the run over (tl_multi_*: replicas + NCCL).  Empty: the
  /// TRILIST_DEVICES environment variable ("0,1,2,3") when set -- so unchanged
  /// reference callers can use every GPU -- else the graph's own device.
  std::vector<int> devices = {};
};

namespace detail {
void validate(const ParallelConfig& cfg);
}

RunStats run_parallel_count(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                            const RunOptions& opt = {});

/// run_parallel (parallel.hpp:25-78): one device run; one sink per worker
/// from the factory (:32-35).  NullSinks count; other sinks receive the
/// emissions in bounded host batches, each batch split across the workers'
/// sinks and replayed on `workers` host threads (the first exception a sink
/// throws is rethrown, :55-72).  Counters are those of the device run, the
/// same for any workers/chunk (test_parallel.cpp:11-40).
template <typename SinkFactory>
RunStats run_parallel(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg, SinkFactory&& make_sink,
                      const RunOptions& opt = {}) {
  detail::validate(cfg);
  using Sink = std::decay_t<decltype(make_sink(0u))>;
  std::vector<Sink> sinks;
  sinks.reserve(cfg.workers);
  for (unsigned w = 0; w < cfg.workers; ++w) sinks.push_back(make_sink(w));
  if constexpr (std::is_same_v<Sink, NullSink>) {
    return run_parallel_count(algo, g, cfg, opt);
  } else {
    return detail::replay_batches(algo, g, sinks, opt);
  }
}

/// Extension: count + order-independent triangle hash, split like run_parallel_count.
RunStats run_parallel_hashing(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                              const RunOptions& opt = {});
namespace detail {
std::vector<int> devices_for(const ParallelConfig& cfg, const OrientedGraph& g);  // cfg.devices / TRILIST_DEVICES
}
RunStats run_parallel_collecting(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                                 std::vector<std::vector<std::array<VertexId, 3>>>& buffers,
                                 const RunOptions& opt = {});

// ------------------------------------------------------------ oracle.hpp
struct OracleOptions {
  VertexId max_vertices = 2000;
};
/// brute_force_triangles (oracle.cpp:8-25) as a device kernel.
std::vector<Triangle> brute_force_triangles(const Graph& g, const OracleOptions& opt = {});

}  // namespace trilist
