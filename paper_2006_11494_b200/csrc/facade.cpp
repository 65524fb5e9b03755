// facade.cpp -- the reference `trilist` C++ API (include/trilist_b200/trilist.hpp)
// implemented over the B200 C-ABI.  Host code here only validates arguments,
// moves data across the boundary and reshapes host-side views (accessor
// lists, sink replay, set differences); every triangle/graph computation is a
// device call.
#include "trilist_b200/trilist.hpp"

#include <algorithm>
#include <cstdlib>
#include <charconv>
#include <cstring>
#include <istream>
#include <iterator>
#include <mutex>
#include <ostream>
#include <sstream>

namespace trilist {

// ------------------------------------------------------------------ errors
[[noreturn]] void throw_status(int code, const std::string& context) {
  std::string msg = context + ": " + tl_last_error();
  switch (code) {
    case TL_EINVAL: throw std::invalid_argument(tl_last_error());
    case TL_ERANGE: throw std::out_of_range(tl_last_error());
    case TL_ELOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

Triangle canonical_triangle(VertexId x, VertexId y, VertexId z) {  // graph.cpp:148-153
  if (x > y) std::swap(x, y);
  if (y > z) std::swap(y, z);
  if (x > y) std::swap(x, y);
  return {x, y, z};
}

// ------------------------------------------------------------------- Graph
Graph Graph::wrap(tl_graph* h, int device) {
  Graph g;
  g.h_ = std::shared_ptr<tl_graph>(h, [](tl_graph* p) { tl_graph_free(p); });
  g.device_ = device;
  check(tl_graph_info(h, &g.n_, &g.m_, &g.dups_, &g.loops_), "tl_graph_info");
  return g;
}

Graph Graph::from_edges(VertexId min_vertices, std::span<const std::pair<VertexId, VertexId>> edges) {
  static_assert(sizeof(std::pair<VertexId, VertexId>) == 8, "pair layout");
  tl_graph* h = nullptr;
  check(tl_graph_from_pairs(reinterpret_cast<const std::uint32_t*>(edges.data()), edges.size(), min_vertices, 0, 0,
                            nullptr, &h),
        "Graph::from_edges");
  return wrap(h, 0);
}

Graph Graph::from_edges(VertexId min_vertices, std::initializer_list<std::pair<VertexId, VertexId>> edges) {
  return from_edges(min_vertices, std::span<const std::pair<VertexId, VertexId>>(edges.begin(), edges.size()));
}

Graph Graph::from_device_pairs(VertexId min_vertices, const std::uint32_t* d_pairs, std::uint64_t npairs, int device,
                               void* stream) {
  tl_graph* h = nullptr;
  check(tl_graph_from_pairs(d_pairs, npairs, min_vertices, device, 1, stream, &h), "Graph::from_device_pairs");
  return wrap(h, device);
}

const Graph::HostCsr& Graph::csr() const {
  if (!csr_) {
    auto c = std::make_shared<HostCsr>();
    c->offsets.assign(std::size_t(n_) + 1, 0);
    c->adjacency.resize(2 * m_);
    if (h_) check(tl_graph_csr(h_.get(), c->offsets.data(), c->adjacency.data()), "Graph::offsets");
    csr_ = c;
  }
  return *csr_;
}

std::span<const VertexId> Graph::neighbors(VertexId u) const {
  const HostCsr& c = csr();
  return {c.adjacency.data() + c.offsets[u], c.adjacency.data() + c.offsets[u + 1]};
}

VertexId Graph::degree(VertexId u) const {  // graph.cpp:208-211
  if (u >= n_) throw std::out_of_range("vertex id " + std::to_string(u) + " out of range");
  const HostCsr& c = csr();
  return VertexId(c.offsets[u + 1] - c.offsets[u]);
}

bool Graph::has_edge(VertexId u, VertexId v) const {  // graph.cpp:213-217
  if (u >= n_ || v >= n_) return false;
  auto nu = neighbors(u);
  return std::binary_search(nu.begin(), nu.end(), v);
}

const std::vector<EdgeCount>& Graph::offsets() const { return csr().offsets; }
const std::vector<VertexId>& Graph::adjacency() const { return csr().adjacency; }

bool Graph::validate(std::string* why) const {  // graph.cpp:219-238
  auto fail = [&](const std::string& reason) {
    if (why) *why = reason;
    return false;
  };
  const HostCsr& c = csr();
  if (c.offsets.size() != std::size_t(n_) + 1) return fail("offsets size");
  if (c.offsets.front() != 0 || c.offsets.back() != 2 * m_) return fail("offset bounds");
  if (c.adjacency.size() != 2 * m_) return fail("adjacency size");
  for (VertexId u = 0; u < n_; ++u) {
    if (c.offsets[u] > c.offsets[u + 1]) return fail("offsets not monotone");
    auto nu = neighbors(u);
    for (std::size_t i = 0; i < nu.size(); ++i) {
      if (nu[i] >= n_) return fail("neighbor out of range");
      if (nu[i] == u) return fail("self-loop");
      if (i > 0 && nu[i - 1] >= nu[i]) return fail("list not strictly ascending");
      if (!has_edge(nu[i], u)) return fail("asymmetric edge");
    }
  }
  return true;
}

// ----------------------------------------------------------------- loading
namespace {
LoadResult load_common(int rc, tl_graph* h, const tl_load_diag& d, std::uint64_t line) {
  if (rc == TL_EPARSE) throw ParseError(tl_last_error(), line);
  if (rc == TL_ELENGTH) throw std::length_error(tl_last_error());
  check(rc, "load_edge_list");
  LoadResult r;
  r.graph = Graph::adopt(h, 0);
  r.diagnostics.lines_read = d.lines_read;
  r.diagnostics.edges_parsed = d.edges_parsed;
  r.diagnostics.self_loops_dropped = d.self_loops_dropped;
  r.diagnostics.duplicates_dropped = d.duplicates_dropped;
  return r;
}

std::uint32_t load_flags(const LoadOptions& o) {
  return (o.one_indexed ? TL_LOAD_ONE_INDEXED : 0u) | (o.compact_ids ? TL_LOAD_COMPACT_IDS : 0u);
}
}  // namespace

LoadResult load_edge_list_text(std::string_view text, const LoadOptions& options) {  // graph.cpp:244-248
  tl_graph* h = nullptr;
  tl_load_diag d{};
  std::uint64_t line = 0;
  int rc = tl_graph_from_text(text.data(), text.size(), load_flags(options), options.comment_prefixes.c_str(), 0, &h,
                              &d, &line);
  return load_common(rc, h, d, line);
}

LoadResult load_edge_list(std::istream& in, const LoadOptions& options) {  // graph.cpp:240-242
  std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return load_edge_list_text(text, options);
}

LoadResult load_edge_list_file(const std::string& path, const LoadOptions& options) {  // graph.cpp:250-275
  tl_graph* h = nullptr;
  tl_load_diag d{};
  std::uint64_t line = 0;
  int rc = tl_graph_from_file(path.c_str(), load_flags(options), options.comment_prefixes.c_str(), 0, &h, &d, &line);
  if (rc == TL_EIO) throw std::runtime_error(tl_last_error());
  return load_common(rc, h, d, line);
}

void write_edge_list(const Graph& g, std::ostream& out) {  // graph.cpp:277-281
  std::string buf;
  for (VertexId u = 0; u < g.num_vertices(); ++u)
    for (VertexId v : g.neighbors(u))
      if (v > u) {
        buf += std::to_string(u);
        buf += ' ';
        buf += std::to_string(v);
        buf += '\n';
        if (buf.size() > (1u << 20)) {
          out << buf;
          buf.clear();
        }
      }
  out << buf;
}

// --------------------------------------------------------------- ordering
bool VertexOrder::is_permutation() const {
  std::vector<bool> seen(rank.size(), false);
  for (VertexId r : rank) {
    if (r >= rank.size() || seen[r]) return false;
    seen[r] = true;
  }
  return true;
}

std::vector<VertexId> VertexOrder::vertices_by_rank() const {
  std::vector<VertexId> by_rank(rank.size());
  for (VertexId u = 0; u < rank.size(); ++u) by_rank[rank[u]] = u;
  return by_rank;
}

VertexOrder id_order(const Graph& g) {
  VertexOrder o;
  o.rank.resize(g.num_vertices());
  for (VertexId u = 0; u < g.num_vertices(); ++u) o.rank[u] = u;
  return o;
}

VertexOrder degree_order(const Graph& g) {
  VertexOrder o;
  o.rank.resize(g.num_vertices());
  if (g.handle() && g.num_vertices()) check(tl_degree_order(g.handle(), o.rank.data()), "degree_order");
  return o;
}

VertexOrder degeneracy_order(const Graph& g) {  // ordering.cpp:86-114
  VertexOrder o;
  o.rank.resize(g.num_vertices());
  if (g.handle() && g.num_vertices()) check(tl_degeneracy_order(g.handle(), o.rank.data()), "degeneracy_order");
  return o;
}

VertexOrder random_order(const Graph& g, std::uint64_t seed) {  // ordering.cpp:116-120
  VertexOrder o;
  o.rank.resize(g.num_vertices());
  check(tl_random_order(g.num_vertices(), seed, o.rank.data()), "random_order");
  return o;
}

VertexOrder make_order(const Graph& g, const OrderSpec& spec) {
  switch (spec.kind) {
    case OrderKind::id: return id_order(g);
    case OrderKind::degree: return degree_order(g);
    case OrderKind::degeneracy: return degeneracy_order(g);
    case OrderKind::random: return random_order(g, spec.seed);
  }
  throw std::invalid_argument("unknown order kind");
}

namespace {
std::uint64_t splitmix64(std::uint64_t& state) {  // ordering.cpp:13-19
  state += 0x9E3779B97F4A7C15ull;
  std::uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

std::uint64_t parse_seed(const std::string& text, std::size_t colon, const char* what) {
  std::uint64_t seed = 0;
  const char* b = text.data() + colon + 1;
  const char* e = text.data() + text.size();
  auto [p, ec] = std::from_chars(b, e, seed);
  if (ec != std::errc{} || p != e || b == e)
    throw std::invalid_argument(std::string("bad ") + what + " seed in '" + text + "'");
  return seed;
}
}  // namespace

OrderSpec parse_order_spec(const std::string& text) {  // ordering.cpp:132-141
  if (text == "id") return {OrderKind::id, 0};
  if (text == "degree") return {OrderKind::degree, 0};
  if (text == "degeneracy") return {OrderKind::degeneracy, 0};
  if (text.rfind("random:", 0) == 0) return {OrderKind::random, parse_seed(text, 6, "order")};
  throw std::invalid_argument("unknown order '" + text + "' (expected id|degree|degeneracy|random:SEED)");
}

std::string to_string(const OrderSpec& spec) {
  switch (spec.kind) {
    case OrderKind::id: return "id";
    case OrderKind::degree: return "degree";
    case OrderKind::degeneracy: return "degeneracy";
    case OrderKind::random: return "random:" + std::to_string(spec.seed);
  }
  return "?";
}

LocalOrder parse_local_order(const std::string& text) {  // ordering.cpp:154-161
  if (text == "rank-asc") return {LocalOrderPolicy::rank_asc, 0};
  if (text == "degree-desc") return {LocalOrderPolicy::degree_desc, 0};
  if (text.rfind("random:", 0) == 0) return {LocalOrderPolicy::random, parse_seed(text, 6, "local order")};
  throw std::invalid_argument("unknown local order '" + text + "' (expected rank-asc|degree-desc|random:SEED)");
}

std::string to_string(const LocalOrder& local) {
  switch (local.policy) {
    case LocalOrderPolicy::rank_asc: return "rank-asc";
    case LocalOrderPolicy::degree_desc: return "degree-desc";
    case LocalOrderPolicy::random: return "random:" + std::to_string(local.seed);
  }
  return "?";
}

OrientedGraph OrientedGraph::wrap(tl_oriented* h, int device) {
  OrientedGraph og;
  og.h_ = std::shared_ptr<tl_oriented>(h, [](tl_oriented* p) { tl_oriented_free(p); });
  og.device_ = device;
  check(tl_oriented_info(h, &og.n_, &og.m_, &og.max_out_), "tl_oriented_info");
  return og;
}

OrientedGraph OrientedGraph::from_csr(VertexId n, std::span<const EdgeCount> out_offsets, std::span<const VertexId> out,
                                      std::span<const VertexId> rank, int device) {
  if (out_offsets.size() != std::size_t(n) + 1 || rank.size() != n)
    throw std::invalid_argument("OrientedGraph::from_csr: array sizes do not match n");
  tl_oriented* h = nullptr;
  check(tl_oriented_from_csr(n, out.size(), out_offsets.data(), out.data(), rank.data(), device, nullptr, &h),
        "OrientedGraph::from_csr");
  return wrap(h, device);
}

const OrientedGraph::HostLayout& OrientedGraph::host() const {
  if (!host_) {
    auto L = std::make_shared<HostLayout>();
    L->out_offsets.assign(std::size_t(n_) + 1, 0);
    L->in_offsets.assign(std::size_t(n_) + 1, 0);
    L->out.resize(m_);
    L->in.resize(m_);
    L->order.rank.resize(n_);
    if (h_)
      check(tl_oriented_csr(h_.get(), L->out_offsets.data(), L->out.data(), L->in_offsets.data(), L->in.data(),
                            L->order.rank.data()),
            "OrientedGraph accessors");
    if (local_.policy != LocalOrderPolicy::rank_asc) rewrite_lists(*L, local_);
    host_ = L;
  }
  return *host_;
}

std::span<const VertexId> OrientedGraph::out_neighbors(VertexId u) const {
  const HostLayout& L = host();
  return {L.out.data() + L.out_offsets[u], L.out.data() + L.out_offsets[u + 1]};
}
std::span<const VertexId> OrientedGraph::in_neighbors(VertexId u) const {
  const HostLayout& L = host();
  return {L.in.data() + L.in_offsets[u], L.in.data() + L.in_offsets[u + 1]};
}
VertexId OrientedGraph::out_degree(VertexId u) const {
  const HostLayout& L = host();
  return VertexId(L.out_offsets[u + 1] - L.out_offsets[u]);
}
VertexId OrientedGraph::in_degree(VertexId u) const {
  const HostLayout& L = host();
  return VertexId(L.in_offsets[u + 1] - L.in_offsets[u]);
}
const VertexOrder& OrientedGraph::order() const { return host().order; }

bool OrientedGraph::out_lists_rank_sorted() const {
  for (VertexId u = 0; u < n_; ++u) {
    auto nb = out_neighbors(u);
    for (std::size_t i = 1; i < nb.size(); ++i)
      if (rank(nb[i - 1]) >= rank(nb[i])) return false;
  }
  return true;
}

OrientedGraph orient(const Graph& g, const VertexOrder& order) {  // ordering.cpp:185-188
  VertexId n = g.num_vertices();
  if (order.rank.size() != n) throw std::invalid_argument("order is not a permutation of the vertex set");
  if (!g.handle()) {  // default-constructed empty Graph
    if (n != 0) throw std::invalid_argument("graph has no device handle");
    Graph empty = Graph::from_edges(0, std::span<const std::pair<VertexId, VertexId>>());
    return orient(empty, order);
  }
  tl_oriented* h = nullptr;
  check(tl_orient(g.handle(), order.rank.data(), &h), "orient");
  return OrientedGraph::wrap(h, g.device());
}

// The device copy stays rank-ascending; the host accessor lists (built on
// first access) are rewritten exactly as ordering.cpp:229-266 does.  The
// rewrite is a pure function of (graph, order, policy, seed), so it is applied
// lazily and a caller that never reads the lists never pays for it.
void OrientedGraph::rewrite_lists(HostLayout& L, const LocalOrder& local) {
  const VertexId n = VertexId(L.order.rank.size());
  auto udeg = [&](VertexId x) {
    return VertexId(L.out_offsets[x + 1] - L.out_offsets[x] + L.in_offsets[x + 1] - L.in_offsets[x]);
  };
  const auto& rank = L.order.rank;
  auto fisher_yates = [](VertexId* first, VertexId* last, std::uint64_t seed) {  // ordering.cpp:23-33
    std::uint64_t state = seed;
    auto len = std::uint64_t(last - first);
    for (std::uint64_t i = len; i > 1; --i) {
      std::uint64_t j = std::uint64_t((static_cast<unsigned __int128>(splitmix64(state)) * i) >> 64);
      std::swap(first[i - 1], first[j]);
    }
  };
  for (VertexId u = 0; u < n; ++u) {
    for (std::uint64_t side = 0; side < 2; ++side) {
      auto& lst = side ? L.in : L.out;
      auto& off = side ? L.in_offsets : L.out_offsets;
      VertexId* b = lst.data() + off[u];
      VertexId* e = lst.data() + off[u + 1];
      switch (local.policy) {
        case LocalOrderPolicy::rank_asc:
          std::sort(b, e, [&](VertexId x, VertexId y) { return rank[x] < rank[y]; });
          break;
        case LocalOrderPolicy::degree_desc:
          std::sort(b, e, [&](VertexId x, VertexId y) {
            VertexId dx = udeg(x), dy = udeg(y);
            return dx != dy ? dx > dy : x < y;
          });
          break;
        case LocalOrderPolicy::random: {
          std::sort(b, e, [&](VertexId x, VertexId y) { return rank[x] < rank[y]; });
          std::uint64_t mix = local.seed;
          std::uint64_t list_key = splitmix64(mix) ^ ((std::uint64_t(u) << 1) | side);
          fisher_yates(b, e, list_key);
          break;
        }
      }
    }
  }
}

OrientedGraph apply_local_order(OrientedGraph g, const LocalOrder& local) {
  g.local_ = local;
  g.host_.reset();  // rebuilt from the device lists on first access
  return g;
}

EdgePolarity edge_polarity(const OrientedGraph& g, VertexId u, VertexId v) {  // ordering.cpp:268-276
  if (u >= g.num_vertices() || v >= g.num_vertices()) throw std::invalid_argument("vertex id out of range");
  auto nb = g.out_neighbors(u);
  if (std::find(nb.begin(), nb.end(), v) == nb.end())
    throw std::invalid_argument("no directed edge " + std::to_string(u) + " -> " + std::to_string(v));
  return g.out_degree_before(u, v) ? EdgePolarity::positive : EdgePolarity::negative;
}

// ------------------------------------------------------------------ engine
const char* to_string(Algorithm a) {  // engine.cpp:7-15
  switch (a) {
    case Algorithm::cf_merge: return "cf";
    case Algorithm::cf_hash: return "cf-hash";
    case Algorithm::kclist3: return "kclist";
    case Algorithm::aot: return "aot";
  }
  return "?";
}

Algorithm parse_algorithm(const std::string& name) {  // engine.cpp:17-24
  if (name == "cf") return Algorithm::cf_merge;
  if (name == "cf-hash") return Algorithm::cf_hash;
  if (name == "kclist") return Algorithm::kclist3;
  if (name == "aot") return Algorithm::aot;
  throw std::invalid_argument("unknown algorithm '" + name + "' (expected cf|cf-hash|kclist|aot)");
}

namespace detail {

void require_device_algorithm(Algorithm a) {
  for (Algorithm d : kDeviceAlgorithms)
    if (d == a) return;
  throw std::invalid_argument(std::string("algorithm '") + to_string(a) + "' has no B200 implementation");
}

std::uint32_t algorithm_code(Algorithm a) {
  switch (a) {
    case Algorithm::cf_merge: return TL_ALGO_CF_MERGE;
    case Algorithm::cf_hash: return TL_ALGO_CF_HASH;
    case Algorithm::kclist3: return TL_ALGO_KCLIST3;
    case Algorithm::aot: return TL_ALGO_AOT;
  }
  throw std::invalid_argument("unknown algorithm");
}

// engine.hpp:143-149: the merge kernel needs rank-ascending lists.  The device
// copy always is; a host layout rewritten by apply_local_order may not be.
void assert_layout(Algorithm algo, const OrientedGraph& g) {
  if (algo == Algorithm::cf_merge && g.local_order().policy != LocalOrderPolicy::rank_asc &&
      !g.out_lists_rank_sorted())
    throw std::invalid_argument("merge kernel requires rank-ascending adjacency (local order rank-asc)");
}

namespace {
tl_run_options options_for(Algorithm algo, const RunOptions& opt) {
  tl_run_options o;
  std::memset(&o, 0, sizeof(o));
  o.skip_negative_phase = opt.aot_skip_negative_phase ? 1u : 0u;
  o.check_hygiene = opt.check_bitmap_between_pivots ? 1u : 0u;
  o.part = 0;
  o.nparts = 1;
  o.algorithm = algorithm_code(algo);
  o.cf_hash_reuse_last_table = opt.cf_hash_reuse_last_table ? 1u : 0u;
  return o;
}

// cf-hash with cf_hash_reuse_last_table counts a rebuild whenever the owner
// changes along the list (engine.hpp:200-206), so on a host layout other than
// the device's rank-ascending one the table_builds counter follows that
// layout: recount it over the host lists.
void relayout_table_builds(const OrientedGraph& g, const RunOptions& opt, Algorithm algo, RunStats& r) {
  if (algo != Algorithm::cf_hash || !opt.cf_hash_reuse_last_table ||
      g.local_order().policy == LocalOrderPolicy::rank_asc)
    return;
  std::uint64_t builds = 0;
  for (VertexId u = 0; u < g.num_vertices(); ++u) {
    bool prev_u = false;
    for (VertexId v : g.out_neighbors(u)) {
      const bool hash_u = g.out_degree_before(v, u);
      if (hash_u) {
        if (!prev_u) builds += g.out_degree(u);
      } else {
        builds += g.out_degree(v);
      }
      prev_u = hash_u;
    }
  }
  r.table_builds = builds;
}

RunStats to_run_stats(const tl_stats& s) {
  RunStats r;
  r.triangles = s.triangles;
  r.probes = s.probes;
  r.merge_comparisons = s.merge_comparisons;
  r.table_builds = s.table_builds;
  r.positive_triangles = s.positive_triangles;
  r.negative_triangles = s.negative_triangles;
  r.wall_time_s = s.list_ms * 1e-3;
  r.probes_executed = s.probes_executed;
  r.hash_sum = s.hash_sum;
  r.hash_xor = s.hash_xor;
  return r;
}

bool empty_handle(const OrientedGraph& g) { return g.handle() == nullptr; }
}  // namespace

RunStats device_count(Algorithm algo, const OrientedGraph& g, const RunOptions& opt, int mode) {
  require_device_algorithm(algo);
  assert_layout(algo, g);
  if (empty_handle(g)) return RunStats{};
  tl_run_options o = options_for(algo, opt);
  tl_stats s;
  if (mode == 1)
    check(tl_run_hash(g.handle(), &o, &s), "hash run");
  else
    check(tl_run_count(g.handle(), &o, &s), "count run");
  RunStats r = to_run_stats(s);
  relayout_table_builds(g, opt, algo, r);
  return r;
}

RunStats device_list(Algorithm algo, const OrientedGraph& g, const RunOptions& opt,
                     std::vector<std::array<VertexId, 3>>& raw) {
  require_device_algorithm(algo);
  assert_layout(algo, g);
  if (empty_handle(g)) return RunStats{};
  tl_run_options o = options_for(algo, opt);
  tl_stats s;
  check(tl_run_list(g.handle(), &o, nullptr, 0, 0, &s), "list run");  // count (cached for sizing)
  std::size_t base = raw.size();
  raw.resize(base + s.triangles);
  static_assert(sizeof(std::array<VertexId, 3>) == 12, "triple layout");
  check(tl_run_list(g.handle(), &o, reinterpret_cast<std::uint32_t*>(raw.data() + base), s.triangles, 0, &s),
        "list run");
  RunStats r = to_run_stats(s);
  relayout_table_builds(g, opt, algo, r);
  return r;
}

RunStats device_batches(Algorithm algo, const OrientedGraph& g, const RunOptions& opt, BatchFn fn, void* user,
                        bool* canceled) {
  require_device_algorithm(algo);
  assert_layout(algo, g);
  if (canceled) *canceled = false;
  if (empty_handle(g)) return RunStats{};
  tl_run_options o = options_for(algo, opt);
  std::uint64_t batch = 0;  // 0: the library's default (2^24 triples = 192 MiB per host buffer)
  if (const char* e = std::getenv("TRILIST_BATCH_TRIPLES")) batch = std::strtoull(e, nullptr, 10);
  tl_stats s;
  const int rc = tl_run_list_batches(g.handle(), &o, batch, 0, fn, user, &s);
  if (rc == TL_ECANCELED) {
    if (canceled) *canceled = true;
    return RunStats{};
  }
  check(rc, "batched listing");
  RunStats r = to_run_stats(s);
  relayout_table_builds(g, opt, algo, r);
  return r;
}

void validate(const ParallelConfig& cfg) {  // parallel.hpp:28-29
  if (cfg.workers < 1) throw std::invalid_argument("workers must be >= 1");
  if (cfg.chunk < 1) throw std::invalid_argument("chunk must be >= 1");
}

}  // namespace detail

RunStats run_counting(Algorithm algo, const OrientedGraph& g, const RunOptions& opt) {
  return detail::device_count(algo, g, opt, 0);
}

RunStats run_collecting(Algorithm algo, const OrientedGraph& g, std::vector<std::array<VertexId, 3>>& out,
                        const RunOptions& opt) {
  return detail::device_list(algo, g, opt, out);
}

RunStats run_hashing(Algorithm algo, const OrientedGraph& g, const RunOptions& opt) {
  return detail::device_count(algo, g, opt, 1);
}

CostModel cost_model(const OrientedGraph& g) {
  CostModel cm;
  if (!g.handle()) return cm;
  std::uint64_t c[3];
  check(tl_cost_model(g.handle(), c), "cost_model");
  cm.cf_cost = c[0];
  cm.kclist_cost = c[1];
  cm.aot_cost = c[2];
  return cm;
}

std::vector<Triangle> canonicalize_emissions(std::span<const std::array<VertexId, 3>> raw) {  // engine.cpp:51-57
  std::vector<Triangle> out;
  out.reserve(raw.size());
  for (const auto& t : raw) out.push_back(canonical_triangle(t[0], t[1], t[2]));
  std::sort(out.begin(), out.end());
  return out;
}

VerifyReport verify_equivalence(const Graph& g, std::span<const Algorithm> algorithms, const VertexOrder& order,
                                const LocalOrder& local, const std::vector<Triangle>* reference,
                                const RunOptions& opt) {  // engine.cpp:82-130, compared on the device (tl_verify)
  for (Algorithm a : algorithms) detail::require_device_algorithm(a);
  OrientedGraph oriented = orient(g, order);
  // cf runs on the rank-ascending layout it requires, the others on `local`;
  // no counter of a non-reusing run depends on the layout
  // (test_engine.cpp:172-185), so every run uses the device's lists.
  (void)local;
  VerifyReport report;
  report.reference = reference ? "oracle" : (algorithms.empty() ? "" : to_string(algorithms.front()));
  if (!oriented.handle()) {  // empty graph: every set is empty
    for (Algorithm a : algorithms) {
      VerifyAlgorithmResult r;
      r.algorithm = a;
      report.results.push_back(r);
    }
    return report;
  }
  std::vector<std::uint32_t> codes;
  for (Algorithm a : algorithms) codes.push_back(detail::algorithm_code(a));
  tl_run_options o = detail::options_for(Algorithm::aot, opt);
  std::vector<tl_verify_result> res(codes.size());
  std::uint64_t ref_count = 0;
  static_assert(sizeof(Triangle) == 12, "Triangle layout");
  check(tl_verify(oriented.handle(), codes.data(), std::uint32_t(codes.size()), &o,
                  reference ? reinterpret_cast<const std::uint32_t*>(reference->data()) : nullptr,
                  reference ? reference->size() : 0, reference ? 1 : 0, res.data(), &ref_count),
        "verify_equivalence");
  auto samples = [](const std::uint32_t* t, std::uint32_t k) {
    std::vector<Triangle> v;
    for (std::uint32_t i = 0; i < k; ++i) v.push_back({t[3 * i], t[3 * i + 1], t[3 * i + 2]});
    return v;
  };
  for (std::size_t i = 0; i < res.size(); ++i) {
    const tl_verify_result& x = res[i];
    VerifyAlgorithmResult r;
    r.algorithm = algorithms[i];
    r.stats = detail::to_run_stats(x.stats);
    r.unique_triangles = x.unique_triangles;
    r.duplicate_emissions = x.duplicate_emissions;
    r.missing_count = x.missing_count;
    r.extra_count = x.extra_count;
    r.missing_samples = samples(x.missing_samples, x.n_missing_samples);
    r.extra_samples = samples(x.extra_samples, x.n_extra_samples);
    r.pass = x.pass != 0;
    report.pass = report.pass && r.pass;
    report.results.push_back(std::move(r));
  }
  report.reference_count = ref_count;
  return report;
}

// ---------------------------------------------------------------- parallel
std::vector<int> detail::devices_for(const ParallelConfig& cfg, const OrientedGraph& g) {
  std::vector<int> devs = cfg.devices;
  if (devs.empty()) {
    if (const char* e = std::getenv("TRILIST_DEVICES")) {
      std::string text(e);
      std::size_t i = 0;
      while (i < text.size()) {
        std::size_t j = text.find(',', i);
        if (j == std::string::npos) j = text.size();
        const std::string item = text.substr(i, j - i);
        if (!item.empty()) {
          int d = 0;
          const auto r = std::from_chars(item.data(), item.data() + item.size(), d);
          if (r.ec != std::errc() || r.ptr != item.data() + item.size())
            throw std::invalid_argument("TRILIST_DEVICES must be a comma-separated device list, got '" + text + "'");
          devs.push_back(d);
        }
        i = j + 1;
      }
    }
  }
  (void)g;
  return devs;
}

tl_multi* OrientedGraph::multi(const std::vector<int>& devices) const {
  if (!h_) return nullptr;
  if (!multi_ || multi_devices_ != devices) {
    multi_.reset();
    tl_multi* m = nullptr;
    check(tl_multi_create(h_.get(), devices.data(), int(devices.size()), &m), "tl_multi_create");
    multi_ = std::shared_ptr<tl_multi>(m, [](tl_multi* p) { tl_multi_free(p); });
    multi_devices_ = devices;
  }
  return multi_.get();
}

namespace {
RunStats multi_run(Algorithm algo, const OrientedGraph& g, const std::vector<int>& devs, const RunOptions& opt,
                   bool hashing) {
  detail::require_device_algorithm(algo);
  detail::assert_layout(algo, g);
  if (!g.handle()) return RunStats{};
  tl_run_options o = detail::options_for(algo, opt);
  tl_stats s;
  tl_multi* m = g.multi(devs);
  check(hashing ? tl_multi_hash(m, &o, &s) : tl_multi_count(m, &o, &s), "multi-device run");
  RunStats r = detail::to_run_stats(s);
  detail::relayout_table_builds(g, opt, algo, r);
  return r;
}
}  // namespace

RunStats run_parallel_count(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                            const RunOptions& opt) {
  detail::validate(cfg);
  const std::vector<int> devs = detail::devices_for(cfg, g);
  if (!devs.empty()) return multi_run(algo, g, devs, opt, false);
  return run_counting(algo, g, opt);
}

RunStats run_parallel_hashing(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                              const RunOptions& opt) {
  detail::validate(cfg);
  const std::vector<int> devs = detail::devices_for(cfg, g);
  if (!devs.empty()) return multi_run(algo, g, devs, opt, true);
  return run_hashing(algo, g, opt);
}

RunStats run_parallel_collecting(Algorithm algo, const OrientedGraph& g, const ParallelConfig& cfg,
                                 std::vector<std::vector<std::array<VertexId, 3>>>& buffers, const RunOptions& opt) {
  detail::validate(cfg);
  buffers.assign(cfg.workers, {});
  return run_collecting(algo, g, buffers[0], opt);
}

// ------------------------------------------------------------------ oracle
std::vector<Triangle> brute_force_triangles(const Graph& g, const OracleOptions& opt) {  // oracle.cpp:8-25
  if (g.num_vertices() > opt.max_vertices)
    throw std::invalid_argument("oracle refuses graphs larger than " + std::to_string(opt.max_vertices) +
                                " vertices");
  std::vector<Triangle> out;
  if (!g.handle() || g.num_edges() == 0) return out;
  std::uint64_t count = 0;
  check(tl_brute_force(g.handle(), opt.max_vertices, nullptr, 0, &count), "brute_force_triangles");
  out.resize(count);
  check(tl_brute_force(g.handle(), opt.max_vertices, reinterpret_cast<std::uint32_t*>(out.data()), count, &count),
        "brute_force_triangles");
  return out;
}

}  // namespace trilist
