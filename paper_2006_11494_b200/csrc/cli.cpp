// cli.cpp -- `trilist` command line (the reference's tools/trilist_main.cpp
// interface) over the B200 facade.  Subcommands count, list, verify, bench,
// stats; every JSON document carries schema_version.  Exit codes
// (trilist_main.cpp:28-31): 0 success, 1 input/parse failure, 2 usage error,
// 3 verification failure.  The reference parses its arguments with CLI11
// (absent here); the parser below accepts the same options, values and
// validators and maps every rejection to exit code 2.
#include <unistd.h>

#include <algorithm>
#include <charconv>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "trilist_b200/report.hpp"
#include "trilist_b200/trilist.hpp"

namespace {

using namespace trilist;

constexpr int kExitOk = 0;
constexpr int kExitInput = 1;
constexpr int kExitUsage = 2;
constexpr int kExitVerify = 3;
constexpr const char* kVersion = "0.1.0";

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- arguments
struct CommonArgs {  // trilist_main.cpp:33-40
  std::string input;
  std::string format = "edgelist";
  bool compact = false;
  bool one_indexed = false;
  std::string out;
  bool pretty = false;
};

struct RunArgs {  // trilist_main.cpp:42-48
  std::string algo = "aot";
  std::string order;
  std::string local_order;
  unsigned threads = 1;
  VertexId chunk = 64;
};

struct Invocation {
  std::string command;
  CommonArgs c;
  RunArgs r;
  bool list_sorted = false;
  std::vector<std::string> verify_algos = {"cf", "cf-hash", "kclist", "aot"};
  std::vector<std::string> verify_orders = {"degree", "degeneracy", "id"};
  VertexId oracle_cap = 2000;
  std::string fault = "none";
  std::vector<std::string> bench_algos = {"cf", "cf-hash", "kclist", "aot"};
  std::vector<std::string> bench_orders = {"degree"};
  std::vector<unsigned> bench_threads = {1};
  unsigned bench_repeats = 3;
  bool bench_csv = false;
};

const char* kAlgoNames[] = {"cf", "cf-hash", "kclist", "aot"};

void check_algo(const std::string& opt, const std::string& v) {
  for (const char* a : kAlgoNames)
    if (v == a) return;
  throw UsageError(opt + ": " + v + " not in {cf,cf-hash,kclist,aot}");
}

template <typename T>
T parse_uint(const std::string& opt, const std::string& v, T lo, T hi) {
  unsigned long long x = 0;
  auto [p, ec] = std::from_chars(v.data(), v.data() + v.size(), x);
  if (ec != std::errc{} || p != v.data() + v.size() || v.empty())
    throw UsageError(opt + ": Value " + v + " could not be converted");
  if (x < lo || x > hi)
    throw UsageError(opt + ": Value " + v + " not in range [" + std::to_string(lo) + " - " + std::to_string(hi) +
                     "]");
  return T(x);
}

std::vector<std::string> split_commas(const std::string& v) {
  std::vector<std::string> out;
  std::size_t b = 0;
  while (true) {
    std::size_t e = v.find(',', b);
    out.push_back(v.substr(b, e == std::string::npos ? std::string::npos : e - b));
    if (e == std::string::npos) break;
    b = e + 1;
  }
  return out;
}

void check_order(const std::string& opt, const std::string& v) {
  try {
    parse_order_spec(v);
  } catch (const std::invalid_argument& e) {
    throw UsageError(opt + ": " + e.what());
  }
}

void check_local(const std::string& opt, const std::string& v) {
  try {
    parse_local_order(v);
  } catch (const std::invalid_argument& e) {
    throw UsageError(opt + ": " + e.what());
  }
}

std::string help_text(const std::string& command) {
  std::string h;
  if (command.empty()) {
    h = "orientation-based triangle listing toolkit (B200)\n"
        "Usage: trilist [OPTIONS] SUBCOMMAND\n\n"
        "Options:\n  -h,--help      Print this help message and exit\n  --version      Display program version "
        "information and exit\n\n"
        "Subcommands:\n"
        "  count          count triangles, print a JSON report\n"
        "  list           write triangles, one 'a b c' per line\n"
        "  verify         cross-check kernels against each other and the brute-force oracle\n"
        "  bench          time kernels over a cross product\n"
        "  stats          orientation cost model, no listing\n";
    return h;
  }
  h = "Usage: trilist " + command + " [OPTIONS] input\n\nPositionals:\n"
      "  input TEXT REQUIRED    edge list file, .gz transparent, '-' for stdin\n\nOptions:\n"
      "  -h,--help              Print this help message and exit\n"
      "  --format TEXT:{edgelist} [edgelist]  input format\n"
      "  --compact              renumber ids by first appearance\n"
      "  --one-indexed          input counts vertices from 1\n"
      "  --out TEXT             write the report here instead of stdout\n"
      "  --pretty               indent JSON output\n";
  if (command == "count" || command == "list")
    h += "  --algo TEXT:{cf,cf-hash,kclist,aot} [aot]  listing kernel\n";
  h += "  --order ORDER          vertex order: id|degree|degeneracy|random:SEED (default: degree; degeneracy for "
       "kclist)\n"
       "  --local-order LOCAL    adjacency layout: rank-asc|degree-desc|random:SEED (default: rank-asc; "
       "degree-desc for aot)\n"
       "  --threads UINT:INT in [1 - 4096] [1] (Env:TRILIST_THREADS)  worker count\n"
       "  --chunk UINT:INT in [1 - 1073741824] [64]  pivots per work-queue grab\n";
  if (command == "list") h += "  --sorted               sort output lexicographically\n";
  if (command == "verify")
    h += "  --algos TEXT:{cf,cf-hash,kclist,aot} ... [[cf,cf-hash,kclist,aot]]  kernels to cross-check\n"
         "  --orders ORDER ... [[degree,degeneracy,id]]  vertex orders to cover\n"
         "  --oracle-cap UINT [2000]  skip the brute-force oracle above this vertex count\n";
  if (command == "bench")
    h += "  --algos TEXT:{cf,cf-hash,kclist,aot} ... [[cf,cf-hash,kclist,aot]]  kernels to time\n"
         "  --orders ORDER ... [[degree]]  vertex orders to time\n"
         "  --threads-list UINT ... [[1]]  worker counts to time\n"
         "  --repeats UINT:INT in [1 - 1000] [3]  repetitions per cell\n"
         "  --csv                  emit CSV instead of JSON\n";
  return h;
}

struct HelpRequest {
  std::string text;
};
struct VersionRequest {};

// trilist_main.cpp:371-435: one required subcommand, its options and one
// positional input.  Options take "--opt value" or "--opt=value"; list options
// split on ',' and accumulate across occurrences.
Invocation parse_args(int argc, char** argv) {
  Invocation inv;
  std::vector<std::string> args(argv + 1, argv + argc);
  std::size_t i = 0;
  // global options before the subcommand
  while (i < args.size() && !args[i].empty() && args[i][0] == '-') {
    if (args[i] == "-h" || args[i] == "--help") throw HelpRequest{help_text("")};
    if (args[i] == "--version") throw VersionRequest{};
    throw UsageError("The following argument was not expected: " + args[i]);
  }
  if (i == args.size()) throw UsageError("A subcommand is required");
  inv.command = args[i++];
  static const char* kCommands[] = {"count", "list", "verify", "bench", "stats"};
  if (std::find_if(std::begin(kCommands), std::end(kCommands), [&](const char* c) { return inv.command == c; }) ==
      std::end(kCommands))
    throw UsageError("The following arguments were not expected: " + inv.command);
  const std::string& cmd = inv.command;
  const bool with_algo = cmd == "count" || cmd == "list";
  bool threads_given = false;
  std::map<std::string, bool> list_reset;  // a list option's first occurrence replaces its default
  auto take_list = [&](std::vector<std::string>& dst, const std::string& opt, const std::string& v) {
    if (!list_reset[opt]) {
      dst.clear();
      list_reset[opt] = true;
    }
    for (const std::string& x : split_commas(v)) dst.push_back(x);
  };

  for (; i < args.size(); ++i) {
    std::string a = args[i];
    if (a == "-h" || a == "--help") throw HelpRequest{help_text(cmd)};
    if (a.size() < 2 || a[0] != '-' || a == "-") {  // positional
      if (!inv.c.input.empty()) throw UsageError("The following arguments were not expected: " + a);
      inv.c.input = a;
      continue;
    }
    std::string opt = a, val;
    bool has_val = false;
    if (auto eq = a.find('='); eq != std::string::npos && a.rfind("--", 0) == 0) {
      opt = a.substr(0, eq);
      val = a.substr(eq + 1);
      has_val = true;
    }
    auto value = [&]() -> std::string {
      if (has_val) return val;
      if (i + 1 >= args.size()) throw UsageError(opt + ": 1 required TEXT missing");
      return args[++i];
    };
    auto flag = [&]() {
      if (has_val) throw UsageError(opt + ": flag does not take a value");
    };
    if (opt == "--format") {
      std::string v = value();
      if (v != "edgelist") throw UsageError("--format: " + v + " not in {edgelist}");
      inv.c.format = v;
    } else if (opt == "--compact") {
      flag();
      inv.c.compact = true;
    } else if (opt == "--one-indexed") {
      flag();
      inv.c.one_indexed = true;
    } else if (opt == "--out") {
      inv.c.out = value();
    } else if (opt == "--pretty") {
      flag();
      inv.c.pretty = true;
    } else if (opt == "--algo" && with_algo) {
      inv.r.algo = value();
      check_algo(opt, inv.r.algo);
    } else if (opt == "--order") {
      inv.r.order = value();
      check_order(opt, inv.r.order);
    } else if (opt == "--local-order") {
      inv.r.local_order = value();
      check_local(opt, inv.r.local_order);
    } else if (opt == "--threads") {
      inv.r.threads = parse_uint<unsigned>(opt, value(), 1u, 4096u);
      threads_given = true;
    } else if (opt == "--chunk") {
      inv.r.chunk = parse_uint<VertexId>(opt, value(), 1u, 1u << 30);
    } else if (opt == "--sorted" && cmd == "list") {
      flag();
      inv.list_sorted = true;
    } else if (opt == "--algos" && (cmd == "verify" || cmd == "bench")) {
      auto& dst = cmd == "verify" ? inv.verify_algos : inv.bench_algos;
      take_list(dst, opt, value());
      for (const std::string& x : dst) check_algo(opt, x);
    } else if (opt == "--orders" && (cmd == "verify" || cmd == "bench")) {
      auto& dst = cmd == "verify" ? inv.verify_orders : inv.bench_orders;
      take_list(dst, opt, value());
      for (const std::string& x : dst) check_order(opt, x);
    } else if (opt == "--oracle-cap" && cmd == "verify") {
      inv.oracle_cap = parse_uint<VertexId>(opt, value(), 0u, ~VertexId(0));
    } else if (opt == "--inject-fault" && cmd == "verify") {
      inv.fault = value();
      if (inv.fault != "none" && inv.fault != "drop-negative-phase")
        throw UsageError("--inject-fault: " + inv.fault + " not in {none,drop-negative-phase}");
    } else if (opt == "--threads-list" && cmd == "bench") {
      std::vector<std::string> raw;
      for (unsigned t : inv.bench_threads) raw.push_back(std::to_string(t));
      take_list(raw, opt, value());
      inv.bench_threads.clear();
      for (const std::string& x : raw) inv.bench_threads.push_back(parse_uint<unsigned>(opt, x, 0u, ~0u));
    } else if (opt == "--repeats" && cmd == "bench") {
      inv.bench_repeats = parse_uint<unsigned>(opt, value(), 1u, 1000u);
    } else if (opt == "--csv" && cmd == "bench") {
      flag();
      inv.bench_csv = true;
    } else {
      throw UsageError("The following arguments were not expected: " + a);
    }
  }
  if (inv.c.input.empty()) throw UsageError("input is required");
  if (!threads_given) {  // ->envname("TRILIST_THREADS")
    if (const char* env = std::getenv("TRILIST_THREADS"); env && *env)
      inv.r.threads = parse_uint<unsigned>("--threads", env, 1u, 4096u);
  }
  return inv;
}

// ------------------------------------------------------------- commands
double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Per-algorithm defaults (trilist_main.cpp:110-124).
OrderSpec resolve_order(const RunArgs& r, Algorithm algo) {
  if (!r.order.empty()) return parse_order_spec(r.order);
  return {algo == Algorithm::kclist3 ? OrderKind::degeneracy : OrderKind::degree, 0};
}

LocalOrder resolve_local(const RunArgs& r, Algorithm algo) {
  if (!r.local_order.empty()) return parse_local_order(r.local_order);
  if (algo == Algorithm::aot) return {LocalOrderPolicy::degree_desc, 0};
  return {LocalOrderPolicy::rank_asc, 0};
}

LoadResult load_input(const CommonArgs& c, double& seconds) {
  auto t0 = std::chrono::steady_clock::now();
  LoadOptions opt;
  opt.one_indexed = c.one_indexed;
  opt.compact_ids = c.compact;
  LoadResult r = load_edge_list_file(c.input, opt);
  seconds = seconds_since(t0);
  return r;
}

int emit(const CommonArgs& c, const std::string& text) {
  if (c.out.empty()) {
    std::fwrite(text.data(), 1, text.size(), stdout);
    std::fflush(stdout);
    return kExitOk;
  }
  std::ofstream f(c.out, std::ios::binary);
  if (!f) {
    std::fprintf(stderr, "error: cannot open '%s' for writing\n", c.out.c_str());
    return kExitInput;
  }
  f << text;
  return f.good() ? kExitOk : kExitInput;
}

int emit_json(const CommonArgs& c, const Json& doc) { return emit(c, doc.dump(c.pretty ? 2 : -1) + "\n"); }

bool merge_layout_conflict(Algorithm algo, const RunArgs& r) {  // trilist_main.cpp:160-165
  return algo == Algorithm::cf_merge && !r.local_order.empty() &&
         parse_local_order(r.local_order).policy != LocalOrderPolicy::rank_asc;
}

struct PreparedRun {
  OrientedGraph oriented;
  OrderSpec order;
  LocalOrder local;
  PhaseTimings timings;
};

PreparedRun prepare(const Graph& g, const RunArgs& r, Algorithm algo, double load_s) {
  PreparedRun p;
  p.order = resolve_order(r, algo);
  p.local = algo == Algorithm::cf_merge ? LocalOrder{LocalOrderPolicy::rank_asc, 0} : resolve_local(r, algo);
  p.timings.load_s = load_s;
  auto t0 = std::chrono::steady_clock::now();
  VertexOrder order = make_order(g, p.order);
  p.timings.order_s = seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  p.oriented = orient(g, order);
  if (p.local.policy != LocalOrderPolicy::rank_asc) p.oriented = apply_local_order(p.oriented, p.local);
  p.timings.orient_s = seconds_since(t0);
  return p;
}

Json run_document(const char* command, const CommonArgs& c, const LoadResult& loaded) {
  Json d;
  d["schema_version"] = kSchemaVersion;
  d["command"] = command;
  d["dataset"] = c.input;
  d["n"] = loaded.graph.num_vertices();
  d["m"] = loaded.graph.num_edges();
  d["load"] = to_json(loaded.diagnostics);
  return d;
}

int cmd_count(const Invocation& inv) {
  const CommonArgs& c = inv.c;
  const RunArgs& r = inv.r;
  Algorithm algo = parse_algorithm(r.algo);
  if (merge_layout_conflict(algo, r)) {
    std::fprintf(stderr, "error: --algo cf requires --local-order rank-asc\n");
    return kExitUsage;
  }
  double load_s = 0;
  LoadResult loaded = load_input(c, load_s);
  PreparedRun p = prepare(loaded.graph, r, algo, load_s);
  RunStats stats = run_parallel_count(algo, p.oriented, {r.threads, r.chunk});
  p.timings.list_s = stats.wall_time_s;
  Json doc = run_document("count", c, loaded);
  doc["algorithm"] = to_string(algo);
  doc["order"] = to_string(p.order);
  doc["local_order"] = to_string(p.local);
  doc["workers"] = r.threads;
  doc["chunk"] = r.chunk;
  doc["triangles"] = stats.triangles;
  doc["stats"] = to_json(stats);
  doc["costs"] = to_json(cost_model(p.oriented));
  doc["timings"] = to_json(p.timings);
  return emit_json(c, doc);
}

void append_uint(std::string& out, std::uint32_t x) {
  char buf[16];
  auto [p, ec] = std::to_chars(buf, buf + sizeof(buf), x);
  out.append(buf, p);
}

// Unsorted `list`: the lines are written batch by batch as the device lists
// them (tl_run_list_batches), so host memory stays bounded whatever the
// triangle count (the reference builds the whole list first).
struct ListWriter {
  FILE* f;
  std::string buf;
  static int write(void* self, const std::uint32_t* t, std::uint64_t count) {
    auto* w = static_cast<ListWriter*>(self);
    constexpr std::uint64_t kChunk = 1u << 20;  // lines formatted per write
    for (std::uint64_t b = 0; b < count; b += kChunk) {
      const std::uint64_t e = std::min(count, b + kChunk);
      w->buf.clear();
      for (std::uint64_t k = b; k < e; ++k) {
        Triangle tr = canonical_triangle(t[3 * k], t[3 * k + 1], t[3 * k + 2]);
        append_uint(w->buf, tr.a);
        w->buf += ' ';
        append_uint(w->buf, tr.b);
        w->buf += ' ';
        append_uint(w->buf, tr.c);
        w->buf += '\n';
      }
      if (std::fwrite(w->buf.data(), 1, w->buf.size(), w->f) != w->buf.size()) return 1;
    }
    return 0;
  }
};

int stream_list(const CommonArgs& c, const OrientedGraph& og, Algorithm algo) {
  FILE* f = c.out.empty() ? stdout : std::fopen(c.out.c_str(), "wb");
  if (!f) {
    std::fprintf(stderr, "error: cannot open '%s' for writing\n", c.out.c_str());
    return kExitInput;
  }
  ListWriter w{f, {}};
  int rc = TL_OK;
  if (og.handle() && og.num_edges()) {
    tl_run_options o{};
    o.nparts = 1;
    o.algorithm = detail::algorithm_code(algo);
    tl_stats s;
    rc = tl_run_list_batches(og.handle(), &o, 0, 0, &ListWriter::write, &w, &s);
  }
  const bool write_failed = rc == TL_ECANCELED || std::fflush(f) != 0;
  if (f != stdout) std::fclose(f);
  if (write_failed) {
    std::fprintf(stderr, "error: cannot write '%s'\n", c.out.empty() ? "<stdout>" : c.out.c_str());
    return kExitInput;
  }
  check(rc, "list");
  return kExitOk;
}

// trilist_main.cpp:227-245: canonical triangles, one "a b c" line each;
// --sorted sorts them lexicographically (on the device here).
int cmd_list(const Invocation& inv) {
  const CommonArgs& c = inv.c;
  const RunArgs& r = inv.r;
  Algorithm algo = parse_algorithm(r.algo);
  if (merge_layout_conflict(algo, r)) {
    std::fprintf(stderr, "error: --algo cf requires --local-order rank-asc\n");
    return kExitUsage;
  }
  double load_s = 0;
  LoadResult loaded = load_input(c, load_s);
  PreparedRun p = prepare(loaded.graph, r, algo, load_s);
  detail::validate(ParallelConfig{r.threads, r.chunk});
  detail::assert_layout(algo, p.oriented);
  if (!inv.list_sorted) return stream_list(c, p.oriented, algo);
  std::vector<std::uint32_t> tri;
  if (p.oriented.handle() && p.oriented.num_edges()) {
    tl_run_options o{};
    o.nparts = 1;
    o.algorithm = detail::algorithm_code(algo);
    tl_stats s;
    const int canonical = inv.list_sorted ? 1 : 0;
    check(tl_run_list(p.oriented.handle(), &o, nullptr, 0, canonical, &s), "list");
    tri.resize(3 * s.triangles);
    check(tl_run_list(p.oriented.handle(), &o, tri.data(), s.triangles, canonical, &s), "list");
  }
  std::string out;
  out.reserve(tri.size() / 3 * 24);
  for (std::size_t k = 0; k < tri.size(); k += 3) {
    Triangle t = canonical_triangle(tri[k], tri[k + 1], tri[k + 2]);
    append_uint(out, t.a);
    out += ' ';
    append_uint(out, t.b);
    out += ' ';
    append_uint(out, t.c);
    out += '\n';
  }
  return emit(c, out);
}

int cmd_verify(const Invocation& inv) {  // trilist_main.cpp:247-303
  const CommonArgs& c = inv.c;
  const RunArgs& r = inv.r;
  std::vector<Algorithm> algos;
  for (const std::string& n : inv.verify_algos) algos.push_back(parse_algorithm(n));
  for (Algorithm a : algos)
    if (merge_layout_conflict(a, r)) {
      std::fprintf(stderr, "error: --algos cf requires --local-order rank-asc\n");
      return kExitUsage;
    }
  LocalOrder local = r.local_order.empty() ? LocalOrder{} : parse_local_order(r.local_order);
  double load_s = 0;
  LoadResult loaded = load_input(c, load_s);
  const Graph& g = loaded.graph;
  RunOptions opt;
  opt.check_bitmap_between_pivots = true;
  opt.aot_skip_negative_phase = inv.fault == "drop-negative-phase";
  std::optional<std::vector<Triangle>> oracle;
  if (g.num_vertices() <= inv.oracle_cap) oracle = brute_force_triangles(g, {inv.oracle_cap});
  Json orders = Json::array();
  bool pass = true, consistent = true, have_first = false;
  std::uint64_t first_count = 0;
  for (const std::string& name : inv.verify_orders) {
    VertexOrder order = make_order(g, parse_order_spec(name));
    VerifyReport report = verify_equivalence(g, algos, order, local, oracle ? &*oracle : nullptr, opt);
    pass = pass && report.pass;
    if (!have_first) {
      first_count = report.reference_count;
      have_first = true;
    } else if (report.reference_count != first_count) {
      consistent = false;
    }
    Json e;
    e["order"] = name;
    e["report"] = to_json(report);
    orders.push_back(e);
  }
  pass = pass && consistent;
  Json doc = run_document("verify", c, loaded);
  Json names = Json::array();
  for (const std::string& n : inv.verify_algos) names.push_back(n);
  doc["algorithms"] = names;
  doc["local_order"] = to_string(local);
  doc["oracle_used"] = bool(oracle);
  doc["oracle_cap"] = inv.oracle_cap;
  if (oracle) doc["oracle_triangles"] = std::uint64_t(oracle->size());
  doc["orders"] = orders;
  doc["cross_order_consistent"] = consistent;
  doc["pass"] = pass;
  int code = emit_json(c, doc);
  if (code != kExitOk) return code;
  return pass ? kExitOk : kExitVerify;
}

int cmd_bench(const Invocation& inv) {  // trilist_main.cpp:305-333
  const CommonArgs& c = inv.c;
  const RunArgs& r = inv.r;
  BenchSettings settings;
  for (const std::string& n : inv.bench_algos) settings.algorithms.push_back(parse_algorithm(n));
  for (const std::string& n : inv.bench_orders) settings.orders.push_back(parse_order_spec(n));
  settings.local_order = r.local_order.empty() ? LocalOrder{} : parse_local_order(r.local_order);
  settings.thread_counts = inv.bench_threads.empty() ? std::vector<unsigned>{1} : inv.bench_threads;
  settings.chunk = r.chunk;
  settings.repeats = inv.bench_repeats;
  double load_s = 0;
  LoadResult loaded = load_input(c, load_s);
  std::vector<BenchRow> rows = run_bench(loaded.graph, c.input, settings, load_s);
  if (inv.bench_csv) return emit(c, bench_rows_to_csv(rows));
  Json arr = Json::array();
  for (const BenchRow& row : rows) arr.push_back(to_json(row));
  Json doc = run_document("bench", c, loaded);
  doc["repeats"] = inv.bench_repeats;
  doc["rows"] = arr;
  return emit_json(c, doc);
}

int cmd_stats(const Invocation& inv) {  // trilist_main.cpp:335-355
  const CommonArgs& c = inv.c;
  double load_s = 0;
  LoadResult loaded = load_input(c, load_s);
  OrderSpec spec = inv.r.order.empty() ? OrderSpec{} : parse_order_spec(inv.r.order);
  auto t0 = std::chrono::steady_clock::now();
  VertexOrder order = make_order(loaded.graph, spec);
  const double order_s = seconds_since(t0);
  t0 = std::chrono::steady_clock::now();
  OrientedGraph og = orient(loaded.graph, order);
  PhaseTimings timings{load_s, order_s, seconds_since(t0), 0};
  Json doc = run_document("stats", c, loaded);
  doc["order"] = to_string(spec);
  doc["max_out_degree"] = og.max_out_degree();
  doc["costs"] = to_json(cost_model(og));
  doc["timings"] = to_json(timings);
  return emit_json(c, doc);
}

}  // namespace

int main(int argc, char** argv) {
  Invocation inv;
  try {
    inv = parse_args(argc, argv);
  } catch (const HelpRequest& h) {
    std::fputs(h.text.c_str(), stdout);
    return kExitOk;
  } catch (const VersionRequest&) {
    std::printf("%s\n", kVersion);
    return kExitOk;
  } catch (const UsageError& e) {
    std::fprintf(stderr, "%s\nRun with --help for more information.\n", e.what());
    return kExitUsage;
  }
  try {
    if (inv.command == "count") return cmd_count(inv);
    if (inv.command == "list") return cmd_list(inv);
    if (inv.command == "verify") return cmd_verify(inv);
    if (inv.command == "bench") return cmd_bench(inv);
    if (inv.command == "stats") return cmd_stats(inv);
  } catch (const ParseError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitInput;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return kExitInput;
  }
  return kExitUsage;
}
