// report.hpp -- the reference's reporting layer (proj/include/trilist/report.hpp,
// src/report.cpp) over the B200 facade: phase timings, the benchmark cross
// product and its JSON/CSV rows.  The reference builds its documents with
// nlohmann::json (an ordered std::map per object); Json below is a small
// value type with the same output: keys in sorted order, dump(-1) compact,
// dump(2) indented, integers exact, doubles in shortest round-trip form.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include "trilist_b200/trilist.hpp"

namespace trilist {

class Json {
 public:
  using Array = std::vector<Json>;
  using Object = std::map<std::string, Json>;

  Json() : v_(nullptr) {}
  Json(std::nullptr_t) : v_(nullptr) {}
  Json(bool b) : v_(b) {}
  Json(int x) : v_(std::int64_t(x)) {}
  Json(long x) : v_(std::int64_t(x)) {}
  Json(long long x) : v_(std::int64_t(x)) {}
  Json(unsigned x) : v_(std::uint64_t(x)) {}
  Json(unsigned long x) : v_(std::uint64_t(x)) {}
  Json(unsigned long long x) : v_(std::uint64_t(x)) {}
  Json(double d) : v_(d) {}
  Json(const char* s) : v_(std::string(s)) {}
  Json(std::string s) : v_(std::move(s)) {}
  Json(Array a) : v_(std::make_shared<Array>(std::move(a))) {}
  Json(Object o) : v_(std::make_shared<Object>(std::move(o))) {}

  // value semantics: copies are deep
  Json(const Json& o) : v_(nullptr) { *this = o; }
  Json& operator=(const Json& o);
  Json(Json&&) noexcept = default;
  Json& operator=(Json&&) noexcept = default;

  static Json array() { return Json(Array{}); }
  static Json object() { return Json(Object{}); }

  Json& operator[](const std::string& key);  // object member (creates; null -> object)
  void push_back(Json x);                    // array append (null -> array)
  std::size_t size() const;

  /// nlohmann-compatible text: indent < 0 compact, else pretty with `indent` spaces.
  std::string dump(int indent = -1) const;

 private:
  void write(std::string& out, int indent, int depth) const;
  std::variant<std::nullptr_t, bool, std::int64_t, std::uint64_t, double, std::string, std::shared_ptr<Array>,
               std::shared_ptr<Object>>
      v_;
};

/// Version stamp carried by every JSON document (report.hpp:14).
inline constexpr int kSchemaVersion = 1;

struct PhaseTimings {  // report.hpp:16-21
  double load_s = 0;
  double order_s = 0;
  double orient_s = 0;
  double list_s = 0;
};

/// One benchmark cell: algorithm x order x worker count on one dataset (report.hpp:23-40).
struct BenchRow {
  std::string dataset;
  VertexId n = 0;
  EdgeCount m = 0;
  std::string algorithm;
  std::string order;
  std::string local_order;
  unsigned workers = 1;
  VertexId chunk = 64;
  unsigned repeats = 1;
  RunStats stats;
  std::vector<double> list_times_s;
  double median_list_s = 0;
  PhaseTimings timings;
  CostModel costs;
};

Json to_json(const RunStats& s);
Json to_json(const CostModel& c);
Json to_json(const LoadDiagnostics& d);
Json to_json(const PhaseTimings& t);
Json to_json(const BenchRow& row);
Json to_json(const VerifyReport& report);

std::string bench_rows_to_csv(const std::vector<BenchRow>& rows);

struct BenchSettings {  // report.hpp:50-58
  std::vector<Algorithm> algorithms;
  std::vector<OrderSpec> orders;
  LocalOrder local_order;
  std::vector<unsigned> thread_counts = {1};
  VertexId chunk = 64;
  unsigned repeats = 1;
  RunOptions run_options;
};

/// Runs the full cross product (report.cpp:114-164); counters must repeat
/// exactly across repeats, else std::logic_error.
std::vector<BenchRow> run_bench(const Graph& g, const std::string& dataset, const BenchSettings& settings,
                                double load_seconds);

}  // namespace trilist
