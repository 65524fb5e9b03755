// stream_sink_check -- a C++ caller of the drop-in facade with a custom sink.
//
// The reference's run_parallel<SinkFactory> (parallel.hpp:25-78) gives every
// worker its own sink (engine.hpp:125-134); oracle/ref_shim.cpp runs the
// reference itself with exactly this HashSink.  Here the same sink runs
// through trilist::run_parallel over the B200 facade, which streams the
// emissions from the device in bounded host batches.  Prints one JSON line:
// the triangle hash (count, sum, xor), the counters, the wall time and the
// process's peak resident set (VmHWM), so a test can check both the
// result (against the reference's golden hash) and the bounded host memory.
//
//   stream_sink_check <er|rmat|chung_lu> <seed> <n or scale> <npairs> [workers] [avg gamma]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <cstdlib>
#include <string>
#include <vector>

#include "trilist_b200.h"
#include "trilist_b200/trilist.hpp"

namespace {

std::uint64_t fmix64(std::uint64_t z) {  // ordering.cpp:16-18
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct HashSink {  // order-independent triangle hash
  std::uint64_t* acc;  // [count, sum, xor]
  void operator()(trilist::VertexId a, trilist::VertexId b, trilist::VertexId c) const {
    // Z(v) = fmix64(v + golden); sum of Z(a) Z(b) Z(c), xor of Z(a) & Z(b) & Z(c)
    const std::uint64_t za = fmix64(a + 0x9E3779B97F4A7C15ull), zb = fmix64(b + 0x9E3779B97F4A7C15ull),
                        zc = fmix64(c + 0x9E3779B97F4A7C15ull);
    acc[0] += 1;
    acc[1] += za * zb * zc;
    acc[2] ^= za & zb & zc;
  }
};

void cuda_ok(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    std::fprintf(stderr, "%s: %s\n", what, cudaGetErrorString(e));
    std::exit(2);
  }
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s <er|rmat|chung_lu> <seed> <n|scale> <npairs> [workers] [avg gamma]\n", argv[0]);
    return 2;
  }
  const std::string kind = argv[1];
  const std::uint64_t seed = std::strtoull(argv[2], nullptr, 10);
  const std::uint64_t size = std::strtoull(argv[3], nullptr, 10);
  const std::uint64_t npairs = std::strtoull(argv[4], nullptr, 10);
  const unsigned workers = argc > 5 ? unsigned(std::strtoul(argv[5], nullptr, 10)) : 8u;
  const double avg = argc > 6 ? std::atof(argv[6]) : 32.0, gamma = argc > 7 ? std::atof(argv[7]) : 2.1;

  std::uint32_t* d_pairs = nullptr;
  cuda_ok(cudaMalloc(&d_pairs, sizeof(std::uint32_t) * 2 * npairs), "cudaMalloc");
  std::uint32_t n = 0;
  int rc = 0;
  if (kind == "er") {
    n = std::uint32_t(size);
    rc = tl_gen_er(seed, n, npairs, d_pairs, nullptr);
  } else if (kind == "rmat") {
    n = std::uint32_t(1u << size);
    rc = tl_gen_rmat(seed, std::uint32_t(size), npairs, d_pairs, nullptr);
  } else {
    n = std::uint32_t(size);
    std::vector<std::uint64_t> prefix(std::uint64_t(n) + 1);
    rc = tl_chung_lu_prefix(seed, n, avg, gamma, prefix.data());
    if (rc == TL_OK) rc = tl_gen_chung_lu(seed, n, prefix.data(), npairs, d_pairs, nullptr);
  }
  if (rc != TL_OK) {
    std::fprintf(stderr, "generator: %s\n", tl_last_error());
    return 2;
  }
  cuda_ok(cudaDeviceSynchronize(), "generate");

  trilist::OrientedGraph og;
  {
    trilist::Graph g = trilist::Graph::from_device_pairs(n, d_pairs, npairs, 0);
    cuda_ok(cudaFree(d_pairs), "cudaFree");
    og = trilist::orient(g, trilist::degree_order(g));
  }

  struct alignas(64) Acc {  // one cache line per worker: no false sharing between the workers' sinks
    std::uint64_t v[3] = {0, 0, 0};
  };
  std::vector<Acc> accs(workers);
  const auto t0 = std::chrono::steady_clock::now();
  const trilist::RunStats s = trilist::run_parallel(
      trilist::Algorithm::aot, og, trilist::ParallelConfig{workers, 64},
      [&](unsigned w) { return HashSink{accs[w].v}; });
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::uint64_t c = 0, sum = 0, x = 0, busy = 0;
  for (auto& a : accs) {
    c += a.v[0];
    sum += a.v[1];
    x ^= a.v[2];
    busy += a.v[0] != 0;
  }
  // Peak resident set of THIS program: VmHWM (reset at exec), not
  // getrusage's ru_maxrss, which Linux carries over from the pre-exec image
  // of a forked parent (a large test runner would show up as ours).
  long hwm_kb = -1;
  {
    std::ifstream status("/proc/self/status");
    std::string line;
    while (std::getline(status, line)) {
      if (line.rfind("VmHWM:", 0) == 0) hwm_kb = std::strtol(line.c_str() + 6, nullptr, 10);
      if (line.rfind("VmHWM", 0) == 0 || line.rfind("VmRSS", 0) == 0 || line.rfind("RssAnon", 0) == 0 ||
          line.rfind("RssFile", 0) == 0 || line.rfind("RssShmem", 0) == 0)
        std::fprintf(stderr, "%s\n", line.c_str());
    }
  }
  std::printf(
      "{\"n\": %u, \"m\": %llu, \"hash_count\": %llu, \"hash_sum\": %llu, \"hash_xor\": %llu, \"triangles\": %llu, "
      "\"probes\": %llu, \"table_builds\": %llu, \"positive_triangles\": %llu, \"negative_triangles\": %llu, "
      "\"workers\": %u, \"workers_with_emissions\": %llu, \"wall_s\": %.3f, \"list_s\": %.3f, \"max_rss_kb\": %ld}\n",
      og.num_vertices(), (unsigned long long)og.num_edges(), (unsigned long long)c, (unsigned long long)sum,
      (unsigned long long)x, (unsigned long long)s.triangles, (unsigned long long)s.probes,
      (unsigned long long)s.table_builds, (unsigned long long)s.positive_triangles,
      (unsigned long long)s.negative_triangles, workers, (unsigned long long)busy, wall, s.wall_time_s,
      hwm_kb);
  return 0;
}
