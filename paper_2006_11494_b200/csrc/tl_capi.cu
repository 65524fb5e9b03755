// tl_capi.cu -- the extern "C" boundary (include/trilist_b200.h).
//
// Each entry point validates its arguments, maps failures onto TL_E* codes
// (the reference's exception types) with a thread-local message,
// and dispatches to the device pipeline.  There is no CPU fallback: without a
// CUDA device every compute entry point fails with TL_ENODEV.
#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "tl_internal.cuh"

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return TL_OK;
  } catch (const tlb::TlError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc& e) {
    g_last_error = std::string("host allocation failed: ") + e.what();
    return TL_ENOMEM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TL_ECUDA;
  }
}

void require_device(int device) {
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    throw tlb::TlError(TL_ENODEV, std::string("no CUDA device available for the B200 trilist path") +
                                      (e != cudaSuccess ? std::string(" (") + cudaGetErrorString(e) + ")" : ""));
  }
  TL_REQUIRE(device >= 0 && device < count, TL_EINVAL, "device index " + std::to_string(device) + " out of range");
}

cudaStream_t pick_stream(void* user, cudaStream_t own) { return user ? static_cast<cudaStream_t>(user) : own; }

tl_run_options defaults() {
  tl_run_options o;
  std::memset(&o, 0, sizeof(o));
  o.nparts = 1;
  return o;
}

}  // namespace

namespace tlb {

void set_last_error(const std::string& msg) { g_last_error = msg; }

void fill_stats_from(const AotResult& r, tl_stats* st) {
  if (!st) return;
  std::memset(st, 0, sizeof(*st));
  st->triangles = r.triangles;
  st->probes = r.probes;
  st->merge_comparisons = r.merge_comparisons;
  st->table_builds = r.table_builds;
  st->positive_triangles = r.report_positive;
  st->negative_triangles = r.report_negative;
  st->probes_executed = r.executed;
  st->hash_sum = r.hash_sum;
  st->hash_xor = r.hash_xor;
  st->tasks = r.tasks;
  st->list_ms = r.list_ms;
  st->prep_ms = r.prep_ms;
  st->kernel_launches = r.launches;
}

void ensure_device_setup(int device) {
  static std::mutex mu;
  static bool done[64] = {false};
  std::lock_guard<std::mutex> lock(mu);
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    // keep freed blocks cached across calls (per-run task buffers, an e2e
    // upload's working set), but never more than a quarter of the device:
    // at each synchronisation the pool releases what it holds beyond that,
    // so orient()'s m-sized sort temporaries go back to the device and a
    // PyTorch allocator in the same process still sees them as free.
    size_t free_b = 0, total_b = 0;
    uint64_t threshold = 16ull << 30;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess && total_b) threshold = total_b / 4;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
  }
  cudaGetLastError();
  done[device] = true;
}

}  // namespace tlb

tl_graph::~tl_graph() {
  keys.reset();
  deg.reset();
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

tl_oriented::~tl_oriented() {
  off.reset();
  col.reset();
  orig.reset();
  rank.reset();
  claim_off.reset();
  win.reset();
  claim_s.reset();
  vword.reset();
  fwd_win.reset();  // every buffer is freed on its stream before the stream goes
  cp.reset();
  plans.clear();
  if (aux) {
    cudaStreamSynchronize(aux);
    cudaStreamDestroy(aux);
  }
  if (stream) {
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

extern "C" {

const char* tl_last_error(void) { return g_last_error.c_str(); }

const char* tl_version(void) { return "trilist-b200 0.1.0 (sm_100a)"; }

int tl_device_count(int* count) {
  return guarded([&] {
    TL_REQUIRE(count, TL_EINVAL, "count is NULL");
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

// ------------------------------------------------------------- generators
static int gen_common(void* stream, uint32_t* d_pairs, const char* what) {
  (void)stream;
  (void)what;
  TL_REQUIRE(d_pairs, TL_EINVAL, "d_pairs is NULL");
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  require_device(dev);
  return dev;
}

int tl_gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint32_t* d_pairs, void* stream) {
  return guarded([&] {
    gen_common(stream, d_pairs, "er");
    tlb::gen_er(seed, n, npairs, d_pairs, static_cast<cudaStream_t>(stream));
  });
}

int tl_gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint32_t* d_pairs, void* stream) {
  return guarded([&] {
    gen_common(stream, d_pairs, "rmat");
    tlb::gen_rmat(seed, scale, npairs, d_pairs, static_cast<cudaStream_t>(stream));
  });
}

int tl_chung_lu_prefix(uint64_t seed, uint32_t n, double avg, double gamma, uint64_t* prefix) {
  return guarded([&] {
    TL_REQUIRE(prefix, TL_EINVAL, "prefix is NULL");
    TL_REQUIRE(gamma > 1.0 && avg > 0.0, TL_EINVAL, "Chung-Lu needs gamma > 1 and avg > 0");
    tlb::chung_lu_prefix_host(seed, n, avg, gamma, prefix);
  });
}

int tl_gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs, uint32_t* d_pairs,
                    void* stream) {
  return guarded([&] {
    TL_REQUIRE(prefix, TL_EINVAL, "prefix is NULL");
    gen_common(stream, d_pairs, "chung_lu");
    tlb::gen_chung_lu(seed, n, prefix, npairs, d_pairs, static_cast<cudaStream_t>(stream));
  });
}

// ------------------------------------------------------------- graph core
int tl_graph_from_pairs(const uint32_t* pairs, uint64_t npairs, uint32_t min_vertices, int device,
                        int pairs_on_device, void* stream, tl_graph** out) {
  return guarded([&] {
    TL_REQUIRE(out, TL_EINVAL, "out is NULL");
    TL_REQUIRE(pairs || npairs == 0, TL_EINVAL, "pairs is NULL");
    *out = nullptr;
    require_device(device);
    tlb::DeviceGuard guard(device);
    tlb::ensure_device_setup(device);
    auto g = std::make_unique<tl_graph>();
    g->device = device;
    TL_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    cudaStream_t s = g->stream;
    if (stream) {  // order after the caller's stream (inputs may be produced there)
      cudaEvent_t ev;
      TL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      TL_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
      TL_CUDA(cudaStreamWaitEvent(s, ev, 0));
      cudaEventDestroy(ev);
    }
    tlb::DBuf<uint32_t> staged;
    const uint32_t* d_pairs = pairs;
    if (!pairs_on_device && npairs) {
      staged.alloc(2 * npairs, s);
      TL_CUDA(cudaMemcpyAsync(staged.p, pairs, sizeof(uint32_t) * 2 * npairs, cudaMemcpyHostToDevice, s));
      d_pairs = staged.p;
    }
    tlb::graph_from_pairs(*g, d_pairs, npairs, min_vertices);
    TL_CUDA(cudaStreamSynchronize(s));
    *out = g.release();
  });
}

static int load_common(const char* text, uint64_t len, uint32_t flags, const char* comments, int device,
                       tl_graph** out, tl_load_diag* diag, uint64_t* error_line, const std::string* owned) {
  (void)owned;
  try {
    TL_REQUIRE(out, TL_EINVAL, "out is NULL");
    TL_REQUIRE(text || len == 0, TL_EINVAL, "text is NULL");
    *out = nullptr;
    if (error_line) *error_line = 0;
    require_device(device);
    tlb::DeviceGuard guard(device);
    tlb::ensure_device_setup(device);
    auto g = std::make_unique<tl_graph>();
    g->device = device;
    TL_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    tlb::graph_from_text(*g, text, len, flags, comments, diag);
    *out = g.release();
    return TL_OK;
  } catch (const tlb::ParseFailure& e) {
    g_last_error = e.what();
    if (error_line) *error_line = e.line;
    return TL_EPARSE;
  } catch (const tlb::TlError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TL_ECUDA;
  }
}

int tl_graph_from_text(const char* text, uint64_t len, uint32_t flags, const char* comment_prefixes, int device,
                       tl_graph** out, tl_load_diag* diag, uint64_t* error_line) {
  return load_common(text, len, flags, comment_prefixes, device, out, diag, error_line, nullptr);
}

int tl_graph_from_file(const char* path, uint32_t flags, const char* comment_prefixes, int device, tl_graph** out,
                       tl_load_diag* diag, uint64_t* error_line) {
  std::string text;
  const int rc = guarded([&] {
    TL_REQUIRE(path, TL_EINVAL, "path is NULL");
    text = tlb::read_text_file(path);
  });
  if (rc != TL_OK) return rc;
  return load_common(text.data(), text.size(), flags, comment_prefixes, device, out, diag, error_line, &text);
}

int tl_graph_free(tl_graph* g) {
  return guarded([&] {
    if (!g) return;
    tlb::DeviceGuard guard(g->device);
    delete g;
  });
}

int tl_graph_info(const tl_graph* g, uint32_t* n, uint64_t* m, uint64_t* duplicates, uint64_t* self_loops) {
  return guarded([&] {
    TL_REQUIRE(g, TL_EINVAL, "graph is NULL");
    if (n) *n = g->n;
    if (m) *m = g->m;
    if (duplicates) *duplicates = g->duplicates;
    if (self_loops) *self_loops = g->self_loops;
  });
}

int tl_graph_degrees(tl_graph* g, uint32_t* degrees) {
  return guarded([&] {
    TL_REQUIRE(g && degrees, TL_EINVAL, "NULL argument");
    tlb::DeviceGuard guard(g->device);
    if (g->n)
      TL_CUDA(cudaMemcpyAsync(degrees, g->deg.p, sizeof(uint32_t) * g->n, cudaMemcpyDeviceToHost, g->stream));
    TL_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int tl_graph_csr(tl_graph* g, uint64_t* offsets, uint32_t* adjacency) {
  return guarded([&] {
    TL_REQUIRE(g, TL_EINVAL, "graph is NULL");
    tlb::DeviceGuard guard(g->device);
    tlb::DBuf<uint64_t> off;
    tlb::DBuf<uint32_t> adj;
    tlb::graph_csr(*g, off, adj);
    if (offsets)
      TL_CUDA(cudaMemcpyAsync(offsets, off.p, sizeof(uint64_t) * (uint64_t(g->n) + 1), cudaMemcpyDeviceToHost,
                              g->stream));
    if (adjacency && g->m)
      TL_CUDA(cudaMemcpyAsync(adjacency, adj.p, sizeof(uint32_t) * 2 * g->m, cudaMemcpyDeviceToHost, g->stream));
    TL_CUDA(cudaStreamSynchronize(g->stream));
  });
}

// ------------------------------------------------------------- ordering
int tl_degree_order(tl_graph* g, uint32_t* rank) {
  return guarded([&] {
    TL_REQUIRE(g && rank, TL_EINVAL, "NULL argument");
    tlb::DeviceGuard guard(g->device);
    tlb::DBuf<uint32_t> d_rank;
    tlb::degree_order(*g, d_rank);
    if (g->n) TL_CUDA(cudaMemcpyAsync(rank, d_rank.p, sizeof(uint32_t) * g->n, cudaMemcpyDeviceToHost, g->stream));
    TL_CUDA(cudaStreamSynchronize(g->stream));
  });
}

int tl_orient(tl_graph* g, const uint32_t* rank, tl_oriented** out) {
  return guarded([&] {
    TL_REQUIRE(g && out, TL_EINVAL, "NULL argument");
    *out = nullptr;
    tlb::DeviceGuard guard(g->device);
    auto og = std::make_unique<tl_oriented>();
    og->device = g->device;
    TL_CUDA(cudaStreamCreateWithFlags(&og->stream, cudaStreamNonBlocking));
    // the graph's work is complete (every graph call synchronises), so the
    // oriented graph's stream may read its buffers directly
    cudaStream_t s = og->stream;
    tlb::DBuf<uint32_t> d_rank;
    if (rank) {
      d_rank.alloc(std::max<uint64_t>(g->n, 1), s);
      if (g->n) TL_CUDA(cudaMemcpyAsync(d_rank.p, rank, sizeof(uint32_t) * g->n, cudaMemcpyHostToDevice, s));
      TL_REQUIRE(tlb::is_permutation(d_rank.p, g->n, s), TL_EINVAL, "order is not a permutation of the vertex set");
    } else {
      cudaStream_t keep = g->stream;
      g->stream = s;  // run the degree order on the new stream
      try {
        tlb::degree_order(*g, d_rank);
      } catch (...) {
        g->stream = keep;
        throw;
      }
      g->stream = keep;
    }
    tlb::orient(*g, d_rank.p, *og);
    TL_CUDA(cudaStreamSynchronize(s));
    *out = og.release();
  });
}

int tl_oriented_from_csr(uint32_t n, uint64_t m, const uint64_t* out_offsets, const uint32_t* out,
                         const uint32_t* rank, int device, void* stream, tl_oriented** out_graph) {
  return guarded([&] {
    TL_REQUIRE(out_graph && out_offsets && rank && (out || m == 0), TL_EINVAL, "NULL argument");
    *out_graph = nullptr;
    require_device(device);
    tlb::DeviceGuard guard(device);
    tlb::ensure_device_setup(device);
    auto og = std::make_unique<tl_oriented>();
    og->device = device;
    TL_CUDA(cudaStreamCreateWithFlags(&og->stream, cudaStreamNonBlocking));
    cudaStream_t s = og->stream;
    if (stream) {
      cudaEvent_t ev;
      TL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      TL_CUDA(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
      TL_CUDA(cudaStreamWaitEvent(s, ev, 0));
      cudaEventDestroy(ev);
    }
    tlb::oriented_from_host_csr(*og, n, m, out_offsets, out, rank);
    TL_CUDA(cudaStreamSynchronize(s));
    *out_graph = og.release();
  });
}

int tl_oriented_free(tl_oriented* og) {
  return guarded([&] {
    if (!og) return;
    tlb::DeviceGuard guard(og->device);
    delete og;
  });
}

int tl_oriented_info(const tl_oriented* og, uint32_t* n, uint64_t* m, uint32_t* max_out_degree) {
  return guarded([&] {
    TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
    if (n) *n = og->n;
    if (m) *m = og->m;
    if (max_out_degree) *max_out_degree = og->max_out_degree;
  });
}

int tl_oriented_csr(tl_oriented* og, uint64_t* out_offsets, uint32_t* out, uint64_t* in_offsets, uint32_t* in,
                    uint32_t* rank) {
  return guarded([&] {
    TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
    tlb::DeviceGuard guard(og->device);
    tlb::oriented_download(*og, out_offsets, out, in_offsets, in, rank);
  });
}

int tl_cost_model(tl_oriented* og, uint64_t* costs) {
  return guarded([&] {
    TL_REQUIRE(og && costs, TL_EINVAL, "NULL argument");
    costs[0] = og->cost[0];
    costs[1] = og->cost[1];
    costs[2] = og->cost[2];
  });
}

// ------------------------------------------------------------- listing
static tlb::RunSpec spec_of(const tl_run_options& o, tlb::AotMode mode, bool any_algorithm) {
  tlb::RunSpec sp;
  if (any_algorithm) {
    TL_REQUIRE(o.algorithm <= TL_ALGO_KCLIST3, TL_EINVAL,
               "unknown algorithm " + std::to_string(o.algorithm) + " (expected TL_ALGO_*)");
    sp.algo = static_cast<tlb::Algo>(o.algorithm);
  }
  sp.mode = mode;
  sp.skip_negative = o.skip_negative_phase != 0;
  sp.reuse = o.cf_hash_reuse_last_table != 0;
  sp.part = o.part;
  sp.nparts = o.nparts ? o.nparts : 1;
  TL_REQUIRE(sp.part < sp.nparts, TL_EINVAL, "part must be < nparts");
  return sp;
}

static std::tuple<uint32_t, uint32_t, uint32_t, uint32_t> cache_key(const tlb::RunSpec& sp) {
  return {uint32_t(sp.algo), uint32_t(sp.algo == tlb::Algo::aot && sp.skip_negative), sp.part, sp.nparts};
}

static void run_checked(tl_oriented* og, const tl_run_options* opt, tlb::AotMode mode, bool any_algorithm,
                        tl_stats* stats) {
  TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
  tl_run_options o = opt ? *opt : defaults();
  tlb::RunSpec sp = spec_of(o, mode, any_algorithm);
  tlb::DeviceGuard guard(og->device);
  tlb::AotResult r = tlb::aot_run(*og, sp, pick_stream(o.stream, og->stream), nullptr, 0);
  og->tri_cache[cache_key(sp)] = r.triangles;
  tlb::fill_stats_from(r, stats);
}

// The emission count of a run (sizes the output): cached per orientation and
// claim set, else one counting pass, whose stats are returned in *counted.
static uint64_t emission_count(tl_oriented* og, const tlb::RunSpec& count_spec, cudaStream_t s,
                               tlb::AotResult* counted) {
  auto key = cache_key(count_spec);
  auto it = og->tri_cache.find(key);
  if (it != og->tri_cache.end() && !counted) return it->second;
  tlb::AotResult c = tlb::aot_run(*og, count_spec, s, nullptr, 0);
  og->tri_cache[key] = c.triangles;
  if (counted) *counted = c;
  return c.triangles;
}

// One listing pass into device memory d_out (cap triples), canonicalised and
// sorted when asked.  Returns the emission count; TL_ECAPACITY (stats still
// filled) when it exceeds cap.
static uint64_t list_into(tl_oriented* og, tlb::RunSpec sp, cudaStream_t s, uint32_t* d_out, uint64_t cap,
                          int canonical, tl_stats* stats) {
  sp.mode = tlb::AotMode::list;
  tlb::AotResult r = tlb::aot_run(*og, sp, s, d_out, cap);
  const uint64_t T = r.emitted;
  TL_REQUIRE(T == r.triangles, TL_ELOGIC, "emission count disagrees with the triangle counters");
  tlb::fill_stats_from(r, stats);
  sp.mode = tlb::AotMode::count;
  og->tri_cache[cache_key(sp)] = T;
  if (T > cap) {
    TL_CUDA(cudaStreamSynchronize(s));
    throw tlb::TlError(TL_ECAPACITY, "output capacity " + std::to_string(cap) + " < " + std::to_string(T) +
                                         " triangles");
  }
  if (canonical && T) {
    tlb::canonicalize_triples(d_out, T, s);
    tlb::sort_triples(d_out, T, og->nb, s);
  }
  return T;
}

static void list_checked(tl_oriented* og, const tl_run_options* opt, bool any_algorithm, uint32_t* triples,
                         uint64_t cap, int canonical, tl_stats* stats) {
  TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
  tl_run_options o = opt ? *opt : defaults();
  tlb::RunSpec sp = spec_of(o, tlb::AotMode::count, any_algorithm);
  tlb::DeviceGuard guard(og->device);
  cudaStream_t s = pick_stream(o.stream, og->stream);
  if (!triples) {  // only count (trilist_b200.h): one counting pass, cached for the sizing call
    tlb::AotResult c;
    emission_count(og, sp, s, &c);
    tlb::fill_stats_from(c, stats);
    return;
  }
  const uint64_t expect = emission_count(og, sp, s, nullptr);
  if (cap < expect)
    throw tlb::TlError(TL_ECAPACITY, "output capacity " + std::to_string(cap) + " < " + std::to_string(expect) +
                                         " triangles");
  tlb::DBuf<uint32_t> d_out;
  d_out.alloc(std::max<uint64_t>(3 * expect, 3), s);
  const uint64_t T = list_into(og, sp, s, d_out.p, expect, canonical, stats);
  if (T) TL_CUDA(cudaMemcpyAsync(triples, d_out.p, sizeof(uint32_t) * 3 * T, cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
}

static void list_device_checked(tl_oriented* og, const tl_run_options* opt, uint32_t* d_triples, uint64_t cap,
                                int canonical, tl_stats* stats) {
  TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
  TL_REQUIRE(d_triples || cap == 0, TL_EINVAL, "d_triples is NULL");
  tl_run_options o = opt ? *opt : defaults();
  tlb::RunSpec sp = spec_of(o, tlb::AotMode::count, true);
  tlb::DeviceGuard guard(og->device);
  cudaStream_t s = pick_stream(o.stream, og->stream);
  list_into(og, sp, s, d_triples, cap, canonical, stats);
  TL_CUDA(cudaStreamSynchronize(s));
}

int tl_aot_count(tl_oriented* og, const tl_run_options* opt, tl_stats* stats) {
  return guarded([&] { run_checked(og, opt, tlb::AotMode::count, false, stats); });
}

int tl_aot_hash(tl_oriented* og, const tl_run_options* opt, tl_stats* stats) {
  return guarded([&] { run_checked(og, opt, tlb::AotMode::hash, false, stats); });
}

int tl_aot_list(tl_oriented* og, const tl_run_options* opt, uint32_t* triples, uint64_t cap, int canonical,
                tl_stats* stats) {
  return guarded([&] { list_checked(og, opt, false, triples, cap, canonical, stats); });
}

int tl_run_count(tl_oriented* og, const tl_run_options* opt, tl_stats* stats) {
  return guarded([&] { run_checked(og, opt, tlb::AotMode::count, true, stats); });
}

int tl_run_hash(tl_oriented* og, const tl_run_options* opt, tl_stats* stats) {
  return guarded([&] { run_checked(og, opt, tlb::AotMode::hash, true, stats); });
}

int tl_run_list(tl_oriented* og, const tl_run_options* opt, uint32_t* triples, uint64_t cap, int canonical,
                tl_stats* stats) {
  return guarded([&] { list_checked(og, opt, true, triples, cap, canonical, stats); });
}

int tl_run_list_batches(tl_oriented* og, const tl_run_options* opt, uint64_t batch_triples, uint32_t host_buffers,
                        tl_batch_fn fn, void* user, tl_stats* stats) {
  return guarded([&] {
    TL_REQUIRE(og, TL_EINVAL, "oriented graph is NULL");
    tl_run_options o = opt ? *opt : defaults();
    tlb::RunSpec sp = spec_of(o, tlb::AotMode::list, true);
    tlb::DeviceGuard guard(og->device);
    tlb::AotResult r = tlb::list_batches(*og, sp, pick_stream(o.stream, og->stream), batch_triples, host_buffers, fn,
                                         user);
    tlb::fill_stats_from(r, stats);
  });
}

int tl_run_list_device(tl_oriented* og, const tl_run_options* opt, uint32_t* d_triples, uint64_t cap, int canonical,
                       tl_stats* stats) {
  return guarded([&] { list_device_checked(og, opt, d_triples, cap, canonical, stats); });
}

int tl_verify(tl_oriented* og, const uint32_t* algorithms, uint32_t nalgos, const tl_run_options* opt,
              const uint32_t* reference, uint64_t nreference, int have_reference, tl_verify_result* results,
              uint64_t* reference_count) {
  return guarded([&] {
    TL_REQUIRE(og && (algorithms || nalgos == 0) && (results || nalgos == 0), TL_EINVAL, "NULL argument");
    TL_REQUIRE(!have_reference || reference || nreference == 0, TL_EINVAL, "NULL reference");
    for (uint32_t i = 0; i < nalgos; ++i)
      TL_REQUIRE(algorithms[i] <= TL_ALGO_KCLIST3, TL_EINVAL, "unknown algorithm " + std::to_string(algorithms[i]));
    tl_run_options o = opt ? *opt : defaults();
    o.algorithm = 0;
    o.part = 0;
    o.nparts = 1;
    tlb::RunSpec sp = spec_of(o, tlb::AotMode::count, true);
    tlb::DeviceGuard guard(og->device);
    tlb::verify_algorithms(*og, algorithms, nalgos, sp, reference, nreference, have_reference != 0,
                           pick_stream(o.stream, og->stream), results, reference_count);
  });
}

// ------------------------------------------------------ sequential orders
int tl_degeneracy_order(tl_graph* g, uint32_t* rank) {
  return guarded([&] {
    TL_REQUIRE(g && (rank || g->n == 0), TL_EINVAL, "NULL argument");
    tlb::DeviceGuard guard(g->device);
    const uint32_t n = g->n;
    std::vector<uint64_t> off(uint64_t(n) + 1);
    std::vector<uint32_t> adj(2 * g->m);
    {
      tlb::DBuf<uint64_t> d_off;
      tlb::DBuf<uint32_t> d_adj;
      tlb::graph_csr(*g, d_off, d_adj);
      TL_CUDA(cudaMemcpyAsync(off.data(), d_off.p, sizeof(uint64_t) * off.size(), cudaMemcpyDeviceToHost, g->stream));
      if (g->m)
        TL_CUDA(cudaMemcpyAsync(adj.data(), d_adj.p, sizeof(uint32_t) * adj.size(), cudaMemcpyDeviceToHost,
                                g->stream));
      TL_CUDA(cudaStreamSynchronize(g->stream));
    }
    tlb::degeneracy_order_host(n, off.data(), adj.data(), rank);
  });
}

int tl_random_order(uint32_t n, uint64_t seed, uint32_t* rank) {
  return guarded([&] {
    TL_REQUIRE(rank || n == 0, TL_EINVAL, "NULL argument");
    tlb::random_order_host(n, seed, rank);
  });
}

int tl_brute_force(tl_graph* g, uint32_t max_vertices, uint32_t* triples, uint64_t cap, uint64_t* count) {
  return guarded([&] {
    TL_REQUIRE(g && count, TL_EINVAL, "NULL argument");
    TL_REQUIRE(g->n <= max_vertices, TL_EINVAL,
               "oracle refuses graphs larger than " + std::to_string(max_vertices) + " vertices");
    tlb::DeviceGuard guard(g->device);
    tlb::DBuf<uint32_t> out;
    uint64_t T = tlb::brute_force(*g, out);
    *count = T;
    if (triples) {
      TL_REQUIRE(cap >= T, TL_ECAPACITY, "output capacity too small");
      if (T) TL_CUDA(cudaMemcpyAsync(triples, out.p, sizeof(uint32_t) * 3 * T, cudaMemcpyDeviceToHost, g->stream));
    }
    TL_CUDA(cudaStreamSynchronize(g->stream));
  });
}

}  // extern "C"
