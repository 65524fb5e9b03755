// tl_verify.cu -- verify_equivalence (engine.cpp:82-130) on the device.
//
// Every algorithm's emissions are canonicalised and sorted on the device
// (tl_run_list's canonical path); duplicates are counted with a device
// unique, and the set differences against the baseline (the oracle's set, or
// the first algorithm's) are device merges.  Only the counters and the first
// VerifyReport::kMaxSamples differences of each side come back to the host.
#include <thrust/execution_policy.h>
#include <thrust/set_operations.h>
#include <thrust/unique.h>

#include <cstring>

#include "tl_internal.cuh"

namespace tlb {

namespace {

struct Tri {
  uint32_t a, b, c;
};
struct TriLess {
  __host__ __device__ bool operator()(const Tri& x, const Tri& y) const {
    return x.a != y.a ? x.a < y.a : (x.b != y.b ? x.b < y.b : x.c < y.c);
  }
};
struct TriEq {
  __host__ __device__ bool operator()(const Tri& x, const Tri& y) const {
    return x.a == y.a && x.b == y.b && x.c == y.c;
  }
};
static_assert(sizeof(Tri) == 12, "triple layout");

// Sorted canonical list (duplicates kept) of one run; returns its length.
uint64_t canonical_list(tl_oriented& og, const RunSpec& base, DBuf<uint32_t>& out, cudaStream_t s, AotResult& r) {
  RunSpec sp = base;
  sp.mode = AotMode::count;
  const AotResult c = aot_run(og, sp, s, nullptr, 0);
  const uint64_t T = c.triangles;
  out.alloc(std::max<uint64_t>(3 * T, 3), s);
  sp.mode = AotMode::list;
  r = aot_run(og, sp, s, out.p, T);
  TL_REQUIRE(r.emitted == T && r.triangles == T, TL_ELOGIC, "listing run disagrees with its counting run");
  if (T) {
    canonicalize_triples(out.p, T, s);
    sort_triples(out.p, T, og.nb, s);
  }
  return T;
}

// |a \ b| for sorted unique lists, plus its first `cap` elements.
uint64_t difference(const Tri* a, uint64_t na, const Tri* b, uint64_t nb, cudaStream_t s, uint32_t* samples,
                    uint32_t cap) {
  if (na == 0) return 0;
  DBuf<uint32_t> diff;
  diff.alloc(3 * na, s);
  Tri* d = reinterpret_cast<Tri*>(diff.p);
  Tri* end = thrust::set_difference(thrust::cuda::par.on(s), a, a + na, b, b + nb, d, TriLess());
  const uint64_t k = uint64_t(end - d);
  if (samples && k) {
    const uint64_t ns = std::min<uint64_t>(k, cap);
    TL_CUDA(cudaMemcpyAsync(samples, diff.p, sizeof(uint32_t) * 3 * ns, cudaMemcpyDeviceToHost, s));
  }
  TL_CUDA(cudaStreamSynchronize(s));
  return k;
}

}  // namespace

void verify_algorithms(tl_oriented& og, const uint32_t* algos, uint32_t nalgos, const RunSpec& base,
                       const uint32_t* h_reference, uint64_t nreference, bool have_reference, cudaStream_t s,
                       tl_verify_result* results, uint64_t* reference_count) {
  DBuf<uint32_t> baseline;
  uint64_t nb = 0;
  bool have_baseline = false;
  if (have_reference) {  // engine.cpp:94-100: the oracle set, sorted and unique
    baseline.alloc(std::max<uint64_t>(3 * nreference, 3), s);
    if (nreference) {
      TL_CUDA(cudaMemcpyAsync(baseline.p, h_reference, sizeof(uint32_t) * 3 * nreference, cudaMemcpyHostToDevice,
                              s));
      sort_triples(baseline.p, nreference, og.nb, s);
      Tri* t = reinterpret_cast<Tri*>(baseline.p);
      nb = uint64_t(thrust::unique(thrust::cuda::par.on(s), t, t + nreference, TriEq()) - t);
    }
    have_baseline = true;
  }
  for (uint32_t i = 0; i < nalgos; ++i) {
    tl_verify_result& res = results[i];
    std::memset(&res, 0, sizeof(res));
    res.algorithm = algos[i];
    RunSpec sp = base;
    sp.algo = static_cast<Algo>(algos[i]);
    DBuf<uint32_t> list;
    AotResult r;
    const uint64_t T = canonical_list(og, sp, list, s, r);
    Tri* t = reinterpret_cast<Tri*>(list.p);
    const uint64_t u = T ? uint64_t(thrust::unique(thrust::cuda::par.on(s), t, t + T, TriEq()) - t) : 0;
    res.unique_triangles = u;
    res.duplicate_emissions = T - u;
    fill_stats_from(r, &res.stats);
    if (!have_baseline) {  // engine.cpp:113-116: the first algorithm anchors the comparison
      baseline = std::move(list);
      nb = u;
      have_baseline = true;
      res.missing_count = res.extra_count = 0;
    } else {
      const Tri* b = reinterpret_cast<const Tri*>(baseline.p);
      res.missing_count = difference(b, nb, t, u, s, res.missing_samples, TL_VERIFY_SAMPLES);
      res.extra_count = difference(t, u, b, nb, s, res.extra_samples, TL_VERIFY_SAMPLES);
    }
    res.n_missing_samples = uint32_t(std::min<uint64_t>(res.missing_count, TL_VERIFY_SAMPLES));
    res.n_extra_samples = uint32_t(std::min<uint64_t>(res.extra_count, TL_VERIFY_SAMPLES));
    res.pass = res.duplicate_emissions == 0 && res.missing_count == 0 && res.extra_count == 0;
    TL_CUDA(cudaStreamSynchronize(s));
  }
  if (reference_count) *reference_count = nb;
}

}  // namespace tlb
