// tl_common.cuh -- shared device/host helpers for the B200 trilist path.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "trilist_b200.h"

namespace tlb {

// ---------------------------------------------------------------------------
// errors: every C-ABI entry point catches TlError and returns its code
// ---------------------------------------------------------------------------
struct TlError : std::runtime_error {
  int code;
  TlError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TL_CUDA(x)                                                                        \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess)                                                                \
      throw ::tlb::TlError(TL_ECUDA, std::string(#x) + " failed: " + cudaGetErrorString(e_) + \
                                         " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define TL_REQUIRE(cond, code, msg)                     \
  do {                                                  \
    if (!(cond)) throw ::tlb::TlError((code), (msg));   \
  } while (0)

// ---------------------------------------------------------------------------
// splitmix64 finaliser (reference ordering.cpp:13-19) and derived functions
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// k-th (0-based) output of the sequential splitmix64 seeded with `seed`.
__host__ __device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t k) {
  return fmix64(seed + (k + 1) * kGolden);
}

// Order-independent triangle hash, round 2.  Every
// vertex has a 64-bit word Z(v) = fmix64(v + golden) of its ORIGINAL id; a
// triangle {a, b, c} contributes
//     Z(a) * Z(b) * Z(c)  (mod 2^64)  to hash_sum   and
//     Z(a) & Z(b) & Z(c)              to hash_xor,
// both symmetric in the three ids (no canonical order needed) and both
// distributive over their accumulation (+ resp. ^): the hits w of one claim
// (l, s) add up to Z(l) Z(s) * sum Z(w) and (Z(l) & Z(s)) & xor Z(w), so the
// hash sink of the device costs one gathered word and four integer
// instructions per triangle instead of two 64-bit mixes, a three-way sort and
// a staged compaction.  The reference side (oracle/ref_shim.cpp's HashSink
// behind run_parallel) evaluates the same two expressions per emitted
// triangle.
__host__ __device__ __forceinline__ uint64_t vertex_word(uint32_t v) { return fmix64(uint64_t(v) + kGolden); }
__host__ __device__ __forceinline__ uint64_t tri_hash_sum(uint32_t a, uint32_t b, uint32_t c) {
  return vertex_word(a) * vertex_word(b) * vertex_word(c);
}
__host__ __device__ __forceinline__ uint64_t tri_hash_xor(uint32_t a, uint32_t b, uint32_t c) {
  return vertex_word(a) & vertex_word(b) & vertex_word(c);
}

// canonical_triangle (reference graph.cpp:148-153).
__host__ __device__ __forceinline__ void canon3(uint32_t& x, uint32_t& y, uint32_t& z) {
  uint32_t lo = min(x, y), hi = max(x, y);
  uint32_t a = min(lo, z), t = max(lo, z);
  uint32_t b = min(t, hi), c = max(t, hi);
  x = a;
  y = b;
  z = c;
}

// Bijection on [0, 2^bits) used to scramble R-MAT ids.
__host__ __device__ __forceinline__ uint32_t permute_id(uint64_t seed, uint32_t bits, uint32_t x) {
  const uint64_t mask = (bits >= 64) ? ~0ull : ((1ull << bits) - 1);
  const uint32_t sh = (bits + 1) / 2;
  uint64_t k1 = fmix64(seed ^ 0xA5A5A5A5A5A5A5A5ull);
  uint64_t k2 = fmix64(seed ^ 0x5A5A5A5A5A5A5A5Aull);
  uint64_t v = (uint64_t(x) ^ k1) & mask;
  v = (v * 0x9E3779B1ull) & mask;
  v ^= v >> sh;
  v = (v * 0x85EBCA77ull) & mask;
  v ^= v >> sh;
  v = (v + k2) & mask;
  return uint32_t(v);
}

// R-MAT quadrant thresholds floor(p * 2^64), p = 0.57, 0.76, 0.95.
constexpr uint64_t kRmatT1 = 10514644122014444421ull;
constexpr uint64_t kRmatT2 = 14019525496019259228ull;
constexpr uint64_t kRmatT3 = 17524406870024074035ull;

inline uint32_t bits_for(uint64_t n) {  // smallest b with n <= 2^b
  uint32_t b = 0;
  while (b < 64 && (1ull << b) < n) ++b;
  return b;
}

inline unsigned grid_for(uint64_t items, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (items + block - 1) / block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return unsigned(g);
}

// ---------------------------------------------------------------------------
// device memory: stream-ordered allocator, RAII buffer
// ---------------------------------------------------------------------------
template <typename T>
struct DBuf {
  T* p = nullptr;
  uint64_t n = 0;
  cudaStream_t s = nullptr;

  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { swap(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      reset();
      swap(o);
    }
    return *this;
  }
  ~DBuf() { reset(); }

  void swap(DBuf& o) noexcept {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(s, o.s);
  }
  void alloc(uint64_t count, cudaStream_t stream) {
    reset();
    s = stream;
    n = count;
    if (count) {
      cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&p), sizeof(T) * count, stream);
      if (e != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        n = 0;
        throw TlError(TL_ENOMEM, "device allocation of " + std::to_string(sizeof(T) * count) +
                                     " bytes failed: " + cudaGetErrorString(e));
      }
    }
  }
  void reset() noexcept {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  uint64_t bytes() const { return sizeof(T) * n; }
};

void ensure_device_setup(int device);  // mempool release threshold etc.

}  // namespace tlb
