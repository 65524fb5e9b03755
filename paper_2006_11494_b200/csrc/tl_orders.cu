// tl_orders.cu -- the two vertex orders that are sequential chains by
// definition (ordering.cpp:86-120), computed on the host over the graph's CSR.
// The AOT path never uses them (it runs on the device degree order); they
// exist so that orient() accepts every OrderSpec the reference accepts.
#include <algorithm>
#include <functional>
#include <vector>

#include "tl_internal.cuh"

namespace tlb {

// degeneracy_order (ordering.cpp:86-114): rank r goes to the remaining vertex
// of least (current degree, id).  Keys (degree << 32 | id) live in a min-heap
// with lazy deletion: a decrement pushes a fresh key, stale keys are dropped
// when they surface.
void degeneracy_order_host(uint32_t n, const uint64_t* off, const uint32_t* adj, uint32_t* rank) {
  std::vector<uint32_t> cur(n);
  std::vector<uint8_t> gone(n, 0);
  std::vector<uint64_t> heap;
  heap.reserve(size_t(n) + (n ? off[n] : 0) / 2 + 1);
  for (uint32_t u = 0; u < n; ++u) {
    cur[u] = uint32_t(off[u + 1] - off[u]);
    heap.push_back((uint64_t(cur[u]) << 32) | u);
  }
  std::make_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
  for (uint32_t r = 0; r < n; ++r) {
    uint32_t u = 0;
    while (true) {
      std::pop_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
      const uint64_t key = heap.back();
      heap.pop_back();
      u = uint32_t(key);
      if (!gone[u] && uint32_t(key >> 32) == cur[u]) break;
    }
    gone[u] = 1;
    rank[u] = r;
    for (uint64_t i = off[u]; i < off[u + 1]; ++i) {
      const uint32_t v = adj[i];
      if (gone[v]) continue;
      heap.push_back((uint64_t(--cur[v]) << 32) | v);
      std::push_heap(heap.begin(), heap.end(), std::greater<uint64_t>());
    }
  }
}

// random_order (ordering.cpp:116-120, :23-34): Fisher-Yates over the
// identity, position i-1 swapped with floor(x * i / 2^64) for the next
// splitmix64 output x.
void random_order_host(uint32_t n, uint64_t seed, uint32_t* rank) {
  for (uint32_t u = 0; u < n; ++u) rank[u] = u;
  uint64_t state = seed;
  for (uint64_t i = n; i > 1; --i) {
    state += 0x9E3779B97F4A7C15ull;
    const uint64_t x = fmix64(state);
    const uint64_t j = uint64_t((static_cast<unsigned __int128>(x) * i) >> 64);
    std::swap(rank[i - 1], rank[j]);
  }
}

}  // namespace tlb
