// tl_build.cu -- graph construction on sm_100a: synthetic generators,
// Graph::from_edges (K1), degree_order (K2), orient + rank-sorted out-lists
// (K3/K4, one global radix sort instead of a per-list sort), the AOT claim
// lists, cost_model, the reference-layout upload/download, triple sorting and
// the brute-force checker kernel.
//
// All integer work is HBM-bound gather/scatter/sort; none of it is reshaped
// into tensor-core work.  Sorting uses CUB's onesweep radix sort restricted to
// the bits the keys actually use (2 * ceil(log2 n) for packed vertex pairs).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "tl_internal.cuh"

namespace tlb {

namespace {

constexpr unsigned kBlock = 256;

#define TL_GRID_STRIDE(i, count) \
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (count); i += uint64_t(gridDim.x) * blockDim.x)

template <typename F>
void cub_call(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TL_CUDA(f(static_cast<void*>(nullptr), bytes));
  DBuf<uint8_t> tmp;
  tmp.alloc(bytes ? bytes : 1, s);
  TL_CUDA(f(static_cast<void*>(tmp.p), bytes));
}

// Sort `a` (count keys) on bits [0, end_bit); `b` is scratch of the same size.
// The sorted keys end up in `a`.
template <typename K>
void radix_sort_keys(DBuf<K>& a, DBuf<K>& b, uint64_t count, int end_bit, cudaStream_t s) {
  if (count < 2) return;
  cub::DoubleBuffer<K> db(a.p, b.p);
  cub_call(s, [&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(t, bytes, db, count, 0, end_bit, s);
  });
  if (db.Current() != a.p) a.swap(b);
}

template <typename K, typename V>
void radix_sort_pairs(DBuf<K>& ka, DBuf<K>& kb, DBuf<V>& va, DBuf<V>& vb, uint64_t count, int end_bit,
                      cudaStream_t s) {
  if (count < 2) return;
  cub::DoubleBuffer<K> dk(ka.p, kb.p);
  cub::DoubleBuffer<V> dv(va.p, vb.p);
  cub_call(s, [&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, count, 0, end_bit, s);
  });
  if (dk.Current() != ka.p) ka.swap(kb);
  if (dv.Current() != va.p) va.swap(vb);
}

template <typename T>
T d2h_scalar(const T* d, cudaStream_t s) {
  T v{};
  TL_CUDA(cudaMemcpyAsync(&v, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  return v;
}

// ---------------------------------------------------------------- generators
__global__ void k_gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint2* out) {
  TL_GRID_STRIDE(i, npairs) {
    uint64_t d = draw(seed, i);
    out[i] = make_uint2(uint32_t((d >> 32) % n), uint32_t((d & 0xFFFFFFFFull) % n));
  }
}

__global__ void k_gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint2* out) {
  TL_GRID_STRIDE(i, npairs) {
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
      uint64_t d = draw(seed, i * scale + l);
      uint32_t ub = d >= kRmatT2;
      uint32_t vb = (d >= kRmatT1 && d < kRmatT2) || d >= kRmatT3;
      u = (u << 1) | ub;
      v = (v << 1) | vb;
    }
    out[i] = make_uint2(permute_id(seed, scale, u), permute_id(seed, scale, v));
  }
}

__device__ __forceinline__ uint32_t upper_slot(const uint64_t* prefix, uint32_t n, uint64_t r) {
  uint32_t lo = 0, hi = n;  // prefix[lo] <= r < prefix[hi]
  while (hi - lo > 1) {
    uint32_t mid = lo + (hi - lo) / 2;
    if (__ldg(prefix + mid) <= r) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void k_gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs,
                               uint2* out) {
  const uint64_t total = prefix[n];
  const uint64_t s2 = fmix64(seed ^ 0xC0FFEEull);
  TL_GRID_STRIDE(i, npairs) {
    uint32_t a = upper_slot(prefix, n, draw(s2, 2 * i) % total);
    uint32_t b = upper_slot(prefix, n, draw(s2, 2 * i + 1) % total);
    out[i] = make_uint2(a, b);
  }
}

// ---------------------------------------------------------------- K1 build
// graph.cpp:191-196: n = max(min_vertices, largest id + 1) over ALL pairs
// (self-loops included); self-loops counted.
__global__ void k_scan_pairs(const uint2* pairs, uint64_t npairs, uint32_t* max_id, unsigned long long* loops) {
  uint32_t mx = 0;
  unsigned long long lp = 0;
  TL_GRID_STRIDE(i, npairs) {
    uint2 p = pairs[i];
    mx = max(mx, max(p.x, p.y));
    lp += p.x == p.y;
  }
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    lp += __shfl_xor_sync(0xFFFFFFFFu, lp, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(max_id, mx);
    if (lp) atomicAdd(loops, lp);
  }
}

// graph.cpp:29-31, :196-197: pack (min, max); self-loops become the sentinel,
// which sorts after every real key and is dropped after unique().
__global__ void k_pack(const uint2* pairs, uint64_t npairs, uint32_t nb, uint64_t sentinel, uint64_t* keys) {
  TL_GRID_STRIDE(i, npairs) {
    uint2 p = pairs[i];
    uint32_t lo = min(p.x, p.y), hi = max(p.x, p.y);
    keys[i] = p.x == p.y ? sentinel : ((uint64_t(lo) << nb) | hi);
  }
}

// graph.cpp:168-171: degree count over the deduplicated pairs.
__global__ void k_degree(const uint64_t* keys, uint64_t m, uint32_t nb, uint32_t* deg) {
  const uint64_t mask = (1ull << nb) - 1;
  TL_GRID_STRIDE(i, m) {
    uint64_t k = keys[i];
    atomicAdd(deg + (k >> nb), 1u);
    atomicAdd(deg + (k & mask), 1u);
  }
}

__global__ void k_max_u32(const uint32_t* a, uint64_t count, uint32_t* out) {
  uint32_t mx = 0;
  TL_GRID_STRIDE(i, count) mx = max(mx, a[i]);
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(out, mx);
}

__global__ void k_iota(uint32_t* a, uint64_t count) {
  TL_GRID_STRIDE(i, count) a[i] = uint32_t(i);
}

// rank[by_rank[r]] = r  (inverse permutation; also used for orig = inverse(rank))
__global__ void k_invert(const uint32_t* perm, uint64_t count, uint32_t* inv) {
  TL_GRID_STRIDE(i, count) inv[perm[i]] = uint32_t(i);
}

__global__ void k_perm_check(const uint32_t* rank, uint64_t n, uint8_t* seen, uint32_t* bad) {
  TL_GRID_STRIDE(i, n) {
    uint32_t r = rank[i];
    if (r >= n) {
      atomicOr(bad, 1u);
    } else {
      // byte-granular test-and-set via a 32-bit CAS on the containing word
      unsigned int* w = reinterpret_cast<unsigned int*>(seen + (r & ~3ull));
      unsigned int bit = 1u << (8 * (r & 3));
      unsigned int old = atomicOr(w, bit);
      if (old & bit) atomicOr(bad, 1u);
    }
  }
}

// Row lengths of a sorted key array (row(e) = key >> shift) from its run
// boundaries: the first element of a run subtracts its index, the last adds
// index + 1 -- one write per run end, no contention, rows without keys stay 0.
template <typename K>
__global__ void k_run_lengths(const K* keys, uint32_t shift, uint64_t m, unsigned long long* len) {
  TL_GRID_STRIDE(e, m) {
    const uint64_t row = uint64_t(keys[e]) >> shift;
    if (e == 0 || (uint64_t(keys[e - 1]) >> shift) != row) atomicAdd(len + row, 0ull - e);
    if (e + 1 == m || (uint64_t(keys[e + 1]) >> shift) != row) atomicAdd(len + row, e + 1);
  }
}

// ---------------------------------------------------------------- K3 orient
// ordering.cpp:198-203: point each edge from lower to higher rank.
__global__ void k_direct(const uint64_t* keys, uint64_t m, uint32_t nb, const uint32_t* rank, uint64_t* dk) {
  const uint64_t mask = (1ull << nb) - 1;
  TL_GRID_STRIDE(i, m) {
    uint64_t k = keys[i];
    uint32_t ra = rank[k >> nb], rb = rank[k & mask];
    dk[i] = (uint64_t(min(ra, rb)) << nb) | max(ra, rb);
  }
}

__global__ void k_low_bits(const uint64_t* keys, uint64_t m, uint32_t nb, uint32_t* col) {
  const uint64_t mask = (1ull << nb) - 1;
  TL_GRID_STRIDE(i, m) col[i] = uint32_t(keys[i] & mask);
}

// Claims + cost model in one pass over the rank-sorted directed edges.
// out_degree_before (ordering.hpp:86-89) decides the traversed side:
//   h < t (positive phase, engine.hpp:247-257): pivot t traverses N+(h) from 0
//   t < h (negative phase, engine.hpp:259-272): pivot h traverses N+(t) after h
// Writes the claim in place over dk: key = pivot, value = pos << 32 | s | neg<<31.
__global__ void k_claims(uint64_t* dk_val, uint32_t* ckey, uint64_t m, uint32_t nb, const uint64_t* off,
                         const uint32_t* orig, unsigned long long* costs, uint32_t* max_out) {
  const uint64_t mask = (1ull << nb) - 1;
  unsigned long long cf = 0, kc = 0, ao = 0;
  uint32_t mx = 0;
  TL_GRID_STRIDE(e, m) {
    uint64_t k = dk_val[e];
    uint32_t t = uint32_t(k >> nb), h = uint32_t(k & mask);
    uint64_t ot = off[t];
    uint32_t dt = uint32_t(off[t + 1] - ot), dh = uint32_t(off[h + 1] - off[h]);
    cf += dt + dh;  // engine.cpp:43-45
    kc += dh;
    ao += min(dt, dh);
    mx = max(mx, dt);
    bool h_first = dh != dt ? dh < dt : orig[h] < orig[t];
    uint32_t pivot, s, pos;
    if (h_first) {
      pivot = t; s = h; pos = 0;
    } else {
      pivot = h; s = t | kNegBit; pos = uint32_t(e - ot) + 1;
    }
    ckey[e] = pivot;
    dk_val[e] = (uint64_t(pos) << 32) | s;
  }
  for (int o = 16; o; o >>= 1) {
    cf += __shfl_xor_sync(0xFFFFFFFFu, cf, o);
    kc += __shfl_xor_sync(0xFFFFFFFFu, kc, o);
    ao += __shfl_xor_sync(0xFFFFFFFFu, ao, o);
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (cf) atomicAdd(costs + 0, cf);
    if (kc) atomicAdd(costs + 1, kc);
    if (ao) atomicAdd(costs + 2, ao);
    if (mx) atomicMax(max_out, mx);
  }
}

// Claim windows: after grouping, each claim (pos << 32 | s | neg << 31)
// becomes the packed traversal window {begin:40 | len:23 | neg:1} (in place)
// plus the traversed vertex id (s | neg << 31) for the hash/list modes.
__global__ void k_windows(uint64_t* val_win, uint64_t m, const uint64_t* off, uint32_t* cs) {
  TL_GRID_STRIDE(i, m) {
    const uint64_t v = val_win[i];
    const uint32_t sflag = uint32_t(v), pos = uint32_t(v >> 32);
    const uint32_t s = sflag & ~kNegBit;
    const uint64_t b = off[s] + pos, len = off[s + 1] - b;
    cs[i] = sflag;
    val_win[i] = b | (len << kWinLenShift) | (uint64_t(sflag >> 31) << 63);
  }
}

// ------------------------------------------------ reference-layout transfer
// Rows [u0, u1) of the reference layout straight to rank-space col + claims
// + cost model (k_rows_to_keys, k_low_bits and k_claims in one pass), valid
// when every row is rank-ascending (flags bit0 clear; else the caller falls
// back to the sorting path).  Eight lanes per row.  orig[t] = u and orig[h] =
// v, so the (deg+, id) tie-break needs no gather.
__global__ void k_rows_claims(const uint64_t* out_off, const uint32_t* out, const uint32_t* rank, uint32_t n,
                              uint32_t u0, uint32_t u1, const uint64_t* off, uint32_t* col, uint32_t* ckey,
                              uint64_t* val, unsigned long long* costs, uint32_t* max_out, uint32_t* flags) {
  constexpr uint32_t G = 8;
  const uint32_t gl = threadIdx.x & (G - 1);
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const uint64_t groups = (uint64_t(gridDim.x) * blockDim.x) / G;
  unsigned long long cf = 0, kc = 0, ao = 0;
  uint32_t mx = 0, f = 0;
  for (uint64_t u = u0 + (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G; u < u1; u += groups) {
    const uint32_t t = rank[u];
    const uint64_t src = out_off[u], len = out_off[u + 1] - src, dst = off[t];
    const uint32_t dt = uint32_t(len);
    mx = max(mx, dt);
    uint32_t carry = t;
    for (uint64_t j0 = 0; j0 < len; j0 += G) {
      const uint64_t j = j0 + gl;
      const bool valid = j < len;
      uint32_t h = 0;
      if (valid) {
        const uint32_t v = out[src + j];
        h = v < n ? rank[v] : 0;
        if (v >= n || h <= t) f |= 2u;
        const uint32_t dh = v < n ? uint32_t(off[h + 1] - off[h]) : 0u;
        cf += dt + dh;  // engine.cpp:43-45
        kc += dh;
        ao += min(dt, dh);
        const bool h_first = dh != dt ? dh < dt : v < uint32_t(u);
        col[dst + j] = h;
        ckey[dst + j] = h_first ? t : h;
        val[dst + j] = h_first ? uint64_t(h) : ((uint64_t(j + 1) << 32) | t | kNegBit);
      }
      uint32_t prev = __shfl_up_sync(gmask, h, 1, G);
      if (gl == 0) prev = carry;
      if (valid && h <= prev) f |= 1u;
      const uint32_t last = uint32_t(len - j0 < G ? len - j0 - 1 : G - 1);
      carry = __shfl_sync(gmask, h, last, G);
    }
  }
  for (int o = 16; o; o >>= 1) {
    cf += __shfl_xor_sync(0xFFFFFFFFu, cf, o);
    kc += __shfl_xor_sync(0xFFFFFFFFu, kc, o);
    ao += __shfl_xor_sync(0xFFFFFFFFu, ao, o);
    mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
    f |= __shfl_xor_sync(0xFFFFFFFFu, f, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (cf) atomicAdd(costs + 0, cf);
    if (kc) atomicAdd(costs + 1, kc);
    if (ao) atomicAdd(costs + 2, ao);
    if (mx) atomicMax(max_out, mx);
    if (f) atomicOr(flags, f);
  }
}


__global__ void k_rank_degrees(const uint32_t* orig, uint32_t n, const uint64_t* out_off, uint64_t* deg) {
  TL_GRID_STRIDE(r, uint64_t(n) + 1) {
    if (r < n) {
      uint32_t u = orig[r];
      deg[r] = out_off[u + 1] - out_off[u];
    } else {
      deg[r] = 0;
    }
  }
}

// Rows of the reference layout (original ids) -> rank-space directed keys at
// each row's rank position.  Eight lanes per row, so reads and writes of a
// row are coalesced (rows average ~16 entries at the BASELINE configs).
// flags: bit0 = some row not rank-ascending, bit1 = an edge against the order
// or an id out of range.
__global__ void k_rows_to_keys(const uint64_t* out_off, const uint32_t* out, const uint32_t* rank, uint32_t n,
                               uint32_t nb, const uint64_t* off, uint64_t* dk, uint32_t* flags) {
  constexpr uint32_t G = 8;
  const uint32_t gl = threadIdx.x & (G - 1);
  const unsigned gmask = 0xFFu << (threadIdx.x & 24);
  const uint64_t groups = (uint64_t(gridDim.x) * blockDim.x) / G;
  uint32_t f = 0;
  for (uint64_t u = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G; u < n; u += groups) {
    const uint32_t t = rank[u];
    const uint64_t src = out_off[u], len = out_off[u + 1] - src, dst = off[t];
    uint32_t carry = t;  // rank of the previous entry (the tail before the first)
    for (uint64_t j0 = 0; j0 < len; j0 += G) {
      const uint64_t j = j0 + gl;
      const bool valid = j < len;
      uint32_t h = 0;
      if (valid) {
        const uint32_t v = out[src + j];
        h = v < n ? rank[v] : 0;
        if (v >= n || h <= t) f |= 2u;
        dk[dst + j] = (uint64_t(t) << nb) | h;
      }
      uint32_t prev = __shfl_up_sync(gmask, h, 1, G);
      if (gl == 0) prev = carry;
      if (valid && h <= prev) f |= 1u;
      const uint32_t last = uint32_t(len - j0 < G ? len - j0 - 1 : G - 1);
      carry = __shfl_sync(gmask, h, last, G);
    }
  }
  if (f) atomicOr(flags, f);
}

__global__ void k_orig_degrees(const uint32_t* rank, uint32_t n, const uint64_t* off, uint64_t* deg) {
  TL_GRID_STRIDE(u, uint64_t(n) + 1) {
    if (u < n) {
      uint32_t r = rank[u];
      deg[u] = off[r + 1] - off[r];
    } else {
      deg[u] = 0;
    }
  }
}

// Copies rank-space rows into original-id rows, mapping ids through orig[].
template <typename K>
__global__ void k_rows_to_orig(const uint32_t* rank, uint32_t n, const uint64_t* off, const K* src_ids,
                               uint64_t src_mask, const uint32_t* orig, const uint64_t* dst_off, uint32_t* dst) {
  TL_GRID_STRIDE(u, uint64_t(n)) {
    uint32_t r = rank[u];
    uint64_t s = off[r], len = off[r + 1] - s, d = dst_off[u];
    for (uint64_t j = 0; j < len; ++j) dst[d + j] = orig[uint32_t(uint64_t(src_ids[s + j]) & src_mask)];
  }
}

// in-list keys: (head << nb | tail) for every directed edge of rank row r.
__global__ void k_in_keys(const uint64_t* off, const uint32_t* col, uint32_t n, uint32_t nb, uint64_t* ik) {
  TL_GRID_STRIDE(r, uint64_t(n)) {
    for (uint64_t e = off[r]; e < off[r + 1]; ++e) ik[e] = (uint64_t(col[e]) << nb) | r;
  }
}

// ---------------------------------------------------------- undirected CSR
__global__ void k_sym_keys(const uint64_t* keys, uint64_t m, uint32_t nb, uint64_t* k2) {
  const uint64_t mask = (1ull << nb) - 1;
  TL_GRID_STRIDE(i, m) {
    uint64_t k = keys[i];
    k2[2 * i] = k;
    k2[2 * i + 1] = ((k & mask) << nb) | (k >> nb);
  }
}

// ---------------------------------------------------------- triple sorting
__global__ void k_canon(uint32_t* t, uint64_t count) {
  TL_GRID_STRIDE(i, count) {
    uint32_t a = t[3 * i], b = t[3 * i + 1], c = t[3 * i + 2];
    canon3(a, b, c);
    t[3 * i] = a;
    t[3 * i + 1] = b;
    t[3 * i + 2] = c;
  }
}

__global__ void k_triple_key_c(const uint32_t* t, uint64_t count, uint32_t* kc) {
  TL_GRID_STRIDE(i, count) kc[i] = t[3 * i + 2];
}
__global__ void k_triple_key_ab(const uint32_t* t, const uint32_t* idx, uint64_t count, uint32_t nb, uint64_t* kab) {
  TL_GRID_STRIDE(i, count) {
    uint32_t j = idx[i];
    kab[i] = (uint64_t(t[3 * j]) << nb) | t[3 * j + 1];
  }
}
__global__ void k_triple_gather(const uint32_t* t, const uint32_t* idx, uint64_t count, uint32_t* out) {
  TL_GRID_STRIDE(i, count) {
    uint32_t j = idx[i];
    out[3 * i] = t[3 * j];
    out[3 * i + 1] = t[3 * j + 1];
    out[3 * i + 2] = t[3 * j + 2];
  }
}

// ------------------------------------------------------ brute force (oracle.cpp:8-25)
__device__ __forceinline__ bool csr_has(const uint64_t* off, const uint32_t* adj, uint32_t v, uint32_t w) {
  uint64_t lo = off[v], hi = off[v + 1];
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (adj[mid] < w) lo = mid + 1; else hi = mid;
  }
  return lo < off[v + 1] && adj[lo] == w;
}

// One thread per undirected pair (u, v), u < v, i.e. per sorted key.
__global__ void k_brute(const uint64_t* keys, uint64_t m, uint32_t nb, const uint64_t* off, const uint32_t* adj,
                        unsigned long long* count, uint32_t* out, uint64_t cap) {
  const uint64_t mask = (1ull << nb) - 1;
  TL_GRID_STRIDE(i, m) {
    uint32_t u = uint32_t(keys[i] >> nb), v = uint32_t(keys[i] & mask);
    for (uint64_t j = off[u]; j < off[u + 1]; ++j) {
      uint32_t w = adj[j];
      if (w <= v) continue;
      if (csr_has(off, adj, v, w)) {
        unsigned long long slot = atomicAdd(count, 1ull);
        if (out && slot < cap) {
          out[3 * slot] = u;
          out[3 * slot + 1] = v;
          out[3 * slot + 2] = w;
        }
      }
    }
  }
}


// off[v] = first index e with row(e) >= v, for v in [0, n] (rows ascending):
// run lengths from the run boundaries, then an exclusive scan.
template <typename K>
void fill_offsets(const K* keys, uint32_t shift, uint64_t m, uint32_t n, uint64_t* off, cudaStream_t s) {
  DBuf<uint64_t> len;
  len.alloc(uint64_t(n) + 1, s);
  TL_CUDA(cudaMemsetAsync(len.p, 0, sizeof(uint64_t) * (uint64_t(n) + 1), s));
  if (m) {
    k_run_lengths<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(
        keys, shift, m, reinterpret_cast<unsigned long long*>(len.p));
    TL_CUDA(cudaGetLastError());
  }
  cub_call(s, [&](void* t, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(t, bytes, len.p, off, uint64_t(n) + 1, s);
  });
}

}  // namespace

// ===================================================================== API
void gen_er(uint64_t seed, uint32_t n, uint64_t npairs, uint32_t* d_pairs, cudaStream_t s) {
  TL_REQUIRE(n > 0, TL_EINVAL, "ER generator needs n > 0");
  if (!npairs) return;
  k_gen_er<<<grid_for(npairs, kBlock, 148u * 64u), kBlock, 0, s>>>(seed, n, npairs, reinterpret_cast<uint2*>(d_pairs));
  TL_CUDA(cudaGetLastError());
}

void gen_rmat(uint64_t seed, uint32_t scale, uint64_t npairs, uint32_t* d_pairs, cudaStream_t s) {
  TL_REQUIRE(scale >= 1 && scale <= 31, TL_EINVAL, "R-MAT scale must be in [1, 31]");
  if (!npairs) return;
  k_gen_rmat<<<grid_for(npairs, kBlock, 148u * 64u), kBlock, 0, s>>>(seed, scale, npairs,
                                                                   reinterpret_cast<uint2*>(d_pairs));
  TL_CUDA(cudaGetLastError());
}

void chung_lu_prefix_host(uint64_t seed, uint32_t n, double avg, double gamma, uint64_t* prefix) {
  // Same definition as oracle/trilist_oracle.c: w_i = (1-U_i)^(-1/(gamma-1)),
  // mean `avg`, capped at sqrt(n*avg), fixed point 2^20.  Computed on the host
  // once so libm and CUDA pow() can never diverge.
  std::vector<double> w(n);
  double sum = 0.0;
  for (uint32_t i = 0; i < n; ++i) {
    double u = double(draw(seed, i) >> 11) * (1.0 / 9007199254740992.0);
    w[i] = std::pow(1.0 - u, -1.0 / (gamma - 1.0));
    sum += w[i];
  }
  double scale = (n && sum > 0) ? avg * double(n) / sum : 0.0;
  double cap = std::sqrt(double(n) * avg);
  prefix[0] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    double x = w[i] * scale;
    if (x > cap) x = cap;
    prefix[i + 1] = prefix[i] + uint64_t(x * 1048576.0);
  }
}

void gen_chung_lu(uint64_t seed, uint32_t n, const uint64_t* prefix, uint64_t npairs, uint32_t* d_pairs,
                  cudaStream_t s) {
  TL_REQUIRE(n > 0 && prefix[n] > 0, TL_EINVAL, "Chung-Lu generator needs positive total weight");
  if (!npairs) return;
  DBuf<uint64_t> dp;
  dp.alloc(uint64_t(n) + 1, s);
  TL_CUDA(cudaMemcpyAsync(dp.p, prefix, sizeof(uint64_t) * (uint64_t(n) + 1), cudaMemcpyHostToDevice, s));
  k_gen_chung_lu<<<grid_for(npairs, kBlock, 148u * 64u), kBlock, 0, s>>>(seed, n, dp.p, npairs,
                                                                       reinterpret_cast<uint2*>(d_pairs));
  TL_CUDA(cudaGetLastError());
  TL_CUDA(cudaStreamSynchronize(s));  // prefix buffer lifetime
}

// Graph::build_from_packed (graph.cpp:158-187) + from_edges (:189-200):
// radix sort + unique of packed pairs, then the degree histogram.  The
// symmetric CSR itself is materialised only on demand (graph_csr).
void graph_from_pairs(tl_graph& g, const uint32_t* d_pairs_u32, uint64_t npairs, uint32_t min_vertices) {
  cudaStream_t s = g.stream;
  const uint2* d_pairs = reinterpret_cast<const uint2*>(d_pairs_u32);
  uint64_t n = min_vertices;
  uint64_t loops = 0;
  if (npairs) {
    DBuf<uint8_t> scal;
    scal.alloc(16, s);
    TL_CUDA(cudaMemsetAsync(scal.p, 0, 16, s));
    auto* d_max = reinterpret_cast<uint32_t*>(scal.p);
    auto* d_loops = reinterpret_cast<unsigned long long*>(scal.p + 8);
    k_scan_pairs<<<grid_for(npairs, kBlock, 148u * 16u), kBlock, 0, s>>>(d_pairs, npairs, d_max, d_loops);
    TL_CUDA(cudaGetLastError());
    uint64_t host[2];
    TL_CUDA(cudaMemcpyAsync(host, scal.p, 16, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    uint32_t max_id = uint32_t(host[0]);
    loops = host[1];
    n = std::max<uint64_t>(n, uint64_t(max_id) + 1);
  }
  TL_REQUIRE(n < (1ull << 31), TL_EINVAL, "the B200 path supports fewer than 2^31 vertices");
  g.n = uint32_t(n);
  g.nb = std::max<uint32_t>(1, bits_for(n));
  g.self_loops = loops;
  g.deg.alloc(std::max<uint64_t>(n, 1), s);
  TL_CUDA(cudaMemsetAsync(g.deg.p, 0, sizeof(uint32_t) * std::max<uint64_t>(n, 1), s));
  g.m = 0;
  g.max_deg = 0;
  if (npairs == 0) {
    g.duplicates = 0;
    return;
  }
  const int end_bit = int(2 * g.nb);
  const uint64_t sentinel = end_bit >= 64 ? ~0ull : ((1ull << end_bit) - 1);
  DBuf<uint64_t> a, b;
  a.alloc(npairs, s);
  b.alloc(npairs, s);
  k_pack<<<grid_for(npairs, kBlock, 148u * 64u), kBlock, 0, s>>>(d_pairs, npairs, g.nb, sentinel, a.p);
  TL_CUDA(cudaGetLastError());
  radix_sort_keys(a, b, npairs, end_bit, s);
  DBuf<uint64_t> d_cnt;
  d_cnt.alloc(1, s);
  cub_call(s, [&](void* t, size_t& bytes) {
    return cub::DeviceSelect::Unique(t, bytes, a.p, b.p, d_cnt.p, int64_t(npairs), s);
  });
  uint64_t uniq = d2h_scalar(d_cnt.p, s);
  uint64_t m = uniq - (loops ? 1 : 0);
  a.reset();
  g.m = m;
  g.duplicates = (npairs - loops) - m;
  g.keys.alloc(std::max<uint64_t>(m, 1), s);
  if (m) TL_CUDA(cudaMemcpyAsync(g.keys.p, b.p, sizeof(uint64_t) * m, cudaMemcpyDeviceToDevice, s));
  b.reset();
  if (m) {
    k_degree<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(g.keys.p, m, g.nb, g.deg.p);
    TL_CUDA(cudaGetLastError());
    DBuf<uint32_t> mx;
    mx.alloc(1, s);
    TL_CUDA(cudaMemsetAsync(mx.p, 0, 4, s));
    k_max_u32<<<grid_for(n, kBlock, 148u * 8u), kBlock, 0, s>>>(g.deg.p, n, mx.p);
    TL_CUDA(cudaGetLastError());
    g.max_deg = d2h_scalar(mx.p, s);
  }
}

// offsets()/adjacency(): symmetric ascending lists (graph.cpp:175-186).
void graph_csr(tl_graph& g, DBuf<uint64_t>& off, DBuf<uint32_t>& adj) {
  cudaStream_t s = g.stream;
  off.alloc(uint64_t(g.n) + 1, s);
  adj.alloc(std::max<uint64_t>(2 * g.m, 1), s);
  if (g.m == 0) {
    TL_CUDA(cudaMemsetAsync(off.p, 0, sizeof(uint64_t) * (uint64_t(g.n) + 1), s));
    return;
  }
  uint64_t m2 = 2 * g.m;
  DBuf<uint64_t> k2, tmp;
  k2.alloc(m2, s);
  tmp.alloc(m2, s);
  k_sym_keys<<<grid_for(g.m, kBlock, 148u * 64u), kBlock, 0, s>>>(g.keys.p, g.m, g.nb, k2.p);
  TL_CUDA(cudaGetLastError());
  radix_sort_keys(k2, tmp, m2, int(2 * g.nb), s);
  fill_offsets(k2.p, g.nb, m2, g.n, off.p, s);
  k_low_bits<<<grid_for(m2, kBlock, 148u * 64u), kBlock, 0, s>>>(k2.p, m2, g.nb, adj.p);
  TL_CUDA(cudaGetLastError());
}

// degree_order (ordering.cpp:69-84): a stable radix sort of (degree, id) pairs
// keyed on degree alone reproduces the counting sort's id tie-break.
void degree_order(tl_graph& g, DBuf<uint32_t>& rank) {
  cudaStream_t s = g.stream;
  uint64_t n = g.n;
  rank.alloc(std::max<uint64_t>(n, 1), s);
  if (n == 0) return;
  DBuf<uint32_t> ka, kb, va, vb;
  ka.alloc(n, s);
  kb.alloc(n, s);
  va.alloc(n, s);
  vb.alloc(n, s);
  TL_CUDA(cudaMemcpyAsync(ka.p, g.deg.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
  k_iota<<<grid_for(n, kBlock), kBlock, 0, s>>>(va.p, n);
  TL_CUDA(cudaGetLastError());
  int end_bit = std::max<int>(1, int(bits_for(uint64_t(g.max_deg) + 1)));
  radix_sort_pairs(ka, kb, va, vb, n, end_bit, s);
  k_invert<<<grid_for(n, kBlock), kBlock, 0, s>>>(va.p, n, rank.p);  // va = by_rank
  TL_CUDA(cudaGetLastError());
}

bool is_permutation(const uint32_t* d_rank, uint32_t n, cudaStream_t s) {
  if (n == 0) return true;
  DBuf<uint8_t> seen;
  uint64_t bytes = (uint64_t(n) + 3) & ~3ull;
  seen.alloc(bytes + 4, s);
  TL_CUDA(cudaMemsetAsync(seen.p, 0, bytes + 4, s));
  uint32_t* bad = reinterpret_cast<uint32_t*>(seen.p + bytes);
  k_perm_check<<<grid_for(n, kBlock), kBlock, 0, s>>>(d_rank, n, seen.p, bad);
  TL_CUDA(cudaGetLastError());
  return d2h_scalar(bad, s) == 0;
}

namespace {

void finish_claims(tl_oriented& og, DBuf<uint32_t>& ckey, DBuf<uint64_t>& dk, DBuf<uint64_t>& scal);

// Shared tail of orient / oriented_from_csr: `dk` holds the m rank-sorted
// directed keys (t << nb | h) and og.off/og.orig/og.rank are set.
void finish_orient(tl_oriented& og, DBuf<uint64_t>& dk) {
  cudaStream_t s = og.stream;
  const PhaseClock clk("finish", s);
  const uint64_t m = og.m;
  og.col.alloc(m + 4, s);  // + 16 B: bulk copies of a window round its end up to 16 B
  og.claim_off.alloc(uint64_t(og.n) + 1, s);
  DBuf<uint64_t> scal;
  scal.alloc(4, s);
  TL_CUDA(cudaMemsetAsync(scal.p, 0, 32, s));
  if (m == 0) {
    TL_CUDA(cudaMemsetAsync(og.claim_off.p, 0, sizeof(uint64_t) * (uint64_t(og.n) + 1), s));
    og.win.alloc(1, s);
    og.claim_s.alloc(1, s);
    og.max_out_degree = 0;
    og.cost[0] = og.cost[1] = og.cost[2] = 0;
    return;
  }
  k_low_bits<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(dk.p, m, og.nb, og.col.p);
  TL_CUDA(cudaGetLastError());
  DBuf<uint32_t> ckey;
  ckey.alloc(m, s);
  k_claims<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(
      dk.p, ckey.p, m, og.nb, og.off.p, og.orig.p, reinterpret_cast<unsigned long long*>(scal.p),
      reinterpret_cast<uint32_t*>(scal.p + 3));
  TL_CUDA(cudaGetLastError());
  clk.mark("low_bits+claims");
  finish_claims(og, ckey, dk, scal);
}

// Claims (ckey = pivot, val = pos << 32 | s | neg << 31, in rank-sorted edge
// order) -> grouped by pivot, windows; scal = {cf, kclist, aot, max deg+}.
void finish_claims(tl_oriented& og, DBuf<uint32_t>& ckey, DBuf<uint64_t>& dk, DBuf<uint64_t>& scal) {
  cudaStream_t s = og.stream;
  const PhaseClock clk("claims", s);
  const uint64_t m = og.m;
  uint64_t host[4];
  TL_CUDA(cudaMemcpyAsync(host, scal.p, 32, cudaMemcpyDeviceToHost, s));
  // group claims by pivot (stable: deterministic order inside a pivot)
  DBuf<uint32_t> ckey2;
  ckey2.alloc(m, s);
  DBuf<uint64_t> val2;
  val2.alloc(m, s);
  radix_sort_pairs(ckey, ckey2, dk, val2, m, int(og.nb), s);
  ckey2.reset();
  val2.reset();
  fill_offsets(ckey.p, 0, m, og.n, og.claim_off.p, s);
  TL_CUDA(cudaStreamSynchronize(s));
  clk.mark("claim_sort");
  og.cost[0] = host[0];
  og.cost[1] = host[1];
  og.cost[2] = host[2];
  og.max_out_degree = uint32_t(host[3]);
  TL_REQUIRE(m < (1ull << kWinLenShift) && og.max_out_degree < (1u << 23), TL_EINVAL,
             "graph exceeds the claim-window encoding (m < 2^40, max out-degree < 2^23)");
  // windows are written over the sorted values; the key buffer becomes claim_s
  k_windows<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(dk.p, m, og.off.p, ckey.p);
  TL_CUDA(cudaGetLastError());
  og.win = std::move(dk);
  og.claim_s = std::move(ckey);
  TL_CUDA(cudaStreamSynchronize(s));
  clk.mark("windows");
}

}  // namespace

// orient (ordering.cpp:185-227) in rank space: one radix sort of the directed
// keys (tail rank, head rank) yields CSR rows in rank order whose lists are
// rank-ascending -- the layout orient() produces and AOT's early exit needs.
void orient(tl_graph& g, const uint32_t* d_rank, tl_oriented& og) {
  cudaStream_t s = og.stream;
  og.n = g.n;
  og.nb = g.nb;
  og.m = g.m;
  uint64_t n = g.n, m = g.m;
  og.rank.alloc(std::max<uint64_t>(n, 1), s);
  og.orig.alloc(std::max<uint64_t>(n, 1), s);
  og.off.alloc(n + 1, s);
  if (n) {
    TL_CUDA(cudaMemcpyAsync(og.rank.p, d_rank, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    k_invert<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.rank.p, n, og.orig.p);
    TL_CUDA(cudaGetLastError());
  }
  DBuf<uint64_t> dk, tmp;
  dk.alloc(std::max<uint64_t>(m, 1), s);
  if (m) {
    k_direct<<<grid_for(m, kBlock, 148u * 64u), kBlock, 0, s>>>(g.keys.p, m, g.nb, og.rank.p, dk.p);
    TL_CUDA(cudaGetLastError());
    tmp.alloc(m, s);
    radix_sort_keys(dk, tmp, m, int(2 * g.nb), s);
    tmp.reset();
  }
  fill_offsets(dk.p, og.nb, m, og.n, og.off.p, s);
  finish_orient(og, dk);
}

void oriented_from_csr(tl_oriented& og, uint32_t n, uint64_t m, const uint64_t* d_out_off, const uint32_t* d_out,
                       const uint32_t* d_rank) {
  cudaStream_t s = og.stream;
  const PhaseClock clk("from_csr", s);
  TL_REQUIRE(n < (1u << 31), TL_EINVAL, "the B200 path supports fewer than 2^31 vertices");
  og.n = n;
  og.nb = std::max<uint32_t>(1, bits_for(n));
  og.m = m;
  TL_REQUIRE(is_permutation(d_rank, n, s), TL_EINVAL, "order is not a permutation of the vertex set");
  uint64_t last = 0;
  TL_CUDA(cudaMemcpyAsync(&last, d_out_off + n, 8, cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  TL_REQUIRE(last == m, TL_EINVAL, "out_offsets[n] does not equal m");
  og.rank.alloc(std::max<uint64_t>(n, 1), s);
  og.orig.alloc(std::max<uint64_t>(n, 1), s);
  og.off.alloc(uint64_t(n) + 1, s);
  if (n) {
    TL_CUDA(cudaMemcpyAsync(og.rank.p, d_rank, sizeof(uint32_t) * n, cudaMemcpyDeviceToDevice, s));
    k_invert<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.rank.p, n, og.orig.p);
  }
  DBuf<uint64_t> deg;
  deg.alloc(uint64_t(n) + 1, s);
  k_rank_degrees<<<grid_for(uint64_t(n) + 1, kBlock), kBlock, 0, s>>>(og.orig.p, n, d_out_off, deg.p);
  TL_CUDA(cudaGetLastError());
  cub_call(s, [&](void* t, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(t, bytes, deg.p, og.off.p, uint64_t(n) + 1, s);
  });
  deg.reset();
  DBuf<uint64_t> dk;
  dk.alloc(std::max<uint64_t>(m, 1), s);
  DBuf<uint32_t> flags;
  flags.alloc(1, s);
  TL_CUDA(cudaMemsetAsync(flags.p, 0, 4, s));
  if (m) {
    k_rows_to_keys<<<grid_for(uint64_t(n) * 8, kBlock, 148u * 64u), kBlock, 0, s>>>(d_out_off, d_out, og.rank.p, n, og.nb, og.off.p, dk.p,
                                                          flags.p);
    TL_CUDA(cudaGetLastError());
  }
  uint32_t f = d2h_scalar(flags.p, s);
  clk.mark("rows_to_keys");
  TL_REQUIRE(!(f & 2u), TL_EINVAL, "out-lists contain an edge that does not point to higher rank");
  if (f & 1u) {  // a local order other than rank-asc: restore rank-ascending lists
    DBuf<uint64_t> tmp;
    tmp.alloc(m, s);
    radix_sort_keys(dk, tmp, m, int(2 * og.nb), s);
  }
  finish_orient(og, dk);
}

// Upload of a host OrientedGraph in the reference layout with the transfer
// of the out-lists overlapped: rows are cut into chunks of about equal edge
// counts on the host offsets, each chunk is copied on a copy stream and, as
// soon as it lands, converted on the graph stream straight to rank-space col
// + claims (k_rows_claims).  Lists that are not rank-ascending (another local
// order) take the sorting path over the resident copy.
void oriented_from_host_csr(tl_oriented& og, uint32_t n, uint64_t m, const uint64_t* h_off, const uint32_t* h_out,
                            const uint32_t* h_rank) {
  cudaStream_t s = og.stream;
  const PhaseClock clk("from_host_csr", s);
  TL_REQUIRE(n < (1u << 31), TL_EINVAL, "the B200 path supports fewer than 2^31 vertices");
  TL_REQUIRE(h_off[n] == m, TL_EINVAL, "out_offsets[n] does not equal m");
  og.n = n;
  og.nb = std::max<uint32_t>(1, bits_for(n));
  og.m = m;
  DBuf<uint64_t> d_off;
  DBuf<uint32_t> d_out, d_rank;
  d_off.alloc(uint64_t(n) + 1, s);
  d_out.alloc(std::max<uint64_t>(m, 1), s);
  d_rank.alloc(std::max<uint64_t>(n, 1), s);
  if (n) TL_CUDA(cudaMemcpyAsync(d_rank.p, h_rank, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, s));
  TL_CUDA(cudaMemcpyAsync(d_off.p, h_off, sizeof(uint64_t) * (uint64_t(n) + 1), cudaMemcpyHostToDevice, s));
  // chunk c = rows [cut[c], cut[c+1]), about m / nchunks edges each
  uint32_t nchunks = uint32_t(std::min<uint64_t>(16, std::max<uint64_t>(1, m >> 26)));
  if (const char* e = getenv("TL_UPLOAD_CHUNKS")) nchunks = uint32_t(std::max(1, std::min(64, atoi(e))));  // tests
  std::vector<uint32_t> cut(nchunks + 1, n);
  cut[0] = 0;
  for (uint32_t c = 1; c < nchunks; ++c)
    cut[c] = uint32_t(std::lower_bound(h_off, h_off + n + 1, m * c / nchunks) - h_off);
  cudaStream_t cs = nullptr;
  std::vector<cudaEvent_t> ev(nchunks + 1, nullptr);
  auto release = [&] {
    if (cs) cudaStreamSynchronize(cs);
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
    if (cs) cudaStreamDestroy(cs);
    cs = nullptr;
    for (auto& e : ev) e = nullptr;
  };
  DBuf<uint32_t> ckey, flags;
  DBuf<uint64_t> val, scal;
  uint32_t f = 0;
  try {
    TL_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (auto& e : ev) TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(ev[nchunks], s));  // the allocations above are stream-ordered on s
    TL_CUDA(cudaStreamWaitEvent(cs, ev[nchunks], 0));
    for (uint32_t c = 0; c < nchunks && m; ++c) {
      const uint64_t b = h_off[cut[c]], e = h_off[cut[c + 1]];
      if (e > b) TL_CUDA(cudaMemcpyAsync(d_out.p + b, h_out + b, sizeof(uint32_t) * (e - b), cudaMemcpyHostToDevice, cs));
      TL_CUDA(cudaEventRecord(ev[c], cs));
    }
    TL_REQUIRE(is_permutation(d_rank.p, n, s), TL_EINVAL, "order is not a permutation of the vertex set");
    og.rank = std::move(d_rank);
    og.orig.alloc(std::max<uint64_t>(n, 1), s);
    og.off.alloc(uint64_t(n) + 1, s);
    if (n) k_invert<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.rank.p, n, og.orig.p);
    {
      DBuf<uint64_t> deg;
      deg.alloc(uint64_t(n) + 1, s);
      k_rank_degrees<<<grid_for(uint64_t(n) + 1, kBlock), kBlock, 0, s>>>(og.orig.p, n, d_off.p, deg.p);
      TL_CUDA(cudaGetLastError());
      cub_call(s, [&](void* t, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(t, bytes, deg.p, og.off.p, uint64_t(n) + 1, s);
      });
    }
    clk.mark("offsets");
    og.col.alloc(m + 4, s);  // + 16 B: bulk copies of a window round its end up to 16 B
    ckey.alloc(std::max<uint64_t>(m, 1), s);
    val.alloc(std::max<uint64_t>(m, 1), s);
    scal.alloc(4, s);
    flags.alloc(1, s);
    TL_CUDA(cudaMemsetAsync(scal.p, 0, 32, s));
    TL_CUDA(cudaMemsetAsync(flags.p, 0, 4, s));
    for (uint32_t c = 0; c < nchunks && m; ++c) {
      TL_CUDA(cudaStreamWaitEvent(s, ev[c], 0));
      const uint64_t rows = cut[c + 1] - cut[c];
      if (!rows) continue;
      k_rows_claims<<<grid_for(rows * 8, kBlock, 148u * 64u), kBlock, 0, s>>>(
          d_off.p, d_out.p, og.rank.p, n, cut[c], cut[c + 1], og.off.p, og.col.p, ckey.p, val.p,
          reinterpret_cast<unsigned long long*>(scal.p), reinterpret_cast<uint32_t*>(scal.p + 3), flags.p);
      TL_CUDA(cudaGetLastError());
    }
    f = d2h_scalar(flags.p, s);
    clk.mark("rows_claims");
  } catch (...) {
    release();
    throw;
  }
  release();
  TL_REQUIRE(!(f & 2u), TL_EINVAL, "out-lists contain an edge that does not point to higher rank");
  if (m == 0 || (f & 1u)) {  // empty, or a local order other than rank-asc: restore rank-ascending lists
    og.col.reset();
    ckey.reset();
    val.reset();
    DBuf<uint64_t> dk;
    dk.alloc(std::max<uint64_t>(m, 1), s);
    TL_CUDA(cudaMemsetAsync(flags.p, 0, 4, s));
    if (m) {
      k_rows_to_keys<<<grid_for(uint64_t(n) * 8, kBlock, 148u * 64u), kBlock, 0, s>>>(
          d_off.p, d_out.p, og.rank.p, n, og.nb, og.off.p, dk.p, flags.p);
      TL_CUDA(cudaGetLastError());
      DBuf<uint64_t> tmp;
      tmp.alloc(m, s);
      radix_sort_keys(dk, tmp, m, int(2 * og.nb), s);
    }
    d_out.reset();
    d_off.reset();
    finish_orient(og, dk);
    return;
  }
  d_out.reset();
  d_off.reset();
  og.claim_off.alloc(uint64_t(n) + 1, s);
  finish_claims(og, ckey, val, scal);
}

// Reference OrientedGraph layout (original ids): out_offsets/out by id, in
// lists (tails ascending by rank, ordering.cpp:220-225), rank[].
void oriented_download(tl_oriented& og, uint64_t* out_off, uint32_t* out, uint64_t* in_off, uint32_t* in,
                       uint32_t* rank) {
  cudaStream_t s = og.stream;
  const uint64_t n = og.n, m = og.m;
  if (rank && n) TL_CUDA(cudaMemcpyAsync(rank, og.rank.p, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost, s));
  if (out_off || out) {
    DBuf<uint64_t> deg, doff;
    deg.alloc(n + 1, s);
    doff.alloc(n + 1, s);
    k_orig_degrees<<<grid_for(n + 1, kBlock), kBlock, 0, s>>>(og.rank.p, og.n, og.off.p, deg.p);
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, deg.p, doff.p, n + 1, s); });
    if (out_off) TL_CUDA(cudaMemcpyAsync(out_off, doff.p, sizeof(uint64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (out && m) {
      DBuf<uint32_t> dout;
      dout.alloc(m, s);
      k_rows_to_orig<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.rank.p, og.n, og.off.p, og.col.p, ~0ull, og.orig.p,
                                                            doff.p, dout.p);
      TL_CUDA(cudaGetLastError());
      TL_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
    }
    TL_CUDA(cudaStreamSynchronize(s));
  }
  if (in_off || in) {
    DBuf<uint64_t> ik, tmp, roff, deg, doff;
    ik.alloc(std::max<uint64_t>(m, 1), s);
    roff.alloc(n + 1, s);
    if (m) {
      k_in_keys<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.off.p, og.col.p, og.n, og.nb, ik.p);
      TL_CUDA(cudaGetLastError());
      tmp.alloc(m, s);
      radix_sort_keys(ik, tmp, m, int(2 * og.nb), s);
      tmp.reset();
    }
    fill_offsets(ik.p, og.nb, m, og.n, roff.p, s);
    deg.alloc(n + 1, s);
    doff.alloc(n + 1, s);
    k_orig_degrees<<<grid_for(n + 1, kBlock), kBlock, 0, s>>>(og.rank.p, og.n, roff.p, deg.p);
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, deg.p, doff.p, n + 1, s); });
    if (in_off) TL_CUDA(cudaMemcpyAsync(in_off, doff.p, sizeof(uint64_t) * (n + 1), cudaMemcpyDeviceToHost, s));
    if (in && m) {
      DBuf<uint32_t> din;
      din.alloc(m, s);
      k_rows_to_orig<<<grid_for(n, kBlock), kBlock, 0, s>>>(og.rank.p, og.n, roff.p, ik.p, (1ull << og.nb) - 1,
                                                            og.orig.p, doff.p, din.p);
      TL_CUDA(cudaGetLastError());
      TL_CUDA(cudaMemcpyAsync(in, din.p, sizeof(uint32_t) * m, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
    }
  }
  TL_CUDA(cudaStreamSynchronize(s));
}

void canonicalize_triples(uint32_t* d_triples, uint64_t count, cudaStream_t s) {
  if (!count) return;
  k_canon<<<grid_for(count, kBlock, 148u * 64u), kBlock, 0, s>>>(d_triples, count);
  TL_CUDA(cudaGetLastError());
}

// Lexicographic sort of uint32 triples: a stable sort on c, then a stable
// sort on (a, b) carrying the permutation.
void sort_triples(uint32_t* d_triples, uint64_t count, uint32_t nb, cudaStream_t s) {
  if (count < 2) return;
  TL_REQUIRE(count < (1ull << 32), TL_EINVAL, "triple sort supports fewer than 2^32 triples");
  DBuf<uint32_t> kc, kc2, idx, idx2;
  kc.alloc(count, s);
  kc2.alloc(count, s);
  idx.alloc(count, s);
  idx2.alloc(count, s);
  k_triple_key_c<<<grid_for(count, kBlock, 148u * 64u), kBlock, 0, s>>>(d_triples, count, kc.p);
  k_iota<<<grid_for(count, kBlock, 148u * 64u), kBlock, 0, s>>>(idx.p, count);
  TL_CUDA(cudaGetLastError());
  radix_sort_pairs(kc, kc2, idx, idx2, count, int(nb), s);
  kc.reset();
  kc2.reset();
  DBuf<uint64_t> kab, kab2;
  kab.alloc(count, s);
  kab2.alloc(count, s);
  k_triple_key_ab<<<grid_for(count, kBlock, 148u * 64u), kBlock, 0, s>>>(d_triples, idx.p, count, nb, kab.p);
  TL_CUDA(cudaGetLastError());
  radix_sort_pairs(kab, kab2, idx, idx2, count, int(2 * nb), s);
  kab.reset();
  kab2.reset();
  DBuf<uint32_t> tmp;
  tmp.alloc(3 * count, s);
  k_triple_gather<<<grid_for(count, kBlock, 148u * 64u), kBlock, 0, s>>>(d_triples, idx.p, count, tmp.p);
  TL_CUDA(cudaGetLastError());
  TL_CUDA(cudaMemcpyAsync(d_triples, tmp.p, sizeof(uint32_t) * 3 * count, cudaMemcpyDeviceToDevice, s));
  TL_CUDA(cudaStreamSynchronize(s));
}

uint64_t brute_force(tl_graph& g, DBuf<uint32_t>& out) {
  cudaStream_t s = g.stream;
  if (g.m == 0) {
    out.alloc(1, s);
    return 0;
  }
  DBuf<uint64_t> off;
  DBuf<uint32_t> adj;
  graph_csr(g, off, adj);
  DBuf<unsigned long long> cnt;
  cnt.alloc(1, s);
  TL_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
  unsigned grid = grid_for(g.m, 128, 148u * 64u);
  k_brute<<<grid, 128, 0, s>>>(g.keys.p, g.m, g.nb, off.p, adj.p, cnt.p, nullptr, 0);
  TL_CUDA(cudaGetLastError());
  uint64_t total = d2h_scalar(cnt.p, s);
  out.alloc(std::max<uint64_t>(3 * total, 1), s);
  if (total) {
    TL_CUDA(cudaMemsetAsync(cnt.p, 0, 8, s));
    k_brute<<<grid, 128, 0, s>>>(g.keys.p, g.m, g.nb, off.p, adj.p, cnt.p, out.p, total);
    TL_CUDA(cudaGetLastError());
    sort_triples(out.p, total, g.nb, s);
  }
  return total;
}

}  // namespace tlb
