// tl_aot.cu -- the AOT intersection on sm_100a.
//
// Reference semantics: aot_pivot (engine.hpp:238-276) driven by run_parallel
// (parallel.hpp:25-78).  For every pivot l the reference sets a bitmap over
// N+(l), then for every claimed edge traverses N+(s) of the (deg+, id)-smaller
// endpoint s and probes the bitmap.  Here:
//
//   * claims (built at orient time, tl_build.cu) list, per pivot l, the
//     traversed vertex s, the phase (positive/negative) and the first useful
//     position in N+(s) (after l for the negative phase: a witness must rank
//     above l);
//   * N+(l) is staged ONCE per work item in shared memory as an open-addressing
//     hash table (the paper's H) -- per warp for
//     deg+(l) <= 1024, per CTA (up to 32K slots) for larger pivots, and a
//     binary search over the sorted global list beyond that;
//   * traversal lists are streamed with coalesced loads: lists longer than 64
//     are swept by the whole warp (early exit as soon as a rank exceeds
//     max N+(l), the list being rank-ascending), shorter ones are packed 32
//     probes per round by a warp-level load-balanced search;
//   * work items ("tasks") are cost-balanced: small pivots are grouped to
//     ~kTaskWarp probes, heavy pivots are split into chunks of their claim
//     list by the claim-cost prefix (the same prefix cuts multi-GPU parts).
#include <cub/cub.cuh>

#include "tl_internal.cuh"

namespace tlb {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
constexpr uint32_t kChunkBit = 0x80000000u;

constexpr int kWarpThreads = 256;  // 8 warps per CTA
constexpr int kWarpsPerCta = kWarpThreads / 32;
constexpr int kWarpSlotsLg = 11;  // 2048-slot table per warp (8 KB)
constexpr int kWarpSlots = 1 << kWarpSlotsLg;
constexpr uint32_t kWarpDegMax = kWarpSlots / 2;
constexpr int kCtaThreads = 512;
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr int kCtaSlotsLg = 15;  // 32K slots (128 KB)
constexpr uint32_t kCtaDegMax = (1u << kCtaSlotsLg) / 2;
constexpr int kEmitCap = 64;      // per-warp staging of listed triangles
constexpr uint32_t kLong = 64;    // claims longer than this are warp-swept
constexpr uint64_t kTaskWarp = 4096;
constexpr uint64_t kTaskCta = 65536;
constexpr uint64_t kBeta = 4;     // hash build weight per N+(l) element
constexpr uint64_t kGamma = 32;   // per-pivot overhead
constexpr uint64_t kKappa = 2;    // per-claim overhead for the multi-GPU cut

struct Task {
  uint32_t pb, pe;  // pivots [pb, pe); pe | kChunkBit = chunk of one heavy pivot
  uint64_t cb, ce;  // claims clipped to [cb, ce)
};

enum Acc : int { kPos = 0, kNeg, kExec, kHsum, kHxor, kEmitted, kWarpCounter, kCtaCounter, kLogical, kAccN };

struct Params {
  const uint64_t* off;
  const uint32_t* col;
  const uint64_t* claim_off;
  const uint2* claims;
  const uint32_t* orig;
  const uint8_t* pskip;  // pivots [pbase, ...): 1 = not processed by group tasks
  uint32_t pbase;
  uint32_t skip_neg;
  const Task* tasks;
  uint64_t ntasks;
  unsigned long long* acc;
  uint32_t* out;
  uint64_t out_cap;
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint32_t hslot(uint32_t x, uint32_t shift) { return (x * 0x9E3779B1u) >> shift; }

// ------------------------------------------------------------ probe sides
struct SmemHash {
  const uint32_t* T;
  uint32_t mask, shift;
  __device__ __forceinline__ bool find(uint32_t x) const {
    uint32_t h = hslot(x, shift);
    while (true) {
      uint32_t v = T[h];
      if (v == x) return true;
      if (v == kEmpty) return false;
      h = (h + 1) & mask;
    }
  }
};

struct GlobalSorted {  // pivots beyond the largest shared-memory table
  const uint32_t* list;
  uint32_t len;
  __device__ __forceinline__ bool find(uint32_t x) const {
    uint32_t lo = 0, hi = len;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (__ldg(list + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo < len && __ldg(list + lo) == x;
  }
};

__device__ __forceinline__ void hash_insert(uint32_t* T, uint32_t mask, uint32_t shift, uint32_t x) {
  uint32_t h = hslot(x, shift);
  while (atomicCAS(T + h, kEmpty, x) != kEmpty) h = (h + 1) & mask;
}

// ------------------------------------------------------------ emission
template <AotMode MODE>
struct Lane {
  unsigned long long pos = 0, neg = 0, exec = 0, hsum = 0, hxor = 0;
  uint32_t* ebuf = nullptr;  // LIST: per-warp staging (kEmitCap triples)
  uint32_t ecount = 0;       // warp-uniform
};

template <AotMode MODE>
__device__ __forceinline__ void flush_emits(Lane<MODE>& st, const Params& P) {
  if constexpr (MODE == AotMode::list) {
    __syncwarp();
    uint32_t cnt = st.ecount;
    if (cnt) {
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd(P.acc + kEmitted, (unsigned long long)cnt);
      base = __shfl_sync(kFull, base, 0);
      for (uint32_t i = lane_id(); i < 3 * cnt; i += 32) {
        uint64_t slot = base + i / 3;
        if (slot < P.out_cap) P.out[3 * base + i] = st.ebuf[i];
      }
    }
    st.ecount = 0;
    __syncwarp();
  }
}

// Warp-collective: every lane calls it once per probe round.
// Emission order (pivot, neighbor, witness) as in engine.hpp:256 / :269.
template <AotMode MODE>
__device__ __forceinline__ void emit(Lane<MODE>& st, const Params& P, bool hit, bool neg, uint32_t a_orig,
                                     uint32_t b_orig, uint32_t w) {
  if constexpr (MODE == AotMode::count) {
    if (hit) {
      if (neg) ++st.neg; else ++st.pos;
    }
  } else {
    uint32_t c_orig = hit ? __ldg(P.orig + w) : 0;
    if (hit) {
      if (neg) ++st.neg; else ++st.pos;
    }
    if constexpr (MODE == AotMode::hash) {
      if (hit) {
        uint32_t x = a_orig, y = b_orig, z = c_orig;
        canon3(x, y, z);
        uint64_t h = tri_hash(x, y, z);
        st.hsum += h;
        st.hxor ^= h;
      }
    } else {
      unsigned hm = __ballot_sync(kFull, hit);
      if (hm) {
        uint32_t k = __popc(hm);
        if (st.ecount + k > kEmitCap) flush_emits(st, P);
        if (hit) {
          uint32_t slot = st.ecount + __popc(hm & lanemask_lt());
          st.ebuf[3 * slot] = a_orig;
          st.ebuf[3 * slot + 1] = b_orig;
          st.ebuf[3 * slot + 2] = c_orig;
        }
        st.ecount += k;
      }
    }
  }
}

// ------------------------------------------------------------ claim batch
// One warp processes claims [base, min(base + 32, ce)) of pivot l against the
// staged probe side.  All 32 lanes must call it.
template <AotMode MODE, typename Probe>
__device__ __forceinline__ void claim_batch(const Params& P, const Probe& probe, uint32_t lmin, uint32_t lmax,
                                            uint32_t a_orig, uint64_t base, uint64_t ce, Lane<MODE>& st) {
  const uint32_t lane = lane_id();
  const uint64_t c = base + lane;
  uint32_t sflag = 0, pos = 0;
  uint64_t b = 0, e = 0;
  if (c < ce) {
    uint2 cl = P.claims[c];
    sflag = cl.x;
    pos = cl.y;
    bool neg = sflag & kNegBit;
    if (!(P.skip_neg && neg)) {
      uint32_t s = sflag & ~kNegBit;
      uint64_t os = P.off[s];
      e = P.off[s + 1];
      b = os + pos;
    }
  }
  const uint32_t len = e > b ? uint32_t(e - b) : 0;
  const bool neg = sflag & kNegBit;
  uint32_t b_orig = 0;
  if constexpr (MODE != AotMode::count) {
    if (len) b_orig = __ldg(P.orig + (sflag & ~kNegBit));
  }

  // ---- short claims: 32 probes per round, load-balanced over the lanes
  const uint32_t slen = len > kLong ? 0 : len;
  uint32_t incl = slen;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= uint32_t(o)) incl += t;
  }
  const uint32_t excl = incl - slen;
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint64_t bm = b - excl;  // element q of the packed stream: col[bm(owner) + q]
  for (uint32_t r0 = 0; r0 < total; r0 += 32) {
    const uint32_t q = r0 + lane;
    uint32_t i = 0;  // owner: the largest lane i with excl_i <= q
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1) {
      uint32_t pv = __shfl_sync(kFull, excl, i + step);
      if (pv <= q) i += step;
    }
    const uint64_t obm = __shfl_sync(kFull, bm, i);
    const uint32_t oflag = __shfl_sync(kFull, sflag, i);
    uint32_t oorig = 0;
    if constexpr (MODE != AotMode::count) oorig = __shfl_sync(kFull, b_orig, i);
    const bool act = q < total;
    const uint32_t x = act ? __ldg(P.col + obm + q) : kEmpty;
    const bool inwin = x <= lmax;  // kEmpty > any rank
    st.exec += inwin;
    const bool hit = inwin && x >= lmin && probe.find(x);
    emit(st, P, hit, oflag & kNegBit, a_orig, oorig, x);
  }

  // ---- long claims: the whole warp sweeps one list, rank-window early exit
  unsigned longm = __ballot_sync(kFull, len > kLong);
  while (longm) {
    const int j = __ffs(longm) - 1;
    longm &= longm - 1;
    const uint64_t bj = __shfl_sync(kFull, b, j);
    const uint64_t ej = __shfl_sync(kFull, e, j);
    const bool nj = __shfl_sync(kFull, neg, j);
    uint32_t oj = 0;
    if constexpr (MODE != AotMode::count) oj = __shfl_sync(kFull, b_orig, j);
    for (uint64_t p0 = bj; p0 < ej; p0 += 128) {
      uint32_t x[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint64_t p = p0 + 32 * k + lane;
        x[k] = p < ej ? __ldg(P.col + p) : kEmpty;
      }
      bool over = false;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool inwin = x[k] <= lmax;
        st.exec += inwin;
        over |= !inwin;
        const bool hit = inwin && x[k] >= lmin && probe.find(x[k]);
        emit(st, P, hit, nj, a_orig, oj, x[k]);
      }
      if (__any_sync(kFull, over)) break;
    }
  }
}

template <AotMode MODE>
__device__ __forceinline__ void reduce_and_flush(Lane<MODE>& st, const Params& P) {
  flush_emits(st, P);
  unsigned long long v[5] = {st.pos, st.neg, st.exec, st.hsum, st.hxor};
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] += __shfl_xor_sync(kFull, v[k], o);
    v[4] ^= __shfl_xor_sync(kFull, v[4], o);
  }
  if (lane_id() == 0) {
    if (v[0]) atomicAdd(P.acc + kPos, v[0]);
    if (v[1]) atomicAdd(P.acc + kNeg, v[1]);
    if (v[2]) atomicAdd(P.acc + kExec, v[2]);
    if (v[3]) atomicAdd(P.acc + kHsum, v[3]);
    if (v[4]) atomicXor(P.acc + kHxor, v[4]);
  }
}

// ------------------------------------------------------------ warp kernel
template <AotMode MODE>
__global__ void __launch_bounds__(kWarpThreads, 3) k_aot_warp(Params P) {
  extern __shared__ uint32_t smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t* T = smem + warp * kWarpSlots;
  Lane<MODE> st;
  if constexpr (MODE == AotMode::list) st.ebuf = smem + kWarpsPerCta * kWarpSlots + warp * (3 * kEmitCap);

  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(P.acc + kWarpCounter, 1ull);
    t = __shfl_sync(kFull, t, 0);
    if (t >= P.ntasks) break;
    const Task tk = P.tasks[t];
    const bool chunk = tk.pe & kChunkBit;
    const uint32_t pe = tk.pe & ~kChunkBit;
    for (uint32_t l = tk.pb; l < pe; ++l) {
      if (!chunk && P.pskip[l - P.pbase]) continue;
      const uint64_t cb = max(P.claim_off[l], tk.cb), ce = min(P.claim_off[l + 1], tk.ce);
      const uint64_t lb = P.off[l], le = P.off[l + 1];
      const uint32_t dl = uint32_t(le - lb);
      if (cb >= ce || dl == 0) continue;
      // table of 2^lg >= 4 deg+(l) slots (load <= 1/4), at most kWarpSlots
      uint32_t lg = 32 - __clz(4 * dl - 1);
      lg = max(5u, min(lg, uint32_t(kWarpSlotsLg)));
      const uint32_t cap = 1u << lg;
      __syncwarp();
      for (uint32_t i = lane; i < cap; i += 32) T[i] = kEmpty;
      __syncwarp();
      for (uint32_t i = lane; i < dl; i += 32) hash_insert(T, cap - 1, 32 - lg, __ldg(P.col + lb + i));
      const uint32_t lmin = __ldg(P.col + lb), lmax = __ldg(P.col + le - 1);
      uint32_t a_orig = 0;
      if constexpr (MODE != AotMode::count) a_orig = __ldg(P.orig + l);
      __syncwarp();
      const SmemHash probe{T, cap - 1, 32 - lg};
      for (uint64_t base = cb; base < ce; base += 32) claim_batch<MODE>(P, probe, lmin, lmax, a_orig, base, ce, st);
    }
  }
  reduce_and_flush(st, P);
}

// ------------------------------------------------------------ CTA kernel
// Heavy pivots (deg+ > kWarpDegMax): one shared table per CTA, the CTA's
// warps split the chunk's claims.
template <AotMode MODE>
__global__ void __launch_bounds__(kCtaThreads, 1) k_aot_cta(Params P) {
  extern __shared__ uint32_t smem[];
  __shared__ unsigned long long s_task;
  const uint32_t warp = threadIdx.x >> 5;
  uint32_t* T = smem;
  Lane<MODE> st;
  if constexpr (MODE == AotMode::list) st.ebuf = smem + (1u << kCtaSlotsLg) + warp * (3 * kEmitCap);

  while (true) {
    if (threadIdx.x == 0) s_task = atomicAdd(P.acc + kCtaCounter, 1ull);
    __syncthreads();
    const unsigned long long t = s_task;
    __syncthreads();
    if (t >= P.ntasks) break;
    const Task tk = P.tasks[t];
    const uint32_t l = tk.pb;
    const uint64_t cb = tk.cb, ce = tk.ce;
    const uint64_t lb = P.off[l], le = P.off[l + 1];
    const uint32_t dl = uint32_t(le - lb);
    if (cb >= ce || dl == 0) continue;
    const uint32_t lmin = __ldg(P.col + lb), lmax = __ldg(P.col + le - 1);
    uint32_t a_orig = 0;
    if constexpr (MODE != AotMode::count) a_orig = __ldg(P.orig + l);
    if (dl <= kCtaDegMax) {
      uint32_t lg = 32 - __clz(2 * dl - 1);
      lg = max(5u, min(lg, uint32_t(kCtaSlotsLg)));
      const uint32_t cap = 1u << lg;
      for (uint32_t i = threadIdx.x; i < cap; i += kCtaThreads) T[i] = kEmpty;
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < dl; i += kCtaThreads) hash_insert(T, cap - 1, 32 - lg, __ldg(P.col + lb + i));
      __syncthreads();
      const SmemHash probe{T, cap - 1, 32 - lg};
      for (uint64_t base = cb + 32 * warp; base < ce; base += 32 * kCtaWarps)
        claim_batch<MODE>(P, probe, lmin, lmax, a_orig, base, ce, st);
    } else {
      const GlobalSorted probe{P.col + lb, dl};
      for (uint64_t base = cb + 32 * warp; base < ce; base += 32 * kCtaWarps)
        claim_batch<MODE>(P, probe, lmin, lmax, a_orig, base, ce, st);
    }
    __syncthreads();
  }
  reduce_and_flush(st, P);
}

// ------------------------------------------------------------ task building
#define TL_GRID_STRIDE(i, count) \
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (count); i += uint64_t(gridDim.x) * blockDim.x)

// Claim cost (window upper bound): deg+(s) - pos; 0 for skipped negative claims.
__global__ void k_claim_cost(const uint2* claims, const uint64_t* off, uint64_t m, uint32_t skip_neg, uint64_t* cost) {
  TL_GRID_STRIDE(i, m + 1) {
    uint64_t c = 0;
    if (i < m) {
      uint2 cl = claims[i];
      bool neg = cl.x & kNegBit;
      if (!(skip_neg && neg)) {
        uint32_t s = cl.x & ~kNegBit;
        c = (off[s + 1] - off[s]) - cl.y;
      }
    }
    cost[i] = c;
  }
}

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Cost-balanced cut of the claim index space: part p owns claims
// [cut(p), cut(p+1)), cut(k) = first i with CP[i] + kKappa*i >= k*Total/nparts.
// out: cb, ce, pb (pivot of cb), pe (one past the pivot of ce-1),
//      vb, ve (pivot attribution range for table_builds).
__global__ void k_split(const uint64_t* CP, uint64_t m, const uint64_t* claim_off, uint32_t n, uint32_t part,
                        uint32_t nparts, uint64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned __int128 total = (unsigned __int128)CP[m] + (unsigned __int128)kKappa * m;
  auto cut = [&](uint32_t k) -> uint64_t {
    if (k == 0) return 0;
    if (k >= nparts) return m;
    unsigned __int128 target = total * k / nparts;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      uint64_t mid = lo + (hi - lo) / 2;
      unsigned __int128 v = (unsigned __int128)CP[mid] + (unsigned __int128)kKappa * mid;
      if (v < target) lo = mid + 1; else hi = mid;
    }
    return lo;
  };
  auto pivot_of = [&](uint64_t c) -> uint64_t {  // l with claim_off[l] <= c < claim_off[l+1]
    return upper_bound_u64(claim_off, 0, uint64_t(n) + 1, c) - 1;
  };
  const uint64_t cb = cut(part), ce = cut(part + 1);
  out[0] = cb;
  out[1] = ce;
  out[2] = cb < ce ? pivot_of(cb) : 0;
  out[3] = cb < ce ? pivot_of(ce - 1) + 1 : 0;
  out[4] = part == 0 ? 0 : (cb < m ? pivot_of(cb) : n);
  out[5] = part + 1 >= nparts ? n : (ce < m ? pivot_of(ce) : n);
}

// Logical probes (engine.hpp:250/:264: one per traversed element of the full
// list) over the part's claims.
__global__ void k_logical(const uint2* claims, const uint64_t* off, uint64_t cb, uint64_t ce, uint32_t skip_neg,
                          unsigned long long* acc) {
  unsigned long long sum = 0;
  TL_GRID_STRIDE(k, ce - cb) {
    uint2 cl = claims[cb + k];
    if (!(skip_neg && (cl.x & kNegBit))) {
      uint32_t s = cl.x & ~kNegBit;
      sum += off[s + 1] - off[s];
    }
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, sum);
}

struct PivotClass {
  uint8_t* skip;
  uint64_t* sw;   // small-pivot weight (grouped)
  uint32_t* nchw; // chunks for the warp kernel
  uint32_t* nchc; // chunks for the CTA kernel
};

__global__ void k_classify(const uint64_t* CP, const uint64_t* claim_off, const uint64_t* off, uint32_t pb, uint32_t np,
                           uint64_t cb, uint64_t ce, PivotClass pc) {
  TL_GRID_STRIDE(i, uint64_t(np) + 1) {
    if (i == np) {
      pc.sw[i] = 0;
      pc.nchw[i] = 0;
      pc.nchc[i] = 0;
      continue;
    }
    const uint32_t l = pb + uint32_t(i);
    const uint64_t a = max(claim_off[l], cb), b = min(claim_off[l + 1], ce);
    const uint64_t W = a < b ? CP[b] - CP[a] : 0;
    const uint64_t dl = off[l + 1] - off[l];
    uint8_t skip = 1;
    uint64_t sw = 0;
    uint32_t nw = 0, nc = 0;
    if (W && dl) {
      const uint64_t weight = W + kBeta * dl + kGamma;
      if (weight <= kTaskWarp && dl <= kWarpDegMax) {
        skip = 0;
        sw = weight;
      } else if (dl <= kWarpDegMax) {
        nw = uint32_t((W + kTaskWarp - 1) / kTaskWarp);
      } else {
        nc = uint32_t((W + kTaskCta - 1) / kTaskCta);
      }
    }
    pc.skip[i] = skip;
    pc.sw[i] = sw;
    pc.nchw[i] = nw;
    pc.nchc[i] = nc;
  }
}

// Chunks of heavy pivots: chunk k of pivot l covers the claims whose cost
// prefix falls in [W*k/nch, W*(k+1)/nch).
__global__ void k_chunks(const uint64_t* CP, const uint64_t* claim_off, uint32_t pb, uint32_t np, uint64_t cb,
                         uint64_t ce, const uint32_t* nch, const uint32_t* nch_off, Task* tasks) {
  TL_GRID_STRIDE(i, uint64_t(np)) {
    const uint32_t k = nch[i];
    if (!k) continue;
    const uint32_t l = pb + uint32_t(i);
    const uint64_t a = max(claim_off[l], cb), b = min(claim_off[l + 1], ce);
    const uint64_t base = CP[a], W = CP[b] - base;
    Task* out = tasks + nch_off[i];
    uint64_t prev = a;
    for (uint32_t j = 0; j < k; ++j) {
      uint64_t next = j + 1 == k ? b : lower_bound_u64(CP, a, b, base + (W * (j + 1)) / k);
      out[j] = Task{l, (l + 1) | kChunkBit, prev, next};
      prev = next;
    }
  }
}

// Group g = small pivots whose weight prefix SP lies in [g*T, (g+1)*T).
__global__ void k_groups(const uint64_t* SP, uint32_t np, uint32_t pb, uint64_t G, uint64_t cb, uint64_t ce,
                         Task* tasks) {
  TL_GRID_STRIDE(g, G) {
    uint64_t lo = lower_bound_u64(SP, 0, np, g * kTaskWarp);
    uint64_t hi = g + 1 == G ? np : lower_bound_u64(SP, 0, np, (g + 1) * kTaskWarp);
    tasks[g] = Task{pb + uint32_t(lo), pb + uint32_t(hi), cb, ce};
  }
}

template <typename F>
void cub_call(cudaStream_t s, F&& f) {
  size_t bytes = 0;
  TL_CUDA(f(static_cast<void*>(nullptr), bytes));
  DBuf<uint8_t> tmp;
  tmp.alloc(bytes ? bytes : 1, s);
  TL_CUDA(f(static_cast<void*>(tmp.p), bytes));
}

int sm_count() {
  static int cached = -1;
  if (cached < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

template <AotMode MODE>
uint64_t launch_kernels(const Params& pw, const Params& pc, cudaStream_t s) {
  uint64_t launches = 0;
  const size_t warp_smem = sizeof(uint32_t) * (kWarpsPerCta * kWarpSlots +
                                               (MODE == AotMode::list ? kWarpsPerCta * 3 * kEmitCap : 0));
  const size_t cta_smem = sizeof(uint32_t) * ((1u << kCtaSlotsLg) +
                                              (MODE == AotMode::list ? kCtaWarps * 3 * kEmitCap : 0));
  static bool configured = false;
  if (!configured) {
    TL_CUDA(cudaFuncSetAttribute(k_aot_warp<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(warp_smem)));
    TL_CUDA(cudaFuncSetAttribute(k_aot_cta<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(cta_smem)));
    configured = true;
  }
  const int sms = sm_count();
  if (pc.ntasks) {
    unsigned grid = unsigned(std::min<uint64_t>(pc.ntasks, uint64_t(sms)));
    k_aot_cta<MODE><<<grid, kCtaThreads, cta_smem, s>>>(pc);
    TL_CUDA(cudaGetLastError());
    ++launches;
  }
  if (pw.ntasks) {
    int per_sm = 0;
    TL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_aot_warp<MODE>, kWarpThreads, warp_smem));
    per_sm = std::max(per_sm, 1);
    uint64_t want = (pw.ntasks + kWarpsPerCta - 1) / kWarpsPerCta;
    unsigned grid = unsigned(std::min<uint64_t>(want, uint64_t(sms) * per_sm));
    k_aot_warp<MODE><<<grid, kWarpThreads, warp_smem, s>>>(pw);
    TL_CUDA(cudaGetLastError());
    ++launches;
  }
  return launches;
}

}  // namespace

AotResult aot_run(tl_oriented& og, AotMode mode, bool skip_negative, uint32_t part, uint32_t nparts, cudaStream_t s,
                  uint32_t* d_out, uint64_t out_cap) {
  AotResult r;
  if (nparts == 0) nparts = 1;
  TL_REQUIRE(part < nparts, TL_EINVAL, "partition index out of range");
  const uint64_t m = og.m;
  if (m == 0) return r;

  cudaEvent_t ev[3];
  for (auto& e : ev) TL_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};
  TL_CUDA(cudaEventRecord(ev[0], s));

  DBuf<unsigned long long> acc;
  acc.alloc(kAccN, s);
  TL_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long) * kAccN, s));

  // claim-cost prefix CP[0..m]
  DBuf<uint64_t> CP;
  CP.alloc(m + 1, s);
  k_claim_cost<<<grid_for(m + 1, 256, 148u * 64u), 256, 0, s>>>(og.claims.p, og.off.p, m, skip_negative, CP.p);
  TL_CUDA(cudaGetLastError());
  cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, CP.p, m + 1, s); });
  r.launches += 1 + 2 + 1;  // k_claim_cost, scan (init + sweep), k_split

  DBuf<uint64_t> split;
  split.alloc(6, s);
  k_split<<<1, 32, 0, s>>>(CP.p, m, og.claim_off.p, og.n, part, nparts, split.p);
  TL_CUDA(cudaGetLastError());
  uint64_t hs[6];
  TL_CUDA(cudaMemcpyAsync(hs, split.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  const uint64_t cb = hs[0], ce = hs[1];
  const uint32_t pb = uint32_t(hs[2]), pe = uint32_t(hs[3]);
  {  // table_builds attribution: sum of deg+ over pivots [vb, ve)
    uint64_t ob = 0, oe = 0;
    TL_CUDA(cudaMemcpyAsync(&ob, og.off.p + hs[4], 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaMemcpyAsync(&oe, og.off.p + hs[5], 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    r.table_builds = oe - ob;
  }
  if (cb < ce) {
    k_logical<<<grid_for(ce - cb, 256, 148u * 32u), 256, 0, s>>>(og.claims.p, og.off.p, cb, ce, skip_negative,
                                                               acc.p + kLogical);
    TL_CUDA(cudaGetLastError());
    ++r.launches;
  }

  const uint32_t np = cb < ce ? pe - pb : 0;
  DBuf<uint8_t> pskip;
  DBuf<uint64_t> SP;
  DBuf<uint32_t> nchw, nchc, ow, oc;
  DBuf<Task> wtasks, ctasks;
  uint64_t nw_chunks = 0, nc_chunks = 0, G = 0;
  if (np) {
    pskip.alloc(np + 1, s);
    SP.alloc(np + 1, s);
    nchw.alloc(np + 1, s);
    nchc.alloc(np + 1, s);
    ow.alloc(np + 1, s);
    oc.alloc(np + 1, s);
    k_classify<<<grid_for(uint64_t(np) + 1, 256, 148u * 32u), 256, 0, s>>>(CP.p, og.claim_off.p, og.off.p, pb, np, cb,
                                                                          ce, PivotClass{pskip.p, SP.p, nchw.p, nchc.p});
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, SP.p, np + 1, s); });
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, nchw.p, ow.p, np + 1, s); });
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, nchc.p, oc.p, np + 1, s); });
    uint64_t sp_total = 0;
    uint32_t tw = 0, tc = 0;
    TL_CUDA(cudaMemcpyAsync(&sp_total, SP.p + np, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaMemcpyAsync(&tw, ow.p + np, 4, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaMemcpyAsync(&tc, oc.p + np, 4, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    nw_chunks = tw;
    nc_chunks = tc;
    G = sp_total ? (sp_total - 1) / kTaskWarp + 1 : 0;
    wtasks.alloc(std::max<uint64_t>(nw_chunks + G, 1), s);
    ctasks.alloc(std::max<uint64_t>(nc_chunks, 1), s);
    if (nw_chunks)
      k_chunks<<<grid_for(np, 256, 148u * 32u), 256, 0, s>>>(CP.p, og.claim_off.p, pb, np, cb, ce, nchw.p, ow.p,
                                                             wtasks.p);
    if (nc_chunks)
      k_chunks<<<grid_for(np, 256, 148u * 32u), 256, 0, s>>>(CP.p, og.claim_off.p, pb, np, cb, ce, nchc.p, oc.p,
                                                             ctasks.p);
    if (G) k_groups<<<grid_for(G, 256, 148u * 32u), 256, 0, s>>>(SP.p, np, pb, G, cb, ce, wtasks.p + nw_chunks);
    TL_CUDA(cudaGetLastError());
    r.launches += 1 + 3 * 2 + (nw_chunks ? 1 : 0) + (nc_chunks ? 1 : 0) + (G ? 1 : 0);
  }
  TL_CUDA(cudaEventRecord(ev[1], s));

  Params P{};
  P.off = og.off.p;
  P.col = og.col.p;
  P.claim_off = og.claim_off.p;
  P.claims = og.claims.p;
  P.orig = og.orig.p;
  P.pskip = pskip.p;
  P.pbase = pb;
  P.skip_neg = skip_negative;
  P.acc = acc.p;
  P.out = d_out;
  P.out_cap = out_cap;
  Params pw = P, pc = P;
  pw.tasks = wtasks.p;
  pw.ntasks = nw_chunks + G;
  pc.tasks = ctasks.p;
  pc.ntasks = nc_chunks;
  switch (mode) {
    case AotMode::count: r.launches += launch_kernels<AotMode::count>(pw, pc, s); break;
    case AotMode::hash: r.launches += launch_kernels<AotMode::hash>(pw, pc, s); break;
    case AotMode::list: r.launches += launch_kernels<AotMode::list>(pw, pc, s); break;
  }
  TL_CUDA(cudaEventRecord(ev[2], s));
  unsigned long long h[kAccN];
  TL_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  TL_CUDA(cudaEventElapsedTime(&r.prep_ms, ev[0], ev[1]));
  TL_CUDA(cudaEventElapsedTime(&r.list_ms, ev[1], ev[2]));
  r.positive = h[kPos];
  r.negative = h[kNeg];
  r.executed = h[kExec];
  r.logical = h[kLogical];
  r.hash_sum = h[kHsum];
  r.hash_xor = h[kHxor];
  r.emitted = h[kEmitted];
  r.tasks = nw_chunks + G + nc_chunks;
  return r;
}

}  // namespace tlb
