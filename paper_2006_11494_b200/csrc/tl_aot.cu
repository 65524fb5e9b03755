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
//   * N+(l) is staged ONCE per work record in shared memory.  Vertices are
//     relabelled by rank, so N+(l) lies in [min, max] of its own ranks; when
//     that span fits, the probe side is a direct bitmap over the span (the
//     reference's bitmap, restricted to the window: one LDS + bit test per
//     probe, no collision loop).  Wider spans use a two-level rank bitmap, then
//     hashes (key + 1 stored, 0 = empty, so every layout shares the all-zero
//     resting state).  Per warp: 4.6 KB (a 37,888-bit span); heavy pivots with
//     a wide span use the CTA's 38 KB, and a binary search over the sorted
//     global list beyond that;
//   * traversal lists are streamed with coalesced loads: lists longer than 64
//     are swept by the whole warp (4 or 8 rounds in flight, early exit once a
//     rank exceeds max N+(l) -- lists are rank-ascending; count mode sweeps a
//     batch's long lists as one software-pipelined stream), shorter ones are
//     packed 32 probes per round by a warp-level load-balanced search;
//   * hash mode accumulates, per claim, the sum and the xor of its witnesses'
//     vertex words (tl_common.cuh: the hash distributes over a claim's hits);
//     list mode stages hits per warp and flushes them per pivot;
//   * work is described by compact records (one per pivot with work, or per
//     chunk of a heavy pivot's claim list cut at the claim-cost prefix) and
//     cost-balanced tasks over consecutive records, fetched dynamically; the
//     same cost prefix cuts the multi-GPU parts.
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "tl_internal.cuh"

namespace tlb {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;  // padding value of an out-of-range load

// Tuning knobs (compile-time; see tools/sweep.py):
// Rounds of 32 traversal loads in flight per warp: 4 for graphs whose mean
// window is short (L2-resident C2, C3), 8 for long windows (C4, C5; 6 in the
// emission modes), chosen per run from the mean window length.
#ifndef TL_UNROLL
#define TL_UNROLL 4
#endif
#ifndef TL_UNROLL_LONG
#define TL_UNROLL_LONG 8
#endif
#ifndef TL_LONG_WINDOW
#define TL_LONG_WINDOW 160
#endif
#ifndef TL_WARP_WORDS
#define TL_WARP_WORDS 1184  // per-warp probe region in 32-bit words (a 37,888-bit span): 5 CTAs then fit the 196 KB carve-out
#endif
#ifndef TL_CTAS_PER_SM
#define TL_CTAS_PER_SM 5
#endif
#ifndef TL_CTA_MIN_WORK
#define TL_CTA_MIN_WORK 65536
#endif
#ifndef TL_EMIT_UNROLL_LONG
#define TL_EMIT_UNROLL_LONG 6
#endif
constexpr int kUnrollShort = TL_UNROLL;
constexpr int kUnrollLong = TL_UNROLL_LONG;
constexpr int kUnrollLongEmit = TL_EMIT_UNROLL_LONG;  // hash / list modes (register budget)
#ifndef TL_WARP_CTA_THREADS
#define TL_WARP_CTA_THREADS 256
#endif
constexpr int kWarpThreads = TL_WARP_CTA_THREADS;  // warps per CTA = kWarpThreads / 32
constexpr int kWarpsPerCta = kWarpThreads / 32;
constexpr uint32_t kWarpWords = TL_WARP_WORDS;
constexpr uint32_t kWarpWordsLg = 31 - __builtin_clz(TL_WARP_WORDS);  // largest hash table: 2^lg <= words
constexpr uint32_t kWarpSpanMax = kWarpWords * 32;                    // bitmap span
constexpr uint32_t kWarpHashDegMax = (1u << kWarpWordsLg) / 2;
constexpr uint32_t kWarpStride = kWarpWords + 32;    // + an always-zero guard word (128 B aligned)
// Phase 1 of the kernel: a CTA works on one heavy record with the union of
// its warps' regions (the last guard stays past the end).
constexpr uint32_t kCtaWords = kWarpsPerCta * kWarpStride - 32;
constexpr uint32_t kCtaSpanMax = kCtaWords * 32;
constexpr uint32_t kCtaWordsLg = 31 - __builtin_clz(kCtaWords);
#ifndef TL_CTA_HASH_DEG
#define TL_CTA_HASH_DEG ((1u << kCtaWordsLg) / 2)
#endif
constexpr uint32_t kCtaHashDegMax = TL_CTA_HASH_DEG;  // larger pivots use the global binary search
constexpr uint64_t kCtaMinWork = TL_CTA_MIN_WORK;  // wide-span pivots below this stay on the warp hash path
#ifndef TL_EMIT_CAP
#define TL_EMIT_CAP 224  // hash mode staging (8-byte hits: 4 CTAs/SM fit; >= 32 x the long unroll; 192: +1%)
#endif
#ifndef TL_EMIT_CTAS
#define TL_EMIT_CTAS 4
#endif
#ifndef TL_CTA_TAIL
#define TL_CTA_TAIL 2048  // C5 -2.7%, C4 -0.8%, C4 hash -1.7% (tools/sweep.py)
#endif
#ifndef TL_CTA_TAIL_BS
#define TL_CTA_TAIL_BS 8
#endif
#ifndef TL_BUCKET_PROBE
#define TL_BUCKET_PROBE 1
#endif
#ifndef TL_LIST_CAP
#define TL_LIST_CAP 224  // list mode staging (hits per warp; >= 32 x the long unroll; 192: +1%)
#endif
#ifndef TL_LIST_CTAS
#define TL_LIST_CTAS 4
#endif
// Optional (measured, off): long windows streamed through a per-warp
// shared-memory ring, so the loads in flight hold no registers and a warp
// keeps TL_RING_STAGES chunks of TL_RING_WORDS ids in flight while it probes
// the oldest one.  TL_RING=1: 1-D bulk copies (cp.async.bulk -> UBLKCP, one
// mbarrier per stage); TL_RING=2: per-thread 16-byte cp.async (LDGSTS, zero
// fill past the window, commit groups).  On a B200 (tools/sweep.py, C4 count,
// DESIGN §4): register path 277 ms; bulk ring 432 ms (the TMA engine's
// per-copy cost caps 512-byte copies near 3 TB/s); LDGSTS ring 348 ms at 4
// CTAs/SM, 353 ms at 5 CTAs/SM with 4 KB probe regions (register path with
// the same regions: 288 ms) -- the ring's per-chunk bookkeeping costs more
// issue slots than the latency it hides.  Parity-tested (TL_RING=1 passed the
// full -m gpu suite); kept for the record and for other GPUs.
#ifndef TL_RING
#define TL_RING 0
#endif
#ifndef TL_RING_STAGES
#define TL_RING_STAGES 3
#endif
#ifndef TL_RING_WORDS
#define TL_RING_WORDS 128  // 512 B per chunk (4 probe rounds)
#endif
#ifndef TL_RING_CTAS
#define TL_RING_CTAS 4
#endif
template <AotMode MODE>
constexpr bool ring_mode() {
  return TL_RING && MODE == AotMode::count;
}
constexpr uint32_t kRingStages = TL_RING_STAGES;
constexpr uint32_t kRingWords = TL_RING_WORDS;
[[maybe_unused]] constexpr uint32_t kRingBytes = 4 * kRingWords;
constexpr bool kRingAsync = TL_RING == 2;  // 2: per-thread cp.async (LDGSTS); 1: cp.async.bulk (TMA engine)
static_assert(!kRingAsync || kRingWords % 128 == 0, "LDGSTS chunks are 128-word multiples");
static_assert((kRingWords & (kRingWords - 1)) == 0 && kRingWords >= 32 && kRingWords <= 256, "ring chunk size");

#ifndef TL_REDUX_FOLD
#define TL_REDUX_FOLD 1
#endif
#ifndef TL_FLUSH_UNROLL
#define TL_FLUSH_UNROLL 4
#endif
constexpr int kFlushUnroll = TL_FLUSH_UNROLL;  // staged hits gathered in flight per lane in a flush
// per-warp staging of hits (hash / list modes)
template <AotMode MODE>
constexpr int emit_cap() {
  return MODE == AotMode::list ? TL_LIST_CAP : TL_EMIT_CAP;
}
#ifndef TL_SHORT
#define TL_SHORT 64  // 32 with 1 round in flight: C3 26.7 -> 24.8 ms (more loads in flight for short windows)
#endif
constexpr uint32_t kShort = TL_SHORT;  // claims of at most this length are packed
#ifndef TL_TASK_MIN
#define TL_TASK_MIN 4096
#endif
#ifndef TL_KAPPA
#define TL_KAPPA 8
#endif
constexpr uint64_t kTaskMin = TL_TASK_MIN;  // minimum work per warp task (adaptive: ~64 tasks per warp)
#ifndef TL_CTA_TASK_SCALE
#define TL_CTA_TASK_SCALE 8
#endif
constexpr uint64_t kCtaTaskScale = TL_CTA_TASK_SCALE;  // a CTA record holds kCtaTaskScale warp tasks of work
constexpr uint64_t kBeta = 2;    // staging weight per N+(l) element
constexpr uint64_t kGamma = 64;  // per-record overhead
constexpr uint64_t kKappa = TL_KAPPA;  // per-claim overhead (scheduling and the multi-GPU cut)

// One unit of work: the claims [cb, ce) of pivot l, whose out-list is
// col[lb, lb + dl).
struct Rec {
  uint64_t lb, cb, ce;
  uint32_t l, dl;
};

enum Acc : int { kPos = 0, kNeg, kExec, kHsum, kHxor, kEmitted, kWarpCounter, kCtaCounter, kLogical, kEdgeCounter, kAccN };

struct Params {
  const uint64_t* off;
  const uint32_t* col;
  const uint64_t* win;     // claim windows {begin:40 | len:23 | neg:1}
  const uint32_t* cs;      // traversed vertex per claim (hash/list modes)
  const uint32_t* orig;
  const uint64_t* vword;  // hash mode: rank -> vertex_word(original id)
  const Rec* recs;      // phase 2 (warp) records
  const uint2* tasks;   // phase 2: [rb, re) record ranges
  uint64_t ntasks;       // this part's warp tasks: global index gtasks - 1 - (toff + t * tstride)
  uint64_t gtasks;
  uint32_t toff, tstride;
  const Rec* crecs;     // phase 1 (CTA) records, one per task
  uint64_t ncta;
  uint32_t skip_neg;
  uint32_t prefetch;    // L2 prefetches of the batch's windows: on when the out-lists do not fit in L2
  uint32_t swap_neg;    // cf-hash: a negative claim emits (tail, head, w) (engine.hpp:212)
  unsigned long long* acc;
  uint32_t* out;
  uint64_t out_cap;
};

extern __shared__ uint32_t dsmem[];  // dynamic shared memory, addressed by word offset

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t hslot(uint32_t x, uint32_t shift) { return (x * 0x9E3779B1u) >> shift; }

// Shared memory is addressed with 32-bit shared::cta byte addresses through
// PTX, so the hot loops never rebuild a generic/cluster-window address.
__device__ __forceinline__ uint32_t sm_addr(uint32_t word) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(dsmem)) + 4u * word;
}
__device__ __forceinline__ uint32_t ld_sm(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void st_sm(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void red_or_sm(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ void red_add_sm64(uint32_t a, unsigned long long v) {
  asm volatile("red.shared.add.u64 [%0], %1;" ::"r"(a), "l"(v));
}
#pragma nv_diag_suppress 177  // the ring helpers are unused when TL_RING=0
// mbarrier + 1-D bulk copy (TMA engine, no tensor map): global -> this CTA's
// shared memory, completion counted in bytes on the stage's mbarrier.
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "TL_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra TL_WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(__cvta_generic_to_global(src)), "r"(bytes), "r"(bar)
               : "memory");
}
// Per-thread asynchronous copies (LDGSTS): 16 bytes, the bytes past `bytes`
// zero-filled; completion tracked per thread by commit groups.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(__cvta_generic_to_global(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(__cvta_generic_to_global(p)));
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// In-kernel count of the traversal ids loaded (TL_EXEC_COUNT=1: a shared
// counter per warp, one add per packed batch / long list).  Off by default:
// it cost 3.7% of the C4 count kernel (277.4 vs 270.7 ms, tools/sweep.py); the
// same number is computed outside the hot loop by k_executed (below), which
// replays the early-exit rule per claim.
#ifndef TL_EXEC_COUNT
#define TL_EXEC_COUNT 0
#endif
// Per-warp count of the traversal ids the kernel actually loads (probes left
// after the rank-window pruning and the in-kernel early exit): one shared
// 64-bit word per warp, added to by lane 0 once per packed round group / long
// list, folded into the run's counters at the end.
__device__ __forceinline__ uint32_t exec_addr() {
  __shared__ unsigned long long s_exec[32];
  return static_cast<uint32_t>(__cvta_generic_to_shared(s_exec)) + 8u * (threadIdx.x >> 5);
}
__device__ __forceinline__ uint32_t cas_sm(uint32_t a, uint32_t cmp, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(v));
  return old;
}

// ------------------------------------------------------------ probe sides
// The C4 count kernel kept the ALU pipe (LOP3 / SHF / IADD3 / ISETP /
// VIADDMNMX) 64% busy under ncu (profiles/r2_ncu_summary_c4.md) while the FMA
// pipe idled; both issue one warp instruction per 2 cycles per SM
// sub-partition and run side by side (tools/pipe_bench.cu, profiles/
// r2_pipe_bench.txt).  TL_FMA_PROBE=1 builds the bitmap probe with fewer ALU
// instructions: the word's byte address is one multiply-add of d >> 5 (IMAD,
// the multiplier read from the constant bank so ptxas keeps it on the FMA
// pipe), the bitmap stores id d at bit 31 - (d & 31) so one rotate (SHF.L.W)
// brings it to bit 31, and the count adds t >> 31 (one LEA.HI): 4 ALU + 1 FMA
// instructions per id instead of 5.5 + 1.  IMAD.HI / mad.hi forms of the
// shift and of the accumulation were also built and are slower: IMAD.HI
// issues at a quarter rate.
#ifndef TL_FMA_PROBE
#define TL_FMA_PROBE 1
#endif
#ifndef TL_OPAQUE_BASE
#define TL_OPAQUE_BASE 1
#endif
__constant__ uint32_t c_mul4 = 4u;
__device__ __forceinline__ uint32_t mad_lo_c4(uint32_t a, uint32_t c) {  // 4 * a + c on the FMA pipe
  uint32_t r;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(c_mul4), "r"(c));
  return r;
}
__device__ __forceinline__ uint32_t rotl_wrap(uint32_t a, uint32_t s) {  // bit 31 - (s & 31) lands in bit 31
  uint32_t r;
  asm("shf.l.wrap.b32 %0, %1, %1, %2;" : "=r"(r) : "r"(a), "r"(s));
  return r;
}

struct BitmapProbe {  // bit (x - lmin) of the words at byte address `base`
  static constexpr bool kRangeChecked = true;  // bit() itself rejects x outside [lmin, lmax]
  uint32_t base, lmin, span;
  // Branch-free membership as 0/1 with one LDS.  Ids outside [lmin, lmax]
  // clamp to bit `span`, which is never set (the region keeps a zero word past
  // the largest span).
#if TL_FMA_PROBE
  static constexpr uint32_t mask(uint32_t d) { return 0x80000000u >> (d & 31); }
  __device__ __forceinline__ uint32_t bit(uint32_t x) const {
    const uint32_t d = min(x - lmin, span);
    return rotl_wrap(ld_sm(mad_lo_c4(d >> 5, base)), d) >> 31;
  }
#else
  static constexpr uint32_t mask(uint32_t d) { return 1u << (d & 31); }
  __device__ __forceinline__ uint32_t bit(uint32_t x) const {
    const uint32_t d = min(x - lmin, span);
    return (ld_sm(base + ((d >> 5) << 2)) >> (d & 31)) & 1u;
  }
#endif
  __device__ __forceinline__ uint32_t add(uint32_t x, uint32_t hits) const { return hits + bit(x); }
  __device__ __forceinline__ bool test(uint32_t x) const { return bit(x) != 0; }
};

struct HashProbe {  // linear probing, stores x + 1, 0 = empty
  static constexpr bool kRangeChecked = false;
  uint32_t base, mask, shift;
  __device__ __forceinline__ uint32_t bit(uint32_t x) const { return test(x); }
  __device__ __forceinline__ bool test(uint32_t x) const {
    const uint32_t key = x + 1;
    uint32_t h = hslot(x, shift);
    while (true) {
      const uint32_t v = ld_sm(base + (h << 2));
      if (v == key) return true;
      if (v == 0) return false;
      h = (h + 1) & mask;
    }
  }
};

// Two-level bitmap for spans too wide for a direct bitmap: level 1 has one
// bit per 32-id bucket of [lmin, lmax], level 2 one 32-bit mask per occupied
// bucket, found by rank (a u16 running count per level-1 word + popc).  A
// miss costs one LDS like the direct bitmap; a candidate two more, with no
// data-dependent loop.  Layout from word 0: level 1 (nbw words, the last one
// all-zero: ids outside the window clamp into it), counts (ceil(nbw/2)
// words), masks (one word per occupied bucket).
struct RankProbe {
  static constexpr bool kRangeChecked = true;
  uint32_t bm, cnt, msk, lmin, dmax;
  __device__ __forceinline__ uint32_t bit(uint32_t x) const {
    const uint32_t d = min(x - lmin, dmax), b = d >> 5, w = b >> 5;
    const uint32_t word = ld_sm(bm + (w << 2));
    uint32_t hit = 0;
    if ((word >> (b & 31)) & 1u) {
      uint16_t c;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(c) : "r"(cnt + (w << 1)));
      const uint32_t idx = uint32_t(c) + __popc(word & ((1u << (b & 31)) - 1u));
      hit = (ld_sm(msk + (idx << 2)) >> (d & 31)) & 1u;
    }
    return hit;
  }
  __device__ __forceinline__ uint32_t add(uint32_t x, uint32_t hits) const { return hits + bit(x); }
  __device__ __forceinline__ bool test(uint32_t x) const { return bit(x) != 0; }
};

struct RankLayout {  // word counts of a RankProbe over `span` >= 1 ids
  uint32_t nbw, ncw;   // level-1 words (incl. the zero guard word), count words
  __device__ __forceinline__ explicit RankLayout(uint32_t span)
      : nbw(((span - 1) >> 10) + 2), ncw((nbw + 1) >> 1) {}
  __device__ __forceinline__ uint32_t words(uint32_t dl) const { return nbw + ncw + dl; }  // dl >= masks
};

#ifndef TL_RANK_PROBE
#define TL_RANK_PROBE 1  // 0: wide windows go straight to the hash / global search (path tests)
#endif
__device__ __forceinline__ bool rank_fits(uint32_t dl, uint32_t span, uint32_t words) {
  return TL_RANK_PROBE && RankLayout(span).words(dl) <= words;
}

__device__ __forceinline__ RankProbe rank_probe(uint32_t base, uint32_t lmin, uint32_t span) {
  const RankLayout L(span);
  RankProbe p;
  p.bm = base;
  p.cnt = base + 4 * L.nbw;
  p.msk = p.cnt + 4 * L.ncw;
  p.lmin = lmin;
  p.dmax = (L.nbw - 1) << 10;  // first id of the all-zero last level-1 word
  return p;
}

// Built by one warp from the sorted list nl[0, dl) into the zeroed region of
// p (rank_probe); returns the number of mask words written.
__device__ __forceinline__ uint32_t rank_build(const RankProbe& p, const uint32_t* nl, uint32_t dl, uint32_t span) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lmin = p.lmin;
  const RankLayout L(span);
  uint32_t carry = 0;  // occupied buckets so far
  for (uint32_t i0 = 0; i0 < dl; i0 += 32) {
    const uint32_t i = i0 + lane;
    const bool valid = i < dl;
    const uint32_t d = valid ? __ldg(nl + i) - lmin : 0u;
    const uint32_t b = d >> 5;
    const uint32_t pb = (valid && i > 0) ? (__ldg(nl + i - 1) - lmin) >> 5 : 0xFFFFFFFFu;
    const bool first = valid && b != pb;
    const unsigned fm = __ballot_sync(kFull, first);
    const uint32_t idx = carry + __popc(fm & ((2u << lane) - 1u)) - 1u;  // this element's bucket rank
    if (first) red_or_sm(p.bm + ((b >> 5) << 2), 1u << (b & 31));
    if (valid) red_or_sm(p.msk + (idx << 2), 1u << (d & 31));
    carry += __popc(fm);
  }
  __syncwarp();
  // counts: exclusive prefix of popc over the level-1 words
  const uint32_t per = (L.nbw + 31) >> 5, w0 = min(lane * per, L.nbw), w1 = min(w0 + per, L.nbw);
  uint32_t local = 0;
  for (uint32_t w = w0; w < w1; ++w) local += __popc(ld_sm(p.bm + (w << 2)));
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= uint32_t(o)) incl += t;
  }
  uint32_t run = incl - local;
  for (uint32_t w = w0; w < w1; ++w) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(p.cnt + (w << 1)), "h"(uint16_t(run)));
    run += __popc(ld_sm(p.bm + (w << 2)));
  }
  __syncwarp();
  return carry;
}

// Two-choice bucketized hash for small pivots with windows too wide for the
// rank bitmap: buckets of four slots (x + 1 stored, 0 = empty), each id in one
// of two buckets, so a lookup is two 16-byte LDS and eight compares with no
// data-dependent loop (the linear-probing hash's probe loops diverge the warp).
// Load <= 1/2; an insertion that finds both buckets full reports failure and
// the record falls back to the linear-probing hash.
__device__ __forceinline__ uint32_t bslot1(uint32_t x, uint32_t shift) { return (x * 0x9E3779B1u) >> shift; }
__device__ __forceinline__ uint32_t bslot2(uint32_t x, uint32_t shift) { return (x * 0x85EBCA77u) >> shift; }
__device__ __forceinline__ uint4 ld_sm4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

struct BucketProbe {
  static constexpr bool kRangeChecked = false;
  uint32_t base, shift;  // 2^(32 - shift) buckets of 16 bytes at byte address base
  __device__ __forceinline__ uint32_t bit(uint32_t x) const { return test(x); }
  __device__ __forceinline__ bool test(uint32_t x) const {
    const uint32_t key = x + 1;
    const uint4 a = ld_sm4(base + (bslot1(x, shift) << 4)), b = ld_sm4(base + (bslot2(x, shift) << 4));
    return (a.x == key) | (a.y == key) | (a.z == key) | (a.w == key) | (b.x == key) | (b.y == key) |
           (b.z == key) | (b.w == key);
  }
};

// lg = log2(buckets) for dl ids at load <= 1/2 (at least 8 buckets)
__device__ __forceinline__ uint32_t bucket_lg(uint32_t dl) { return max(3u, 32u - __clz(max(dl, 2u) / 2u - 1u | 1u)); }

// Inserts x (any thread set may call it concurrently); false if both of its
// buckets are full.
#ifndef TL_BUCKET_FORCE_FAIL
#define TL_BUCKET_FORCE_FAIL 0  // path tests: report some insertions as failed
#endif
__device__ __forceinline__ bool bucket_insert(uint32_t base, uint32_t shift, uint32_t x) {
  const uint32_t key = x + 1;
  if (TL_BUCKET_FORCE_FAIL && x % 7 == 3) return false;
  const uint32_t b1 = base + (bslot1(x, shift) << 4), b2 = base + (bslot2(x, shift) << 4);
#pragma unroll
  for (uint32_t k = 0; k < 8; ++k) {
    const uint32_t a = (k < 4 ? b1 : b2) + 4 * (k & 3);
    if (cas_sm(a, 0u, key) == 0u) return true;
  }
  return false;
}

struct GlobalProbe {  // pivots beyond every shared-memory layout
  static constexpr bool kRangeChecked = false;
  const uint32_t* list;
  uint32_t len;
  __device__ __forceinline__ uint32_t bit(uint32_t x) const { return test(x); }
  __device__ __forceinline__ bool test(uint32_t x) const {
    uint32_t lo = 0, hi = len;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(list + mid) < x) lo = mid + 1; else hi = mid;
    }
    return lo < len && __ldg(list + lo) == x;
  }
};

__device__ __forceinline__ void bitmap_set(uint32_t base, uint32_t lmin, uint32_t x) {
  const uint32_t d = x - lmin;
  red_or_sm(base + ((d >> 5) << 2), BitmapProbe::mask(d));
}
__device__ __forceinline__ void bitmap_clear(uint32_t base, uint32_t lmin, uint32_t x) {
  st_sm(base + (((x - lmin) >> 5) << 2), 0u);
}
__device__ __forceinline__ void hash_insert(uint32_t base, uint32_t mask, uint32_t shift, uint32_t x) {
  uint32_t h = hslot(x, shift);
  while (cas_sm(base + (h << 2), 0u, x + 1) != 0u) h = (h + 1) & mask;
}

// ------------------------------------------------------------ emission
// Hash / list modes stage hits per warp as 8-byte entries {neighbour id |
// swap << 31, witness rank}; the pivot's original id is warp-uniform for a
// whole record (`a_orig`), so a record's hits are flushed before the next
// record starts.  Original ids are < 2^31 (n < 2^31), which frees bit 31 for
// the cf-hash role swap of list mode (engine.hpp:212).
constexpr uint32_t kSwapBit = 0x80000000u;

template <AotMode MODE>
struct Lane {
  uint32_t pos = 0, neg = 0;  // per record
  unsigned long long pos64 = 0, neg64 = 0, hsum = 0, hxor = 0;
  uint32_t ebase = 0;   // hash/list: byte address of the per-warp staging buffer
  uint32_t ecount = 0;  // warp-uniform
  uint32_t a_orig = 0;  // the current record's pivot (original id)
  unsigned long long zl = 0;  // hash mode: the pivot's vertex word
  uint32_t ring = 0;    // ring modes: byte address of the warp's chunk ring
  uint32_t bars = 0;    //             and of its per-stage mbarriers
  uint32_t phases = 0;  //             bit s = parity of stage s's next completion
  // Per record: the lanes' 32-bit counts go to 64-bit totals.  TL_REDUX_FOLD=1
  // sums them across the warp first (REDUX.SUM), so the totals are
  // warp-uniform and live in uniform registers instead of four registers per
  // lane (the 48-register count kernel then keeps all U loads of a group in
  // flight).  A record's hits fit 32 bits: its weight is bounded by the task
  // size plus one claim window (< 2^23 ids), and tasks are sized far below 2^31.
  __device__ __forceinline__ void fold() {
#if TL_REDUX_FOLD
    pos64 += __reduce_add_sync(kFull, pos);
    neg64 += __reduce_add_sync(kFull, neg);
#else
    pos64 += pos;
    neg64 += neg;
#endif
    pos = neg = 0;
  }
};

__device__ __forceinline__ void st_sm2(uint32_t a, uint32_t x, uint32_t y) {
  asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(a), "r"(x), "r"(y));
}
__device__ __forceinline__ uint2 ld_sm2(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}

// List mode: a flush maps the witnesses to original ids with independent
// gathers (all in flight at once) and writes the whole batch.  (Hash mode
// stages nothing: tl_common.cuh's hash distributes over a claim's hits.)
template <AotMode MODE>
__device__ __forceinline__ void flush_emits(Lane<MODE>& st, const Params& P) {
  if constexpr (MODE == AotMode::list) {
    __syncwarp();
    const uint32_t cnt = st.ecount;
    if (cnt) {
      unsigned long long base = 0;
      if (lane_id() == 0) base = atomicAdd(P.acc + kEmitted, (unsigned long long)cnt);
      base = __shfl_sync(kFull, base, 0);
#pragma unroll kFlushUnroll
      for (uint32_t i = lane_id(); i < cnt; i += 32) {
        const uint2 e = ld_sm2(st.ebase + 8 * i);
        const uint32_t c = __ldg(P.orig + e.y);
        const uint32_t b = e.x & ~kSwapBit;
        const bool sw = e.x & kSwapBit;
        if (base + i < P.out_cap) {
          uint32_t* o = P.out + 3 * (base + i);
          o[0] = sw ? b : st.a_orig;
          o[1] = sw ? st.a_orig : b;
          o[2] = c;
        }
      }
    }
    st.ecount = 0;
    __syncwarp();
  }
}

// Starts a record: the previous record's hits go out with its pivot.
template <AotMode MODE>
__device__ __forceinline__ void begin_record(Lane<MODE>& st, const Params& P, uint32_t l) {
  if constexpr (MODE == AotMode::list) {
    const uint32_t a = __ldg(P.orig + l);
    if (a != st.a_orig && st.ecount) flush_emits(st, P);
    st.a_orig = a;
  }
  if constexpr (MODE == AotMode::hash) st.zl = __ldg(P.vword + l);
}

// Warp-collective: the hits of one group of U sweep rounds of one list (bit
// k of `hm` = round k hit on this lane), all with the same neighbour word.
template <int U>
struct SameWord {  // one neighbour word for every round (a long sweep of one list)
  uint32_t w;
  __device__ __forceinline__ uint32_t operator[](int) const { return w; }
};
template <int U>
struct RoundWords {  // a neighbour word per round (packed claims)
  const uint32_t (&w)[U];
  __device__ __forceinline__ uint32_t operator[](int k) const { return w[k]; }
};

// Warp-collective: the hits of one group of U probe rounds (bit k of `hm` =
// round k hit on this lane); bw[k] = the neighbour word of round k.
template <AotMode MODE, int U, typename Words>
__device__ __forceinline__ void emit_group(Lane<MODE>& st, const Params& P, uint32_t hm, const uint32_t (&x)[U],
                                           const Words& bw) {
  static_assert(32 * U <= emit_cap<MODE>(), "a group's hits must fit the staging buffer");
  const uint32_t lane = lane_id();
  const uint32_t c = __popc(hm);
  uint32_t incl = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= uint32_t(o)) incl += t;
  }
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  if (total == 0) return;
  if (st.ecount + total > emit_cap<MODE>()) flush_emits(st, P);
  uint32_t slot = st.ebase + 8 * (st.ecount + incl - c);
#pragma unroll
  for (int k = 0; k < U; ++k) {
    if ((hm >> k) & 1u) {
      st_sm2(slot, bw[k], x[k]);
      slot += 8;
    }
  }
  st.ecount += total;
}

// ------------------------------------------------------------ claim batch
// TL_PREFETCH: L2 prefetches of the traversal windows a claim batch is about
// to read -- 1: the next long list while the current one is swept; 2: also
// the batch's first long list, under the packed rounds; 3: also the first and
// last line of every packed (short) claim.  0 = off.
#ifndef TL_PREFETCH
#define TL_PREFETCH 3
#endif
// TL_PIPE=1: count mode sweeps a batch's long lists as one software-pipelined
// stream of groups (claim_batch); 0: one list at a time, load then probe.
#ifndef TL_PIPE
#define TL_PIPE 1
#endif
template <AotMode MODE, int U>
constexpr bool kOverLast() {
  return !(MODE == AotMode::count && U == kUnrollLong);
}

// Long claims (lanes set in longm) through the warp's chunk ring.  Each
// window [b, b + len) of col is read as 16-byte-aligned chunks of at most
// kRingWords words (col is padded by 16 B): the words before b and past the
// window's end are overwritten with kEmpty (never a hit) before probing.  The
// chunk stream runs across the batch's long claims, kRingStages chunks ahead
// of the probing.  No early exit: the windows end at the list's end, and the
// ids past max N+(l) cost one probe each (measured: windows are nearly tight).
template <AotMode MODE, typename Probe>
__device__ __forceinline__ void ring_sweep(const Params& P, const Probe& probe, uint32_t lmax, unsigned longm,
                                           uint64_t b, uint32_t len, bool neg, Lane<MODE>& st) {
  const uint32_t lane = lane_id();
  const uint64_t a0 = b & ~3ull;                                       // 16-byte-aligned chunk origin
  const uint32_t wtot = uint32_t(((b + len + 3) & ~3ull) - a0);        // words to copy (multiple of 4)
  const uint32_t nch = (wtot + kRingWords - 1) / kRingWords;           // chunks of this lane's claim
  // producer cursor: claim lane pj, chunk pc of pn
  unsigned pm = longm;
  int pj = __ffs(pm) - 1;
  uint32_t pc = 0, pn = __shfl_sync(kFull, nch, pj);
  const uint32_t wend = uint32_t(b + len - a0);                       // one past the window, from a0
  auto issue = [&](uint32_t slot) {
    if constexpr (kRingAsync) {
      if (pj < 0) {
        cp_async_commit();  // an empty group keeps one group per chunk slot
        return;
      }
      const uint64_t pa = __shfl_sync(kFull, a0, pj);
      const uint32_t pe = __shfl_sync(kFull, wend, pj);
#pragma unroll
      for (uint32_t v = 0; v < kRingWords / 128; ++v) {
        // lane copies words [w, w + 4) of the window's copy; past the window's
        // end the bytes are zero-filled (id 0 is never in a probe side: every
        // out-list holds ids above its owner)
        const uint32_t w = pc * kRingWords + 128 * v + 4 * lane;
        const uint32_t nb = w < pe ? min(16u, 4 * (pe - w)) : 0u;
        cp_async16(st.ring + slot * kRingBytes + 512 * v + 16 * lane, P.col + pa + (nb ? w : 0u), nb);
      }
      cp_async_commit();
    } else {
      if (pj < 0) return;
      const uint64_t pa = __shfl_sync(kFull, a0, pj);
      const uint32_t pw = __shfl_sync(kFull, wtot, pj);
      if (lane == 0) {
        const uint32_t words = min(kRingWords, pw - pc * kRingWords);
        const uint32_t bar = st.bars + 8 * slot;
        mbar_expect_tx(bar, 4 * words);
        bulk_g2s(st.ring + slot * kRingBytes, P.col + pa + uint64_t(pc) * kRingWords, 4 * words, bar);
      }
    }
    if (++pc == pn) {
      pm &= pm - 1;
      pj = pm ? __ffs(pm) - 1 : -1;
      pc = 0;
      pn = __shfl_sync(kFull, nch, pj < 0 ? 0 : pj);
    }
  };
#pragma unroll
  for (uint32_t i = 0; i < kRingStages; ++i) issue(i);
  // consumer cursor
  unsigned cm = longm;
  int cj = __ffs(cm) - 1;
  uint32_t cc = 0, hits = 0, s = 0;
  uint32_t cn = __shfl_sync(kFull, nch, cj), head = __shfl_sync(kFull, uint32_t(b - a0), cj);
  uint32_t cl = __shfl_sync(kFull, len, cj);
  bool cneg = __shfl_sync(kFull, neg, cj);
  while (true) {
    if constexpr (kRingAsync) {
      cp_async_wait<kRingStages - 1>();  // this lane's copies of the oldest chunk have landed
    } else {
      mbar_wait(st.bars + 8 * s, (st.phases >> s) & 1u);
      st.phases ^= 1u << s;
    }
    const uint32_t wb = cc * kRingWords;                     // chunk origin within the window's copy
    const uint32_t lo = cc == 0 ? head : 0u;                 // valid words [lo, hi) of this chunk
    const uint32_t hi = min(kRingWords, head + cl - wb);
    const uint32_t rounds = (hi + 31) >> 5;
    const uint32_t sb = st.ring + s * kRingBytes;
    if constexpr (kRingAsync) {
      __syncwarp();  // every lane's copies of the chunk are visible to the warp
      if (lane < lo) st_sm(sb + 4 * lane, kEmpty);
    } else {
      if (lane < lo) st_sm(sb + 4 * lane, kEmpty);
      if (hi + lane < 32 * rounds) st_sm(sb + 4 * (hi + lane), kEmpty);
    }
    __syncwarp();
#pragma unroll
    for (uint32_t k = 0; k < kRingWords / 32; ++k) {
      if (k < rounds) {
        const uint32_t x = ld_sm(sb + 4 * (32 * k + lane));
        hits += Probe::kRangeChecked ? probe.bit(x) : uint32_t(x <= lmax && probe.test(x));
      }
    }
    if constexpr (!kRingAsync) fence_proxy_async();  // reads / masks of the slot precede the next bulk write
    __syncwarp();
    issue(s);
    s = s + 1 == kRingStages ? 0u : s + 1;
    if (++cc == cn) {
      if (cneg) st.neg += hits; else st.pos += hits;
      if (TL_EXEC_COUNT && lane == 0) red_add_sm64(exec_addr(), cl);
      cm &= cm - 1;
      if (!cm) break;
      cj = __ffs(cm) - 1;
      cc = 0;
      hits = 0;
      cn = __shfl_sync(kFull, nch, cj);
      head = __shfl_sync(kFull, uint32_t(b - a0), cj);
      cl = __shfl_sync(kFull, len, cj);
      cneg = __shfl_sync(kFull, neg, cj);
    }
  }
}

// One warp processes claims [base, min(base + 32, ce)) of a pivot against the
// staged probe side.  All 32 lanes must call it.
template <AotMode MODE, int U, typename Probe>
__device__ __forceinline__ void claim_batch(const Params& P, const Probe& probe, uint32_t lmax, uint64_t base,
                                            uint64_t ce, Lane<MODE>& st) {
  const uint32_t lane = lane_id();
  const uint64_t c = base + lane;
  uint64_t b = 0;
  uint32_t len = 0;
  bool neg = false;
  if (c < ce) {
    const uint64_t w = P.win[c];
    b = w & kWinBeginMask;
    neg = w >> 63;
    len = (P.skip_neg && neg) ? 0u : uint32_t((w >> kWinLenShift) & kWinLenMask);
  }
  const uint32_t sflag = neg ? kNegBit : 0u;
  uint32_t b_orig = 0;  // list mode's neighbour word: original id | swap (cf-hash negative claim)
  if constexpr (MODE == AotMode::list) {
    if (len) b_orig = __ldg(P.orig + (P.cs[c] & ~kNegBit)) | (P.swap_neg && neg ? kSwapBit : 0u);
  }
  // hash mode: the claim's factors Z(l) Z(s) and Z(l) & Z(s); its hits w add
  // Z(w) times the first to hash_sum and Z(w) & the second to hash_xor
  unsigned long long fmul = 0, fand = 0;
  if constexpr (MODE == AotMode::hash) {
    if (len) {
      const unsigned long long zs = __ldg(P.vword + (P.cs[c] & ~kNegBit));
      fmul = st.zl * zs;
      fand = st.zl & zs;
    }
  }

#if TL_PREFETCH
  // The next long list's lines are requested into L2 while the current one is
  // swept (lane i asks for the line of its i-th round: up to 1024 ids), so its
  // demand loads find them there or on their way: more bytes in flight per
  // warp without holding registers.
  auto prefetch_list = [&](unsigned m) {
    if (m && P.prefetch) {
      const int jn = __ffs(m) - 1;
      const uint64_t bn = __shfl_sync(kFull, b, jn);
      const uint32_t ln = __shfl_sync(kFull, len, jn);
      if (32 * lane < ln + 31) prefetch_l2(P.col + bn + 32 * lane);
    }
  };
  if (TL_PREFETCH >= 2) prefetch_list(__ballot_sync(kFull, len > kShort));  // the first long list, under the packed rounds
  if (TL_PREFETCH >= 3 && P.prefetch && len && len <= kShort) {  // the packed claims' lines (rounds after the first find them in L2)
    prefetch_l2(P.col + b);
    prefetch_l2(P.col + b + len - 1);
  }
#endif
  // ---- short claims: 32 probes per round, load-balanced over the lanes
  const uint32_t slen = len > kShort ? 0 : len;
  uint32_t incl = slen;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(kFull, incl, o);
    if (lane >= uint32_t(o)) incl += t;
  }
  const uint32_t excl = incl - slen;
  const uint32_t total = __shfl_sync(kFull, incl, 31);
  const uint64_t bm = b - excl;  // element q of the packed stream: col[bm(owner) + q]
  if (TL_EXEC_COUNT && lane == 0 && total) red_add_sm64(exec_addr(), total);
#ifndef TL_SHORT_UNROLL
#define TL_SHORT_UNROLL 4
#endif
  constexpr int kSU = TL_SHORT_UNROLL;  // packed rounds in flight
  for (uint32_t r0 = 0; r0 < total; r0 += 32 * kSU) {
    uint32_t x[kSU], of[kSU], oo[kSU];  // oo: list mode the owner's neighbour word, hash mode the owner lane
#pragma unroll
    for (int k = 0; k < kSU; ++k) {
      const uint32_t q = r0 + 32 * k + lane;
      uint32_t i = 0;  // owner: the largest lane i with excl_i <= q
#pragma unroll
      for (uint32_t step = 16; step; step >>= 1) {
        const uint32_t pv = __shfl_sync(kFull, excl, i + step);
        if (pv <= q) i += step;
      }
      const uint64_t obm = __shfl_sync(kFull, bm, i);
      of[k] = __shfl_sync(kFull, sflag, i);
      oo[k] = 0;
      if constexpr (MODE == AotMode::list) oo[k] = __shfl_sync(kFull, b_orig, i);
      if constexpr (MODE == AotMode::hash) oo[k] = i;
      x[k] = q < total ? __ldg(P.col + obm + q) : kEmpty;
    }
    uint32_t hm = 0;
#pragma unroll
    for (int k = 0; k < kSU; ++k) {
      const uint32_t hit = Probe::kRangeChecked ? probe.bit(x[k]) : uint32_t(x[k] <= lmax && probe.test(x[k]));
      if (of[k] & kNegBit) st.neg += hit; else st.pos += hit;
      if constexpr (MODE != AotMode::count) hm |= hit << k;
    }
    if constexpr (MODE == AotMode::list) emit_group<MODE, kSU>(st, P, hm, x, RoundWords<kSU>{oo});
    if constexpr (MODE == AotMode::hash) {
      unsigned long long z[kSU];
#pragma unroll
      for (int k = 0; k < kSU; ++k) z[k] = (hm >> k) & 1u ? __ldg(P.vword + x[k]) : 0ull;
#pragma unroll
      for (int k = 0; k < kSU; ++k) {
        st.hsum += z[k] * __shfl_sync(kFull, fmul, oo[k]);
        st.hxor ^= z[k] & __shfl_sync(kFull, fand, oo[k]);
      }
    }
    (void)hm;
  }

  unsigned longm = __ballot_sync(kFull, len > kShort);
  if constexpr (ring_mode<MODE>()) {
    if (longm) ring_sweep<MODE>(P, probe, lmax, longm, b, len, neg, st);
    return;
  }
  // ---- long claims: the whole warp sweeps one list, U rounds of 32
  // loads in flight; lists are rank-ascending, so a list is abandoned once a
  // group reaches past max N+(l)
  if constexpr (TL_PIPE && MODE == AotMode::count) {
    // Software-pipelined over the batch's long lists as one stream of groups:
    // a group's registers are reloaded with the next group -- of the same
    // list, or the first group of the next list once this one ends -- while
    // the group is probed, so the next loads fly under this group's probes
    // and a list's first round trip overlaps the previous list's last group.
    // The group's last round decides the early exit first (ids ascend across
    // rounds and lanes; kEmpty past the window's end also ends the list),
    // which also orders all U loads of a group before their first use.
    // (Measured and left out, profiles/r2_sweep_count_pipeline.md: the same
    // stream for hash mode, unpredicated reloads for groups wholly inside
    // their window, skipping the empty rounds of a list's last group.)
    if (!longm) return;
    int j = __ffs(longm) - 1;
    longm &= longm - 1;
    const uint32_t* p = P.col + __shfl_sync(kFull, b, j) + lane;
    uint32_t lcur = __shfl_sync(kFull, len, j);
    int rem = int(lcur) - int(lane);  // this lane reads p[32k] while 32k < rem
    bool nj = __shfl_sync(kFull, neg, j);
    uint32_t x[U];
#pragma unroll
    for (int k = 0; k < U; ++k) x[k] = 32 * k < rem ? __ldg(p + 32 * k) : kEmpty;
    uint32_t hits = 0, groups = 0;
    while (true) {
      const bool stop = __any_sync(kFull, x[U - 1] > lmax);  // the current list's last group
      const bool cneg = nj;
      const uint32_t lprev = lcur;
      bool more = true;
      if (stop) {
        more = longm != 0;
        if (more) {
          j = __ffs(longm) - 1;
          longm &= longm - 1;
          p = P.col + __shfl_sync(kFull, b, j) + lane - 32 * U;
          lcur = __shfl_sync(kFull, len, j);
          rem = int(lcur) - int(lane) + 32 * U;
          nj = __shfl_sync(kFull, neg, j);
        } else {
          rem = 0;  // nothing left to load
        }
      }
      p += 32 * U;
      rem -= 32 * U;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if constexpr (Probe::kRangeChecked) hits = probe.add(x[k], hits);
        else hits += uint32_t(x[k] <= lmax && probe.test(x[k]));
        x[k] = 32 * k < rem ? __ldg(p + 32 * k) : kEmpty;
      }
      ++groups;
      if (stop) {
        if (cneg) st.neg += hits; else st.pos += hits;
        if (TL_EXEC_COUNT && lane == 0) red_add_sm64(exec_addr(), min(lprev, 32 * U * groups));  // ids loaded
        hits = 0;
        groups = 0;
        if (!more) break;
      }
    }
    return;
  }
  while (longm) {
    const int j = __ffs(longm) - 1;
    longm &= longm - 1;
#if TL_PREFETCH
    prefetch_list(longm);
#endif
    const uint64_t bj = __shfl_sync(kFull, b, j);
    const uint32_t lj = __shfl_sync(kFull, len, j);
    const bool nj = __shfl_sync(kFull, neg, j);
    uint32_t oj = 0;
    if constexpr (MODE == AotMode::list) oj = __shfl_sync(kFull, b_orig, j);
    unsigned long long zsum = 0, zxor = 0;  // hash mode: this lane's witnesses' words of list j
    const uint32_t* p = P.col + bj + lane;
    int rem = int(lj) - int(lane);  // this lane reads p[32k] while 32k < rem
    uint32_t hits = 0;
    for (uint32_t r0 = 0; r0 < lj; r0 += 32 * U) {
      uint32_t x[U];
#pragma unroll
      for (int k = 0; k < U; ++k) x[k] = 32 * k < rem ? __ldg(p + 32 * k) : kEmpty;
      bool over = false;
      uint32_t hm = 0;
#pragma unroll
      for (int k = 0; k < U; ++k) {
        // lists ascend across rounds and lanes, so only the last round can
        // hold the group's largest id (kEmpty past the window's end).  Per
        // instantiation, measured: C2/C3 count -1.5%, C4 hash -1.5%, but the
        // U = 6 count kernel +8.5% (its schedule changes), which keeps the
        // per-round test.
        if constexpr (kOverLast<MODE, U>()) {
          if (k == U - 1) over = x[k] > lmax;
        } else {
          over |= x[k] > lmax;
        }
        if constexpr (MODE == AotMode::count && Probe::kRangeChecked) {
          hits = probe.add(x[k], hits);
        } else {
          const uint32_t hit = Probe::kRangeChecked ? probe.bit(x[k]) : uint32_t(x[k] <= lmax && probe.test(x[k]));
          hits += hit;
          if constexpr (MODE != AotMode::count) hm |= hit << k;
        }
      }
      if constexpr (MODE == AotMode::list) emit_group<MODE, U>(st, P, hm, x, SameWord<U>{oj});
      if constexpr (MODE == AotMode::hash) {
        unsigned long long z[U];
#pragma unroll
        for (int k = 0; k < U; ++k) z[k] = (hm >> k) & 1u ? __ldg(P.vword + x[k]) : 0ull;
#pragma unroll
        for (int k = 0; k < U; ++k) {
          zsum += z[k];
          zxor ^= z[k];
        }
      }
      p += 32 * U;
      rem -= 32 * U;
      if (__any_sync(kFull, over)) break;
    }
    if (nj) st.neg += hits; else st.pos += hits;
    if constexpr (MODE == AotMode::hash) {
      st.hsum += zsum * __shfl_sync(kFull, fmul, j);
      st.hxor ^= zxor & __shfl_sync(kFull, fand, j);
    }
    if (TL_EXEC_COUNT && lane == 0) red_add_sm64(exec_addr(), min(lj, uint32_t(int(lj) - rem)));  // ids loaded
  }
}

template <AotMode MODE>
__device__ __forceinline__ void reduce_and_flush(Lane<MODE>& st, const Params& P) {
  st.fold();
  flush_emits(st, P);
  unsigned long long v[4] = {st.pos64, st.neg64, st.hsum, st.hxor};
#pragma unroll
  for (int o = 16; o; o >>= 1) {
#pragma unroll
    for (int k = TL_REDUX_FOLD ? 2 : 0; k < 3; ++k) v[k] += __shfl_xor_sync(kFull, v[k], o);  // folded totals are already the warp's
    v[3] ^= __shfl_xor_sync(kFull, v[3], o);
  }
  if (lane_id() == 0) {
    if constexpr (TL_EXEC_COUNT) {
      const unsigned long long ex =
          *reinterpret_cast<volatile unsigned long long*>(__cvta_shared_to_generic(exec_addr()));
      if (ex) atomicAdd(P.acc + kExec, ex);
    }
    if (v[0]) atomicAdd(P.acc + kPos, v[0]);
    if (v[1]) atomicAdd(P.acc + kNeg, v[1]);
    if (v[2]) atomicAdd(P.acc + kHsum, v[2]);
    if (v[3]) atomicXor(P.acc + kHxor, v[3]);
  }
}

// ------------------------------------------------------------ warp kernel
template <AotMode MODE, int U>
__device__ __forceinline__ void warp_record(const Params& P, const Rec& R, uint32_t wbase, Lane<MODE>& st) {
  const uint32_t lane = lane_id();
  const uint32_t* nl = P.col + R.lb;
  const uint32_t lmin = __ldg(nl), lmax = __ldg(nl + R.dl - 1);
  const uint32_t span = lmax - lmin + 1;
  begin_record(st, P, R.l);
  if (span <= kWarpSpanMax) {
    for (uint32_t i = lane; i < R.dl; i += 32) bitmap_set(wbase, lmin, __ldg(nl + i));
    __syncwarp();
    const BitmapProbe probe{wbase, lmin, span};
    for (uint64_t base = R.cb; base < R.ce; base += 32) claim_batch<MODE, U>(P, probe, lmax, base, R.ce, st);
    __syncwarp();
    const uint32_t nwords = (span + 31) >> 5;
    if (nwords <= max(64u, 2 * R.dl))
      for (uint32_t i = lane; i < nwords; i += 32) st_sm(wbase + 4 * i, 0u);
    else
      for (uint32_t i = lane; i < R.dl; i += 32) bitmap_clear(wbase, lmin, __ldg(nl + i));
  } else if (rank_fits(R.dl, span, kWarpWords)) {
    const RankProbe probe = rank_probe(wbase, lmin, span);
    const uint32_t nmask = rank_build(probe, nl, R.dl, span);
    for (uint64_t base = R.cb; base < R.ce; base += 32) claim_batch<MODE, U>(P, probe, lmax, base, R.ce, st);
    __syncwarp();
    const RankLayout L(span);
    for (uint32_t i = lane; i < L.nbw + L.ncw + nmask; i += 32) st_sm(wbase + 4 * i, 0u);
  } else {
    bool done = false;
    const uint32_t blg = bucket_lg(R.dl);
    if (TL_BUCKET_PROBE && (4u << blg) <= kWarpWords) {
      bool ok = true;
      for (uint32_t i = lane; i < R.dl; i += 32) ok &= bucket_insert(wbase, 32 - blg, __ldg(nl + i));
      done = __all_sync(kFull, ok);
      if (done) {
        const BucketProbe probe{wbase, 32 - blg};
        for (uint64_t base = R.cb; base < R.ce; base += 32)
          claim_batch<MODE, U>(P, probe, lmax, base, R.ce, st);
      }
      __syncwarp();
      for (uint32_t i = lane; i < (4u << blg); i += 32) st_sm(wbase + 4 * i, 0u);
      __syncwarp();
    }
    if (!done) {
      uint32_t lg = 32 - __clz(4 * R.dl - 1);
      lg = max(5u, min(lg, kWarpWordsLg));
      const uint32_t cap = 1u << lg;
      for (uint32_t i = lane; i < R.dl; i += 32) hash_insert(wbase, cap - 1, 32 - lg, __ldg(nl + i));
      __syncwarp();
      const HashProbe probe{wbase, cap - 1, 32 - lg};
      for (uint64_t base = R.cb; base < R.ce; base += 32)
        claim_batch<MODE, U>(P, probe, lmax, base, R.ce, st);
      __syncwarp();
      for (uint32_t i = lane; i < cap; i += 32) st_sm(wbase + 4 * i, 0u);
    }
  }
  __syncwarp();
  st.fold();
}

// ------------------------------------------------------------ the kernel
// Persistent, two phases.  Phase 1: each CTA takes heavy records (wide spans
// on big pivots) one at a time and probes them with all its warps against one
// probe side built in the union of the warps' regions.  Phase 2: every warp
// independently takes cost-balanced tasks of records with its own region.
// The CTA's warps take the record's claim batches dynamically from a shared
// cursor, so the barrier closing the record waits for at most one batch.
__device__ unsigned long long* cta_cursor() {
  __shared__ unsigned long long cursor;
  return &cursor;
}

template <AotMode MODE, int U, typename Probe>
__device__ __forceinline__ void cta_claims(const Params& P, const Rec& R, const Probe& probe, uint32_t lmax,
                                           Lane<MODE>& st) {
  unsigned long long* cur = cta_cursor();
  while (true) {
    // batches of 32 claims, then of TL_CTA_TAIL_BS once fewer than
    // TL_CTA_TAIL remain: the closing barrier waits for at most a short batch
    unsigned long long base = 0, bs = 32;
    if (lane_id() == 0) {
      const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(cur);
      if (c + TL_CTA_TAIL >= R.ce) bs = TL_CTA_TAIL_BS;
      base = atomicAdd(cur, bs);
    }
    base = __shfl_sync(kFull, base, 0);
    bs = __shfl_sync(kFull, bs, 0);
    if (base >= R.ce) break;
    claim_batch<MODE, U>(P, probe, lmax, base, min(uint64_t(base + bs), R.ce), st);
  }
}

template <AotMode MODE, int U>
__device__ __forceinline__ void cta_record(const Params& P, const Rec& R, uint32_t cbase, Lane<MODE>& st) {
  const uint32_t* nl = P.col + R.lb;
  const uint32_t lmin = __ldg(nl), lmax = __ldg(nl + R.dl - 1);
  const uint32_t span = lmax - lmin + 1;
  begin_record(st, P, R.l);
  if (threadIdx.x == 0) *cta_cursor() = R.cb;  // published by the barrier after the build
  if (span <= kCtaSpanMax) {
    for (uint32_t i = threadIdx.x; i < R.dl; i += kWarpThreads) bitmap_set(cbase, lmin, __ldg(nl + i));
    __syncthreads();
    cta_claims<MODE, U>(P, R, BitmapProbe{cbase, lmin, span}, lmax, st);
    __syncthreads();
    const uint32_t nwords = (span + 31) >> 5;
    if (nwords <= max(uint32_t(kWarpThreads), 2 * R.dl))
      for (uint32_t i = threadIdx.x; i < nwords; i += kWarpThreads) st_sm(cbase + 4 * i, 0u);
    else
      for (uint32_t i = threadIdx.x; i < R.dl; i += kWarpThreads) bitmap_clear(cbase, lmin, __ldg(nl + i));
  } else if (rank_fits(R.dl, span, kCtaWords)) {
    const RankProbe probe = rank_probe(cbase, lmin, span);
    if (threadIdx.x < 32) rank_build(probe, nl, R.dl, span);
    __syncthreads();
    cta_claims<MODE, U>(P, R, probe, lmax, st);
    __syncthreads();
    const RankLayout L(span);
    for (uint32_t i = threadIdx.x; i < L.words(R.dl); i += kWarpThreads) st_sm(cbase + 4 * i, 0u);
  } else if (R.dl <= kCtaHashDegMax) {
    const uint32_t blg = bucket_lg(R.dl);
    bool done = false;
    if (TL_BUCKET_PROBE && (4u << blg) <= kCtaWords) {
      bool ok = true;
      for (uint32_t i = threadIdx.x; i < R.dl; i += kWarpThreads) ok &= bucket_insert(cbase, 32 - blg, __ldg(nl + i));
      done = __syncthreads_and(ok) != 0;
      if (done) cta_claims<MODE, U>(P, R, BucketProbe{cbase, 32 - blg}, lmax, st);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < (4u << blg); i += kWarpThreads) st_sm(cbase + 4 * i, 0u);
      __syncthreads();
      if (!done && threadIdx.x == 0) *cta_cursor() = R.cb;  // the fallback restarts the record's claims
    }
    if (!done) {
      uint32_t lg = 32 - __clz(2 * R.dl - 1);
      lg = max(5u, min(lg, kCtaWordsLg));
      const uint32_t cap = 1u << lg;
      for (uint32_t i = threadIdx.x; i < R.dl; i += kWarpThreads) hash_insert(cbase, cap - 1, 32 - lg, __ldg(nl + i));
      __syncthreads();
      cta_claims<MODE, U>(P, R, HashProbe{cbase, cap - 1, 32 - lg}, lmax, st);
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < cap; i += kWarpThreads) st_sm(cbase + 4 * i, 0u);
    }
  } else {
    __syncthreads();
    cta_claims<MODE, U>(P, R, GlobalProbe{nl, R.dl}, lmax, st);
  }
  st.fold();
}

template <AotMode MODE, int U>
__global__ void __launch_bounds__(kWarpThreads, MODE == AotMode::count  ? (ring_mode<MODE>() ? TL_RING_CTAS : TL_CTAS_PER_SM)
                                                          : MODE == AotMode::hash ? TL_EMIT_CTAS
                                                                                  : TL_LIST_CTAS) k_aot(Params P) {
  __shared__ unsigned long long s_task;
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  uint32_t wbase = sm_addr(warp * kWarpStride);
#if TL_OPAQUE_BASE
  asm volatile("mov.u32 %0, %0;" : "+r"(wbase));  // held in a register, not rebuilt from SR_CgaCtaId in the hot loop
#endif
  for (uint32_t i = lane; i < kWarpStride; i += 32) st_sm(wbase + 4 * i, 0u);
  if constexpr (TL_EXEC_COUNT)
    if (lane == 0) *reinterpret_cast<volatile unsigned long long*>(__cvta_shared_to_generic(exec_addr())) = 0ull;
  Lane<MODE> st;
  st.ebase = sm_addr(kWarpsPerCta * kWarpStride + warp * (2 * emit_cap<MODE>()));
  if constexpr (ring_mode<MODE>()) {
    constexpr uint32_t off =
        (kWarpsPerCta * kWarpStride + (MODE == AotMode::list ? kWarpsPerCta * 2 * emit_cap<MODE>() : 0) + 31) & ~31u;
    st.bars = sm_addr(off + warp * 2 * kRingStages);
    st.ring = sm_addr(off + ((kWarpsPerCta * 2 * kRingStages + 31) & ~31u) + warp * kRingStages * kRingWords);
    if (lane == 0) {
      for (uint32_t i = 0; i < kRingStages; ++i) mbar_init(st.bars + 8 * i, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  __syncthreads();
  // ---- phase 1: CTA records
  if (P.ncta) {
    uint32_t cbase = sm_addr(0);
#if TL_OPAQUE_BASE
    asm volatile("mov.u32 %0, %0;" : "+r"(cbase));
#endif
    while (true) {
      if (threadIdx.x == 0) s_task = atomicAdd(P.acc + kCtaCounter, 1ull);
      __syncthreads();  // also orders the previous record's clear before the next build
      const unsigned long long t = s_task;
      __syncthreads();
      if (t >= P.ncta) break;
      cta_record<MODE, U>(P, P.crecs[P.toff + t * P.tstride], cbase, st);
    }
  }
  // ---- phase 2: warp tasks
  while (true) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(P.acc + kWarpCounter, 1ull);
    t = __shfl_sync(kFull, t, 0);
    if (t >= P.ntasks) break;
    const uint2 tk = P.tasks[P.gtasks - 1 - (P.toff + t * P.tstride)];  // heaviest pivots (highest ranks) first
    for (uint32_t r = tk.x; r < tk.y; ++r) warp_record<MODE, U>(P, P.recs[r], wbase, st);
  }
  reduce_and_flush(st, P);
}

// ------------------------------------------------------------ work building
#define TL_GRID_STRIDE(i, count) \
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < (count); i += uint64_t(gridDim.x) * blockDim.x)

// rank -> vertex_word(original id) (tl_common.cuh): the hash sink gathers one per triangle
__global__ void k_vertex_words(const uint32_t* orig, uint32_t n, uint64_t* vword) {
  TL_GRID_STRIDE(i, uint64_t(n)) vword[i] = vertex_word(orig[i]);
}

// Claim cost (the window's length, an upper bound of its probes; 0 for a
// skipped negative claim), for claim i < m; 0 at i = m so an exclusive scan of
// m + 1 items ends in the total.
struct WindowLength {
  const uint64_t* win;
  uint64_t m;
  uint32_t skip_neg;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    if (i >= m) return 0;
    const uint64_t w = win[i];
    return (skip_neg && (w >> 63)) ? 0 : (w >> kWinLenShift) & kWinLenMask;
  }
};

__device__ __forceinline__ uint64_t lower_bound_u64(const uint64_t* a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t* a, uint64_t lo, uint64_t hi, uint64_t x) {
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Cost cut of the claim index space: part p owns claims [cut(p), cut(p+1)),
// cut(k) = first i with CP[i] + kKappa*i >= k*Total/nparts.  The parts'
// logical-probe / table-build counters are attributed by this cut; the
// execution is interleaved (aot_run) unless TL_SPLIT_MODE=range.
// out: cb, ce, pb (pivot of cb), pe (one past the pivot of ce-1),
//      vb, ve (pivot range attributed to this part), table_builds.
__global__ void k_split(const uint64_t* CP, uint64_t m, const uint64_t* claim_off, const uint64_t* off, uint32_t n,
                        uint32_t part, uint32_t nparts, uint64_t* out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned __int128 total = (unsigned __int128)CP[m] + (unsigned __int128)kKappa * m;
  auto cut = [&](uint32_t k) -> uint64_t {
    if (k == 0) return 0;
    if (k >= nparts) return m;
    const unsigned __int128 target = total * k / nparts;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = lo + (hi - lo) / 2;
      const unsigned __int128 v = (unsigned __int128)CP[mid] + (unsigned __int128)kKappa * mid;
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
  out[6] = off[out[5]] - off[out[4]];  // table_builds: sum of deg+ over the attributed pivots
}

// Logical probes (engine.hpp:250/:264: one per element of the full traversed
// list) over the part's claims.
__global__ void k_logical(const uint32_t* cs, const uint64_t* off, uint64_t cb, uint64_t ce, uint32_t skip_neg,
                          unsigned long long* acc) {
  unsigned long long sum = 0;
  TL_GRID_STRIDE(k, ce - cb) {
    const uint32_t sflag = cs[cb + k];
    if (!(skip_neg && (sflag & kNegBit))) {
      const uint32_t s = sflag & ~kNegBit;
      sum += off[s + 1] - off[s];
    }
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if ((threadIdx.x & 31) == 0 && sum) atomicAdd(acc, sum);
}

// Traversal ids the listing kernel loads (probes_executed) for the records
// this run executes, by the rule of claim_batch's register path: a window of
// at most kShort ids is loaded whole (packed rounds); a longer one in groups
// of G = 32U ids, group g being loaded iff no earlier group held an id above
// max N+(l) (lists ascend): min(len, G * (g* + 1)) ids, g* = the group of the
// first id above max N+(l).  Windows are nearly tight, so one load of the
// window's last id settles most of them.  One warp per warp task (its records)
// and per CTA record of this part; run once per plan and part, cached.
__device__ __forceinline__ unsigned long long executed_of_record(const Rec& R, const uint64_t* win,
                                                                 const uint32_t* col, uint32_t G, uint32_t skip_neg,
                                                                 uint32_t t0, uint32_t step) {
  unsigned long long sum = 0;
  if (R.dl == 0) return 0;
  const uint32_t lmax = __ldg(col + R.lb + R.dl - 1);
  for (uint64_t c = R.cb + t0; c < R.ce; c += step) {
    const uint64_t wv = win[c];
    if (skip_neg && (wv >> 63)) continue;
    const uint64_t s = wv & kWinBeginMask;
    const uint32_t len = uint32_t((wv >> kWinLenShift) & kWinLenMask);
    if (len <= kShort || __ldg(col + s + len - 1) <= lmax) {
      sum += len;
      continue;
    }
    uint32_t lo = 0, hi = len - 1;  // first position with an id above lmax (the last one is)
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(col + s + mid) <= lmax) lo = mid + 1; else hi = mid;
    }
    sum += min(len, G * (lo / G + 1));
  }
  return sum;
}

// A CTA record (many claims) gets a whole block, a warp task a warp.
__global__ void k_executed(Params P, uint32_t G, unsigned long long* out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t wpb = blockDim.x >> 5, tblocks = (P.ntasks + wpb - 1) / wpb;
  unsigned long long sum = 0;
  for (uint64_t b = blockIdx.x; b < P.ncta + tblocks; b += gridDim.x) {
    if (b < P.ncta) {
      sum += executed_of_record(P.crecs[P.toff + b * P.tstride], P.win, P.col, G, P.skip_neg, threadIdx.x,
                                blockDim.x);
    } else {
      const uint64_t w = (b - P.ncta) * wpb + (threadIdx.x >> 5);
      if (w < P.ntasks) {
        const uint2 tk = P.tasks[P.gtasks - 1 - (P.toff + w * P.tstride)];
        for (uint32_t r = tk.x; r < tk.y; ++r)
          sum += executed_of_record(P.recs[r], P.win, P.col, G, P.skip_neg, lane, 32);
      }
    }
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if (lane == 0 && sum) atomicAdd(out, sum);
}

// Warp path: the span fits the warp bitmap, or a small pivot (warp hash) with
// too little work to occupy a CTA.  Everything else is a phase-1 CTA record.
// (Sending every record whose two-level bitmap fits a warp region to the
// warp path measured the same at C2/C3/C5 and 5% slower at C4.)
__device__ __forceinline__ bool warp_path(uint32_t dl, uint32_t span, uint64_t work) {
  return span <= kWarpSpanMax || (dl <= kWarpHashDegMax && work < kCtaMinWork);
}

// Per pivot of the part: number of warp records / CTA records.
__global__ void k_classify(const uint64_t* CP, const uint64_t* claim_off, const uint64_t* off, const uint32_t* col,
                           uint32_t pb, uint32_t np, uint64_t cb, uint64_t ce, uint64_t T, uint32_t* nrw,
                           uint32_t* nrc) {
  TL_GRID_STRIDE(i, uint64_t(np) + 1) {
    uint32_t nw = 0, nc = 0;
    if (i < np) {
      const uint32_t l = pb + uint32_t(i);
      const uint64_t a = max(claim_off[l], cb), b = min(claim_off[l + 1], ce);
      const uint64_t W = a < b ? CP[b] - CP[a] : 0;
      const uint64_t Wk = W + kKappa * (b - a);  // work incl. per-claim overhead
      const uint64_t lb = off[l];
      const uint32_t dl = uint32_t(off[l + 1] - lb);
      if (W && dl) {
        const uint32_t span = col[lb + dl - 1] - col[lb] + 1;
        if (warp_path(dl, span, Wk))
          nw = uint32_t((Wk + T - 1) / T);
        else
          nc = uint32_t((Wk + kCtaTaskScale * T - 1) / (kCtaTaskScale * T));
      }
    }
    nrw[i] = nw;
    nrc[i] = nc;
  }
}

// Diagnostic (TL_DEBUG_PATHS=1): windowed work W per probe path and per
// log2(span) bucket.  out[0..6] = warp bitmap, warp rank, warp hash, CTA bitmap, CTA rank, CTA
// hash, global search; out[8 + b] = work with ceil(log2(span)) == b.
__global__ void k_path_stats(const uint64_t* CP, const uint64_t* claim_off, const uint64_t* off, const uint32_t* col,
                             uint32_t pb, uint32_t np, uint64_t cb, uint64_t ce, unsigned long long* out) {
  TL_GRID_STRIDE(i, uint64_t(np)) {
    const uint32_t l = pb + uint32_t(i);
    const uint64_t a = max(claim_off[l], cb), b = min(claim_off[l + 1], ce);
    const uint64_t W = a < b ? CP[b] - CP[a] : 0;
    const uint64_t lb = off[l];
    const uint32_t dl = uint32_t(off[l + 1] - lb);
    if (!W || !dl) continue;
    const uint32_t span = col[lb + dl - 1] - col[lb] + 1;
    int path;
    if (span <= kWarpSpanMax) path = 0;
    else if (warp_path(dl, span, W + kKappa * (b - a))) path = rank_fits(dl, span, kWarpWords) ? 1 : 2;
    else if (span <= kCtaSpanMax) path = 3;
    else if (rank_fits(dl, span, kCtaWords)) path = 4;
    else if (dl <= kCtaHashDegMax) path = 5;
    else path = 6;
    atomicAdd(out + path, (unsigned long long)W);
    atomicAdd(out + 8 + (32 - __clz(span - 1 | 1)), (unsigned long long)W);
  }
}

// Record j (one thread each): pivot i = the one whose record range contains
// j; its chunk jj covers the claims whose cost prefix falls in
// [W*jj/k, W*(jj+1)/k).  Warp records also get their scheduling weight.
__global__ void k_records(const uint64_t* CP, const uint64_t* claim_off, const uint64_t* off, uint32_t pb, uint32_t np,
                          uint64_t cb, uint64_t ce, const uint32_t* nr, const uint32_t* nr_off, uint64_t nrec, Rec* recs,
                          uint64_t* weight) {
  TL_GRID_STRIDE(j, nrec) {
    uint32_t lo = 0, hi = np;  // largest i with nr_off[i] <= j
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (nr_off[mid] <= j) lo = mid; else hi = mid;
    }
    const uint32_t i = lo, k = nr[i], jj = uint32_t(j - nr_off[i]);
    const uint32_t l = pb + i;
    const uint64_t a = max(claim_off[l], cb), b = min(claim_off[l + 1], ce);
    // cut at the weighted prefix CP[i] + kKappa * i (monotone in i)
    const uint64_t base = CP[a] + kKappa * a, W = CP[b] + kKappa * b - base;
    auto cut = [&](uint64_t target) {
      uint64_t lo = a, hi = b;
      while (lo < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (CP[mid] + kKappa * mid < target) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    const uint64_t from = jj == 0 ? a : cut(base + (W * jj) / k);
    const uint64_t to = jj + 1 == k ? b : cut(base + (W * (jj + 1)) / k);
    const uint64_t lb = off[l];
    const uint32_t dl = uint32_t(off[l + 1] - lb);
    recs[j] = Rec{lb, from, to, l, dl};
    if (weight) weight[j] = (CP[to] - CP[from]) + kKappa * (to - from) + kBeta * dl + kGamma;
  }
}

// Task g = the warp records whose weight prefix RP lies in [g*T, (g+1)*T).
__global__ void k_tasks(const uint64_t* RP, uint32_t nrec, uint64_t G, uint64_t T, uint2* tasks) {
  TL_GRID_STRIDE(g, G) {
    const uint64_t lo = lower_bound_u64(RP, 0, nrec, g * T);
    const uint64_t hi = g + 1 == G ? nrec : lower_bound_u64(RP, 0, nrec, (g + 1) * T);
    tasks[g] = make_uint2(uint32_t(lo), uint32_t(hi));
  }
}

// Forward claims (kclist3_pivot / cf_merge_pivot, engine.hpp:164-236): the
// claim of edge e = t->h is pivot t traversing all of N+(h).
__global__ void k_fwd_windows(const uint64_t* off, const uint32_t* col, uint64_t m, uint64_t* win) {
  TL_GRID_STRIDE(e, m) {
    const uint32_t h = col[e];
    const uint64_t b = off[h];
    win[e] = b | ((off[h + 1] - b) << kWinLenShift);
  }
}

__device__ __forceinline__ uint32_t count_le(const uint32_t* a, uint32_t len, uint32_t x) {  // #{a[i] <= x}
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (__ldg(a + mid) <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Per-edge counters of the comparison kernels over the out-edges [eb, ee) of
// the vertices [vb, ve), one warp per vertex:
//  * cf-hash table builds (engine.hpp:194-206): the build side of u->v is
//    N+(u) when v precedes u in (deg+, id) order, else N+(v); with
//    cf_hash_reuse_last_table a build of N+(u) is skipped when the previous
//    edge of the list also built N+(u);
//  * cf merge comparisons (engine.hpp:166-181): the merge loop of N+(u) and
//    N+(v) (rank-ascending) runs #{a <= M} + #{b <= M} - |common| times,
//    M = min(max N+(u), max N+(v)); this pass sums the first two terms and
//    the caller subtracts the triangles.
__global__ void k_edge_counters(const uint64_t* off, const uint32_t* col, const uint32_t* orig, uint32_t vb,
                                uint32_t ve, uint64_t eb, uint64_t ee, uint32_t algo, uint32_t reuse,
                                unsigned long long* acc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  unsigned long long sum = 0;
  for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < uint64_t(ve - vb); w += nwarps) {
    const uint32_t u = vb + uint32_t(w);
    const uint64_t ub = off[u], ue = off[u + 1];
    const uint64_t lo = max(ub, eb), hi = min(ue, ee);
    if (lo >= hi) continue;
    const uint32_t du = uint32_t(ue - ub), ou = __ldg(orig + u);
    const uint32_t maxA = __ldg(col + ue - 1);
    auto hash_u = [&](uint32_t v, uint32_t dv) { return dv < du || (dv == du && __ldg(orig + v) < ou); };
    for (uint64_t e = lo + lane; e < hi; e += 32) {
      const uint32_t v = __ldg(col + e);
      const uint64_t vb0 = off[v];
      const uint32_t dv = uint32_t(off[v + 1] - vb0);
      if (algo == uint32_t(Algo::cf_hash)) {
        const bool hu = hash_u(v, dv);
        uint32_t build = hu ? du : dv;
        if (reuse && hu && e > ub) {
          const uint32_t p = __ldg(col + e - 1);
          if (hash_u(p, uint32_t(off[p + 1] - off[p]))) build = 0;
        }
        sum += build;
      } else if (dv) {
        const uint32_t maxB = __ldg(col + vb0 + dv - 1);
        if (maxA <= maxB)
          sum += du + count_le(col + vb0, dv, maxA);
        else
          sum += dv + count_le(col + ub, du, maxB);
      }
    }
  }
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(kFull, sum, o);
  if (lane == 0 && sum) atomicAdd(acc, sum);
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
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// Dynamic shared memory: the warps' probe regions, then (hash / list) the
// warps' hit staging, then (ring modes) the stage mbarriers and the rings.
template <AotMode MODE>
__host__ __device__ constexpr uint32_t ring_words_offset() {  // 32-word (128 B) aligned
  return (kWarpsPerCta * kWarpStride + (MODE == AotMode::list ? kWarpsPerCta * 2 * emit_cap<MODE>() : 0) + 31) & ~31u;
}
template <AotMode MODE>
size_t kernel_smem() {
  uint32_t words = kWarpsPerCta * kWarpStride + (MODE == AotMode::list ? kWarpsPerCta * 2 * emit_cap<MODE>() : 0);
  if (ring_mode<MODE>())
    words = ring_words_offset<MODE>() + ((kWarpsPerCta * 2 * kRingStages + 31) & ~31u) +
            kWarpsPerCta * kRingStages * kRingWords;
  return sizeof(uint32_t) * words;
}

template <AotMode MODE>
constexpr int unroll_long() {
  return MODE == AotMode::count ? kUnrollLong : kUnrollLongEmit;
}

template <AotMode MODE>
int resident_warps() {  // warps of k_aot<MODE, *> the current device keeps resident (cached per device)
  static int cache[64] = {0};
  int dev = 0;
  TL_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  TL_CUDA(cudaFuncSetAttribute(k_aot<MODE, kUnrollShort>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kernel_smem<MODE>())));
  TL_CUDA(cudaFuncSetAttribute(k_aot<MODE, unroll_long<MODE>()>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(kernel_smem<MODE>())));
  int per_sm = 0;
  TL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_aot<MODE, kUnrollShort>, kWarpThreads,
                                                        kernel_smem<MODE>()));
  const int w = sm_count() * std::max(per_sm, 1) * kWarpsPerCta;
  if (dev >= 0 && dev < 64) cache[dev] = w;
  return w;
}

template <AotMode MODE>
uint64_t launch_kernels(const Params& P, bool long_lists, cudaStream_t s) {
  if (!P.ntasks && !P.ncta) return 0;
  const uint64_t ctas = uint64_t(resident_warps<MODE>()) / kWarpsPerCta;
  const uint64_t want = std::max<uint64_t>(P.ncta, (P.ntasks + kWarpsPerCta - 1) / kWarpsPerCta);
  const unsigned grid = unsigned(std::min<uint64_t>(want, ctas));
  if (long_lists)
    k_aot<MODE, unroll_long<MODE>()><<<grid, kWarpThreads, kernel_smem<MODE>(), s>>>(P);
  else
    k_aot<MODE, kUnrollShort><<<grid, kWarpThreads, kernel_smem<MODE>(), s>>>(P);
  TL_CUDA(cudaGetLastError());
  return 1;
}

}  // namespace

// A run's work: warp records + cost-balanced warp tasks, CTA records.
struct AotPlan {
  DBuf<Rec> wrecs, crecs;
  DBuf<uint2> tasks;
  uint64_t nw = 0, nc = 0, G = 0;
  // probes_executed of the part (toff, tstride) at group size G (k_executed)
  std::map<std::tuple<uint32_t, uint32_t, uint32_t>, uint64_t> executed;
};

namespace {
// Builds the work records of claims [cb, ce) (pivots [pb, pe)) at task size T
// into `plan` (buffers on stream ps; the temporaries and kernels on s).
void build_plan(tl_oriented& og, AotPlan& plan, const uint64_t* CP, const uint64_t* claim_off, uint32_t pb,
                uint32_t pe, uint64_t cb, uint64_t ce, uint64_t T, cudaStream_t ps, cudaStream_t s, bool debug_paths,
                uint64_t& launches) {
  const uint32_t np = cb < ce ? pe - pb : 0;
  if (!np) return;
  DBuf<uint32_t> nrw, nrc, ow, oc;
  DBuf<uint64_t> wgt;
  nrw.alloc(np + 1, s);
  nrc.alloc(np + 1, s);
  ow.alloc(np + 1, s);
  oc.alloc(np + 1, s);
  k_classify<<<grid_for(uint64_t(np) + 1, 256, 148u * 32u), 256, 0, s>>>(CP, claim_off, og.off.p, og.col.p, pb, np,
                                                                        cb, ce, T, nrw.p, nrc.p);
  TL_CUDA(cudaGetLastError());
  cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, nrw.p, ow.p, np + 1, s); });
  cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, nrc.p, oc.p, np + 1, s); });
  if (debug_paths) {
    DBuf<unsigned long long> pst;
    pst.alloc(48, s);
    TL_CUDA(cudaMemsetAsync(pst.p, 0, 48 * 8, s));
    k_path_stats<<<grid_for(np, 256, 148u * 32u), 256, 0, s>>>(CP, claim_off, og.off.p, og.col.p, pb, np, cb, ce,
                                                              pst.p);
    unsigned long long hp[48];
    TL_CUDA(cudaMemcpyAsync(hp, pst.p, sizeof(hp), cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    fprintf(stderr,
            "[tl paths] warp-bitmap %llu warp-rank %llu warp-hash %llu cta-bitmap %llu cta-rank %llu cta-hash %llu "
            "global %llu\n",
            hp[0], hp[1], hp[2], hp[3], hp[4], hp[5], hp[6]);
    fprintf(stderr, "[tl span log2 buckets]");
    for (int b = 0; b < 40; ++b)
      if (hp[8 + b]) fprintf(stderr, " %d:%llu", b, hp[8 + b]);
    fprintf(stderr, "\n");
  }
  uint32_t tw = 0, tc = 0;
  TL_CUDA(cudaMemcpyAsync(&tw, ow.p + np, 4, cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaMemcpyAsync(&tc, oc.p + np, 4, cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  plan.nw = tw;
  plan.nc = tc;
  launches += 1 + 2 * 2;
  // plan buffers are allocated on ps, before the kernels on s use them
  if (plan.nw) plan.wrecs.alloc(plan.nw, ps);
  if (plan.nc) plan.crecs.alloc(plan.nc, ps);
  if (ps != s) {
    cudaEvent_t e;
    TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(e, ps));
    TL_CUDA(cudaStreamWaitEvent(s, e, 0));
    cudaEventDestroy(e);
  }
  if (plan.nw) {
    const uint64_t nw = plan.nw;
    wgt.alloc(nw + 1, s);
    TL_CUDA(cudaMemsetAsync(wgt.p + nw, 0, 8, s));
    k_records<<<grid_for(nw, 256, 148u * 32u), 256, 0, s>>>(CP, claim_off, og.off.p, pb, np, cb, ce, nrw.p, ow.p, nw,
                                                            plan.wrecs.p, wgt.p);
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, wgt.p, nw + 1, s); });
    uint64_t total = 0;
    TL_CUDA(cudaMemcpyAsync(&total, wgt.p + nw, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    plan.G = total ? (total - 1) / T + 1 : 0;
    // the task list is written on s; allocate it there and move ownership to ps after
    plan.tasks.alloc(std::max<uint64_t>(plan.G, 1), ps);
    if (ps != s) {
      cudaEvent_t e;
      TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TL_CUDA(cudaEventRecord(e, ps));
      TL_CUDA(cudaStreamWaitEvent(s, e, 0));
      cudaEventDestroy(e);
    }
    if (plan.G) k_tasks<<<grid_for(plan.G, 256, 148u * 32u), 256, 0, s>>>(wgt.p, uint32_t(nw), plan.G, T, plan.tasks.p);
    TL_CUDA(cudaGetLastError());
    launches += 1 + 2 + (plan.G ? 1 : 0);
  }
  if (plan.nc) {
    k_records<<<grid_for(plan.nc, 256, 148u * 32u), 256, 0, s>>>(CP, claim_off, og.off.p, pb, np, cb, ce, nrc.p, oc.p,
                                                                 plan.nc, plan.crecs.p, nullptr);
    TL_CUDA(cudaGetLastError());
    ++launches;
  }
  if (ps != s) {  // the plan's writes are complete before ps may free it
    cudaEvent_t e;
    TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(e, s));
    TL_CUDA(cudaStreamWaitEvent(ps, e, 0));
    cudaEventDestroy(e);
  }
}

void ensure_forward_claims(tl_oriented& og, cudaStream_t s) {
  if (og.fwd_win.p || og.m == 0) return;
  og.fwd_win.alloc(og.m, og.stream);  // owned by the handle's stream
  k_fwd_windows<<<grid_for(og.m, 256, 148u * 64u), 256, 0, og.stream>>>(og.off.p, og.col.p, og.m, og.fwd_win.p);
  TL_CUDA(cudaGetLastError());
  if (s != og.stream) {
    cudaEvent_t ev;
    TL_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(ev, og.stream));
    TL_CUDA(cudaStreamWaitEvent(s, ev, 0));
    cudaEventDestroy(ev);
  }
}
}  // namespace

// One run of `spec.algo` on the device.  aot and cf-hash share the adaptive
// claims (cf-hash traverses the min side and probes the other, engine.hpp:
// 194-215 -- the same pairs of lists as aot_pivot's two phases); kclist3 and
// cf merge use the forward claims (every edge t->h: pivot t, all of N+(h)).
AotResult aot_run(tl_oriented& og, const RunSpec& spec, cudaStream_t s, uint32_t* d_out, uint64_t out_cap) {
  AotResult r;
  const AotMode mode = spec.mode;
  const uint32_t nparts = spec.nparts ? spec.nparts : 1, part = spec.part;
  TL_REQUIRE(part < nparts, TL_EINVAL, "partition index out of range");
  const bool skip_negative = spec.algo == Algo::aot && spec.skip_negative;
  const bool fwd = spec.algo == Algo::kclist3 || spec.algo == Algo::cf_merge;
  const uint64_t m = og.m;
  if (m == 0) return r;
  if (fwd) ensure_forward_claims(og, s);
  const uint64_t* claim_off = fwd ? og.off.p : og.claim_off.p;
  const uint64_t* cwin = fwd ? og.fwd_win.p : og.win.p;
  const uint32_t* cs = fwd ? og.col.p : og.claim_s.p;

  cudaEvent_t ev[3];
  for (auto& e : ev) TL_CUDA(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 3; ++i) cudaEventDestroy(e[i]);
    }
  } evg{ev};
  TL_CUDA(cudaEventRecord(ev[0], s));
  // TL_DEBUG_PREP=1: host-side phase timeline of the task construction
  const bool dbg = getenv("TL_DEBUG_PREP") != nullptr;
  auto t_start = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!dbg) return;
    cudaStreamSynchronize(s);
    fprintf(stderr, "[tl prep] %-12s %8.3f ms\n", what,
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count());
  };

  DBuf<unsigned long long> acc;
  acc.alloc(kAccN, s);
  TL_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long) * kAccN, s));

  // claim-cost prefix CP[0..m]: the exclusive scan of the window lengths,
  // read straight from the packed windows.  A function of the orientation's
  // claims alone (like the claims, built once): kept on the handle for the
  // claim set / fault flag it was built for.
  const uint32_t cp_key = (uint32_t(fwd) << 1) | uint32_t(skip_negative);
  if (!og.cp.p || og.cp_key != cp_key) {
    og.cp.reset();
    og.cp.alloc(m + 1, og.stream);  // owned by the handle's stream
    TL_CUDA(cudaStreamSynchronize(og.stream));
    auto lens =
        thrust::make_transform_iterator(thrust::counting_iterator<uint64_t>(0), WindowLength{cwin, m, skip_negative});
    uint64_t* dst = og.cp.p;
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::ExclusiveSum(t, bytes, lens, dst, m + 1, s); });
    TL_CUDA(cudaMemcpyAsync(&og.cp_total, dst + m, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    og.cp_key = cp_key;
    og.cuts.clear();  // cuts and plans belong to the previous claim set's prefix
    og.plans.clear();
    r.launches += 2;  // scan (init + sweep)
  }
  struct {
    const uint64_t* p;
  } CP{og.cp.p};
  mark("alloc");
  const bool whole = nparts == 1;
  // logical probes (engine.hpp:250/:264): the orientation's cost model when
  // the run covers every claim, else a pass over the part's claims (once per
  // handle and part: the cut and its counters are cached with it)
  const bool logical_from_cost = whole && !skip_negative;
  // Multi-GPU execution: the cut attributes the logical-probe and table-build
  // counters (they only need to partition exactly); with interleaving (the
  // default) every part then works from the whole graph's work records and
  // runs every nparts-th task and CTA record, so each GPU gets an even mix of
  // every probe path.  TL_SPLIT_MODE=range runs the cut's own claim range
  // instead.  cf merge runs its counter cut's own edges (range mode), so a
  // part's merge comparisons (per-edge pass minus the part's triangles) are
  // over one edge set; it is a comparison kernel, not the balanced hot path.
  const char* split_mode = getenv("TL_SPLIT_MODE");
  const bool interleave = !whole && !spec.range && !(split_mode && std::string(split_mode) == "range") &&
                          spec.algo != Algo::cf_merge;
  const bool cache = !spec.range;  // batched listing walks thousands of ranges once each
  // ---- the part's cost cut: {cb, ce, pb, pe, table_builds, logical, has_logical, CP[cb], CP[ce]}
  std::array<uint64_t, 9> cut_local{};
  std::array<uint64_t, 9>* cutp = nullptr;
  const auto cut_key = std::make_tuple(cp_key, whole ? 0u : part, whole ? 1u : nparts);
  if (cache) {
    auto it = og.cuts.find(cut_key);
    if (it != og.cuts.end()) cutp = &it->second;
  }
  if (!cutp) {
    std::array<uint64_t, 9> c{};
    uint64_t hs[8] = {0, m, 0, og.n, 0, 0, m, 0};
    DBuf<uint64_t> split;
    split.alloc(8, s);
    if (!whole) {
      k_split<<<1, 32, 0, s>>>(CP.p, m, claim_off, og.off.p, og.n, part, nparts, split.p);
      TL_CUDA(cudaGetLastError());
      TL_CUDA(cudaMemcpyAsync(hs, split.p, sizeof(hs), cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
      ++r.launches;
    }
    c[0] = hs[0];
    c[1] = hs[1];
    c[2] = hs[2];
    c[3] = hs[3];
    c[4] = hs[6];  // table_builds: sum of deg+ over the attributed pivots (m for the whole graph)
    if (logical_from_cost) {
      c[5] = fwd ? og.cost[1] : og.cost[2];
      c[6] = 1;
    }
    TL_CUDA(cudaMemcpyAsync(&c[7], CP.p + c[0], 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaMemcpyAsync(&c[8], CP.p + c[1], 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    if (cache) {
      cutp = &og.cuts.emplace(cut_key, c).first->second;
    } else {
      cut_local = c;
      cutp = &cut_local;
    }
  }
  std::array<uint64_t, 9>& cut = *cutp;
  const uint64_t ccb = cut[0], cce = cut[1];
  const uint32_t cpb = uint32_t(cut[2]), cpe = uint32_t(cut[3]);
  r.table_builds = cut[4];
  const bool need_logical = cut[6] == 0;
  if (need_logical && ccb < cce) {
    k_logical<<<grid_for(cce - ccb, 256, 148u * 32u), 256, 0, s>>>(cs, og.off.p, ccb, cce, skip_negative,
                                                                   acc.p + kLogical);
    TL_CUDA(cudaGetLastError());
    ++r.launches;
  }
  mark("cut");

  // ---- work records over [cb, ce): the whole graph when interleaving
  const uint64_t cb = interleave ? 0 : ccb, ce = interleave ? m : cce;
  const uint32_t pb = interleave ? 0 : cpb, pe = interleave ? og.n : cpe;
  const uint64_t wsum = interleave ? og.cp_total : cut[8] - cut[7];  // window lengths over [cb, ce)
  // adaptive task size: ~64 warp tasks per resident warp (per part).  A
  // part's work must not depend on the mode: listing sizes its buffer by a
  // counting pass over the same part (and the ranks of one job may run
  // different modes), so a partitioned run sizes tasks for the count
  // kernel's residency in every mode.
  int warps = resident_warps<AotMode::count>();
  if (nparts == 1) {
    switch (mode) {
      case AotMode::count: break;
      case AotMode::hash: warps = resident_warps<AotMode::hash>(); break;
      case AotMode::list: warps = resident_warps<AotMode::list>(); break;
    }
  }
  const uint64_t work = wsum + kKappa * (ce - cb);
  const uint64_t T =
      std::max<uint64_t>(kTaskMin, work / (interleave ? nparts : 1) / (uint64_t(std::max(warps, 1)) * 64));
  const bool long_lists = ce > cb && wsum / (ce - cb) >= TL_LONG_WINDOW;
  mark("task size");

  std::shared_ptr<AotPlan> plan;
  const auto plan_key = std::make_tuple(cp_key, cb, ce, T);
  if (cache) {
    auto it = og.plans.find(plan_key);
    if (it != og.plans.end()) plan = it->second;
  }
  const bool debug_paths = getenv("TL_DEBUG_PATHS") != nullptr;
  if (!plan || debug_paths) {
    plan = std::make_shared<AotPlan>();
    // plan buffers belong to the handle's stream (they may outlive s)
    cudaStream_t ps = cache ? og.stream : s;
    if (ps != s) {
      cudaEvent_t e;
      TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      TL_CUDA(cudaEventRecord(e, s));
      TL_CUDA(cudaStreamWaitEvent(ps, e, 0));
      cudaEventDestroy(e);
    }
    build_plan(og, *plan, CP.p, claim_off, pb, pe, cb, ce, T, ps, s, debug_paths, r.launches);
    if (cache) {
      if (og.plans.size() >= 16) og.plans.clear();
      og.plans[plan_key] = plan;
    }
  }
  const uint64_t nw = plan->nw, nc = plan->nc, G = plan->G;
  mark("records");
  TL_CUDA(cudaEventRecord(ev[1], s));

  Params P{};
  P.off = og.off.p;
  P.col = og.col.p;
  P.win = cwin;
  P.cs = cs;
  P.orig = og.orig.p;
  if (mode == AotMode::hash && !og.vword.p && og.n) {  // the hash sink's vertex words, once per orientation
    og.vword.alloc(og.n, s);
    k_vertex_words<<<grid_for(og.n, 256, 148u * 64u), 256, 0, s>>>(og.orig.p, og.n, og.vword.p);
    TL_CUDA(cudaGetLastError());
    ++r.launches;
  }
  P.vword = og.vword.p;
  {  // an L2-resident CSR (C2) gains nothing from L2 prefetches and pays their issue slots (C2 list +3%)
    static int l2_bytes[64] = {0};
    int dev = 0;
    TL_CUDA(cudaGetDevice(&dev));
    int& l2 = l2_bytes[dev >= 0 && dev < 64 ? dev : 0];
    if (!l2) TL_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    P.prefetch = 4 * m > uint64_t(l2) ? 1u : 0u;
  }
  P.skip_neg = skip_negative;
  P.swap_neg = spec.algo == Algo::cf_hash;
  P.acc = acc.p;
  P.out = d_out;
  P.out_cap = out_cap;
  P.recs = plan->wrecs.p;
  P.tasks = plan->tasks.p;
  P.gtasks = G;
  P.crecs = plan->crecs.p;
  P.toff = interleave ? part : 0;
  P.tstride = interleave ? nparts : 1;
  P.ntasks = G > P.toff ? (G - P.toff + P.tstride - 1) / P.tstride : 0;
  P.ncta = nc > P.toff ? (nc - P.toff + P.tstride - 1) / P.tstride : 0;
  // probes_executed of the records this part runs, at this run's group size:
  // once per plan and part, on the handle's side stream overlapped with the
  // listing kernel; s joins it before the counters are read back
  const uint32_t group =
      32u * uint32_t(long_lists ? (mode == AotMode::count ? kUnrollLong : kUnrollLongEmit) : kUnrollShort);
  const auto exec_key = std::make_tuple(P.toff, P.tstride, group);
  auto exec_it = plan->executed.find(exec_key);
  const bool need_executed = !TL_EXEC_COUNT && exec_it == plan->executed.end();
  cudaEvent_t exec_done = nullptr;
  struct ExecEvGuard {
    cudaEvent_t& e;
    ~ExecEvGuard() {
      if (e) cudaEventDestroy(e);
    }
  } exec_guard{exec_done};
  if (need_executed && P.ntasks + P.ncta) {
    if (!og.aux) TL_CUDA(cudaStreamCreateWithFlags(&og.aux, cudaStreamNonBlocking));
    cudaEvent_t ready;
    TL_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(ready, s));  // acc zeroed, the plan built
    TL_CUDA(cudaStreamWaitEvent(og.aux, ready, 0));
    cudaEventDestroy(ready);
    k_executed<<<unsigned(std::min<uint64_t>(P.ncta + (P.ntasks + 7) / 8, 148u * 64u)), 256, 0, og.aux>>>(
        P, group, acc.p + kExec);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaEventCreateWithFlags(&exec_done, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(exec_done, og.aux));
    ++r.launches;
  }
  switch (mode) {
    case AotMode::count: r.launches += launch_kernels<AotMode::count>(P, long_lists, s); break;
    case AotMode::hash: r.launches += launch_kernels<AotMode::hash>(P, long_lists, s); break;
    case AotMode::list: r.launches += launch_kernels<AotMode::list>(P, long_lists, s); break;
  }
  if (spec.algo == Algo::cf_hash || spec.algo == Algo::cf_merge) {
    // edges of this part: the claim range for forward claims (claim index =
    // edge index), a vertex share for the adaptive claims of cf-hash
    uint32_t vb = 0, ve = og.n;
    uint64_t eb = 0, ee = m;
    if (fwd) {  // the counter cut's claims (= edges)
      vb = ccb < cce ? cpb : 0;
      ve = ccb < cce ? cpe : 0;
      eb = ccb;
      ee = cce;
    } else if (nparts > 1) {
      vb = uint32_t(uint64_t(og.n) * part / nparts);
      ve = uint32_t(uint64_t(og.n) * (part + 1) / nparts);
    }
    if (vb < ve) {
      k_edge_counters<<<grid_for(uint64_t(ve - vb) * 32, 256, 148u * 64u), 256, 0, s>>>(
          og.off.p, og.col.p, og.orig.p, vb, ve, eb, ee, uint32_t(spec.algo), spec.reuse, acc.p + kEdgeCounter);
      TL_CUDA(cudaGetLastError());
      ++r.launches;
    }
  }
  TL_CUDA(cudaEventRecord(ev[2], s));
  if (exec_done) TL_CUDA(cudaStreamWaitEvent(s, exec_done, 0));
  unsigned long long h[kAccN];
  TL_CUDA(cudaMemcpyAsync(h, acc.p, sizeof(h), cudaMemcpyDeviceToHost, s));
  TL_CUDA(cudaStreamSynchronize(s));
  TL_CUDA(cudaEventElapsedTime(&r.prep_ms, ev[0], ev[1]));
  TL_CUDA(cudaEventElapsedTime(&r.list_ms, ev[1], ev[2]));
  r.positive = h[kPos];
  r.negative = h[kNeg];
  // traversal ids loaded (after the rank-window pruning and the early exit)
  if (need_executed) exec_it = plan->executed.emplace(exec_key, h[kExec]).first;
  r.executed = TL_EXEC_COUNT ? h[kExec] : exec_it->second;
  r.windowed = cut[8] - cut[7];
  if (need_logical) {
    cut[5] = h[kLogical];
    cut[6] = 1;
  }
  r.logical = cut[5];
  r.hash_sum = h[kHsum];
  r.hash_xor = h[kHxor];
  r.emitted = h[kEmitted];
  r.tasks = P.ntasks + P.ncta;
  r.triangles = r.positive + r.negative;
  switch (spec.algo) {  // the counters each kernel keeps (engine.hpp:164-276)
    case Algo::aot:
      r.probes = r.logical;
      r.report_positive = r.positive;
      r.report_negative = r.negative;
      break;
    case Algo::kclist3:
      r.probes = r.logical;  // sum of deg+(head) = kclist_cost
      break;
    case Algo::cf_hash:
      r.probes = r.logical;  // sum of min(deg+) = aot_cost
      r.table_builds = h[kEdgeCounter];
      break;
    case Algo::cf_merge:
      r.table_builds = 0;
      r.merge_comparisons = h[kEdgeCounter] - r.triangles;
      break;
  }
  return r;
}

}  // namespace tlb
