// tl_parse.cu -- edge-list ingestion on sm_100a: load_edge_list /
// load_edge_list_text / load_edge_list_file (reference graph.cpp:40-146,
// :240-275) feeding Graph::from_edges on the device.
//
// The text is uploaded once; line starts come from one device select over the
// '\n' positions; each line is parsed by one thread with the reference's rules
// (graph.cpp:61-101): leading whitespace, comment prefixes, a '-' is a negative
// id, std::from_chars digits with overflow = malformed, two ids, nothing after
// them, one-indexed shift (0 rejected), 32-bit range unless compacting.  The
// reference stops at the first bad line; here every line is checked in
// parallel and the smallest failing line number wins (atomicMin), which is the
// same line and message.  Compaction renumbers ids by first appearance
// (graph.cpp:103-120) with two stable radix sorts.  Self-loops are dropped at
// parse time (graph.cpp:94-97), so, as in the reference, they do not count
// towards n.  gzip / stdin are inflated on the host with zlib (text I/O only).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <zlib.h>

#include <cstdio>
#include <string>
#include <vector>

#include "tl_internal.cuh"

namespace tlb {

namespace {

constexpr unsigned kBlock = 256;
constexpr uint64_t kNoError = ~0ull;
constexpr uint64_t kMaxVertexId = 0xFFFFFFFEull;  // graph.cpp:27

enum ParseCode : uint32_t {
  kNegative = 1,
  kMalformed = 2,
  kTwoIds = 3,
  kTrailing = 4,
  kZeroOneIndexed = 5,
  kRange = 6,
};

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

struct CommentMask {
  uint32_t bits[8];
  __device__ __forceinline__ bool has(uint8_t c) const { return (bits[c >> 5] >> (c & 31)) & 1u; }
};

__device__ __forceinline__ bool is_space(uint8_t c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

__global__ void k_line_flags(const uint8_t* text, uint64_t len, uint8_t* flags) {
  TL_GRID_STRIDE(i, len) flags[i] = (i == 0 || text[i - 1] == '\n');
}

// graph.cpp:38-55 parse_id: returns false with *code set on a bad token.
__device__ __forceinline__ bool parse_id(const uint8_t* text, uint64_t& p, uint64_t end, uint64_t& value,
                                         uint32_t& code) {
  if (p < end && text[p] == '-') {
    code = kNegative;
    return false;
  }
  uint64_t v = 0;
  uint32_t digits = 0;
  bool overflow = false;
  while (p < end && text[p] >= '0' && text[p] <= '9') {
    const uint64_t d = text[p] - '0';
    if (v > (~0ull - d) / 10) overflow = true;
    v = v * 10 + d;
    ++p;
    ++digits;
  }
  if (!digits || overflow || (p < end && !is_space(text[p]))) {
    code = kMalformed;
    return false;
  }
  value = v;
  return true;
}

// One thread per line (graph.cpp:61-101).  kind: 0 none, 1 edge, 2 self-loop.
__global__ void k_parse(const uint8_t* text, uint64_t len, const uint64_t* starts, uint64_t L, CommentMask comments,
                        uint32_t one_indexed, uint32_t compact, ulonglong2* edges, uint8_t* kind, uint64_t* tokpos,
                        unsigned long long* err, unsigned long long* counts) {
  unsigned long long parsed = 0, loops = 0;
  TL_GRID_STRIDE(j, L) {
    uint64_t p = starts[j];
    const uint64_t end = j + 1 < L ? starts[j + 1] : len;
    uint8_t k = 0;
    uint32_t code = 0;
    uint64_t tok = 0, u = 0, v = 0;
    while (p < end && is_space(text[p])) ++p;
    if (p < end && !comments.has(text[p])) {
      tok = p;
      if (parse_id(text, p, end, u, code)) {
        while (p < end && is_space(text[p])) ++p;
        if (p == end) {
          code = kTwoIds;
        } else {
          tok = p;
          if (parse_id(text, p, end, v, code)) {
            while (p < end && is_space(text[p])) ++p;
            if (p != end) {
              code = kTrailing;
            } else if (one_indexed && (u == 0 || v == 0)) {
              code = kZeroOneIndexed;
            } else {
              if (one_indexed) {
                --u;
                --v;
              }
              if (!compact && (u > kMaxVertexId || v > kMaxVertexId)) code = kRange;
            }
          }
        }
      }
      if (code) {
        tokpos[j] = tok;
        atomicMin(err, ((j + 1) << 8) | code);
      } else {
        ++parsed;
        k = u == v ? 2 : 1;
        loops += u == v;
        edges[j] = make_ulonglong2(u, v);
      }
    }
    kind[j] = k;
  }
  for (int o = 16; o; o >>= 1) {
    parsed += __shfl_xor_sync(0xFFFFFFFFu, parsed, o);
    loops += __shfl_xor_sync(0xFFFFFFFFu, loops, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (parsed) atomicAdd(counts, parsed);
    if (loops) atomicAdd(counts + 1, loops);
  }
}

struct IsEdge {
  __device__ __forceinline__ bool operator()(uint8_t k) const { return k == 1; }
};

// Verbatim ids: to uint32 pairs, n = largest id + 1 (graph.cpp:121-128).
__global__ void k_verbatim(const ulonglong2* e, uint64_t count, uint2* pairs, unsigned long long* max_id) {
  unsigned long long mx = 0;
  TL_GRID_STRIDE(i, count) {
    const ulonglong2 x = e[i];
    pairs[i] = make_uint2(uint32_t(x.x), uint32_t(x.y));
    mx = max(mx, (unsigned long long)max(x.x, x.y) + 1);
  }
  for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xFFFFFFFFu, mx, o));
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(max_id, mx);
}

// Compaction: endpoint 2i / 2i+1 of edge i, keyed by raw id.
__global__ void k_endpoints(const ulonglong2* e, uint64_t count, uint64_t* key, uint64_t* pos) {
  TL_GRID_STRIDE(i, count) {
    key[2 * i] = e[i].x;
    key[2 * i + 1] = e[i].y;
    pos[2 * i] = 2 * i;
    pos[2 * i + 1] = 2 * i + 1;
  }
}

// Run heads of the id-sorted endpoints: the first element of a run carries the
// id's first appearance (stable sort over ascending positions).
__global__ void k_run_heads(const uint64_t* key, const uint64_t* pos, uint64_t count, uint64_t* run_of,
                            uint64_t* head_pos, uint64_t* run_id, const uint64_t* run_scan) {
  TL_GRID_STRIDE(i, count) {
    const uint64_t r = run_scan[i] - 1;  // inclusive scan of head flags
    run_of[i] = r;
    if (i == 0 || key[i] != key[i - 1]) {
      head_pos[r] = pos[i];
      run_id[r] = r;
    }
  }
}

__global__ void k_head_flags(const uint64_t* key, uint64_t count, uint64_t* flag) {
  TL_GRID_STRIDE(i, count) flag[i] = (i == 0 || key[i] != key[i - 1]);
}

__global__ void k_new_ids(const uint64_t* runs_by_appearance, uint64_t D, uint32_t* new_id) {
  TL_GRID_STRIDE(i, D) new_id[runs_by_appearance[i]] = uint32_t(i);
}

__global__ void k_scatter_dense(const uint64_t* pos, const uint64_t* run_of, const uint32_t* new_id, uint64_t count,
                                uint32_t* dense) {
  TL_GRID_STRIDE(i, count) dense[pos[i]] = new_id[run_of[i]];
}

std::string error_message(uint32_t code, const char* text, uint64_t len, uint64_t tok) {
  switch (code) {
    case kNegative: return "negative vertex id";
    case kMalformed: {  // graph.cpp:46-49: up to 16 chars of the token
      uint64_t stop = tok;
      auto space = [](char c) { return c == ' ' || (c >= '\t' && c <= '\r'); };
      while (stop < len && !space(text[stop]) && stop - tok < 16) ++stop;
      return "malformed vertex id '" + std::string(text + tok, stop - tok) + "'";
    }
    case kTwoIds: return "expected two vertex ids";
    case kTrailing: return "unexpected trailing content";
    case kZeroOneIndexed: return "vertex id 0 in one-indexed input";
    case kRange: return "vertex id exceeds 32-bit range; use compact ids";
  }
  return "parse error";
}

}  // namespace

ParseFailure::ParseFailure(uint64_t line_no, const std::string& msg)
    : TlError(TL_EPARSE, "line " + std::to_string(line_no) + ": " + msg), line(line_no) {}

void graph_from_text(tl_graph& g, const char* text, uint64_t len, uint32_t flags, const char* comment_prefixes,
                     tl_load_diag* diag) {
  cudaStream_t s = g.stream;
  CommentMask cm{};
  for (const char* c = comment_prefixes ? comment_prefixes : "#%"; *c; ++c) {
    const uint8_t b = uint8_t(*c);
    cm.bits[b >> 5] |= 1u << (b & 31);
  }
  const bool one_indexed = flags & TL_LOAD_ONE_INDEXED, compact = flags & TL_LOAD_COMPACT_IDS;
  tl_load_diag d{};
  DBuf<uint8_t> dtext;
  dtext.alloc(std::max<uint64_t>(len, 1), s);
  if (len) TL_CUDA(cudaMemcpyAsync(dtext.p, text, len, cudaMemcpyHostToDevice, s));
  // line starts
  DBuf<uint8_t> lflags;
  DBuf<uint64_t> starts, nsel;
  lflags.alloc(std::max<uint64_t>(len, 1), s);
  starts.alloc(std::max<uint64_t>(len, 1), s);
  nsel.alloc(1, s);
  uint64_t L = 0;
  if (len) {
    k_line_flags<<<grid_for(len, kBlock, 148u * 64u), kBlock, 0, s>>>(dtext.p, len, lflags.p);
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) {
      return cub::DeviceSelect::Flagged(t, bytes, thrust::counting_iterator<uint64_t>(0), lflags.p, starts.p, nsel.p,
                                        int64_t(len), s);
    });
    TL_CUDA(cudaMemcpyAsync(&L, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
  }
  lflags.reset();
  d.lines_read = L;
  // parse
  DBuf<ulonglong2> edges, kept;
  DBuf<uint8_t> kind;
  DBuf<uint64_t> tokpos;
  DBuf<unsigned long long> scal;
  scal.alloc(4, s);
  TL_CUDA(cudaMemsetAsync(scal.p, 0, 32, s));
  TL_CUDA(cudaMemsetAsync(scal.p, 0xFF, 8, s));  // err = no error
  uint64_t E = 0;
  if (L) {
    edges.alloc(L, s);
    kind.alloc(L, s);
    tokpos.alloc(L, s);
    k_parse<<<grid_for(L, kBlock, 148u * 64u), kBlock, 0, s>>>(dtext.p, len, starts.p, L, cm, one_indexed, compact,
                                                             edges.p, kind.p, tokpos.p, scal.p, scal.p + 1);
    TL_CUDA(cudaGetLastError());
    unsigned long long h[3];
    TL_CUDA(cudaMemcpyAsync(h, scal.p, 24, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    if (h[0] != kNoError) {
      const uint64_t line = h[0] >> 8;
      uint64_t tok = 0;
      TL_CUDA(cudaMemcpyAsync(&tok, tokpos.p + (line - 1), 8, cudaMemcpyDeviceToHost, s));
      TL_CUDA(cudaStreamSynchronize(s));
      throw ParseFailure(line, error_message(uint32_t(h[0] & 0xFF), text, len, tok));
    }
    d.edges_parsed = h[1];
    d.self_loops_dropped = h[2];
    kept.alloc(L, s);
    cub_call(s, [&](void* t, size_t& bytes) {
      return cub::DeviceSelect::FlaggedIf(t, bytes, edges.p, kind.p, kept.p, nsel.p, int64_t(L), IsEdge{}, s);
    });
    TL_CUDA(cudaMemcpyAsync(&E, nsel.p, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
  }
  edges.reset();
  kind.reset();
  tokpos.reset();
  starts.reset();
  dtext.reset();
  DBuf<uint32_t> pairs;
  pairs.alloc(std::max<uint64_t>(2 * E, 2), s);
  uint64_t n = 0;
  if (E && !compact) {
    TL_CUDA(cudaMemsetAsync(scal.p + 3, 0, 8, s));
    k_verbatim<<<grid_for(E, kBlock, 148u * 64u), kBlock, 0, s>>>(kept.p, E, reinterpret_cast<uint2*>(pairs.p),
                                                                scal.p + 3);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaMemcpyAsync(&n, scal.p + 3, 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
  } else if (E) {  // graph.cpp:107-118: renumber by first appearance
    const uint64_t N2 = 2 * E;
    DBuf<uint64_t> key, key2, pos, pos2;
    key.alloc(N2, s);
    key2.alloc(N2, s);
    pos.alloc(N2, s);
    pos2.alloc(N2, s);
    k_endpoints<<<grid_for(E, kBlock, 148u * 64u), kBlock, 0, s>>>(kept.p, E, key.p, pos.p);
    TL_CUDA(cudaGetLastError());
    {
      cub::DoubleBuffer<uint64_t> dk(key.p, key2.p), dv(pos.p, pos2.p);
      cub_call(s, [&](void* t, size_t& bytes) {
        return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, N2, 0, 64, s);
      });
      if (dk.Current() != key.p) key.swap(key2);
      if (dv.Current() != pos.p) pos.swap(pos2);
    }
    // run ids (inclusive scan of head flags), first position of each run
    DBuf<uint64_t> scan, run_of;
    scan.alloc(N2, s);
    run_of.alloc(N2, s);
    k_head_flags<<<grid_for(N2, kBlock, 148u * 64u), kBlock, 0, s>>>(key.p, N2, key2.p);
    TL_CUDA(cudaGetLastError());
    cub_call(s, [&](void* t, size_t& bytes) { return cub::DeviceScan::InclusiveSum(t, bytes, key2.p, scan.p, N2, s); });
    uint64_t D = 0;
    TL_CUDA(cudaMemcpyAsync(&D, scan.p + (N2 - 1), 8, cudaMemcpyDeviceToHost, s));
    TL_CUDA(cudaStreamSynchronize(s));
    TL_REQUIRE(D <= kMaxVertexId + 1, TL_ELENGTH, "too many distinct vertices for 32-bit ids");
    DBuf<uint64_t> head_pos, run_id, hp2, ri2;
    head_pos.alloc(D, s);
    run_id.alloc(D, s);
    k_run_heads<<<grid_for(N2, kBlock, 148u * 64u), kBlock, 0, s>>>(key.p, pos.p, N2, run_of.p, head_pos.p, run_id.p,
                                                                  scan.p);
    TL_CUDA(cudaGetLastError());
    key.reset();
    key2.reset();
    scan.reset();
    hp2.alloc(D, s);
    ri2.alloc(D, s);
    {
      cub::DoubleBuffer<uint64_t> dk(head_pos.p, hp2.p), dv(run_id.p, ri2.p);
      cub_call(s, [&](void* t, size_t& bytes) {
        return cub::DeviceRadixSort::SortPairs(t, bytes, dk, dv, D, 0, int(bits_for(N2) + 1), s);
      });
      if (dv.Current() != run_id.p) run_id.swap(ri2);
    }
    DBuf<uint32_t> new_id;
    new_id.alloc(D, s);
    k_new_ids<<<grid_for(D, kBlock, 148u * 64u), kBlock, 0, s>>>(run_id.p, D, new_id.p);
    k_scatter_dense<<<grid_for(N2, kBlock, 148u * 64u), kBlock, 0, s>>>(pos.p, run_of.p, new_id.p, N2, pairs.p);
    TL_CUDA(cudaGetLastError());
    TL_CUDA(cudaStreamSynchronize(s));
    n = D;
  }
  kept.reset();
  TL_REQUIRE(n <= kMaxVertexId + 1, TL_EINVAL, "vertex count exceeds 32-bit ids");
  graph_from_pairs(g, pairs.p, E, uint32_t(n));
  TL_CUDA(cudaStreamSynchronize(s));
  d.duplicates_dropped = g.duplicates;
  if (diag) *diag = d;
}

std::string read_text_file(const std::string& path) {  // graph.cpp:250-275, gzip-transparent
  gzFile f = path == "-" ? gzdopen(0, "rb") : gzopen(path.c_str(), "rb");
  if (!f) throw TlError(TL_EIO, "cannot open '" + path + "'");
  struct Closer {
    gzFile f;
    ~Closer() { gzclose(f); }
  } closer{f};
  gzbuffer(f, 1 << 20);
  std::string out;
  std::vector<char> buf(1 << 22);
  while (true) {
    const int got = gzread(f, buf.data(), unsigned(buf.size()));
    if (got < 0) {
      int err = 0;
      const char* msg = gzerror(f, &err);
      throw TlError(TL_EIO, "error reading '" + path + "': " + (msg ? msg : ""));
    }
    if (got == 0) break;
    out.append(buf.data(), size_t(got));
  }
  return out;
}

}  // namespace tlb
