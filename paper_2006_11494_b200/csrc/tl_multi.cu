// tl_multi.cu -- one process, several GPUs: the oriented graph replicated on
// a device list, the run's directed edges split into cost-balanced parts (one
// per device), and the per-device results combined over NVLink by NCCL.
//
// Reference semantics: run_parallel (parallel.hpp:25-78) with ParallelConfig
// (parallel.hpp:14-17) as the only knob; counters are the sums of the parts'
// (parallel.hpp:74-75) and identical for any split (test_parallel.cpp:11-40).
// Here part d of ndev is aot_run's cost cut (tl_aot.cu k_split + interleaved
// work records), each device works on its own replica with no exchange during
// compute, and the only communication is
//   * ncclAllReduce(sum, uint64) of the counters and the hash sum,
//   * ncclAllGather of the per-device hash xor (NCCL has no XOR) and of the
//     per-device emission counts (-> each device's listing offset),
// folded by tl_fold_parts, the same host function a torch.distributed caller
// uses.  NCCL is loaded at run time (dlopen): the library has no link-time
// NCCL dependency, and a process that already loaded NCCL (PyTorch) shares
// that copy -- a process that loads PyTorch should import it first.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tl_internal.cuh"

struct tl_multi {
  std::vector<int> devs;
  std::vector<tl_oriented*> reps;  // reps[d] on devs[d]
  std::vector<bool> owned;         // false: the caller's handle, borrowed
  std::vector<ncclComm_t> comms;
  std::vector<cudaStream_t> streams;               // per device: the collectives' own streams
  std::vector<tlb::DBuf<unsigned long long>> red;  // per device (on streams[d]): 8 sums + ndev xors + ndev counts
  ~tl_multi();
};

namespace tlb {
namespace {

struct Nccl {
  decltype(&ncclCommInitAll) comm_init_all = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclAllGather) all_gather = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  std::string load_error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    // an NCCL the process already loaded (PyTorch's) first, then TL_NCCL_LIB,
    // then the system library -- loading a second copy of libnccl.so.2 first
    // would shadow a framework's newer one
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* path = getenv("TL_NCCL_LIB")) h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      n.load_error = std::string("NCCL not available: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(sym("ncclCommInitAll"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    if (!n.comm_init_all || !n.comm_destroy || !n.all_reduce || !n.all_gather || !n.group_start || !n.group_end)
      n.load_error = "NCCL library lacks the collectives this path needs";
  });
  if (!n.load_error.empty()) throw TlError(TL_ECUDA, n.load_error);
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) {
    const char* msg = nccl().error_string ? nccl().error_string(r) : "unknown";
    throw TlError(TL_ECUDA, std::string(what) + ": NCCL error " + std::to_string(int(r)) + " (" + msg + ")");
  }
}

// The counters aot_run reports, in the order they are reduced.
enum : int { kSumTri, kSumPos, kSumNeg, kSumProbes, kSumExec, kSumBuilds, kSumMerge, kSumHash, kNSums };

void to_sums(const AotResult& r, unsigned long long* v) {
  v[kSumTri] = r.triangles;
  v[kSumPos] = r.report_positive;
  v[kSumNeg] = r.report_negative;
  v[kSumProbes] = r.probes;
  v[kSumExec] = r.executed;
  v[kSumBuilds] = r.table_builds;
  v[kSumMerge] = r.merge_comparisons;
  v[kSumHash] = r.hash_sum;
}

// Replica of og on `device`: the resident buffers copied device to device
// (over NVLink when the devices are peers; the claims are a function of the
// graph, so the replica needs no rebuild).
tl_oriented* replicate(const tl_oriented& og, int device) {
  DeviceGuard guard(device);
  ensure_device_setup(device);
  auto r = std::make_unique<tl_oriented>();
  r->device = device;
  TL_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
  r->n = og.n;
  r->nb = og.nb;
  r->m = og.m;
  r->max_out_degree = og.max_out_degree;
  std::copy(og.cost, og.cost + 3, r->cost);
  auto copy = [&](auto& dst, const auto& src) {
    if (!src.p) return;
    dst.alloc(src.n, r->stream);
    TL_CUDA(cudaMemcpyPeerAsync(dst.p, device, src.p, og.device, sizeof(*src.p) * src.n, r->stream));
  };
  copy(r->off, og.off);
  copy(r->col, og.col);
  copy(r->orig, og.orig);
  copy(r->rank, og.rank);
  copy(r->claim_off, og.claim_off);
  copy(r->win, og.win);
  copy(r->claim_s, og.claim_s);
  TL_CUDA(cudaStreamSynchronize(r->stream));
  return r.release();
}

// Runs part d of ndev of `spec` on every replica, one host thread per device.
std::vector<AotResult> run_parts(tl_multi& mg, RunSpec spec, const std::vector<uint32_t*>& outs,
                                 const std::vector<uint64_t>& caps) {
  const int nd = int(mg.devs.size());
  std::vector<AotResult> res(nd);
  std::vector<std::exception_ptr> err(nd);
  std::vector<std::thread> th;
  for (int d = 0; d < nd; ++d)
    th.emplace_back([&, d] {
      try {
        DeviceGuard guard(mg.devs[d]);
        RunSpec sp = spec;
        sp.part = uint32_t(d);
        sp.nparts = uint32_t(nd);
        tl_oriented& rep = *mg.reps[d];
        res[d] = aot_run(rep, sp, rep.stream, outs.empty() ? nullptr : outs[d], caps.empty() ? 0 : caps[d]);
      } catch (...) {
        err[d] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
  return res;
}

// NCCL: every device contributes its sums, its xor and its emission count;
// afterwards every device holds the totals, all xors and all counts.  The
// device-0 copy is read back and folded.
void reduce_parts(tl_multi& mg, const std::vector<AotResult>& parts, tl_stats* out, std::vector<uint64_t>* offsets) {
  const int nd = int(mg.devs.size());
  const Nccl& N = nccl();
  const size_t words = kNSums + 2 * size_t(nd);
  for (int d = 0; d < nd; ++d) {
    DeviceGuard guard(mg.devs[d]);
    std::vector<unsigned long long> h(words, 0);
    to_sums(parts[d], h.data());
    h[kNSums + d] = parts[d].hash_xor;       // gathered into slot d
    h[kNSums + nd + d] = parts[d].emitted ? parts[d].emitted : parts[d].triangles;
    TL_CUDA(cudaMemcpyAsync(mg.red[d].p, h.data(), words * 8, cudaMemcpyHostToDevice, mg.streams[d]));
  }
  nccl_check(N.group_start(), "ncclGroupStart");
  for (int d = 0; d < nd; ++d) {
    cudaStream_t st = mg.streams[d];
    unsigned long long* b = mg.red[d].p;
    nccl_check(N.all_reduce(b, b, kNSums, ncclUint64, ncclSum, mg.comms[d], st), "ncclAllReduce");
    nccl_check(N.all_gather(b + kNSums + d, b + kNSums, 1, ncclUint64, mg.comms[d], st), "ncclAllGather(xor)");
    nccl_check(N.all_gather(b + kNSums + nd + d, b + kNSums + nd, 1, ncclUint64, mg.comms[d], st),
               "ncclAllGather(counts)");
  }
  nccl_check(N.group_end(), "ncclGroupEnd");
  std::vector<unsigned long long> h(words);
  {
    DeviceGuard guard(mg.devs[0]);
    TL_CUDA(cudaMemcpyAsync(h.data(), mg.red[0].p, words * 8, cudaMemcpyDeviceToHost, mg.streams[0]));
    TL_CUDA(cudaStreamSynchronize(mg.streams[0]));
  }
  for (int d = 1; d < nd; ++d) {
    DeviceGuard guard(mg.devs[d]);
    TL_CUDA(cudaStreamSynchronize(mg.streams[d]));
  }
  // per-part stats as the devices reported them, the collective's sums checked against the host fold
  std::vector<tl_stats> ps(nd);
  for (int d = 0; d < nd; ++d) {
    fill_stats_from(parts[d], &ps[d]);
    ps[d].hash_xor = h[kNSums + d];  // the gathered xor (what device d contributed)
  }
  std::vector<uint64_t> offs(nd);
  TL_REQUIRE(tl_fold_parts(ps.data(), uint32_t(nd), out, offs.data()) == TL_OK, TL_ELOGIC, tl_last_error());
  const uint64_t sums[kNSums] = {out->triangles, out->positive_triangles, out->negative_triangles, out->probes,
                                 out->probes_executed, out->table_builds, out->merge_comparisons, out->hash_sum};
  for (int k = 0; k < kNSums; ++k)
    TL_REQUIRE(h[k] == sums[k], TL_ELOGIC, "NCCL all-reduce disagrees with the per-device counters");
  for (int d = 0; d < nd; ++d)
    TL_REQUIRE(h[kNSums + nd + d] == (parts[d].emitted ? parts[d].emitted : parts[d].triangles), TL_ELOGIC,
               "NCCL all-gather of the emission counts disagrees");
  if (offsets) *offsets = offs;
}

}  // namespace
}  // namespace tlb

tl_multi::~tl_multi() {
  if (!comms.empty() && tlb::nccl().comm_destroy)
    for (auto c : comms)
      if (c) tlb::nccl().comm_destroy(c);
  // never touches a borrowed handle: it may already be gone (garbage collectors
  // do not order finalizers)
  for (size_t d = 0; d < devs.size(); ++d) {
    tlb::DeviceGuard guard(devs[d]);
    if (d < red.size()) red[d].reset();
    if (d < streams.size() && streams[d]) {
      cudaStreamSynchronize(streams[d]);
      cudaStreamDestroy(streams[d]);
    }
    if (d < reps.size() && owned[d]) delete reps[d];
  }
}

namespace {
template <typename F>
int guarded_multi(F&& f) {
  try {
    f();
    return TL_OK;
  } catch (const tlb::TlError& e) {
    tlb::set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc& e) {
    tlb::set_last_error(std::string("host allocation failed: ") + e.what());
    return TL_ENOMEM;
  } catch (const std::exception& e) {
    tlb::set_last_error(e.what());
    return TL_ECUDA;
  }
}

tlb::RunSpec multi_spec(const tl_run_options* opt, tlb::AotMode mode) {
  tlb::RunSpec sp;
  if (opt) {
    TL_REQUIRE(opt->algorithm <= TL_ALGO_KCLIST3, TL_EINVAL, "unknown algorithm");
    TL_REQUIRE(opt->nparts <= 1 && opt->part == 0, TL_EINVAL,
               "tl_multi_* partitions the run itself: opt->part/nparts must be 0/1");
    TL_REQUIRE(opt->stream == nullptr, TL_EINVAL, "tl_multi_* runs on the replicas' own streams");
    sp.algo = static_cast<tlb::Algo>(opt->algorithm);
    sp.skip_negative = opt->skip_negative_phase != 0;
    sp.reuse = opt->cf_hash_reuse_last_table != 0;
  }
  sp.mode = mode;
  return sp;
}
}  // namespace

extern "C" {

int tl_fold_parts(const tl_stats* parts, uint32_t nparts, tl_stats* total, uint64_t* offsets) {
  return guarded_multi([&] {
    TL_REQUIRE((parts || nparts == 0) && total, TL_EINVAL, "NULL argument");
    tl_stats t;
    std::memset(&t, 0, sizeof(t));
    uint64_t off = 0;
    for (uint32_t d = 0; d < nparts; ++d) {
      const tl_stats& p = parts[d];
      t.triangles += p.triangles;  // sums wrap mod 2^64 like the reference's uint64 counters
      t.probes += p.probes;
      t.merge_comparisons += p.merge_comparisons;
      t.table_builds += p.table_builds;
      t.positive_triangles += p.positive_triangles;
      t.negative_triangles += p.negative_triangles;
      t.probes_executed += p.probes_executed;
      t.hash_sum += p.hash_sum;
      t.hash_xor ^= p.hash_xor;
      t.tasks += p.tasks;
      t.kernel_launches += p.kernel_launches;
      t.list_ms = std::max(t.list_ms, p.list_ms);  // the parts run concurrently: the slowest bounds the run
      t.prep_ms = std::max(t.prep_ms, p.prep_ms);
      if (offsets) offsets[d] = off;  // exclusive scan of the emission counts
      off += p.triangles;
    }
    *total = t;
  });
}

int tl_multi_create(tl_oriented* og, const int* devs, int ndev, tl_multi** out) {
  return guarded_multi([&] {
    TL_REQUIRE(og && devs && out && ndev >= 1, TL_EINVAL, "NULL argument or empty device list");
    *out = nullptr;
    int count = 0;
    TL_CUDA(cudaGetDeviceCount(&count));
    for (int d = 0; d < ndev; ++d) {
      TL_REQUIRE(devs[d] >= 0 && devs[d] < count, TL_EINVAL, "device index out of range");
      for (int e = 0; e < d; ++e) TL_REQUIRE(devs[e] != devs[d], TL_EINVAL, "duplicate device in the device list");
    }
    const tlb::Nccl& N = tlb::nccl();
    auto mg = std::make_unique<tl_multi>();
    mg->devs.assign(devs, devs + ndev);
    for (int d = 0; d < ndev; ++d) {
      // enable peer access where the hardware allows it (NVLink copies)
      tlb::DeviceGuard guard(devs[d]);
      if (devs[d] != og->device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devs[d], og->device);
        if (can) {
          cudaError_t e = cudaDeviceEnablePeerAccess(og->device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) TL_CUDA(e);
          cudaGetLastError();
        }
      }
    }
    for (int d = 0; d < ndev; ++d) {
      const bool same = devs[d] == og->device;
      mg->reps.push_back(same ? og : tlb::replicate(*og, devs[d]));
      mg->owned.push_back(!same);
      tlb::DeviceGuard guard(devs[d]);
      cudaStream_t st = nullptr;
      TL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      mg->streams.push_back(st);
      mg->red.emplace_back();
      mg->red.back().alloc(8 + 2 * size_t(ndev), st);
    }
    mg->comms.assign(ndev, nullptr);
    tlb::nccl_check(N.comm_init_all(mg->comms.data(), ndev, devs), "ncclCommInitAll");
    *out = mg.release();
  });
}

int tl_multi_free(tl_multi* mg) {
  return guarded_multi([&] { delete mg; });
}

int tl_multi_count(tl_multi* mg, const tl_run_options* opt, tl_stats* stats) {
  return guarded_multi([&] {
    TL_REQUIRE(mg && stats, TL_EINVAL, "NULL argument");
    auto parts = tlb::run_parts(*mg, multi_spec(opt, tlb::AotMode::count), {}, {});
    tlb::reduce_parts(*mg, parts, stats, nullptr);
  });
}

int tl_multi_hash(tl_multi* mg, const tl_run_options* opt, tl_stats* stats) {
  return guarded_multi([&] {
    TL_REQUIRE(mg && stats, TL_EINVAL, "NULL argument");
    auto parts = tlb::run_parts(*mg, multi_spec(opt, tlb::AotMode::hash), {}, {});
    tlb::reduce_parts(*mg, parts, stats, nullptr);
  });
}

int tl_multi_list(tl_multi* mg, const tl_run_options* opt, uint32_t* triples, uint64_t cap, tl_stats* stats) {
  return guarded_multi([&] {
    TL_REQUIRE(mg && stats, TL_EINVAL, "NULL argument");
    const int nd = int(mg->devs.size());
    tlb::RunSpec sp = multi_spec(opt, tlb::AotMode::count);
    // every device counts its part; the gathered counts give the offsets
    auto counted = tlb::run_parts(*mg, sp, {}, {});
    std::vector<uint64_t> offs;
    tl_stats total;
    tlb::reduce_parts(*mg, counted, &total, &offs);
    if (!triples) {
      *stats = total;
      return;
    }
    TL_REQUIRE(cap >= total.triangles, TL_ECAPACITY,
               "output capacity " + std::to_string(cap) + " < " + std::to_string(total.triangles) + " triangles");
    std::vector<tlb::DBuf<uint32_t>> bufs(nd);
    std::vector<uint32_t*> outs(nd);
    std::vector<uint64_t> caps(nd);
    for (int d = 0; d < nd; ++d) {
      tlb::DeviceGuard guard(mg->devs[d]);
      caps[d] = counted[d].triangles;
      bufs[d].alloc(std::max<uint64_t>(3 * caps[d], 3), mg->reps[d]->stream);
      outs[d] = bufs[d].p;
    }
    sp.mode = tlb::AotMode::list;
    auto listed = tlb::run_parts(*mg, sp, outs, caps);
    for (int d = 0; d < nd; ++d) {
      TL_REQUIRE(listed[d].emitted == counted[d].triangles, TL_ELOGIC, "a part emitted a different count");
      tlb::DeviceGuard guard(mg->devs[d]);
      if (caps[d])
        TL_CUDA(cudaMemcpyAsync(triples + 3 * offs[d], bufs[d].p, 12 * caps[d], cudaMemcpyDeviceToHost,
                                mg->reps[d]->stream));
    }
    for (int d = 0; d < nd; ++d) {
      tlb::DeviceGuard guard(mg->devs[d]);
      TL_CUDA(cudaStreamSynchronize(mg->reps[d]->stream));
    }
    tlb::reduce_parts(*mg, listed, stats, nullptr);
  });
}

}  // extern "C"
