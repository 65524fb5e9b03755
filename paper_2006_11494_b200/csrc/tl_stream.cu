// tl_stream.cu -- batched listing into arbitrary host sinks in bounded memory.
//
// Reference semantics: run_parallel<SinkFactory> (parallel.hpp:25-78) hands
// every emission of aot_pivot (engine.hpp:256, :269) to a per-worker sink
// (engine.hpp:125-134) as it is found, so host memory stays O(workers).  Here
// the device lists a run in consecutive claim ranges of the claim-cost cut
// (RunSpec::range: part b of K), each into a device batch buffer; a range
// whose emissions overflow the buffer is split in two (part 2b, 2b+1 of 2K --
// the same cut points, so the ranges stay an exact cover) and listed again.
// A producer thread drives the device and copies each batch into a ring of
// pinned host buffers; the calling thread consumes them in order and calls
// the user's callback, which may take as long as it likes (the device keeps
// listing ahead while the ring has a free buffer).
#include <condition_variable>
#include <deque>
#include <exception>
#include <mutex>
#include <thread>
#include <utility>
#include <vector>

#include "tl_internal.cuh"

namespace tlb {

namespace {

struct HostSlot {
  uint32_t* p = nullptr;
  cudaEvent_t copied = nullptr;
  uint64_t count = 0;
};

struct Ring {
  std::mutex mu;
  std::condition_variable cv;
  std::deque<uint32_t> free_slots, ready;  // slot indices
  bool done = false, cancel = false;
  std::exception_ptr error;
};

void add_counters(AotResult& a, const AotResult& r) {
  a.positive += r.positive;
  a.negative += r.negative;
  a.executed += r.executed;
  a.logical += r.logical;
  a.windowed += r.windowed;
  a.emitted += r.emitted;
  a.tasks += r.tasks;
  a.table_builds += r.table_builds;
  a.launches += r.launches;
  a.triangles += r.triangles;
  a.probes += r.probes;
  a.merge_comparisons += r.merge_comparisons;
  a.report_positive += r.report_positive;
  a.report_negative += r.report_negative;
  a.list_ms += r.list_ms;
  a.prep_ms += r.prep_ms;
}

}  // namespace

AotResult list_batches(tl_oriented& og, const RunSpec& spec, cudaStream_t s, uint64_t batch_triples,
                       uint32_t host_buffers, tl_batch_fn fn, void* user) {
  TL_REQUIRE(fn, TL_EINVAL, "batch callback is NULL");
  const uint64_t cap = batch_triples ? batch_triples : (1ull << 24);
  const uint32_t R = host_buffers ? std::max(host_buffers, 2u) : 3u;
  const uint32_t nparts = spec.nparts ? spec.nparts : 1, part = spec.part;
  TL_REQUIRE(part < nparts, TL_EINVAL, "partition index out of range");
  AotResult total;
  if (og.m == 0) return total;

  // Top-level ranges from the whole run's emission count (one counting pass
  // over the whole graph; ~3/4 full batches, the cut balances probe cost,
  // not triangles): range b of K belongs to this caller when b % nparts == part.
  const auto key = std::make_tuple(uint32_t(spec.algo), uint32_t(spec.algo == Algo::aot && spec.skip_negative), 0u, 1u);
  uint64_t T;
  if (auto it = og.tri_cache.find(key); it != og.tri_cache.end()) {
    T = it->second;
  } else {
    RunSpec cs = spec;
    cs.mode = AotMode::count;
    cs.part = 0;
    cs.nparts = 1;
    cs.range = false;
    T = aot_run(og, cs, s, nullptr, 0).triangles;
    og.tri_cache[key] = T;
  }
  const uint64_t target = std::max<uint64_t>(1, cap - cap / 4);
  uint64_t K = std::max<uint64_t>(1, (T + target - 1) / target);
  K = std::min<uint64_t>(K, og.m);
  K = ((K + nparts - 1) / nparts) * nparts;  // every part gets the same number of top-level ranges
  TL_REQUIRE(K <= 0xFFFFFFFFull, TL_EINVAL, "batch size too small for this graph");

  DBuf<uint32_t> dbuf[2];  // batch i lists into dbuf[i % 2] while batch i-1 is copied out
  dbuf[0].alloc(3 * cap, s);
  dbuf[1].alloc(3 * cap, s);
  std::vector<HostSlot> slots(R);
  struct SlotGuard {
    std::vector<HostSlot>& v;
    ~SlotGuard() {
      for (auto& h : v) {
        if (h.copied) cudaEventSynchronize(h.copied), cudaEventDestroy(h.copied);
        if (h.p) cudaFreeHost(h.p);
      }
    }
  } slot_guard{slots};
  for (auto& h : slots) {
    TL_CUDA(cudaMallocHost(&h.p, sizeof(uint32_t) * 3 * cap));
    TL_CUDA(cudaEventCreateWithFlags(&h.copied, cudaEventDisableTiming));
  }
  cudaStream_t copy_stream = nullptr;
  TL_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t st;
    ~StreamGuard() {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  } stream_guard{copy_stream};
  cudaEvent_t dbuf_free[2] = {nullptr, nullptr};  // the last D2H out of dbuf[i] has finished
  struct EventGuard {
    cudaEvent_t* e;
    ~EventGuard() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } event_guard{dbuf_free};
  for (auto& e : dbuf_free) {
    TL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    TL_CUDA(cudaEventRecord(e, copy_stream));
  }

  Ring ring;
  for (uint32_t i = 0; i < R; ++i) ring.free_slots.push_back(i);
  int device = og.device;

  auto producer = [&] {
    try {
      TL_CUDA(cudaSetDevice(device));
      std::vector<std::pair<uint64_t, uint64_t>> work;  // (b, K) stack, next range at the back
      uint64_t issued = 0;
      for (uint64_t b = K; b-- > 0;)
        if (b % nparts == part) work.emplace_back(b, K);
      while (!work.empty()) {
        const auto [b, k] = work.back();
        work.pop_back();
        uint32_t slot;
        {
          std::unique_lock<std::mutex> lock(ring.mu);
          ring.cv.wait(lock, [&] { return !ring.free_slots.empty() || ring.cancel; });
          if (ring.cancel) return;
          slot = ring.free_slots.front();
          ring.free_slots.pop_front();
        }
        RunSpec ls = spec;
        ls.mode = AotMode::list;
        ls.part = uint32_t(b);
        ls.nparts = uint32_t(k);
        ls.range = true;
        const int db = int(issued & 1);
        TL_CUDA(cudaStreamWaitEvent(s, dbuf_free[db], 0));  // the batch before last has left dbuf[db]
        const AotResult r = aot_run(og, ls, s, dbuf[db].p, cap);  // synchronises s
        TL_REQUIRE(r.emitted == r.triangles, TL_ELOGIC, "emission count disagrees with the triangle counters");
        if (r.emitted > cap) {  // split the range at the cut's midpoint and list both halves
          TL_REQUIRE(k <= 0x7FFFFFFFull, TL_ELOGIC, "a single claim range exceeds the batch buffer");
          work.emplace_back(2 * b + 1, 2 * k);
          work.emplace_back(2 * b, 2 * k);
          std::lock_guard<std::mutex> lock(ring.mu);
          ring.free_slots.push_front(slot);
          continue;
        }
        HostSlot& h = slots[slot];
        h.count = r.emitted;
        if (r.emitted)
          TL_CUDA(cudaMemcpyAsync(h.p, dbuf[db].p, sizeof(uint32_t) * 3 * r.emitted, cudaMemcpyDeviceToHost,
                                  copy_stream));
        TL_CUDA(cudaEventRecord(h.copied, copy_stream));
        TL_CUDA(cudaEventRecord(dbuf_free[db], copy_stream));
        ++issued;
        {
          std::lock_guard<std::mutex> lock(ring.mu);
          add_counters(total, r);
          ring.ready.push_back(slot);
        }
        ring.cv.notify_all();
      }
    } catch (...) {
      std::lock_guard<std::mutex> lock(ring.mu);
      ring.error = std::current_exception();
    }
    {
      std::lock_guard<std::mutex> lock(ring.mu);
      ring.done = true;
    }
    ring.cv.notify_all();
  };

  std::thread prod(producer);
  std::exception_ptr consumer_error;
  bool canceled = false;
  while (true) {
    uint32_t slot;
    {
      std::unique_lock<std::mutex> lock(ring.mu);
      ring.cv.wait(lock, [&] { return !ring.ready.empty() || ring.done; });
      if (ring.ready.empty()) break;
      slot = ring.ready.front();
      ring.ready.pop_front();
    }
    HostSlot& h = slots[slot];
    int rc = 0;
    try {
      if (cudaEventSynchronize(h.copied) != cudaSuccess) throw TlError(TL_ECUDA, "batch copy failed");
      if (h.count) rc = fn(user, h.p, h.count);
    } catch (...) {
      consumer_error = std::current_exception();
    }
    std::lock_guard<std::mutex> lock(ring.mu);
    if (rc != 0 || consumer_error) {
      canceled = rc != 0;
      ring.cancel = true;
      ring.cv.notify_all();
      break;
    }
    ring.free_slots.push_back(slot);
    ring.cv.notify_all();
  }
  prod.join();
  if (consumer_error) std::rethrow_exception(consumer_error);
  if (canceled) throw TlError(TL_ECANCELED, "the batch callback stopped the run");
  if (ring.error) std::rethrow_exception(ring.error);
  // logical probes and table builds were attributed by the cut, once per
  // range, so the sums are the run's counters as tl_run_count reports them
  return total;
}

}  // namespace tlb
