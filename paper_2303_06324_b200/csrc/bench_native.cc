// bench_native.cc -- end-to-end latency harness over the public C-ABI (bench /
// test infrastructure, libocclbench.so; not part of the product library).
//
// The paper measures a collective's end-to-end latency as the host time from
// submission to completion (§5; fig:nccl "latency").  With n
// virtual ranks in one process, submitting them one after another from Python
// would add the interpreter's per-call cost n times to every sample, so this
// harness runs one native thread per rank: each iteration the threads are
// released by a shared flag, stamp CLOCK_MONOTONIC, call the rank's submit
// (occlAllReduce / ...) and occlWait, and stamp again.  Sample = max(done) -
// min(submit) over ranks.  Everything goes through include/occl.h.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/occl.h"

namespace {
inline uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}
inline void relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}
occlResult_t submit(occlComm_t c, int kind, const void* s, void* r, size_t count, int dtype, int op, int root,
                    int id) {
  switch (kind) {
    case 0: return occlAllReduce(s, r, count, (occlDataType_t)dtype, (occlRedOp_t)op, id, c);
    case 1: return occlAllGather(s, r, count, (occlDataType_t)dtype, id, c);
    case 2: return occlReduceScatter(s, r, count, (occlDataType_t)dtype, (occlRedOp_t)op, id, c);
    case 3: return occlBroadcast(s, r, count, (occlDataType_t)dtype, root, id, c);
    default: return occlReduce(s, r, count, (occlDataType_t)dtype, (occlRedOp_t)op, root, id, c);
  }
}
}  // namespace

extern "C" int occlBenchLatency(occlComm_t* comms, int n, int kind, size_t count, int dtype, int op, int root,
                                void* const* sends, void* const* recvs, int collId, int reps, double* outNs) {
  if (!comms || n < 1 || reps < 1 || !outNs) return (int)occlInvalidArgument;
  std::atomic<int> go{0};
  std::atomic<int> done{0};
  std::atomic<int> err{0};
  std::atomic<int> stop{0};
  std::vector<uint64_t> tsub((size_t)n * reps), tdone((size_t)n * reps);
  std::vector<std::thread> ts;
  for (int r = 0; r < n; ++r) {
    ts.emplace_back([&, r]() {
      for (int it = 0; it < reps; ++it) {
        while (go.load(std::memory_order_acquire) <= it) relax();
        if (stop.load()) break;
        const uint64_t t0 = now_ns();
        occlResult_t e = submit(comms[r], kind, sends[r], recvs[r], count, dtype, op, root, collId);
        if (e == occlSuccess) e = occlWait(comms[r], collId, 60'000'000'000ll);
        const uint64_t t1 = now_ns();
        if (e != occlSuccess) err.store((int)e);
        tsub[(size_t)it * n + r] = t0;
        tdone[(size_t)it * n + r] = t1;
        done.fetch_add(1, std::memory_order_acq_rel);
      }
    });
  }
  for (int it = 0; it < reps; ++it) {
    // a short pause between samples: every rank has finished the previous one
    const uint64_t t = now_ns();
    while (now_ns() - t < 20'000) relax();
    go.store(it + 1, std::memory_order_release);
    while (done.load(std::memory_order_acquire) < (it + 1) * n) relax();
    uint64_t lo = ~0ull, hi = 0;
    for (int r = 0; r < n; ++r) {
      lo = tsub[(size_t)it * n + r] < lo ? tsub[(size_t)it * n + r] : lo;
      hi = tdone[(size_t)it * n + r] > hi ? tdone[(size_t)it * n + r] : hi;
    }
    outNs[it] = (double)(hi - lo);
    if (err.load()) break;
  }
  stop.store(1);
  go.store(reps + 1);
  for (auto& th : ts) th.join();
  return err.load();
}
