// occl_host.cc -- host runtime behind include/occl.h.
//
// CPU part of the DFCE framework (Fig. "fig:df"):
//   * registration = a fixed registry of maxColl ids with dedicated context slots
//     and connectors prepared at communicator creation;
//   * SQ: single-producer ring of 64-B SQEs in pinned, mapped host memory
//     (PAPER.md:394, :483-484); every daemon block consumes every SQE with its own
//     cursor, mirrored to host memory; a slot is free once all cursors passed it
//     (the paper's per-SQE consumer counter, R8);
//   * CQ: one slot per collId holding the last completed submission number
//     (the paper's "optimized CQ", R9);
//   * poller + callback map and the event-driven (re)start of
//     the daemon kernel run in one supervisor thread;
//   * connectors of the ring neighbours are mapped through CUDA IPC (other
//     processes) or used directly (same process), with peer access enabled.
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "../../include/occl.h"
#include "occl_internal.h"

using namespace occl;

namespace {

constexpr uint32_t kHandleMagic = 0x4f43434cu;   // "OCCL"
constexpr uint32_t kHandleVersion = 2;

struct Handle {
  uint32_t magic, version;
  int32_t nranks, rank, dev, pid;
  uint64_t hostId;
  uint64_t arenaPtr;
  uint64_t dataBytes, flagsOffset, llOffset;
  uint64_t cfgFingerprint;
  cudaIpcMemHandle_t ipc;
};
static_assert(sizeof(Handle) <= OCCL_HANDLE_BYTES, "handle too large");

uint64_t now_ns() {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

inline void cpu_relax() {
#if defined(__x86_64__)
  __builtin_ia32_pause();
#endif
}

int elem_size(int dt) { return (dt == kBF16 || dt == kF16) ? 2 : ((dt == kI64 || dt == kF64) ? 8 : 4); }

uint64_t fingerprint(const occlConfig_t& c) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  mix(c.maxColl); mix(c.gridBlocks); mix(c.connSlots); mix(c.slicesPerChunk); mix(c.sliceBytes);
  mix(c.minBlockBytes);
  mix(c.directMode);
  mix(c.directRead);
  mix(c.forceSysScope);
  mix(c.llSliceBytes);
  mix(c.llMaxBytes);
  return h;
}

}  // namespace


namespace occl {
// One daemon kernel launch serves every member communicator (one member unless
// occlCommFuse merged the virtual ranks of a device).  Owns the stream, the
// launch events and the supervisor thread (poller + event-driven restart).
struct Launcher {
  int dev = 0;
  std::vector<occlComm*> members;
  DaemonParams* paramsDev = nullptr;            // [members]
  cudaStream_t stream = nullptr;
  cudaEvent_t evStart = nullptr, evDone = nullptr;
  bool launched = false;
  uint64_t launches = 0;
  float lastLaunchMs = 0.f;
  uint64_t lastExitNs = 0;
  std::mutex mu;                                 // guards launch state and members
  std::condition_variable cv;
  std::thread sup;
  std::atomic<bool> stop{false};
  std::atomic<int> autoLaunch{1};
  std::atomic<int> sticky{0};
  int quitUploaded = -1;                         // effective quitEnabled in paramsDev
  uint32_t* quitWord = nullptr;                  // device: the launch's voluntary-quit votes (zeroed per launch)
  int lastLaunchQuit = 0;                        // the current/last launch may quit voluntarily
};
}  // namespace occl

struct occlComm {
  int nranks = 0, rank = 0, dev = 0;
  occlConfig_t cfg{};
  // device memory
  char* arena = nullptr;
  size_t dataBytes = 0, flagsBytes = 0, llBytes = 0;
  CtxSlot* ctx = nullptr;
  Sqe* sqMirror = nullptr;                       // device copy of the SQ (+ tail, fetch lock)
  uint64_t* mirrorTail = nullptr;
  BlockState* blk = nullptr;
  uint32_t* tqSave = nullptr;
  uint32_t* complCnt = nullptr;
  CollStat* collStats = nullptr;
  BlockStat* blkStats = nullptr;
  TraceRec* trace = nullptr;
  uint32_t* traceCount = nullptr;
  // pinned + mapped host memory
  SqeWire* sqHost = nullptr;
  SqeWire* sqDev = nullptr;
  uint64_t* sqCurHost = nullptr;
  uint64_t* sqCurDev = nullptr;
  uint64_t* cqHost = nullptr;                    // [maxColl] last completed subSeq (device-written in
  uint64_t* cqDev = nullptr;                     //   cqMode 0, poller-maintained in the ring modes)
  uint64_t* cqRingHost = nullptr;                // ring CQ (cqMode 1 / 2): entries + vanilla tail
  uint64_t* cqRingDev = nullptr;
  uint64_t* cqTailHost = nullptr;
  uint64_t* cqTailDev = nullptr;
  uint64_t* cqReserve = nullptr;                 // device: next ring slot
  uint32_t cqDepth = 0;
  uint64_t cqHead = 0;                           // poller: next ring entry to read
  std::mutex cqMu;
  std::atomic<uint64_t> sqTail{0};
  // per-collective host state
  // per collId: submission token = subSeq << 1 | in-flight bit.  Completion
  // CASes the exact token it observed, so a completion can never be applied to
  // a newer submission of the same id (wait + resubmit racing the poller).
  std::unique_ptr<std::atomic<uint64_t>[]> tok;
  std::vector<int> boundSub;                     // root: ring each collId is bound to (-1 free, -2 retired)
  std::vector<occlCallback_t> cb;
  std::vector<void*> cbArg;
  std::vector<int32_t> prio;                     // per-collective priority (default: collId)
  std::atomic<int> inflight{0};
  // peers
  char* nextArena = nullptr;
  char* prevArena = nullptr;
  bool nextIpc = false, prevIpc = false;
  int sysScope = 0;
  DaemonParams params{};
  bool connected = false;
  cudaStream_t statsStream = nullptr;
  std::mutex sqMu;                               // single submitter: guards the SQ tail
  std::atomic<int> sticky{0};
  occl::Launcher* L = nullptr;                   // daemon lifecycle (own, or shared after occlCommFuse)
  // sub-communicators (occlCommSplit): a child shares its root's daemon, SQ, CQ
  // and collId registry and runs its collectives on its own ring (RingDesc)
  occlComm* parent = nullptr;
  int sub = 0;                                   // ring index in the root's daemon
  std::vector<Handle> handles;                   // root: every rank's handle (kept for splits)
  std::vector<char*> peerArena;                  // root: opened arenas by rank
  std::vector<char> peerIpc;                     // root: 1 if opened through CUDA IPC
  RingDesc* ringsDev = nullptr;                  // root: [kMaxRings]
  int nrings = 0;
  std::vector<int> freeRings;                    // root: ring slots of destroyed sub-communicators
  int children = 0;                              // root: live sub-communicators
  std::vector<occlComm*> owner;                  // root: per collId, the comm that submitted it
};

namespace {
inline occlComm* root_of(occlComm* c) { return c && c->parent ? c->parent : c; }
}

namespace {

occlResult_t cuda_fail(occlComm* c, cudaError_t e) {
  if (c) c->sticky.store((int)e);
  return occlCudaError;
}
#define CUDACHECK(comm, call)                          \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(comm, e_); \
  } while (0)

// SQ slots below this index were copied into the daemon's device-memory mirror
// (the fetching block publishes it) and may be rewritten.
uint64_t min_cursor(occlComm* c) {
  return reinterpret_cast<volatile uint64_t*>(c->sqCurHost)[0];
}

bool comm_sticky(occlComm* c) { return c->sticky.load() || (c->L && c->L->sticky.load()); }

// caller holds L->mu
bool daemon_running(Launcher* L) {
  if (!L->launched) return false;
  cudaError_t q = cudaEventQuery(L->evDone);
  if (q == cudaErrorNotReady) return true;
  if (q == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, L->evStart, L->evDone) == cudaSuccess) L->lastLaunchMs = ms;
    L->launched = false;
    L->lastExitNs = now_ns();
    return false;
  }
  L->sticky.store((int)q);                       // asynchronous device fault: sticky
  L->launched = false;
  return false;
}

// caller holds L->mu.  One kernel launch serves every member communicator.
occlResult_t launch_locked(Launcher* L) {
  if (L->sticky.load()) return occlCudaError;
  if (daemon_running(L)) return occlSuccess;
  if (L->members.empty()) return occlInvalidUsage;
  occlComm* c0 = L->members[0];
  cudaError_t e;
  // A voluntary quit is only safe while the host restarts the daemon on pending
  // work (event-driven start); without autoLaunch it would
  // strand queued collectives, so the daemon is told not to quit.
  const int quit = L->autoLaunch.load() ? 1 : 0;
  if (quit != L->quitUploaded) {
    std::vector<DaemonParams> ps;
    for (occlComm* m : L->members) {
      DaemonParams q = m->params;
      q.quitEnabled = m->cfg.quitEnabled && quit;
      ps.push_back(q);
    }
    if ((e = cudaMemcpy(L->paramsDev, ps.data(), ps.size() * sizeof(DaemonParams), cudaMemcpyHostToDevice)) !=
        cudaSuccess) { L->sticky.store((int)e); return occlCudaError; }
    L->quitUploaded = quit;
  }
  if ((e = cudaMemsetAsync(L->quitWord, 0, sizeof(uint32_t), L->stream)) != cudaSuccess) {
    L->sticky.store((int)e);
    return occlCudaError;
  }
  if ((e = cudaEventRecord(L->evStart, L->stream)) != cudaSuccess) { L->sticky.store((int)e); return occlCudaError; }
  int r = occl_internal_launch_daemon(&c0->params, L->paramsDev, (int)L->members.size(), c0->cfg.blockThreads,
                                      L->stream);
  if (r != 0) { L->sticky.store(r); return occlCudaError; }
  if ((e = cudaEventRecord(L->evDone, L->stream)) != cudaSuccess) { L->sticky.store((int)e); return occlCudaError; }
  L->launched = true;
  L->launches++;
  L->lastLaunchQuit = quit;
  return occlSuccess;
}

// Ring CQ modes: the poller drains CQEs (collective ids) into the per-id
// completion counters; one CQE per submission, so the counter equals the subSeq
// of the last completed submission, as the id-slot CQ reports it directly.
void drain_cq(occlComm* c) {
  if (c->cfg.cqMode == 0) return;
  std::lock_guard<std::mutex> g(c->cqMu);
  volatile uint64_t* ring = c->cqRingHost;
  volatile uint64_t* cq = c->cqHost;
  for (;;) {
    const uint64_t h = c->cqHead;
    uint64_t id;
    if (c->cfg.cqMode == 2) {
      const uint64_t e = ring[h % c->cqDepth];
      if ((e >> 32) != ((h + 1) & 0xffffffffull)) break;       // stamp: written for this slot?
      id = e & 0xffffffffull;
    } else {
      if (h >= *reinterpret_cast<volatile uint64_t*>(c->cqTailHost)) break;
      std::atomic_thread_fence(std::memory_order_acquire);
      id = ring[h % c->cqDepth];
    }
    if (id < (uint64_t)c->cfg.maxColl) cq[id] = cq[id] + 1;
    c->cqHead = h + 1;
  }
}

inline bool tok_inflight(uint64_t t) { return (t & 1) != 0; }
inline uint64_t tok_seq(uint64_t t) { return t >> 1; }

bool try_complete(occlComm* c, int id) {
  uint64_t t = c->tok[id].load(std::memory_order_acquire);
  if (!tok_inflight(t)) return false;
  drain_cq(c);
  const uint64_t done = reinterpret_cast<volatile uint64_t*>(c->cqHost)[id];
  if (done < tok_seq(t)) return false;
  // complete exactly the submission observed: fails if the id was completed and
  // resubmitted in between (ABA between the poller and occlWait)
  if (!c->tok[id].compare_exchange_strong(t, t & ~1ull)) return false;
  c->inflight.fetch_sub(1);
  if (!c->owner.empty() && c->owner[id] && c->owner[id] != c) c->owner[id]->inflight.fetch_sub(1);
  occlCallback_t f = c->cb[id];
  if (f) f(id, c->cbArg[id]);                   // exactly once per completion
  return true;
}

// Supervisor: poller + callback map + event-driven (re)start.
void supervisor_main(Launcher* L) {
  cudaSetDevice(L->dev);
  const uint64_t backoffNs = 50'000;
  std::vector<occlComm*> ms;
  while (!L->stop.load()) {
    bool pending = false;
    {
      std::lock_guard<std::mutex> lk(L->mu);
      ms = L->members;
      bool newSqe = false;
      for (occlComm* c : ms) {
        if (c->sqTail.load() > min_cursor(c)) newSqe = true;
        if (c->inflight.load() > 0) pending = true;
      }
      pending = pending || newSqe;
      // event-driven start; a launch that could quit voluntarily is always
      // restarted while work is pending, even if autoLaunch was switched off since
      if ((L->autoLaunch.load() || L->lastLaunchQuit) && pending && !daemon_running(L) && !L->sticky.load()) {
        // new SQEs start the daemon at once; collectives that are merely stuck
        // (the daemon quit voluntarily) restart after a back-off so that device
        // synchronisation on the host can complete in between
        if (newSqe || now_ns() - L->lastExitNs > backoffNs) launch_locked(L);
      }
    }
    for (occlComm* c : ms)
      for (int id = 0; id < c->cfg.maxColl && c->inflight.load() > 0; ++id)
        if (c->cb[id] && tok_inflight(c->tok[id].load())) try_complete(c, id);
    if (!pending) {
      std::unique_lock<std::mutex> lk(L->mu);
      L->cv.wait_for(lk, std::chrono::milliseconds(5));
    } else {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
}

occlResult_t launcher_start(Launcher* L, const std::vector<occlComm*>& members) {
  L->dev = members[0]->dev;
  L->members = members;
  cudaSetDevice(L->dev);
  if (cudaMalloc(&L->quitWord, sizeof(uint32_t)) != cudaSuccess) return occlCudaError;
  if (cudaMemset(L->quitWord, 0, sizeof(uint32_t)) != cudaSuccess) return occlCudaError;
  std::vector<DaemonParams> ps;
  for (occlComm* c : members) {
    c->params.quitWord = L->quitWord;
    c->params.quitTotal = (uint32_t)(c->cfg.gridBlocks * members.size());
    ps.push_back(c->params);
  }
  if (cudaMalloc(&L->paramsDev, ps.size() * sizeof(DaemonParams)) != cudaSuccess) return occlCudaError;
  if (cudaMemcpy(L->paramsDev, ps.data(), ps.size() * sizeof(DaemonParams), cudaMemcpyHostToDevice) != cudaSuccess)
    return occlCudaError;
  if (cudaStreamCreateWithFlags(&L->stream, cudaStreamNonBlocking) != cudaSuccess) return occlCudaError;
  if (cudaEventCreate(&L->evStart) != cudaSuccess) return occlCudaError;
  if (cudaEventCreate(&L->evDone) != cudaSuccess) return occlCudaError;
  L->autoLaunch.store(members[0]->cfg.autoLaunch ? 1 : 0);
  try {
    L->sup = std::thread(supervisor_main, L);
  } catch (...) {
    return occlSystemError;
  }
  for (occlComm* c : members) c->L = L;
  return occlSuccess;
}

// Stop the supervisor and wait for the daemon to be idle; frees the launcher.
void launcher_stop(Launcher* L) {
  L->stop.store(true);
  L->cv.notify_all();
  if (L->sup.joinable()) L->sup.join();
  cudaSetDevice(L->dev);
  if (L->launched) cudaEventSynchronize(L->evDone);
  if (L->paramsDev) cudaFree(L->paramsDev);
  if (L->quitWord) cudaFree(L->quitWord);
  if (L->evStart) cudaEventDestroy(L->evStart);
  if (L->evDone) cudaEventDestroy(L->evDone);
  if (L->stream) cudaStreamDestroy(L->stream);
  for (occlComm* c : L->members)
    if (c->L == L) c->L = nullptr;
  delete L;
}

occlResult_t validate_config(const occlConfig_t& c) {
  if (c.maxColl < 1 || c.maxColl > 65535) return occlInvalidArgument;
  if (c.gridBlocks < 1 || c.gridBlocks > 1024) return occlInvalidArgument;
  if (c.blockThreads < 128 || c.blockThreads > 608 || c.blockThreads % 32) return occlInvalidArgument;
  if (c.slicesPerChunk < 1 || c.connSlots <= c.slicesPerChunk) return occlInvalidArgument;  // invariant I7
  if (c.sliceBytes < 16 || c.sliceBytes % 16 || c.sliceBytes > (1ull << 30)) return occlInvalidArgument;
  if (c.minBlockBytes < 1) return occlInvalidArgument;
  if (c.sqDepth < 2) return occlInvalidArgument;
  if (c.cacheWays < 1 || c.cacheWays > kMaxCacheWays) return occlInvalidArgument;
  if (c.spinMin < 1 || c.spinBase < c.spinMin || c.spinCap < c.spinBase || c.spinBoost < 1) return occlInvalidArgument;
  if (c.spinNs < 1) return occlInvalidArgument;
  if (c.priorityCadence < 1) return occlInvalidArgument;
  if (c.stallLimit < 1) return occlInvalidArgument;
  if (c.pipeDepth < 1 || c.pipeDepth > 8) return occlInvalidArgument;
  if (c.llSpeculate < 0 || c.llSpeculate > 2) return occlInvalidArgument;
  if (c.prefetchSlices != 0) return occlInvalidArgument;       // reserved (the L2 prefetch was removed)
  if (c.readyFirst < 0 || c.readyFirst > 2) return occlInvalidArgument;
  if (c.stagingTiles < 1 || c.stagingTiles > 6) return occlInvalidArgument;
  if (c.l2Hints < 0 || c.l2Hints > 3) return occlInvalidArgument;
  if (c.cqMode < 0 || c.cqMode > 2) return occlInvalidArgument;
  if (c.blocksPerSM < 1 || c.blocksPerSM > 2) return occlInvalidArgument;
  if (c.traceCap > (1u << 24)) return occlInvalidArgument;
  if (c.llSliceBytes < 8 || c.llSliceBytes % 8 || c.llSliceBytes > (1u << 20)) return occlInvalidArgument;
  if (c.blocksPerSM == 2 && (c.blockThreads > 384 || c.stagingTiles > 3)) return occlInvalidArgument;
  return occlSuccess;
}

int coll_blocks(const occlComm* c, int kind, size_t count, int dtype) {
  const int isz = elem_size(dtype);
  const uint64_t A = 16 / isz;
  uint64_t seg = count;
  if (c->nranks > 1 && kind == kAllReduce) {
    const uint64_t per = (count + c->nranks - 1) / c->nranks;
    seg = (per + A - 1) / A * A;
  }
  const uint64_t bytes = seg * isz;
  const uint64_t G = (uint64_t)c->cfg.gridBlocks;
  uint64_t nb = (bytes + c->cfg.minBlockBytes - 1) / c->cfg.minBlockBytes;
  if (nb < 1) nb = 1;
  if (nb > G) nb = G;
  // Latency-bound collectives -- those the block rule above already sends over
  // LL (per-block part <= llMaxBytes) -- are spread so every block moves ONE LL
  // slice per step: a ring step then costs one LL hop (~3 us at 8 ranks), where
  // a single block would chain several slices per step (a 256 KiB all-reduce at
  // 8 ranks: 4 slices x 14 steps on one block, slower than 1 MiB on Simple).
  // Collectives the block rule sends over Simple keep their block count: LL on
  // the whole grid would cut a 1 MiB all-reduce's single-op latency but also
  // its pipelined throughput (4.6x, several ops can no longer share the grid).
  // Same on every rank: a function of (count, dtype, nranks, config).
  const uint64_t partBytes = (bytes + nb - 1) / nb;
  if (c->cfg.llMaxBytes && c->nranks > 1 && partBytes <= c->cfg.llMaxBytes &&
      bytes <= G * (uint64_t)c->cfg.llSliceBytes) {
    uint64_t nbLL = (bytes + c->cfg.llSliceBytes - 1) / c->cfg.llSliceBytes;
    if (nbLL > nb) nb = nbLL;
  }
  return (int)nb;
}

void write_sqe(occlComm* c, Sqe& e) {
  const uint64_t t = c->sqTail.load();
  SqeWire* s = &c->sqHost[t % c->cfg.sqDepth];
  uint32_t w[15];
  sqe_to_words(e, w);
  const uint32_t stamp = (uint32_t)(t + 1);
  // one aligned 16-B store per chunk: the device sees each chunk old or new
  for (int k = 0; k < kWireChunks; ++k) {
    const __m128i v = _mm_set_epi32((int)w[3 * k + 2], (int)w[3 * k + 1], (int)w[3 * k], (int)stamp);
    _mm_store_si128(reinterpret_cast<__m128i*>(s->c[k]), v);
  }
  std::atomic_thread_fence(std::memory_order_release);
  c->sqTail.store(t + 1);
}

occlResult_t push_sqe(occlComm* c, Sqe& e, bool launchNow) {
  Launcher* L = c->L;
  std::unique_lock<std::mutex> lk(c->sqMu);
  // wait for a free slot: the daemon always drains the SQ (invariant I4)
  while (c->sqTail.load() - min_cursor(c) >= (uint64_t)c->cfg.sqDepth) {
    if (comm_sticky(c)) return occlCudaError;
    if (L->autoLaunch.load()) {
      std::lock_guard<std::mutex> g(L->mu);
      if (!daemon_running(L)) launch_locked(L);
    }
    lk.unlock();
    std::this_thread::yield();
    lk.lock();
  }
  write_sqe(c, e);
  lk.unlock();
  occlResult_t r = occlSuccess;
  if (launchNow && L->autoLaunch.load()) {       // the first SQE starts the daemon
    std::lock_guard<std::mutex> g(L->mu);
    if (!daemon_running(L)) r = launch_locked(L);
  }
  L->cv.notify_one();
  return r;
}

occlResult_t submit(occlComm* sc, int kind, int dtype, int op, int root, size_t count, const void* send,
                    void* recv, int collId) {
  if (!sc) return occlInvalidArgument;
  occlComm* c = root_of(sc);                          // SQ, CQ and registry of the daemon's owner
  if (!sc->connected || !c->connected || !c->L) return occlInvalidUsage;
  if (comm_sticky(c)) return occlCudaError;
  if (collId < 0) return occlInvalidArgument;
  if (collId >= c->cfg.maxColl) return occlRegistryFull;
  if (dtype < 0 || dtype > 5) return occlInvalidArgument;
  if (op < occlSum || op > occlMin) return occlInvalidArgument;
  if ((kind == kBroadcast || kind == kReduce) && (root < 0 || root >= sc->nranks)) return occlInvalidArgument;
  if (count > 0 && (!send || !recv)) return occlInvalidArgument;
  if (tok_inflight(c->tok[collId].load()) && !try_complete(c, collId)) return occlDuplicateSubmit;
  // a collId is bound to the ring of its first submission: its connector head /
  // credit counters are per (collId, block) on each member, so moving the id to
  // another rank set would pair counters of different edges
  int& bound = c->boundSub[collId];
  if (bound == -1) bound = sc->sub;
  else if (bound != sc->sub) return occlInvalidUsage;
  const uint64_t seq = tok_seq(c->tok[collId].load()) + 1;
  if (count == 0) {                                   // completes at submission (reading Q18)
    reinterpret_cast<volatile uint64_t*>(c->cqHost)[collId] = seq;
    c->tok[collId].store(seq << 1, std::memory_order_release);
    if (c->cb[collId]) c->cb[collId](collId, c->cbArg[collId]);
    return occlSuccess;
  }
  Sqe e{};
  e.sub = (uint16_t)sc->sub;
  e.subSeq = seq;
  e.count = count;
  e.sendbuff = (uint64_t)(uintptr_t)send;
  e.recvbuff = (uint64_t)(uintptr_t)recv;
  e.collId = (uint32_t)collId;
  e.kind = (uint16_t)kind;
  e.dtype = (uint16_t)dtype;
  e.op = (uint16_t)op;
  e.nblocks = (uint16_t)coll_blocks(sc, kind, count, dtype);   // the collective's own ring size
  e.root = root;
  e.priority = c->prio[collId];
  c->owner[collId] = sc;
  if (sc != c) sc->inflight.fetch_add(1);
  c->tok[collId].store((seq << 1) | 1, std::memory_order_release);
  c->inflight.fetch_add(1);
  return push_sqe(c, e, true);
}

void free_comm(occlComm* c) {
  for (size_t q = 0; q < c->peerArena.size(); ++q)
    if (c->peerIpc[q] && c->peerArena[q]) cudaIpcCloseMemHandle(c->peerArena[q]);
  if (c->ringsDev) cudaFree(c->ringsDev);
  if (c->arena) cudaFree(c->arena);
  if (c->ctx) cudaFree(c->ctx);
  if (c->sqMirror) cudaFree(c->sqMirror);
  if (c->mirrorTail) cudaFree(c->mirrorTail);
  if (c->blk) cudaFree(c->blk);
  if (c->tqSave) cudaFree(c->tqSave);
  if (c->complCnt) cudaFree(c->complCnt);
  if (c->collStats) cudaFree(c->collStats);
  if (c->blkStats) cudaFree(c->blkStats);
  if (c->trace) cudaFree(c->trace);
  if (c->traceCount) cudaFree(c->traceCount);
  if (c->sqHost) cudaFreeHost(c->sqHost);
  if (c->sqCurHost) cudaFreeHost(c->sqCurHost);
  if (c->cqHost) cudaFreeHost(c->cqHost);
  if (c->cqRingHost) cudaFreeHost(c->cqRingHost);
  if (c->cqTailHost) cudaFreeHost(c->cqTailHost);
  if (c->cqReserve) cudaFree(c->cqReserve);
  if (c->statsStream) cudaStreamDestroy(c->statsStream);
}

}  // namespace

// =============================================================================
// C-ABI
// =============================================================================
extern "C" {

const char* occlGetErrorString(occlResult_t r) {
  switch (r) {
    case occlSuccess: return "success";
    case occlInvalidArgument: return "invalid argument";
    case occlInvalidUsage: return "invalid usage";
    case occlRegistryFull: return "collective id out of registry range";
    case occlQueueFull: return "submission queue full";
    case occlDuplicateSubmit: return "collective already in flight";
    case occlUnknownId: return "collective id never submitted";
    case occlCudaError: return "CUDA error";
    case occlSystemError: return "system error";
    case occlTimeout: return "timeout";
    case occlInProgress: return "in progress";
    case occlInternalError: return "internal error";
  }
  return "unknown error";
}

occlResult_t occlConfigDefault(occlConfig_t* c) {
  if (!c) return occlInvalidArgument;
  std::memset(c, 0, sizeof(*c));
  c->maxColl = 128;
  c->gridBlocks = 16;
  c->blockThreads = 608;                 // 3 role warps + 16 compute warps
  c->connSlots = 4;
  c->slicesPerChunk = 2;
  c->sliceBytes = 192 << 10;
  c->minBlockBytes = 128 << 10;
  c->sqDepth = 1024;
  c->orderPolicy = occlOrderPriority;   // priority = collId unless set (reading R10)
  c->priorityCadence = 1;
  c->stickiness = 1;
  // thresholds in failed connector polls; the daemon's probes measure ~40 ns
  // per failed poll on B200 (cycPoll / polls), so: queue front ~150 us, floor
  // ~5 us, cap ~2.5 ms for a collective that keeps making progress (R1)
  c->spinBase = 4096;
  c->spinStep = 512;
  c->spinMin = 128;
  c->spinBoost = 2;
  c->spinCap = 65536;
  c->bulkStores = 0;
  c->directRead = 1;
  c->spinNs = 150;                        // one spin ~ an L2 round trip of a flag poll under load (R1)
  c->stallLimit = 2;
  c->quitEnabled = 1;
  c->quitIdleNs = 1'000'000;
  c->idleSleepNs = 256;
  c->autoLaunch = 1;
  c->cacheWays = 8;
  c->pipeDepth = 4;
  c->prefetchSlices = 0;
  c->discardConsumed = 1;
  c->directMode = 1;
  c->stagingTiles = 6;
  c->llSliceBytes = 8 << 10;
  c->llMaxBytes = 64 << 10;
  c->blocksPerSM = 1;
  c->l2Hints = 2;
  c->sqYieldNs = 20'000;
  c->llSpeculate = 2;
  c->readyFirst = 2;
  return occlSuccess;
}

occlResult_t occlCommCreate(occlComm_t* out, int nranks, int rank, int cudaDev, const occlConfig_t* cfgIn) {
  if (!out || nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks || cudaDev < 0)
    return occlInvalidArgument;
  occlConfig_t cfg;
  if (cfgIn) cfg = *cfgIn; else occlConfigDefault(&cfg);
  occlResult_t v = validate_config(cfg);
  if (v != occlSuccess) return v;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cudaDev >= ndev) return occlCudaError;
  std::unique_ptr<occlComm> c(new occlComm());
  c->nranks = nranks;
  c->rank = rank;
  c->dev = cudaDev;
  c->cfg = cfg;
  const size_t M = cfg.maxColl, G = cfg.gridBlocks;
  c->dataBytes = M * G * cfg.connSlots * cfg.sliceBytes;
  c->flagsBytes = M * G * kFlagStride;
  c->llBytes = M * G * cfg.connSlots * 2ull * cfg.llSliceBytes;
  c->tok.reset(new std::atomic<uint64_t>[M]);
  for (size_t i = 0; i < M; ++i) c->tok[i].store(0);
  c->boundSub.assign(M, -1);
  c->cb.assign(M, nullptr);
  c->cbArg.assign(M, nullptr);
  c->prio.resize(M);
  for (size_t i = 0; i < M; ++i) c->prio[i] = (int32_t)i;
  occlComm* cp = c.get();
  auto fail = [&](cudaError_t) { free_comm(cp); return occlCudaError; };
  cudaError_t e;
  if ((e = cudaSetDevice(cudaDev)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->arena, c->dataBytes + c->flagsBytes + c->llBytes)) != cudaSuccess) return fail(e);
  // flags and LL lines start at 0: LL flags are message sequence numbers >= 1
  if ((e = cudaMemset(cp->arena + c->dataBytes, 0, c->flagsBytes + c->llBytes)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->ctx, M * G * sizeof(CtxSlot))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->ctx, 0, M * G * sizeof(CtxSlot))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->sqMirror, cfg.sqDepth * sizeof(Sqe))) != cudaSuccess) return fail(e);
  // tail, fetch lock, cached minimum block cursor
  if ((e = cudaMalloc(&cp->mirrorTail, 4 * sizeof(uint64_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->mirrorTail, 0, 4 * sizeof(uint64_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->blk, G * sizeof(BlockState))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->blk, 0, G * sizeof(BlockState))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->tqSave, G * M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->complCnt, M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->complCnt, 0, M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->collStats, M * G * sizeof(CollStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->collStats, 0, M * G * sizeof(CollStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->blkStats, G * sizeof(BlockStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->blkStats, 0, G * sizeof(BlockStat))) != cudaSuccess) return fail(e);
  if (cfg.traceCap) {
    if ((e = cudaMalloc(&cp->trace, G * cfg.traceCap * sizeof(TraceRec))) != cudaSuccess) return fail(e);
    if ((e = cudaMemset(cp->trace, 0, G * cfg.traceCap * sizeof(TraceRec))) != cudaSuccess) return fail(e);
  }
  if ((e = cudaMalloc(&cp->traceCount, G * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->traceCount, 0, G * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  const unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable;
  if ((e = cudaHostAlloc(&cp->sqHost, cfg.sqDepth * sizeof(SqeWire), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->sqHost, 0, cfg.sqDepth * sizeof(SqeWire));
  if ((e = cudaHostGetDevicePointer(&cp->sqDev, cp->sqHost, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaHostAlloc(&cp->sqCurHost, G * sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->sqCurHost, 0, G * sizeof(uint64_t));
  if ((e = cudaHostGetDevicePointer(&cp->sqCurDev, cp->sqCurHost, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaHostAlloc(&cp->cqHost, M * sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->cqHost, 0, M * sizeof(uint64_t));
  if ((e = cudaHostGetDevicePointer(&cp->cqDev, cp->cqHost, 0)) != cudaSuccess) return fail(e);
  if (cfg.cqMode != 0) {
    // ring CQ: depth >= maxColl -- at most one CQE per in-flight id, so it never fills
    cp->cqDepth = (uint32_t)(2 * M);
    if ((e = cudaHostAlloc(&cp->cqRingHost, cp->cqDepth * sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
    std::memset(cp->cqRingHost, 0, cp->cqDepth * sizeof(uint64_t));
    if ((e = cudaHostGetDevicePointer(&cp->cqRingDev, cp->cqRingHost, 0)) != cudaSuccess) return fail(e);
    if ((e = cudaHostAlloc(&cp->cqTailHost, sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
    *cp->cqTailHost = 0;
    if ((e = cudaHostGetDevicePointer(&cp->cqTailDev, cp->cqTailHost, 0)) != cudaSuccess) return fail(e);
    if ((e = cudaMalloc(&cp->cqReserve, sizeof(uint64_t))) != cudaSuccess) return fail(e);
    if ((e = cudaMemset(cp->cqReserve, 0, sizeof(uint64_t))) != cudaSuccess) return fail(e);
  }
  if ((e = cudaStreamCreateWithFlags(&cp->statsStream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
  *out = c.release();
  return occlSuccess;
}

occlResult_t occlCommGetHandle(occlComm_t c, void* out, size_t* len) {
  if (!c || !out || !len || *len < sizeof(Handle)) return occlInvalidArgument;
  Handle h;
  std::memset(&h, 0, sizeof(h));
  h.magic = kHandleMagic;
  h.version = kHandleVersion;
  h.nranks = c->nranks;
  h.rank = c->rank;
  h.dev = c->dev;
  h.pid = (int32_t)getpid();
  h.hostId = (uint64_t)gethostid();
  h.arenaPtr = (uint64_t)(uintptr_t)c->arena;
  h.dataBytes = c->dataBytes;
  h.flagsOffset = c->dataBytes;
  h.llOffset = c->dataBytes + c->flagsBytes;
  h.cfgFingerprint = fingerprint(c->cfg);
  cudaSetDevice(c->dev);
  if (cudaIpcGetMemHandle(&h.ipc, c->arena) != cudaSuccess) {
    cudaGetLastError();     // same-process peers do not need IPC
  }
  std::memcpy(out, &h, sizeof(h));
  *len = sizeof(h);
  return occlSuccess;
}

occlResult_t occlCommConnect(occlComm_t c, const void* all, size_t lenPerRank) {
  if (!c || !all || lenPerRank < sizeof(Handle)) return occlInvalidArgument;
  if (c->connected) return occlInvalidUsage;
  std::vector<Handle> hs(c->nranks);
  const int mypid = (int)getpid();
  const uint64_t myhost = (uint64_t)gethostid();
  const uint64_t fp = fingerprint(c->cfg);
  bool local = true;
  for (int r = 0; r < c->nranks; ++r) {
    std::memcpy(&hs[r], static_cast<const char*>(all) + r * lenPerRank, sizeof(Handle));
    const Handle& h = hs[r];
    if (h.magic != kHandleMagic || h.version != kHandleVersion || h.nranks != c->nranks || h.rank != r ||
        h.cfgFingerprint != fp)
      return occlInvalidArgument;
    if (h.pid != mypid || h.hostId != myhost || h.dev != c->dev) local = false;
  }
  cudaSetDevice(c->dev);
  auto open = [&](const Handle& h, char** ptr, bool* ipc) -> occlResult_t {
    if (h.pid == mypid && h.hostId == myhost) {
      *ptr = reinterpret_cast<char*>(h.arenaPtr);
      *ipc = false;
      if (h.dev != c->dev) {
        cudaError_t e = cudaDeviceEnablePeerAccess(h.dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_fail(c, e);
      }
      return occlSuccess;
    }
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(c, e);
    *ptr = static_cast<char*>(p);
    *ipc = true;
    return occlSuccess;
  };
  const int next = (c->rank + 1) % c->nranks, prev = (c->rank - 1 + c->nranks) % c->nranks;
  c->handles = hs;
  c->peerArena.assign(c->nranks, nullptr);
  c->peerIpc.assign(c->nranks, 0);
  occlResult_t r;
  if ((r = open(hs[next], &c->nextArena, &c->nextIpc)) != occlSuccess) return r;
  if (prev == next) {
    c->prevArena = c->nextArena;
    c->prevIpc = c->nextIpc;           // closed once, through nextArena (free_comm)
  } else if ((r = open(hs[prev], &c->prevArena, &c->prevIpc)) != occlSuccess) {
    return r;
  }
  c->sysScope = (local && !c->cfg.forceSysScope) ? 0 : 1;
  c->peerArena[next] = c->nextArena;
  c->peerIpc[next] = c->nextIpc;
  if (prev != next) {
    c->peerArena[prev] = c->prevArena;
    c->peerIpc[prev] = c->prevIpc;
  }
  if (c->peerArena[c->rank] == nullptr) c->peerArena[c->rank] = c->arena;   // n == 1: own arena, not opened
  // every other member's arena too: each rank reads all members' admissions on
  // the readiness board (their flags, R29)
  for (int q = 0; q < c->nranks; ++q) {
    if (c->peerArena[q]) continue;
    bool ipc = false;
    if ((r = open(hs[q], &c->peerArena[q], &ipc)) != occlSuccess) return r;
    c->peerIpc[q] = ipc ? 1 : 0;
  }
  c->owner.assign(c->cfg.maxColl, nullptr);
  // ring 0: this communicator's own ring
  RingDesc rd{};
  rd.dataNext = c->nextArena;
  rd.llNext = c->nextArena + hs[next].llOffset;
  rd.flagsNext = c->nextArena + hs[next].flagsOffset;
  rd.flagsPrev = c->prevArena + hs[prev].flagsOffset;
  rd.nranks = c->nranks;
  rd.rank = c->rank;
  rd.directNext = c->cfg.directMode && !c->nextIpc && !c->cfg.forceSysScope;
  rd.directPrev = c->cfg.directMode && !c->prevIpc && !c->cfg.forceSysScope;
  for (int q = 0; q < c->nranks; ++q)
    rd.flagsOf[q] = (q == c->rank ? c->arena : c->peerArena[q]) + hs[q].flagsOffset;
  if (cudaMalloc(&c->ringsDev, kMaxRings * sizeof(RingDesc)) != cudaSuccess) return occlCudaError;
  if (cudaMemcpy(c->ringsDev, &rd, sizeof(rd), cudaMemcpyHostToDevice) != cudaSuccess) return occlCudaError;
  c->nrings = 1;
  DaemonParams& p = c->params;
  p.sq = c->sqDev;
  p.sqCursorHost = c->sqCurDev;
  p.sqMirror = c->sqMirror;
  p.mirrorTail = c->mirrorTail;
  p.fetchLock = reinterpret_cast<uint32_t*>(c->mirrorTail + 1);
  p.cqDone = c->cqDev;
  p.cqMode = c->cfg.cqMode;
  p.cqDepth = c->cqDepth;
  p.cqReserve = c->cqReserve;
  p.cqRing = c->cqRingDev;
  p.cqTail = c->cqTailDev;
  p.blk = c->blk;
  p.tqSave = c->tqSave;
  p.ctx = c->ctx;
  p.complCnt = c->complCnt;
  p.collStats = c->collStats;
  p.blkStats = c->blkStats;
  p.dataLocal = c->arena;
  p.dataNext = c->nextArena;
  p.flagsLocal = c->arena + c->dataBytes;
  p.flagsNext = c->nextArena + hs[next].flagsOffset;
  p.flagsPrev = c->prevArena + hs[prev].flagsOffset;
  p.sliceBytes = c->cfg.sliceBytes;
  p.sqDepth = (uint32_t)c->cfg.sqDepth;
  p.nranks = c->nranks;
  p.rank = c->rank;
  p.G = c->cfg.gridBlocks;
  p.maxColl = c->cfg.maxColl;
  p.K = c->cfg.connSlots;
  p.slicesPerChunk = c->cfg.slicesPerChunk;
  p.orderPolicy = c->cfg.orderPolicy;
  p.priorityCadence = c->cfg.priorityCadence;
  p.stickiness = c->cfg.stickiness;
  p.spinBase = c->cfg.spinBase;
  p.spinStep = c->cfg.spinStep;
  p.spinMin = c->cfg.spinMin;
  p.spinBoost = c->cfg.spinBoost;
  p.spinCap = c->cfg.spinCap;
  p.spinNs = c->cfg.spinNs;
  p.stallLimit = c->cfg.stallLimit;
  p.quitEnabled = c->cfg.quitEnabled;
  p.quitIdleNs = c->cfg.quitIdleNs;
  p.idleSleepNs = c->cfg.idleSleepNs;
  p.cacheWays = c->cfg.cacheWays;
  p.sysScope = c->sysScope;
  p.pipeDepth = c->cfg.pipeDepth;
  p.prefetchSlices = c->cfg.prefetchSlices;
  p.discardConsumed = c->cfg.discardConsumed;
  // direct mode on an edge iff both ends live in this process (raw device
  // pointers of the peer's buffers are valid here); both ends compute the same
  p.directNext = rd.directNext;
  p.directPrev = rd.directPrev;
  p.rings = c->ringsDev;
  p.llLocal = c->arena + c->dataBytes + c->flagsBytes;
  p.llSliceBytes = c->cfg.llSliceBytes;
  p.llMaxBytes = c->cfg.llMaxBytes;
  p.trace = c->trace;
  p.traceCount = c->traceCount;
  p.traceCap = c->cfg.traceCap;
  p.stages = c->cfg.stagingTiles;
  p.bulkStores = c->cfg.bulkStores;
  p.directRead = c->cfg.directRead && c->cfg.directMode;
  p.blocksPerSM = c->cfg.blocksPerSM;
  p.l2Hints = c->cfg.l2Hints;
  p.stallNs = c->cfg.stallNs;
  p.sqYieldNs = c->cfg.sqYieldNs;
  p.llSpeculate = c->cfg.llSpeculate;
  p.readyFirst = c->cfg.readyFirst;
  Launcher* L = new Launcher();
  if ((r = launcher_start(L, {c})) != occlSuccess) {
    launcher_stop(L);
    return r;
  }
  c->connected = true;
  return occlSuccess;
}

occlResult_t occlCommFuse(occlComm_t* comms, int n) {
  if (!comms || n < 1) return occlInvalidArgument;
  std::vector<occlComm*> ms(comms, comms + n);
  for (occlComm* c : ms) {
    if (!c || !c->connected || !c->L || c->parent || c->children) return occlInvalidUsage;
    if (c->dev != ms[0]->dev || c->cfg.gridBlocks != ms[0]->cfg.gridBlocks ||
        c->cfg.maxColl != ms[0]->cfg.maxColl || c->cfg.cacheWays != ms[0]->cfg.cacheWays ||
        c->cfg.blockThreads != ms[0]->cfg.blockThreads || c->cfg.pipeDepth != ms[0]->cfg.pipeDepth ||
        c->cfg.stagingTiles != ms[0]->cfg.stagingTiles || c->cfg.blocksPerSM != ms[0]->cfg.blocksPerSM)
      return occlInvalidArgument;
    if (c->L->members.size() != 1) return occlInvalidUsage;   // fuse single-member launchers only
    if (c->inflight.load() > 0) return occlInvalidUsage;
  }
  for (occlComm* c : ms) {
    Launcher* old = c->L;
    {
      std::lock_guard<std::mutex> lk(old->mu);
      if (daemon_running(old)) return occlInvalidUsage;
    }
  }
  for (occlComm* c : ms) launcher_stop(c->L);
  Launcher* L = new Launcher();
  occlResult_t r = launcher_start(L, ms);
  if (r != occlSuccess) launcher_stop(L);
  return r;
}

occlResult_t occlCommSplit(occlComm_t parent, int nmembers, const int* members, occlComm_t* out) {
  if (!parent || !members || !out || nmembers < 1) return occlInvalidArgument;
  occlComm* P = parent;
  if (P->parent || !P->connected) return occlInvalidUsage;          // split a root communicator
  if (P->freeRings.empty() && P->nrings >= kMaxRings) return occlInvalidUsage;
  std::vector<char> seen(P->nranks, 0);
  int me = -1;
  for (int i = 0; i < nmembers; ++i) {
    const int q = members[i];
    if (q < 0 || q >= P->nranks || seen[q]) return occlInvalidArgument;
    seen[q] = 1;
    if (q == P->rank) me = i;
  }
  if (me < 0) return occlInvalidArgument;                            // callers are members
  cudaSetDevice(P->dev);
  const int mypid = (int)getpid();
  const uint64_t myhost = (uint64_t)gethostid();
  auto peer = [&](int q, char** ptr) -> occlResult_t {              // open (once) the arena of parent rank q
    if (P->peerArena[q]) { *ptr = P->peerArena[q]; return occlSuccess; }
    const Handle& h = P->handles[q];
    if (h.pid == mypid && h.hostId == myhost) {
      if (h.dev != P->dev) {
        cudaError_t e = cudaDeviceEnablePeerAccess(h.dev, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else if (e != cudaSuccess) return cuda_fail(P, e);
      }
      P->peerArena[q] = reinterpret_cast<char*>(h.arenaPtr);
    } else {
      void* p = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&p, h.ipc, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) return cuda_fail(P, e);
      P->peerArena[q] = static_cast<char*>(p);
      P->peerIpc[q] = 1;
    }
    *ptr = P->peerArena[q];
    return occlSuccess;
  };
  const int nq = members[(me + 1) % nmembers], pq = members[(me - 1 + nmembers) % nmembers];
  char *na = nullptr, *pa = nullptr;
  occlResult_t r;
  if ((r = peer(nq, &na)) != occlSuccess) return r;
  if ((r = peer(pq, &pa)) != occlSuccess) return r;
  RingDesc rd{};
  rd.dataNext = na;
  rd.llNext = na + P->handles[nq].llOffset;
  rd.flagsNext = na + P->handles[nq].flagsOffset;
  rd.flagsPrev = pa + P->handles[pq].flagsOffset;
  rd.nranks = nmembers;
  rd.rank = me;
  rd.directNext = P->cfg.directMode && !P->peerIpc[nq] && !P->cfg.forceSysScope;
  rd.directPrev = P->cfg.directMode && !P->peerIpc[pq] && !P->cfg.forceSysScope;
  for (int i = 0; i < nmembers; ++i) {                                // readiness board of every member
    char* a = nullptr;
    if (members[i] == P->rank) a = P->arena;
    else if ((r = peer(members[i], &a)) != occlSuccess) return r;
    rd.flagsOf[i] = a + P->handles[members[i]].flagsOffset;
  }
  // the new entry is written before any submission names it (the SQE's release
  // store orders it for the daemon)
  // a destroyed child's slot is reused: the ids bound to it were retired
  const int slot = P->freeRings.empty() ? P->nrings : P->freeRings.back();
  if (cudaMemcpy(P->ringsDev + slot, &rd, sizeof(rd), cudaMemcpyHostToDevice) != cudaSuccess)
    return occlCudaError;
  if (slot == P->nrings) P->nrings++;
  else P->freeRings.pop_back();
  occlComm* c = new occlComm();
  c->parent = P;
  c->sub = slot;
  c->nranks = nmembers;
  c->rank = me;
  c->dev = P->dev;
  c->cfg = P->cfg;
  c->connected = true;
  P->children++;
  *out = c;
  return occlSuccess;
}

occlResult_t occlCommInit(occlComm_t* out, int nranks, int rank, int cudaDev, occlAllGatherFn ag, void* agCtx,
                          const occlConfig_t* cfg) {
  if (!out || !ag) return occlInvalidArgument;
  occlComm_t c = nullptr;
  occlResult_t r = occlCommCreate(&c, nranks, rank, cudaDev, cfg);
  if (r != occlSuccess) return r;
  std::vector<char> mine(OCCL_HANDLE_BYTES, 0), all((size_t)OCCL_HANDLE_BYTES * nranks, 0);
  size_t len = OCCL_HANDLE_BYTES;
  if ((r = occlCommGetHandle(c, mine.data(), &len)) != occlSuccess) { occlCommDestroy(c); return r; }
  if (ag(mine.data(), all.data(), OCCL_HANDLE_BYTES, agCtx) != 0) { occlCommDestroy(c); return occlSystemError; }
  if ((r = occlCommConnect(c, all.data(), OCCL_HANDLE_BYTES)) != occlSuccess) { occlCommDestroy(c); return r; }
  *out = c;
  return occlSuccess;
}

occlResult_t occlCommDestroy(occlComm_t c) {
  if (!c) return occlInvalidArgument;
  if (c->parent) {                                     // sub-communicator: bookkeeping only
    occlComm* R = c->parent;
    if (c->inflight.load() > 0 && !comm_sticky(R)) {
      for (int id = 0; id < R->cfg.maxColl; ++id)
        if (R->owner[id] == c) try_complete(R, id);
      if (c->inflight.load() > 0) return occlInvalidUsage;
    }
    for (int id = 0; id < R->cfg.maxColl; ++id) {
      if (R->owner[id] == c) R->owner[id] = nullptr;
      if (R->boundSub[id] == c->sub) R->boundSub[id] = -2;   // retired: its counters belong to that ring
    }
    R->freeRings.push_back(c->sub);
    R->children--;
    delete c;
    return occlSuccess;
  }
  if (c->children > 0) return occlInvalidUsage;        // destroy the sub-communicators first
  // a sticky-errored communicator cannot complete its in-flight work: it may be
  // destroyed regardless (there is no daemon to drain)
  if (c->inflight.load() > 0 && !comm_sticky(c)) {
    for (int id = 0; id < c->cfg.maxColl; ++id) try_complete(c, id);
    if (c->inflight.load() > 0) return occlInvalidUsage;
  }
  cudaSetDevice(c->dev);
  Launcher* L = c->L;
  if (L) {
    {
      std::lock_guard<std::mutex> lk(L->mu);
      if (daemon_running(L)) {
        // Exiting SQE to every member: the daemon drains and exits.
        // Each waits for a free SQ slot as push_sqe does (a running daemon always
        // drains the SQ, invariant I4); a daemon that stopped needs no Exiting SQE.
        for (occlComm* m : L->members) {
          Sqe e{};
          e.kind = kExit;
          std::lock_guard<std::mutex> g(m->sqMu);
          bool room = true;
          while (m->sqTail.load() - min_cursor(m) >= (uint64_t)m->cfg.sqDepth) {
            if (!daemon_running(L)) { room = false; break; }
            std::this_thread::yield();
          }
          if (room) write_sqe(m, e);
        }
      }
    }
    if (L->members.size() <= 1) {
      launcher_stop(L);
    } else {
      // a fused member leaves: relaunch-capable launcher keeps serving the others
      L->stop.store(true);
      L->cv.notify_all();
      if (L->sup.joinable()) L->sup.join();
      if (L->launched) cudaEventSynchronize(L->evDone);
      std::vector<occlComm*> rest;
      for (occlComm* m : L->members)
        if (m != c) rest.push_back(m);
      launcher_stop(L);
      Launcher* L2 = new Launcher();
      if (launcher_start(L2, rest) != occlSuccess) launcher_stop(L2);
    }
  }
  free_comm(c);
  delete c;
  return occlSuccess;
}

occlResult_t occlAllReduce(const void* s, void* r, size_t count, occlDataType_t dt, occlRedOp_t op, int id,
                           occlComm_t c) {
  return submit(c, kAllReduce, dt, op, 0, count, s, r, id);
}
occlResult_t occlAllGather(const void* s, void* r, size_t sendcount, occlDataType_t dt, int id, occlComm_t c) {
  return submit(c, kAllGather, dt, occlSum, 0, sendcount, s, r, id);
}
occlResult_t occlReduceScatter(const void* s, void* r, size_t recvcount, occlDataType_t dt, occlRedOp_t op, int id,
                               occlComm_t c) {
  return submit(c, kReduceScatter, dt, op, 0, recvcount, s, r, id);
}
occlResult_t occlBroadcast(const void* s, void* r, size_t count, occlDataType_t dt, int root, int id, occlComm_t c) {
  return submit(c, kBroadcast, dt, occlSum, root, count, s, r, id);
}
occlResult_t occlReduce(const void* s, void* r, size_t count, occlDataType_t dt, occlRedOp_t op, int root, int id,
                        occlComm_t c) {
  return submit(c, kReduce, dt, op, root, count, s, r, id);
}

occlResult_t occlTest(occlComm_t c, int id, int* done) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !done || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (tok_seq(c->tok[id].load()) == 0) return occlUnknownId;
  if (tok_inflight(c->tok[id].load())) try_complete(c, id);
  *done = !tok_inflight(c->tok[id].load());
  if (!*done && comm_sticky(c)) return occlCudaError;
  return occlSuccess;
}

occlResult_t occlWait(occlComm_t c, int id, int64_t timeoutNs) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (tok_seq(c->tok[id].load()) == 0) return occlUnknownId;
  const uint64_t t0 = now_ns();
  uint64_t it = 0;
  for (;;) {
    if (!tok_inflight(c->tok[id].load(std::memory_order_acquire))) return occlSuccess;
    if (try_complete(c, id)) return occlSuccess;
    if (!tok_inflight(c->tok[id].load())) return occlSuccess;
    if (comm_sticky(c)) return occlCudaError;
    if ((++it & 1023) == 0) {
      if (c->L) {
        std::lock_guard<std::mutex> lk(c->L->mu);
        daemon_running(c->L);                    // surfaces asynchronous device faults
      }
      if (timeoutNs >= 0 && now_ns() - t0 > (uint64_t)timeoutNs) return occlTimeout;
      std::this_thread::yield();
    } else {
      cpu_relax();
    }
  }
}

occlResult_t occlSetCallback(occlComm_t c, int id, occlCallback_t cb, void* arg) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (tok_inflight(c->tok[id].load())) return occlInvalidUsage;   // rebinding only between submissions
  c->cbArg[id] = arg;
  c->cb[id] = cb;
  return occlSuccess;
}

occlResult_t occlGetStats(occlComm_t c, occlStats_t* out) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !out) return occlInvalidArgument;
  std::memset(out, 0, sizeof(*out));
  const size_t M = c->cfg.maxColl, G = c->cfg.gridBlocks;
  std::vector<BlockStat> bs(G);
  std::vector<CollStat> cs(M * G);
  cudaSetDevice(c->dev);
  CUDACHECK(c, cudaMemcpyAsync(bs.data(), c->blkStats, G * sizeof(BlockStat), cudaMemcpyDeviceToHost, c->statsStream));
  CUDACHECK(c, cudaMemcpyAsync(cs.data(), c->collStats, M * G * sizeof(CollStat), cudaMemcpyDeviceToHost,
                               c->statsStream));
  CUDACHECK(c, cudaStreamSynchronize(c->statsStream));
  for (auto& b : bs) {
    out->quits += b.quits;
    out->exits += b.exits;
    out->sqeFetched += b.fetched;
    out->cqeWritten += b.cqes;
  }
  for (auto& s : cs) {
    out->preemptions += s.preemptions;
    out->ctxLoads += s.ctxLoads;
    out->ctxSaves += s.ctxSaves;
    out->slices += s.slices;
  }
  if (c->L) {
    std::lock_guard<std::mutex> lk(c->L->mu);
    daemon_running(c->L);
    out->launches = c->L->launches;
    out->lastLaunchMs = c->L->lastLaunchMs;
  }
  return occlSuccess;
}

occlResult_t occlGetCollStats(occlComm_t c, int id, occlCollStats_t* out) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !out || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  const size_t G = c->cfg.gridBlocks;
  std::vector<CollStat> cs(G);
  cudaSetDevice(c->dev);
  CUDACHECK(c, cudaMemcpyAsync(cs.data(), c->collStats + (size_t)id * G, G * sizeof(CollStat),
                               cudaMemcpyDeviceToHost, c->statsStream));
  CUDACHECK(c, cudaStreamSynchronize(c->statsStream));
  std::memset(out, 0, sizeof(*out));
  for (auto& s : cs) {
    out->preemptions += s.preemptions;
    out->ctxLoads += s.ctxLoads;
    out->ctxSaves += s.ctxSaves;
    out->slices += s.slices;
    out->completions += s.completions;
  }
  return occlSuccess;
}

occlResult_t occlGetProbes(occlComm_t c, occlProbes_t* out) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !out) return occlInvalidArgument;
  const size_t G = c->cfg.gridBlocks;
  std::vector<BlockStat> bs(G);
  cudaSetDevice(c->dev);
  CUDACHECK(c, cudaMemcpyAsync(bs.data(), c->blkStats, G * sizeof(BlockStat), cudaMemcpyDeviceToHost, c->statsStream));
  CUDACHECK(c, cudaStreamSynchronize(c->statsStream));
  std::memset(out, 0, sizeof(*out));
  for (auto& b : bs) {
    out->cycRun += b.cycRun;
    out->cycPoll += b.cycPoll;
    out->cycAcqFence += b.cycAcqFence;
    out->cycRelFence += b.cycRelFence;
    out->nFence += b.nFence;
    out->cycCtxLoad += b.cycCtxLoad;
    out->nCtxLoad += b.nCtxLoad;
    out->cycCtxSave += b.cycCtxSave;
    out->nCtxSave += b.nCtxSave;
    out->cycCqe += b.cycCqe;
    out->nCqe += b.nCqe;
    out->cycData += b.cycData;
    out->cycDataWait += b.cycDataWait;
    out->nData += b.nData;
    out->nCommit += b.nCommit;
  }
  return occlSuccess;
}

occlResult_t occlGetTrace(occlComm_t c, int block, occlTraceRec_t* out, size_t cap, size_t* n) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !n || block < 0 || block >= c->cfg.gridBlocks || (cap && !out)) return occlInvalidArgument;
  *n = 0;
  if (!c->cfg.traceCap) return occlSuccess;
  cudaSetDevice(c->dev);
  uint32_t cnt = 0;
  const size_t tc = c->cfg.traceCap;
  std::vector<TraceRec> ring(tc);
  CUDACHECK(c, cudaMemcpyAsync(&cnt, c->traceCount + block, sizeof(cnt), cudaMemcpyDeviceToHost, c->statsStream));
  CUDACHECK(c, cudaMemcpyAsync(ring.data(), c->trace + (size_t)block * tc, tc * sizeof(TraceRec),
                               cudaMemcpyDeviceToHost, c->statsStream));
  CUDACHECK(c, cudaStreamSynchronize(c->statsStream));
  const size_t have = cnt < tc ? cnt : tc;
  const size_t first = cnt - have;                 // oldest record still in the ring
  size_t k = 0;
  for (; k < have && k < cap; ++k) {
    const TraceRec& r = ring[(first + k) % tc];
    out[k].t = r.t;
    out[k].tag = r.tag;
    out[k].arg = r.arg;
  }
  *n = k;
  return occlSuccess;
}

occlResult_t occlTraceReset(occlComm_t c) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c) return occlInvalidArgument;
  cudaSetDevice(c->dev);
  if (c->L) {
    std::lock_guard<std::mutex> lk(c->L->mu);
    if (daemon_running(c->L)) return occlInvalidUsage;
  }
  CUDACHECK(c, cudaMemsetAsync(c->traceCount, 0, c->cfg.gridBlocks * sizeof(uint32_t), c->statsStream));
  CUDACHECK(c, cudaStreamSynchronize(c->statsStream));
  return occlSuccess;
}

occlResult_t occlGetFootprint(occlComm_t c, occlFootprint_t* out) {
  if (!c || !out) return occlInvalidArgument;
  c = root_of(c);
  const size_t M = c->cfg.maxColl, G = c->cfg.gridBlocks;
  std::memset(out, 0, sizeof(*out));
  out->connectorData = c->dataBytes;
  out->connectorFlags = c->flagsBytes;
  out->llLines = c->llBytes;
  out->contexts = M * G * sizeof(CtxSlot);
  out->other = c->cfg.sqDepth * sizeof(Sqe) + 3 * sizeof(uint64_t) + G * sizeof(BlockState) +
               G * M * sizeof(uint32_t) + M * sizeof(uint32_t) + M * G * sizeof(CollStat) + G * sizeof(BlockStat) +
               (size_t)G * c->cfg.traceCap * sizeof(TraceRec) + G * sizeof(uint32_t) +
               (c->ringsDev ? kMaxRings * sizeof(RingDesc) : 0);
  out->device = out->connectorData + out->connectorFlags + out->llLines + out->contexts + out->other;
  out->pinnedHost = c->cfg.sqDepth * sizeof(SqeWire) + G * sizeof(uint64_t) + M * sizeof(uint64_t) +
                    (c->cqDepth ? (c->cqDepth + 1) * sizeof(uint64_t) : 0);
  out->perBlockPerColl = (double)(out->device) / (double)(M * G);
  return occlSuccess;
}

occlResult_t occlSetPriority(occlComm_t c, int id, int32_t priority) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  c->prio[id] = priority;
  return occlSuccess;
}

occlResult_t occlCommExit(occlComm_t c) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c) return occlInvalidArgument;
  if (!c->connected || !c->L) return occlInvalidUsage;
  Sqe e{};
  e.kind = kExit;
  return push_sqe(c, e, true);
}

occlResult_t occlCommLaunch(occlComm_t c) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c) return occlInvalidArgument;
  if (!c->connected || !c->L) return occlInvalidUsage;
  cudaSetDevice(c->dev);
  std::lock_guard<std::mutex> lk(c->L->mu);
  return launch_locked(c->L);
}

occlResult_t occlCommSetAutoLaunch(occlComm_t c, int enable) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !c->L) return occlInvalidArgument;
  c->L->autoLaunch.store(enable ? 1 : 0);
  c->L->cv.notify_one();
  return occlSuccess;
}

occlResult_t occlCommQuiesce(occlComm_t c, int64_t timeoutNs) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !c->L) return occlInvalidArgument;
  const uint64_t t0 = now_ns();
  for (;;) {
    {
      std::lock_guard<std::mutex> lk(c->L->mu);
      if (!daemon_running(c->L)) return comm_sticky(c) ? occlCudaError : occlSuccess;
    }
    if (timeoutNs >= 0 && now_ns() - t0 > (uint64_t)timeoutNs) return occlTimeout;
    std::this_thread::sleep_for(std::chrono::microseconds(10));
  }
}

occlResult_t occlCommGetStream(occlComm_t c, void** stream) {
  c = root_of(c);                                      // sub-communicators use their root's daemon
  if (!c || !stream || !c->L) return occlInvalidArgument;
  *stream = (void*)c->L->stream;
  return occlSuccess;
}

occlResult_t occlCollBlocks(occlComm_t c, int kind, size_t count, occlDataType_t dt, int* nblocks) {
  if (!c || !nblocks || kind < 0 || kind > 4 || dt < 0 || dt > 5) return occlInvalidArgument;
  *nblocks = coll_blocks(c, kind, count, dt);
  return occlSuccess;
}

}  // extern "C"
