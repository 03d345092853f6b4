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
constexpr uint32_t kHandleVersion = 1;

struct Handle {
  uint32_t magic, version;
  int32_t nranks, rank, dev, pid;
  uint64_t hostId;
  uint64_t arenaPtr;
  uint64_t dataBytes, flagsOffset;
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

int elem_size(int dt) { return dt == kBF16 ? 2 : 4; }

uint64_t fingerprint(const occlConfig_t& c) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  mix(c.maxColl); mix(c.gridBlocks); mix(c.connSlots); mix(c.slicesPerChunk); mix(c.sliceBytes);
  mix(c.minBlockBytes);
  return h;
}

}  // namespace

struct occlComm {
  int nranks = 0, rank = 0, dev = 0;
  occlConfig_t cfg{};
  // device memory
  char* arena = nullptr;
  size_t dataBytes = 0, flagsBytes = 0;
  CtxSlot* ctx = nullptr;
  BlockState* blk = nullptr;
  uint32_t* tqSave = nullptr;
  uint32_t* complCnt = nullptr;
  CollStat* collStats = nullptr;
  BlockStat* blkStats = nullptr;
  DaemonParams* paramsDev = nullptr;
  // pinned + mapped host memory
  Sqe* sqHost = nullptr;
  Sqe* sqDev = nullptr;
  uint64_t* sqCurHost = nullptr;
  uint64_t* sqCurDev = nullptr;
  uint64_t* cqHost = nullptr;
  uint64_t* cqDev = nullptr;
  uint64_t sqTail = 0;
  // per-collective host state
  std::vector<uint64_t> subSeq;
  std::unique_ptr<std::atomic<int>[]> state;     // 0 idle, 1 in flight
  std::vector<occlCallback_t> cb;
  std::vector<void*> cbArg;
  std::atomic<int> inflight{0};
  // peers
  char* nextArena = nullptr;
  char* prevArena = nullptr;
  bool nextIpc = false, prevIpc = false;
  int sysScope = 0;
  DaemonParams params{};
  bool connected = false;
  // daemon lifecycle
  cudaStream_t stream = nullptr, statsStream = nullptr;
  cudaEvent_t evStart = nullptr, evDone = nullptr;
  bool launched = false;
  uint64_t launches = 0;
  float lastLaunchMs = 0.f;
  uint64_t lastExitNs = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::thread sup;
  std::atomic<bool> stop{false};
  std::atomic<int> autoLaunch{1};
  std::atomic<int> sticky{0};
};

namespace {

occlResult_t cuda_fail(occlComm* c, cudaError_t e) {
  if (c) c->sticky.store((int)e);
  return occlCudaError;
}
#define CUDACHECK(comm, call)                      \
  do {                                             \
    cudaError_t e_ = (call);                       \
    if (e_ != cudaSuccess) return cuda_fail(comm, e_); \
  } while (0)

uint64_t min_cursor(occlComm* c) {
  uint64_t m = UINT64_MAX;
  for (int b = 0; b < c->cfg.gridBlocks; ++b) {
    uint64_t v = reinterpret_cast<volatile uint64_t*>(c->sqCurHost)[b];
    if (v < m) m = v;
  }
  return m;
}

// caller holds mu
bool daemon_running(occlComm* c) {
  if (!c->launched) return false;
  cudaError_t q = cudaEventQuery(c->evDone);
  if (q == cudaErrorNotReady) return true;
  if (q == cudaSuccess) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->evStart, c->evDone) == cudaSuccess) c->lastLaunchMs = ms;
    c->launched = false;
    c->lastExitNs = now_ns();
    return false;
  }
  c->sticky.store((int)q);
  c->launched = false;
  return false;
}

// caller holds mu
occlResult_t launch_locked(occlComm* c) {
  if (c->sticky.load()) return occlCudaError;
  if (daemon_running(c)) return occlSuccess;
  CUDACHECK(c, cudaEventRecord(c->evStart, c->stream));
  int e = occl_internal_launch_daemon(&c->params, c->paramsDev, c->cfg.blockThreads, c->stream);
  if (e != 0) return cuda_fail(c, (cudaError_t)e);
  CUDACHECK(c, cudaEventRecord(c->evDone, c->stream));
  c->launched = true;
  c->launches++;
  return occlSuccess;
}

bool try_complete(occlComm* c, int id) {
  if (c->state[id].load(std::memory_order_acquire) != 1) return false;
  const uint64_t done = reinterpret_cast<volatile uint64_t*>(c->cqHost)[id];
  if (done < c->subSeq[id]) return false;
  int one = 1;
  if (!c->state[id].compare_exchange_strong(one, 0)) return false;
  c->inflight.fetch_sub(1);
  occlCallback_t f = c->cb[id];
  if (f) f(id, c->cbArg[id]);                   // exactly once per completion
  return true;
}

// Supervisor: poller + callback map + event-driven (re)start.
void supervisor_main(occlComm* c) {
  cudaSetDevice(c->dev);
  uint64_t backoffNs = 50'000;
  while (!c->stop.load()) {
    bool pending;
    {
      std::lock_guard<std::mutex> lk(c->mu);
      const bool newSqe = c->sqTail > min_cursor(c);
      pending = newSqe || c->inflight.load() > 0;
      if (c->autoLaunch.load() && pending && !daemon_running(c) && !c->sticky.load()) {
        // new SQEs start the daemon at once; collectives that are merely stuck
        // (the daemon quit voluntarily) restart after a back-off so that device
        // synchronisation on the host can complete in between
        if (newSqe || now_ns() - c->lastExitNs > backoffNs) launch_locked(c);
      }
    }
    for (int id = 0; id < c->cfg.maxColl && c->inflight.load() > 0; ++id)
      if (c->cb[id] && c->state[id].load() == 1) try_complete(c, id);
    if (!pending) {
      std::unique_lock<std::mutex> lk(c->mu);
      c->cv.wait_for(lk, std::chrono::milliseconds(5));
    } else {
      std::this_thread::sleep_for(std::chrono::microseconds(20));
    }
  }
}

occlResult_t validate_config(const occlConfig_t& c) {
  if (c.maxColl < 1 || c.maxColl > 65535) return occlInvalidArgument;
  if (c.gridBlocks < 1 || c.gridBlocks > 1024) return occlInvalidArgument;
  if (c.blockThreads < 32 || c.blockThreads > 512 || c.blockThreads % 32) return occlInvalidArgument;
  if (c.slicesPerChunk < 1 || c.connSlots <= c.slicesPerChunk) return occlInvalidArgument;  // invariant I7
  if (c.sliceBytes < 16 || c.sliceBytes % 16 || c.sliceBytes > (1ull << 30)) return occlInvalidArgument;
  if (c.minBlockBytes < 1) return occlInvalidArgument;
  if (c.sqDepth < 2) return occlInvalidArgument;
  if (c.cacheWays < 1 || c.cacheWays > kMaxCacheWays) return occlInvalidArgument;
  if (c.spinMin < 1 || c.spinBase < c.spinMin || c.spinCap < c.spinBase || c.spinBoost < 1) return occlInvalidArgument;
  if (c.priorityCadence < 1) return occlInvalidArgument;
  if (c.stallLimit < 1) return occlInvalidArgument;
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
  uint64_t nb = (bytes + c->cfg.minBlockBytes - 1) / c->cfg.minBlockBytes;
  if (nb < 1) nb = 1;
  if (nb > (uint64_t)c->cfg.gridBlocks) nb = c->cfg.gridBlocks;
  return (int)nb;
}

occlResult_t push_sqe(occlComm* c, Sqe& e, bool launchNow) {
  std::unique_lock<std::mutex> lk(c->mu);
  // wait for a free slot: the daemon always drains the SQ (invariant I4)
  while (c->sqTail - min_cursor(c) >= (uint64_t)c->cfg.sqDepth) {
    if (c->sticky.load()) return occlCudaError;
    if (c->autoLaunch.load() && !daemon_running(c)) launch_locked(c);
    lk.unlock();
    std::this_thread::yield();
    lk.lock();
  }
  Sqe* s = &c->sqHost[c->sqTail % c->cfg.sqDepth];
  e.seq = 0;
  std::memcpy(reinterpret_cast<char*>(s) + 8, reinterpret_cast<const char*>(&e) + 8, sizeof(Sqe) - 8);
  std::atomic_thread_fence(std::memory_order_release);
  reinterpret_cast<std::atomic<uint64_t>*>(&s->seq)->store(c->sqTail + 1, std::memory_order_release);
  c->sqTail++;
  occlResult_t r = occlSuccess;
  if (launchNow && c->autoLaunch.load() && !daemon_running(c)) r = launch_locked(c);
  lk.unlock();
  c->cv.notify_one();
  return r;
}

occlResult_t submit(occlComm* c, int kind, int dtype, int op, int root, size_t count, const void* send,
                    void* recv, int collId) {
  if (!c) return occlInvalidArgument;
  if (!c->connected) return occlInvalidUsage;
  if (c->sticky.load()) return occlCudaError;
  if (collId < 0) return occlInvalidArgument;
  if (collId >= c->cfg.maxColl) return occlRegistryFull;
  if (dtype < 0 || dtype > 2) return occlInvalidArgument;
  if (op != occlSum) return occlInvalidArgument;
  if (kind == kBroadcast && (root < 0 || root >= c->nranks)) return occlInvalidArgument;
  if (count > 0 && (!send || !recv)) return occlInvalidArgument;
  if (c->state[collId].load() == 1 && !try_complete(c, collId)) return occlDuplicateSubmit;
  c->subSeq[collId]++;
  if (count == 0) {                                   // completes at submission (reading Q18)
    reinterpret_cast<volatile uint64_t*>(c->cqHost)[collId] = c->subSeq[collId];
    if (c->cb[collId]) c->cb[collId](collId, c->cbArg[collId]);
    return occlSuccess;
  }
  Sqe e{};
  e.subSeq = c->subSeq[collId];
  e.count = count;
  e.sendbuff = (uint64_t)(uintptr_t)send;
  e.recvbuff = (uint64_t)(uintptr_t)recv;
  e.collId = (uint32_t)collId;
  e.kind = (uint16_t)kind;
  e.dtype = (uint16_t)dtype;
  e.op = (uint16_t)op;
  e.nblocks = (uint16_t)coll_blocks(c, kind, count, dtype);
  e.root = root;
  c->state[collId].store(1, std::memory_order_release);
  c->inflight.fetch_add(1);
  return push_sqe(c, e, true);
}

void free_all(occlComm* c) {
  if (c->nextIpc && c->nextArena) cudaIpcCloseMemHandle(c->nextArena);
  if (c->prevIpc && c->prevArena && c->prevArena != c->nextArena) cudaIpcCloseMemHandle(c->prevArena);
  if (c->arena) cudaFree(c->arena);
  if (c->ctx) cudaFree(c->ctx);
  if (c->blk) cudaFree(c->blk);
  if (c->tqSave) cudaFree(c->tqSave);
  if (c->complCnt) cudaFree(c->complCnt);
  if (c->collStats) cudaFree(c->collStats);
  if (c->blkStats) cudaFree(c->blkStats);
  if (c->paramsDev) cudaFree(c->paramsDev);
  if (c->sqHost) cudaFreeHost(c->sqHost);
  if (c->sqCurHost) cudaFreeHost(c->sqCurHost);
  if (c->cqHost) cudaFreeHost(c->cqHost);
  if (c->evStart) cudaEventDestroy(c->evStart);
  if (c->evDone) cudaEventDestroy(c->evDone);
  if (c->stream) cudaStreamDestroy(c->stream);
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
  c->blockThreads = 512;
  c->connSlots = 4;
  c->slicesPerChunk = 2;
  c->sliceBytes = 64 << 10;
  c->minBlockBytes = 128 << 10;
  c->sqDepth = 1024;
  c->orderPolicy = occlOrderFifo;
  c->priorityCadence = 8;
  c->stickiness = 1;
  c->spinBase = 1 << 14;
  c->spinStep = 1 << 10;
  c->spinMin = 1 << 10;
  c->spinBoost = 2;
  c->spinCap = 1 << 16;
  c->stallLimit = 2;
  c->quitEnabled = 1;
  c->quitIdleNs = 1'000'000;
  c->idleSleepNs = 256;
  c->autoLaunch = 1;
  c->cacheWays = 8;
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
  c->subSeq.assign(M, 0);
  c->state.reset(new std::atomic<int>[M]);
  for (size_t i = 0; i < M; ++i) c->state[i].store(0);
  c->cb.assign(M, nullptr);
  c->cbArg.assign(M, nullptr);
  occlComm* cp = c.get();
  auto fail = [&](cudaError_t e) { free_all(cp); (void)e; return occlCudaError; };
  cudaError_t e;
  if ((e = cudaSetDevice(cudaDev)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->arena, c->dataBytes + c->flagsBytes)) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->arena + c->dataBytes, 0, c->flagsBytes)) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->ctx, M * G * sizeof(CtxSlot))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->ctx, 0, M * G * sizeof(CtxSlot))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->blk, G * sizeof(BlockState))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->blk, 0, G * sizeof(BlockState))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->tqSave, G * M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->complCnt, M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->complCnt, 0, M * sizeof(uint32_t))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->collStats, M * G * sizeof(CollStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->collStats, 0, M * G * sizeof(CollStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->blkStats, G * sizeof(BlockStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMemset(cp->blkStats, 0, G * sizeof(BlockStat))) != cudaSuccess) return fail(e);
  if ((e = cudaMalloc(&cp->paramsDev, sizeof(DaemonParams))) != cudaSuccess) return fail(e);
  const unsigned flags = cudaHostAllocMapped | cudaHostAllocPortable;
  if ((e = cudaHostAlloc(&cp->sqHost, cfg.sqDepth * sizeof(Sqe), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->sqHost, 0, cfg.sqDepth * sizeof(Sqe));
  if ((e = cudaHostGetDevicePointer(&cp->sqDev, cp->sqHost, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaHostAlloc(&cp->sqCurHost, G * sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->sqCurHost, 0, G * sizeof(uint64_t));
  if ((e = cudaHostGetDevicePointer(&cp->sqCurDev, cp->sqCurHost, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaHostAlloc(&cp->cqHost, M * sizeof(uint64_t), flags)) != cudaSuccess) return fail(e);
  std::memset(cp->cqHost, 0, M * sizeof(uint64_t));
  if ((e = cudaHostGetDevicePointer(&cp->cqDev, cp->cqHost, 0)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&cp->stream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaStreamCreateWithFlags(&cp->statsStream, cudaStreamNonBlocking)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&cp->evStart)) != cudaSuccess) return fail(e);
  if ((e = cudaEventCreate(&cp->evDone)) != cudaSuccess) return fail(e);
  if ((e = cudaDeviceSynchronize()) != cudaSuccess) return fail(e);
  cp->autoLaunch.store(cfg.autoLaunch ? 1 : 0);
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
  h.cfgFingerprint = fingerprint(c->cfg);
  cudaSetDevice(c->dev);
  if (cudaIpcGetMemHandle(&h.ipc, c->arena) != cudaSuccess) {
    // IPC may be unavailable (e.g. some virtualised setups); same-process peers
    // do not need it.
    cudaGetLastError();
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
  occlResult_t r;
  if ((r = open(hs[next], &c->nextArena, &c->nextIpc)) != occlSuccess) return r;
  if (prev == next) {
    c->prevArena = c->nextArena;
  } else if ((r = open(hs[prev], &c->prevArena, &c->prevIpc)) != occlSuccess) {
    return r;
  }
  c->sysScope = local ? 0 : 1;
  DaemonParams& p = c->params;
  p.sq = c->sqDev;
  p.sqCursorHost = c->sqCurDev;
  p.cqDone = c->cqDev;
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
  p.stallLimit = c->cfg.stallLimit;
  p.quitEnabled = c->cfg.quitEnabled;
  p.quitIdleNs = c->cfg.quitIdleNs;
  p.idleSleepNs = c->cfg.idleSleepNs;
  p.cacheWays = c->cfg.cacheWays;
  p.sysScope = c->sysScope;
  CUDACHECK(c, cudaMemcpy(c->paramsDev, &p, sizeof(p), cudaMemcpyHostToDevice));
  c->connected = true;
  try {
    c->sup = std::thread(supervisor_main, c);
  } catch (...) {
    c->connected = false;
    return occlSystemError;
  }
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
  if (c->inflight.load() > 0) {
    for (int id = 0; id < c->cfg.maxColl; ++id) try_complete(c, id);
    if (c->inflight.load() > 0) return occlInvalidUsage;
  }
  c->stop.store(true);
  c->cv.notify_all();
  if (c->sup.joinable()) c->sup.join();
  cudaSetDevice(c->dev);
  {
    std::lock_guard<std::mutex> lk(c->mu);
    if (c->connected && daemon_running(c)) {
      // Exiting SQE: the daemon drains and exits
      Sqe e{};
      e.kind = kExit;
      Sqe* s = &c->sqHost[c->sqTail % c->cfg.sqDepth];
      std::memcpy(reinterpret_cast<char*>(s) + 8, reinterpret_cast<const char*>(&e) + 8, sizeof(Sqe) - 8);
      std::atomic_thread_fence(std::memory_order_release);
      reinterpret_cast<std::atomic<uint64_t>*>(&s->seq)->store(c->sqTail + 1, std::memory_order_release);
      c->sqTail++;
    }
  }
  if (c->launched) cudaEventSynchronize(c->evDone);
  free_all(c);
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

occlResult_t occlTest(occlComm_t c, int id, int* done) {
  if (!c || !done || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (c->subSeq[id] == 0) return occlUnknownId;
  if (c->state[id].load() == 1) try_complete(c, id);
  *done = c->state[id].load() == 0;
  if (!*done && c->sticky.load()) return occlCudaError;
  return occlSuccess;
}

occlResult_t occlWait(occlComm_t c, int id, int64_t timeoutNs) {
  if (!c || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (c->subSeq[id] == 0) return occlUnknownId;
  const uint64_t t0 = now_ns();
  uint64_t it = 0;
  for (;;) {
    if (c->state[id].load(std::memory_order_acquire) == 0) return occlSuccess;
    if (try_complete(c, id)) return occlSuccess;
    if (c->state[id].load() == 0) return occlSuccess;
    if (c->sticky.load()) return occlCudaError;
    if ((++it & 1023) == 0) {
      {
        std::lock_guard<std::mutex> lk(c->mu);
        daemon_running(c);                       // surfaces asynchronous device faults
      }
      if (timeoutNs >= 0 && now_ns() - t0 > (uint64_t)timeoutNs) return occlTimeout;
      std::this_thread::yield();
    } else {
      cpu_relax();
    }
  }
}

occlResult_t occlSetCallback(occlComm_t c, int id, occlCallback_t cb, void* arg) {
  if (!c || id < 0) return occlInvalidArgument;
  if (id >= c->cfg.maxColl) return occlRegistryFull;
  if (c->state[id].load() == 1) return occlInvalidUsage;   // rebinding only between submissions
  c->cbArg[id] = arg;
  c->cb[id] = cb;
  return occlSuccess;
}

occlResult_t occlGetStats(occlComm_t c, occlStats_t* out) {
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
  std::lock_guard<std::mutex> lk(c->mu);
  daemon_running(c);
  out->launches = c->launches;
  out->lastLaunchMs = c->lastLaunchMs;
  return occlSuccess;
}

occlResult_t occlGetCollStats(occlComm_t c, int id, occlCollStats_t* out) {
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

occlResult_t occlCommExit(occlComm_t c) {
  if (!c) return occlInvalidArgument;
  if (!c->connected) return occlInvalidUsage;
  Sqe e{};
  e.kind = kExit;
  return push_sqe(c, e, true);
}

occlResult_t occlCommLaunch(occlComm_t c) {
  if (!c) return occlInvalidArgument;
  if (!c->connected) return occlInvalidUsage;
  cudaSetDevice(c->dev);
  std::lock_guard<std::mutex> lk(c->mu);
  return launch_locked(c);
}

occlResult_t occlCommSetAutoLaunch(occlComm_t c, int enable) {
  if (!c) return occlInvalidArgument;
  c->autoLaunch.store(enable ? 1 : 0);
  c->cv.notify_one();
  return occlSuccess;
}

occlResult_t occlCommQuiesce(occlComm_t c, int64_t timeoutNs) {
  if (!c) return occlInvalidArgument;
  const uint64_t t0 = now_ns();
  for (;;) {
    {
      std::lock_guard<std::mutex> lk(c->mu);
      if (!daemon_running(c)) return c->sticky.load() ? occlCudaError : occlSuccess;
    }
    if (timeoutNs >= 0 && now_ns() - t0 > (uint64_t)timeoutNs) return occlTimeout;
    std::this_thread::sleep_for(std::chrono::microseconds(10));
  }
}

occlResult_t occlCommGetStream(occlComm_t c, void** stream) {
  if (!c || !stream) return occlInvalidArgument;
  *stream = (void*)c->stream;
  return occlSuccess;
}

occlResult_t occlCollBlocks(occlComm_t c, int kind, size_t count, occlDataType_t dt, int* nblocks) {
  if (!c || !nblocks || kind < 0 || kind > 3 || dt < 0 || dt > 2) return occlInvalidArgument;
  *nblocks = coll_blocks(c, kind, count, dt);
  return occlSuccess;
}

}  // extern "C"
