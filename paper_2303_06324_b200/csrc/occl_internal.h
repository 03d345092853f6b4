// occl_internal.h -- layouts shared by the host runtime (occl_host.cc) and the
// daemon kernel (occl_daemon.cu).  Product code; shares nothing with the CPU reference.
#pragma once
#include <stdint.h>
#include <stddef.h>

namespace occl {

enum Kind : uint16_t { kAllReduce = 0, kAllGather = 1, kReduceScatter = 2, kBroadcast = 3, kReduce = 4, kExit = 15 };
enum Dtype : uint16_t { kI32 = 0, kF32 = 1, kBF16 = 2, kF16 = 3, kI64 = 4, kF64 = 5 };

constexpr int kMaxRanks = 64;
constexpr int kFlagStride = 384;        // per (coll, block): head @+0, credit @+128, direct @+256 (own lines)
constexpr int kDirectOff = 256;         // {u64 recvbuff, u64 subSeq} written by the downstream rank,
                                        // then {u64 sendbuff, u64 subSeq} written by the upstream (direct read)
constexpr int kCtxBytes = 128;          // one context slot (static + dynamic), 16 B aligned
constexpr int kMaxCacheWays = 32;

// Submission queue entry: 64 B, lives in pinned+mapped host memory.
// `seq` is written LAST by the host (release); the daemon accepts the slot iff
// seq == its cursor + 1.
struct alignas(64) Sqe {
  uint64_t seq;        // 1-based index of this SQE in the SQ stream
  uint64_t subSeq;     // per-collective submission number (what the CQ reports)
  uint64_t count;      // AR/BC: elements; AG: sendcount; RS: recvcount
  uint64_t sendbuff;
  uint64_t recvbuff;
  uint32_t collId;
  uint16_t kind;
  uint16_t dtype;
  uint16_t op;
  uint16_t nblocks;    // the collective's grid size
  int32_t root;
  int32_t priority;    // user-defined priority (lower runs first) for the priority order policy
  uint16_t sub;        // ring of this rank's daemon the collective runs on (0: the communicator,
                       // k: its k-th sub-communicator, occlCommSplit); local to this rank
  uint16_t pad;
};
static_assert(sizeof(Sqe) == 64, "Sqe must be 64 B");

// The SQE as it sits in the pinned host SQ: five 16-B chunks, each stamped with
// the low 32 bits of the SQE's 1-based sequence number.  The host writes every
// chunk with ONE aligned 16-B store, so a device read of a chunk sees either
// the old or the new chunk, never a mix; a slot is valid iff all five stamps
// equal the expected sequence number.  The daemon thus reads an SQE in a single
// PCIe round trip -- no "seq first, payload after an acquire" second trip.
constexpr int kWireChunks = 5;
struct alignas(128) SqeWire {
  uint32_t c[8][4];    // chunk k = {stamp, w0, w1, w2}; chunks 5..7 unused (128-B slot stride)
};
static_assert(sizeof(SqeWire) == 128, "SqeWire must be 128 B");
// Payload words of an Sqe in chunk order (15 x 32 bit; seq travels as the stamp).
#if defined(__CUDACC__)
#define OCCL_HD __host__ __device__ __forceinline__
#else
#define OCCL_HD inline
#endif
OCCL_HD void sqe_to_words(const Sqe& e, uint32_t w[15]) {
  w[0] = e.collId;
  w[1] = (uint32_t)e.kind | ((uint32_t)e.dtype << 16);
  w[2] = (uint32_t)e.op | ((uint32_t)e.nblocks << 16);
  w[3] = (uint32_t)e.subSeq; w[4] = (uint32_t)(e.subSeq >> 32);
  w[5] = (uint32_t)e.root;
  w[6] = (uint32_t)e.count; w[7] = (uint32_t)(e.count >> 32);
  w[8] = (uint32_t)e.priority;
  w[9] = (uint32_t)e.sendbuff; w[10] = (uint32_t)(e.sendbuff >> 32);
  w[11] = (uint32_t)e.sub;
  w[12] = (uint32_t)e.recvbuff; w[13] = (uint32_t)(e.recvbuff >> 32);
  w[14] = 0;
}
OCCL_HD void sqe_from_words(const uint32_t w[15], uint64_t seq, Sqe& e) {
  e.seq = seq;
  e.collId = w[0];
  e.kind = (uint16_t)w[1]; e.dtype = (uint16_t)(w[1] >> 16);
  e.op = (uint16_t)w[2]; e.nblocks = (uint16_t)(w[2] >> 16);
  e.subSeq = (uint64_t)w[3] | ((uint64_t)w[4] << 32);
  e.root = (int32_t)w[5];
  e.count = (uint64_t)w[6] | ((uint64_t)w[7] << 32);
  e.priority = (int32_t)w[8];
  e.sendbuff = (uint64_t)w[9] | ((uint64_t)w[10] << 32);
  e.sub = (uint16_t)w[11];
  e.pad = 0;
  e.recvbuff = (uint64_t)w[12] | ((uint64_t)w[13] << 32);
}

constexpr int kMaxRings = 32;           // communicator + sub-communicators served by one daemon
// One ring the daemon serves (the static context carries the
// collective's own nranks / rank).  Connectors and flags of a collective live at
// (collId, block) in every member's arena, so only the neighbours differ.
struct alignas(16) RingDesc {
  char* dataNext;      // downstream member's connector data
  char* llNext;        // downstream member's LL connector lines
  char* flagsNext;     // downstream member's flags
  char* flagsPrev;     // upstream member's flags
  int32_t nranks, rank;
  int32_t directNext, directPrev;
  char* flagsOf[kMaxRanks];   // every member's flags base, ring order (readiness board, R29)
};

// Static context: constant for one submission.  48 B.
struct alignas(16) StaticCtx {
  uint64_t sendbuff;
  uint64_t recvbuff;
  uint64_t subSeq;
  uint64_t segLen;     // elements per segment (AR: L; RS/AG: count; BC: count)
  uint64_t part;       // elements of each segment handled by one block (Pb)
  uint64_t count;
};
// Dynamic context: chunk (loop) id, primitive (step) id,
// slice id, plus the connector sequence numbers (heads/credits are monotonic per
// (collective, block) across submissions).  32 B.
struct alignas(16) DynCtx {
  uint32_t loop;
  uint16_t step;
  uint16_t slc;
  uint32_t nloops;
  uint16_t kind;
  uint8_t dtype;
  uint8_t progressed;
  uint64_t nsent;      // slices pushed into the downstream connector so far
  uint64_t nrecv;      // slices consumed from the upstream connector so far
};
struct alignas(16) CtxSlot {
  StaticCtx s;         // 48
  DynCtx d;            // 32
  int32_t root;        // meta that also belongs to the static part
  uint16_t nblocks;
  uint16_t nsteps;
  int32_t priority;
  uint32_t lane;       // this block's lane in the collective: (block - collId) mod G
  uint32_t sub;        // ring (RingDesc index) of the collective
  uint32_t proto;      // 0 = Simple (TMA slices, head/credit flags), 1 = LL (flags inside the data)
  uint32_t spc;        // slices per chunk of this collective: min(cfg, slices a block's part needs)
  uint32_t op;         // reducing function (occlRedOp_t)
  uint32_t pad[2];
};
static_assert(sizeof(CtxSlot) == kCtxBytes, "CtxSlot must be 128 B");

// Per-block state that survives a voluntary quit.
struct alignas(16) BlockState {
  uint64_t sqCursor;   // SQEs consumed by this block
  uint32_t qlen;       // task queue length at quit
  uint32_t pos;
  uint32_t exiting;    // Exiting SQE consumed, not yet drained
  uint32_t pad;
};

struct alignas(16) CollStat {   // per (collective, block), device memory
  unsigned long long preemptions, ctxLoads, ctxSaves, slices, completions, pad[3];
};
struct alignas(16) BlockStat {  // per block
  unsigned long long quits, exits, fetched, cqes, launches, idlePolls, pad[1];
  // in-kernel timing probes (SM clock cycles), flushed when the block exits
  // (the paper's "core execution time" probes)
  unsigned long long cycRun;        // control thread inside collective runs
  unsigned long long cycPoll;       // ... in failed connector polls (waiting for peers)
  unsigned long long cycAcqFence;   // ... in the acquire fence after a successful poll
  unsigned long long cycRelFence;   // publisher lane in release fences
  unsigned long long nFence;        // release fences issued by the publisher lane
  unsigned long long cycData;       // data group leaders: moving slices
  unsigned long long cycDataWait;   // data group leaders: waiting for a descriptor
  unsigned long long nData;         // slices timed by data group leaders
  unsigned long long nCommit;       // slices committed
  unsigned long long cycCtxLoad, nCtxLoad;   // context loads (cache misses) by the control lane
  unsigned long long cycCtxSave, nCtxSave;   // lazy dynamic-context saves
  unsigned long long cycCqe, nCqe;           // CQE write: from the completing increment to the host store issued
};

// Device event trace (one ring of `traceCap` records per block, %globaltimer
// stamped): slice issue / publish, context switches, preemptions, completions.
// Used for the paper's context-switch traces and for the
// per-hop latency analysis of the ring.
enum TraceEv : uint32_t {
  kEvFetch = 1, kEvSwitchIn = 2, kEvIssue = 3, kEvPublish = 4, kEvPreempt = 5, kEvDone = 6, kEvCqe = 7,
  kEvQuit = 8, kEvExit = 9, kEvSdone = 10, kEvStart = 11, kEvMark = 12
};
struct alignas(16) TraceRec {
  uint64_t t;          // %globaltimer (ns)
  uint32_t tag;        // ev << 24 | collId (16 bits)
  uint32_t arg;        // event argument (slice sequence, queue position, ...)
};

struct DaemonParams {
  const SqeWire* sq;                // mapped host SQ (stamped wire format)
  volatile uint64_t* sqCursorHost;  // mapped host [G]: [0] = SQEs copied to the mirror (slots below are free)
  Sqe* sqMirror;                    // device [sqDepth]: copy of the host SQ read by every block
  uint64_t* mirrorTail;             // device: [0] SQEs in the mirror, [1] fetch lock, [2] cached min block cursor,
                                    //         [3] %globaltimer of the last host-SQ poll by a blocked collective
  uint32_t* fetchLock;              // device: the block copying host SQEs holds it
  volatile uint64_t* cqDone;        // mapped host [maxColl]: last completed subSeq
  BlockState* blk;                  // [G]
  uint32_t* tqSave;                 // [G][maxColl] packed (id | stall << 16)
  CtxSlot* ctx;                     // [maxColl][G]
  uint32_t* complCnt;               // [maxColl]
  CollStat* collStats;              // [maxColl][G]
  BlockStat* blkStats;              // [G]
  char* dataLocal;                  // this rank's connector data [maxColl][G][K][sliceBytes]
  char* dataNext;                   // downstream rank's connector data
  char* flagsLocal;                 // [maxColl][G] x kFlagStride
  char* flagsNext;
  char* flagsPrev;
  uint64_t sliceBytes;
  uint32_t sqDepth;
  int nranks, rank, G, maxColl, K, slicesPerChunk;
  int orderPolicy, priorityCadence, stickiness;
  uint32_t spinBase, spinStep, spinMin, spinBoost, spinCap, stallLimit;
  uint32_t spinNs;                  // duration of one spin (failed poll) in ns
  int quitEnabled;
  uint64_t quitIdleNs;
  uint32_t idleSleepNs;
  int cacheWays;
  int sysScope;                     // 1: peers in other processes/devices -> .sys fences
  int pipeDepth;                    // slices in flight control -> data warps (<= 8)
  int prefetchSlices;               // reserved (0): the L2 prefetch of the send-buffer operand was removed
  int discardConsumed;              // invalidate consumed connector lines in L2 (no write-back)
  int directNext;                   // downstream's buffers are addressable: final data goes straight there
  int directPrev;                   // upstream writes final data straight into our recv buffer
  const RingDesc* rings;            // [kMaxRings] ring 0 = this communicator, then sub-communicators
  TraceRec* trace;                  // [G][traceCap] or null
  uint32_t* traceCount;             // [G] records written (monotonic; ring index = count % traceCap)
  uint32_t traceCap;
  char* llLocal;                    // this rank's LL connector lines [maxColl][G][K][2 * llSliceBytes]
  uint32_t llSliceBytes;            // LL payload per slice (lines carry 8 B payload + 8 B flags)
  uint32_t llMaxBytes;              // a collective uses LL when its per-block part is at most this
  int stages;                       // TMA staging tiles per block (x 2 x 16 KiB of shared memory)
  int bulkStores;                   // 1: staged tiles leave through cp.async.bulk stores (publisher lane)
  int directRead;                   // 1: the first reduce step reads a same-process upstream's send buffer
  int blocksPerSM;                  // 1 or 2 co-resident daemon blocks per SM
  int l2Hints;                      // evict-first L2 policy for user-buffer loads / stores
  uint32_t* quitWord;               // device, per launch: quit votes | latch (zeroed before each launch)
  uint32_t quitTotal;               // blocks of the launch (G x fused members)
  uint64_t stallNs;                 // FIFO: all entries stuck when none progressed for this long (0: off)
  uint64_t sqYieldNs;               // priority: host-SQ poll period of blocked collectives (0: no yield)
  int llSpeculate;                  // LL: issue recv slices before their lines arrived (abortable)
  int readyFirst;                   // priority: run the highest-priority collective admitted by every member
  // CQ variant (NEXT-3 ablation): 0 = id slots (cqDone, default),
  // 1 = vanilla MPSC ring (entry, fence, in-order tail update), 2 = packed 64-bit
  // ring entries {stamp, id} (one host write, no fence between entry and tail)
  int cqMode;
  uint32_t cqDepth;                 // ring entries (>= maxColl: one CQE per in-flight id, never full)
  uint64_t* cqReserve;              // device: next ring slot (gpu-scope atomic)
  volatile uint64_t* cqRing;        // mapped host [cqDepth]
  volatile uint64_t* cqTail;        // mapped host: vanilla ring tail (entries published in order)
};

}  // namespace occl

// Launch entry implemented in occl_daemon.cu (internal, not part of the C-ABI).
extern "C" int occl_internal_launch_daemon(const occl::DaemonParams* p, const occl::DaemonParams* pDev,
                                           int nranks, int blockThreads, void* stream);
extern "C" size_t occl_internal_daemon_smem(int maxColl, int cacheWays, int stages);
