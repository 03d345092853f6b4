/*
 * occl.h -- C-ABI of the B200-native OCCL hot path (arXiv 2303.06324).
 *
 * A persistent, preemptible daemon kernel (one per rank) runs ring AllReduce /
 * AllGather / ReduceScatter / Broadcast slice by slice over peer memory
 * (NVLink 5 / NVSwitch through CUDA IPC or peer access; plain HBM when several
 * ranks share one device).  Ranks may submit collectives in ANY per-rank order.
 *
 * Paper passages each call follows (PAPER.md = /root/reference/PAPER.md, LaTeX):
 *   - registration with unique ids, prepared before execution ... PAPER.md:373-375 (§3.1.1)
 *   - SQE = collective id + send/recv buffer addresses ........... PAPER.md:397-398 (§3.1.2)
 *   - Exiting SQE ................................................ PAPER.md:399     (§3.1.2)
 *   - CQE + poller + callback map ................................ PAPER.md:401-404 (§3.1.2)
 *   - voluntary quit / event-driven start ........................ PAPER.md:406-416 (§3.1.3)
 *   - stickiness (order + spin-threshold policies) ............... PAPER.md:422-457 (§3.2)
 *   - per-collective grid size, SPMC SQ, completion counters ..... PAPER.md:464-506 (§4)
 *   - context-switch optimisations ............................... PAPER.md:509-515 (§4)
 *
 * Conventions (all calls):
 *   - Every call returns occlResult_t; nothing throws or aborts across the ABI.
 *   - Argument errors are reported synchronously.  An asynchronous device fault
 *     makes the communicator sticky-errored; it then surfaces from
 *     occlWait / occlTest / occlCommQuiesce as occlCudaError.
 *   - Pointers named send/recv are DEVICE pointers on the communicator's device,
 *     owned by the caller.  They must stay allocated, and `send` unmodified, until
 *     occlWait / occlTest reports completion.  `send` must already hold its data
 *     when the call is made (the invoker submits when its tensor is ready,
 *     PAPER.md:525): synchronise the producing stream first.
 *   - The communicator owns connectors, SQ/CQ, context buffer and daemon stream.
 *   - collId in [0, maxColl) is GLOBALLY AGREED: every rank uses the same id for
 *     the same logical collective with identical (kind, count, dtype, op, root).
 *     Mismatched metadata across ranks is undefined behaviour.  An id may be
 *     resubmitted (with new buffers) only after it completed locally
 *     (PAPER.md:382-383); resubmitting an in-flight id returns occlDuplicateSubmit.
 *     Local completion means this rank's buffers are free: no peer reads `send`
 *     or writes `recv` of that submission any more (a direct-reading downstream
 *     acknowledges its last read before the CQE is posted).
 *   - In-place (NCCL conventions): send == recv (AllReduce, Broadcast);
 *     send == recv + rank*sendcount (AllGather); recv == send + rank*recvcount
 *     (ReduceScatter).
 *   - count == 0 completes at submission.  One submitting host thread per
 *     communicator at a time.  A full SQ blocks the submitter
 *     until the daemon frees a slot.
 */
#ifndef OCCL_H_
#define OCCL_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct occlComm* occlComm_t;

typedef enum {
  occlSuccess = 0,
  occlInvalidArgument = 1,   /* bad pointer/size/dtype/root/collId (SPEC.md:56 InvalidMeta)   */
  occlInvalidUsage = 2,      /* wrong state: destroy with work in flight, not connected, ...  */
  occlRegistryFull = 3,      /* collId >= maxColl                                              */
  occlQueueFull = 4,         /* reserved (submission blocks instead)                           */
  occlDuplicateSubmit = 5,   /* collId already in flight                         */
  occlUnknownId = 6,         /* wait/test on an id never submitted               */
  occlCudaError = 7,         /* CUDA runtime error or asynchronous device fault (sticky)       */
  occlSystemError = 8,       /* host allocation / thread failure                               */
  occlTimeout = 9,           /* occlWait / occlCommQuiesce timeout                              */
  occlInProgress = 10,       /* returned by occlTest-like helpers when not complete            */
  occlInternalError = 11     /* corrupt context or invariant violation                         */
} occlResult_t;

typedef enum { occlInt32 = 0, occlFloat32 = 1, occlBfloat16 = 2, occlFloat16 = 3, occlInt64 = 4,
               occlFloat64 = 5 } occlDataType_t;
/* The collective's reducing function ("a specified reducing
 * function").  Results are bit-exact with the ring's fold order: IEEE
 * round-to-nearest-even per hop for f64 / f32 / bf16 / f16, two's-complement wrap
 * for integer sum and prod, exact max / min. */
typedef enum { occlSum = 0, occlProd = 1, occlMax = 2, occlMin = 3 } occlRedOp_t;
typedef enum { occlOrderFifo = 0, occlOrderPriority = 1 } occlOrderPolicy_t;

/* Configuration.  Every rank of a communicator MUST use identical values (the
 * per-collective block count and the slice geometry derive from them). */
typedef struct {
  int maxColl;            /* registry size: collId in [0, maxColl) ("up to 1,000")   */
  int gridBlocks;         /* G: daemon grid = max blocks any collective uses        */
  int blockThreads;       /* threads per block: control, TMA and publisher warps + compute warps (128..608) */
  int connSlots;          /* K: slots per connector; must exceed slicesPerChunk                    */
  int slicesPerChunk;     /* slices each primitive moves per loop             */
  size_t sliceBytes;      /* bytes per connector slot (multiple of 16)                             */
  size_t minBlockBytes;   /* a collective uses ceil(segmentBytes / minBlockBytes) blocks (<= G)   */
  int sqDepth;            /* SQ ring entries                                                       */
  int orderPolicy;        /* occlOrderFifo | occlOrderPriority (queue sorted by priority)       */
  int priorityCadence;    /* priority policy: poll the SQ every N scheduling rounds                */
  int stickiness;         /* 1 = paper's spin-threshold policy; 0 = constant    */
  uint32_t spinBase;      /* initial threshold (failed connector polls) at queue position 0       */
  uint32_t spinStep;      /* decrement per queue position                                         */
  uint32_t spinMin;       /* floor                                                                 */
  uint32_t spinBoost;     /* multiply on each successful primitive                                */
  uint32_t spinCap;       /* ceiling                                                               */
  uint32_t stallLimit;    /* preemptions without progress => "cannot progress"     */
  int quitEnabled;        /* voluntary quit                                     */
  uint64_t quitIdleNs;    /* quit horizon: queue empty/all stuck and no SQE for this long         */
  uint32_t idleSleepNs;   /* back-off between empty SQ polls                                       */
  int autoLaunch;         /* 1 = event-driven (re)start by the host supervisor */
  int cacheWays;          /* direct-mapped shared-memory context cache ways        */
  int pipeDepth;          /* slices in flight between the control warp and the data warps (1..8)   */
  int prefetchSlices;     /* reserved, must be 0 (an L2 prefetch of the send-buffer operand measured
                             8-14 % slower and was removed)                          */
  int discardConsumed;    /* 1 = drop consumed connector lines from L2 without write-back         */
  int l2Hints;            /* 1 = evict-first L2 policy for send/recv-buffer streams; 2 = also evict-last for connector stores;
                             3 = also evict-last for direct sends the downstream forwards (demoted once read) */
  int directMode;         /* 1 = final data goes straight into a same-process peer's recv buffer  */
  int stagingTiles;       /* TMA staging ring depth per block (1..6), 32 KiB of shared memory each */
  int blocksPerSM;        /* 1 (up to 608 threads) or 2 (up to 384 threads, <= 3 staging tiles)    */
  uint32_t traceCap;      /* device event-trace records kept per block (0 = tracing off)          */
  uint32_t llSliceBytes;  /* LL protocol: payload bytes per slice (multiple of 8; lines are 16 B) */
  uint32_t llMaxBytes;    /* a collective whose per-block part is <= this uses LL (0 = never)   */
  uint32_t spinNs;        /* one spin = this many ns of failed polling (thresholds are in spins)  */
  int bulkStores;         /* 1 = staged tiles are stored with cp.async.bulk by the publisher lane  */
  int directRead;         /* 1 = AR/RS first reduce step reads a same-process upstream's send buffer */
  uint64_t stallNs;       /* FIFO fetch gate: 0 = an entry is stuck after stallLimit preemptions without
                             progress; > 0 = also when no queued entry progressed for this long (reading R3) */
  int forceSysScope;      /* 1 = treat every peer as another process (CUDA IPC): system-scope fences,
                             connector-only edges (no direct mode / direct read) -- the one-process-per-GPU
                             data path, selectable on one device for testing and benchmarking */
  int cqMode;             /* CQ variant: 0 = one slot per collId (default), 1 = vanilla
                             MPSC ring (entry, fence, in-order tail), 2 = packed 64-bit {stamp, id} ring */
  uint64_t sqYieldNs;     /* priority policy: a collective blocked on a peer for >= spinMin spins yields to
                             newly submitted SQEs; its rank polls the host SQ for them at most once per
                             sqYieldNs (0 = never: new SQEs are seen only between runs) */
  int llSpeculate;        /* LL slice driving (DESIGN.md §LL runs).  2 (default) = LL runs: a collective
                             whose blocks move one LL slice per ring step is handed to the data warps
                             as ONE descriptor; they walk its whole slice schedule, polling their own
                             lines, and stop when a slice's lines do not come within the spin threshold
                             (the control lane resumes from the reported cursor); longer LL schedules
                             use mode 0.  1 = LL slices are handed to the data warps one by one before
                             their lines arrived (abortable speculation).  0 = the control lane polls
                             each slice's last line, then issues it.  All modes are wire-compatible.
                             Other values: occlInvalidArgument */
  int readyFirst;         /* priority policy: 1/2 = run the highest-priority collective that EVERY member
                             rank has admitted (each rank publishes its admissions on a readiness
                             board in its flags; R29); a collective not yet admitted
                             everywhere waits at most spinMin (1), or -- when the whole queue is in
                             the scan window and nothing in it is ready -- is not run at all while
                             the block waits for admissions (2).  0 = the queue front first (R10) */
} occlConfig_t;

/* Aggregate counters (device counters summed over blocks/collectives). */
typedef struct {
  uint64_t launches;      /* daemon kernel launches (event-driven starts)                          */
  uint64_t quits;         /* block-level voluntary quits                                           */
  uint64_t exits;         /* block-level exits after the Exiting SQE                               */
  uint64_t preemptions;   /* collective preemptions (context switches out)                         */
  uint64_t ctxLoads;      /* context loads from the context buffer (cache misses)                  */
  uint64_t ctxSaves;      /* lazy dynamic-context saves                                            */
  uint64_t slices;        /* connector slices executed                                             */
  uint64_t sqeFetched;    /* SQEs admitted into task queues                                        */
  uint64_t cqeWritten;    /* CQEs posted                                                           */
  float lastLaunchMs;     /* device time of the last completed daemon launch (CUDA events)         */
} occlStats_t;

typedef struct {
  uint64_t preemptions, ctxLoads, ctxSaves, slices, completions;
} occlCollStats_t;

/* In-kernel timing probes summed over the communicator's blocks, in SM clock
 * cycles (the paper's "core execution time" probes).  Values
 * accumulate over daemon launches; each block flushes them when it exits. */
typedef struct {
  uint64_t cycRun;        /* control thread inside collective runs                  */
  uint64_t cycPoll;       /* ... in failed connector polls (waiting for peers)      */
  uint64_t cycAcqFence;   /* ... in the acquire fence after a successful poll       */
  uint64_t cycRelFence;   /* publisher lanes in release fences                      */
  uint64_t cycData;       /* data-group leader threads moving slices                */
  uint64_t cycDataWait;   /* data-group leader threads waiting for a descriptor     */
  uint64_t nData;         /* slices timed by data-group leaders                     */
  uint64_t nCommit;       /* slices committed                                       */
  uint64_t nFence;        /* release fences issued by publisher lanes               */
  uint64_t cycCtxLoad;    /* context loads into the shared-memory cache */
  uint64_t nCtxLoad;
  uint64_t cycCtxSave;    /* lazy dynamic-context saves              */
  uint64_t nCtxSave;
  uint64_t cycCqe;        /* CQE writes: completing increment -> host store issued (cfg.cqMode) */
  uint64_t nCqe;
} occlProbes_t;

/* One device trace record (%globaltimer ns).  tag = event << 24 | collId; for
 * occlEvPublish the low 16 bits hold the number of slices the fence covered.
 * arg: Issue = nsent | nrecv << 14 | actions << 28 (connector sequence numbers,
 *      low 14 bits; actions: 1 recv, 2 reduce, 4 copy, 8 send);
 * Publish / Sdone (slices moved, before the release fence) = head | credit << 16; SwitchIn / Preempt = task-queue position;
 * Fetch / Cqe = submission number. */
typedef struct {
  uint64_t t;
  uint32_t tag;
  uint32_t arg;
} occlTraceRec_t;
enum { occlEvFetch = 1, occlEvSwitchIn = 2, occlEvIssue = 3, occlEvPublish = 4, occlEvPreempt = 5,
       occlEvDone = 6, occlEvCqe = 7, occlEvQuit = 8, occlEvExit = 9, occlEvSdone = 10, occlEvStart = 11, occlEvMark = 12 };

/* Memory footprint of one rank (PAPER.md:581-582 reports "about 4 MB of global
 * memory per block for 1,000 collectives"; reading Q15 of SURVEY.md).  Bytes. */
typedef struct {
  uint64_t device;          /* total device memory of the communicator           */
  uint64_t connectorData;   /* maxColl x G x K x sliceBytes (Simple connectors)  */
  uint64_t connectorFlags;  /* maxColl x G x 384 B (head, credit, direct line)   */
  uint64_t llLines;         /* maxColl x G x K x 2 x llSliceBytes                */
  uint64_t contexts;        /* maxColl x G x 128 B context buffer                */
  uint64_t other;           /* SQ mirror, block state, stats, trace, ring table  */
  uint64_t pinnedHost;      /* SQ, SQ cursors, CQ                                */
  double perBlockPerColl;   /* device / (maxColl x G)                            */
} occlFootprint_t;

/* Bootstrap all-gather: gather `bytesPerRank` bytes from every rank into `out`
 * (rank-major).  Return 0 on success. */
typedef int (*occlAllGatherFn)(const void* in, void* out, size_t bytesPerRank, void* ctx);
typedef void (*occlCallback_t)(int collId, void* arg);

#define OCCL_HANDLE_BYTES 256

/* Static description of a result code.  Never NULL. */
const char* occlGetErrorString(occlResult_t result);

/* Fill *cfg with the library defaults (thresholds of reading R1, slices of 192 KiB,
 * K = 4 slots, priority order policy).  Errors: occlInvalidArgument (cfg NULL). */
occlResult_t occlConfigDefault(occlConfig_t* cfg);

/* --- communicator setup: registration before execution (§3.1.1;
 *     dedicated connectors per collective and block, §5) ---------- */

/* Create rank `rank` (0 <= rank < nranks <= 64) of an `nranks` ring on CUDA device
 * `cudaDev`.  Allocates, owned by the communicator: the connector arena
 * (maxColl x G x K x sliceBytes data + maxColl x G x 384 B flags, device), the
 * context buffer (maxColl x G x 128 B), completion counters, and the SQ / CQ /
 * SQ cursors in pinned mapped host memory.  cfg == NULL => occlConfigDefault;
 * *cfg is copied.  Every rank of a ring must pass identical cfg values.  Not
 * usable for collectives until occlCommConnect.
 * Errors: occlInvalidArgument (bad rank/nranks/device, invalid cfg),
 * occlCudaError (allocation, no such device). */
occlResult_t occlCommCreate(occlComm_t* comm, int nranks, int rank, int cudaDev,
                            const occlConfig_t* cfg);

/* Serialise this rank's handle into `out` (caller-owned, *len bytes of
 * capacity >= OCCL_HANDLE_BYTES); on return *len = bytes written.  The handle is
 * plain bytes: the arena's CUDA IPC handle, its raw device pointer, pid and
 * device (a same-process peer uses the raw pointer directly).
 * Errors: occlInvalidArgument (NULL pointer, capacity too small). */
occlResult_t occlCommGetHandle(occlComm_t comm, void* out, size_t* len);

/* Open the ring neighbours' arenas (rank r pushes into r+1 and returns credits
 * to r-1: the send side of r is the receive side of r+1) from
 * `allHandles`: nranks handles, rank-major, lenPerRank bytes each, caller-owned,
 * read during the call only.  Enables peer access / opens IPC mappings and
 * starts the host supervisor thread (poller + event-driven launcher).
 * Errors: occlInvalidArgument (NULL, short handles, a handle of another ring
 * geometry), occlInvalidUsage (already connected), occlCudaError (IPC open,
 * peer access). */
occlResult_t occlCommConnect(occlComm_t comm, const void* allHandles, size_t lenPerRank);

/* occlCommCreate + occlCommGetHandle + ag(...) + occlCommConnect: the paper's
 * registration step over a rank set.  `ag` gathers
 * OCCL_HANDLE_BYTES from every rank, rank-major, into its `out` (e.g. an MPI or
 * torch.distributed all-gather); it is called once, synchronously, with agCtx.
 * Errors: those of the three calls; occlSystemError if ag returns non-zero (the
 * half-built communicator is destroyed, *comm untouched). */
occlResult_t occlCommInit(occlComm_t* comm, int nranks, int rank, int cudaDev,
                          occlAllGatherFn ag, void* agCtx, const occlConfig_t* cfg);

/* Serve `n` connected communicators of THIS process that live on the same device
 * with ONE daemon kernel launch: blocks [i*G, (i+1)*G) run comms[i]'s daemon,
 * each with its own SQ, CQ, contexts and connectors (virtual ranks sharing one
 * B200: co-resident by construction, started, stopped and timed together).  All
 * must share gridBlocks, maxColl, cacheWays and blockThreads, be idle and have
 * nothing in flight.  The array is read during the call only.
 * Errors: occlInvalidArgument (NULL, n < 1, mismatched geometry or devices),
 * occlInvalidUsage (not connected, a sub-communicator, already fused, busy). */
occlResult_t occlCommFuse(occlComm_t* comms, int n);

/* Sub-communicator (§3.1.1: a collective's static context carries
 * its own nranks / rank, so one daemon per GPU serves collectives of overlapping
 * rank sets).  `members` (caller-owned, nmembers distinct parent ranks, read
 * during the call) lists the new ring in its rank order; every member calls this
 * with the same list (globally agreed, like collId) and the caller must be a
 * member.  The child shares the parent's daemon, SQ, CQ and collId registry; its
 * collectives use dedicated connectors at (collId, block) in the members' arenas,
 * opened from the handles the parent received at occlCommConnect.  A collId is
 * BOUND to the (sub-)communicator of its first submission -- its connector
 * sequence numbers belong to that ring's edges -- and submitting it on another
 * returns occlInvalidUsage; destroying a child retires the ids bound to it.
 * Destroy children before their parent.  Up to 31 live sub-communicators per
 * communicator (a destroyed child's slot is reused).
 * Errors: occlInvalidArgument (NULL, duplicate / out-of-range member, caller not
 * a member), occlInvalidUsage (parent not a connected root, no free slot),
 * occlCudaError. */
occlResult_t occlCommSplit(occlComm_t parent, int nmembers, const int* members, occlComm_t* child);

/* Push the Exiting SQE (§3.1.2), wait for the daemon to drain and
 * exit, free everything the communicator owns.  A sticky-errored communicator
 * can still be destroyed.
 * Errors: occlInvalidArgument (NULL), occlInvalidUsage (collectives still in
 * flight, or live sub-communicators). */
occlResult_t occlCommDestroy(occlComm_t comm);

/* --- collectives: asynchronous submission of one SQE = {collective id, send /
 *     recv buffer addresses, shape} (§3.1.2), any per-rank order
 *     (§3.1).  Each returns once the SQE is in the SQ (a full SQ
 *     blocks until the daemon frees a slot); completion is reported by the CQE
 *     (occlWait / occlTest / occlSetCallback).  Buffers: DEVICE pointers on the
 *     communicator's device, caller-owned, contiguous, element type `datatype`;
 *     `send` must hold its data at the call and stay unmodified, and both must stay
 *     allocated, until local completion.  The ring primitive sequences follow
 *     NCCL's Ring/Simple; the reduction order is the
 *     ring's left fold of DESIGN.md R6/R7, so results are bit-exact with oracle O1.
 * Common errors: occlInvalidArgument (NULL buffer with count > 0, bad datatype /
 * op / root, collId < 0), occlRegistryFull (collId >= maxColl),
 * occlDuplicateSubmit (collId still in flight), occlInvalidUsage
 * (not connected; collId bound to another sub-communicator), occlCudaError
 * (sticky device fault).  count == 0 completes at submission. */

/* AllReduce: recvbuff[i] = (+) over ranks of sendbuff[i], i < count (count
 * elements per rank in both buffers; in place iff send == recv). */
occlResult_t occlAllReduce(const void* sendbuff, void* recvbuff, size_t count,
                           occlDataType_t datatype, occlRedOp_t op, int collId, occlComm_t comm);
/* AllGather: recvbuff[q*sendcount + j] = rank q's sendbuff[j]; recvbuff holds
 * nranks*sendcount elements (in place iff send == recv + rank*sendcount). */
occlResult_t occlAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                           occlDataType_t datatype, int collId, occlComm_t comm);
/* ReduceScatter: recvbuff[j] = (+) over ranks q of q's sendbuff[rank*recvcount + j];
 * sendbuff holds nranks*recvcount elements (in place iff recv == send + rank*recvcount). */
occlResult_t occlReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                               occlDataType_t datatype, occlRedOp_t op, int collId, occlComm_t comm);
/* Broadcast: every rank's recvbuff = the root's sendbuff (count elements; the
 * root may pass send == recv).  0 <= root < nranks. */
occlResult_t occlBroadcast(const void* sendbuff, void* recvbuff, size_t count,
                           occlDataType_t datatype, int root, int collId, occlComm_t comm);
/* Reduce (beyond the paper's four, R23): NCCL's ring Reduce, the chain
 * root+1 -> ... -> root folds the inputs in that order; only the root's recvbuff
 * (count elements) is written, other ranks' recvbuff may be NULL. */
occlResult_t occlReduce(const void* sendbuff, void* recvbuff, size_t count, occlDataType_t datatype,
                        occlRedOp_t op, int root, int collId, occlComm_t comm);

/* --- completion: CQE, poller, callback map (§3.1.2; the CQ
 *     variants of PAPER.md:496-506, §4, cfg.cqMode) ---------------------------- */

/* Block until the latest submission of collId completed locally: its CQE was
 * posted, so this rank's buffers are free (no peer still reads `send` or writes
 * `recv`).  timeoutNs < 0 waits forever.
 * Errors: occlInvalidArgument, occlRegistryFull, occlUnknownId (never
 * submitted), occlTimeout, occlCudaError (sticky fault). */
occlResult_t occlWait(occlComm_t comm, int collId, int64_t timeoutNs);

/* Non-blocking completion test: *done = 1 when the latest submission of collId
 * completed locally, else 0.  Errors: as occlWait, minus occlTimeout. */
occlResult_t occlTest(occlComm_t comm, int collId, int* done);

/* Bind cb(collId, arg), fired exactly once per completion of collId by the host
 * poller thread; it must not block and must not call back
 * into this communicator's submit / wait functions.  cb == NULL unbinds.
 * Errors: occlInvalidArgument, occlRegistryFull, occlInvalidUsage (collId in
 * flight: rebinding only between submissions). */
occlResult_t occlSetCallback(occlComm_t comm, int collId, occlCallback_t cb, void* arg);

/* User-defined priority of collId for the priority order policy (PAPER.md:438-446,
 * §3.2; reading R10): lower values run first; the task queues are kept sorted by
 * it.  Like collId it must be globally agreed.  Default: priority = collId.
 * Takes effect at the next submission of collId.
 * Errors: occlInvalidArgument, occlRegistryFull. */
occlResult_t occlSetPriority(occlComm_t comm, int collId, int32_t priority);

/* --- observability (the paper's probes and traces) */
/* Counters summed over blocks (a snapshot; the daemon may be running); *out is
 * caller-owned.  Errors: occlInvalidArgument (NULL), occlRegistryFull (collId). */
occlResult_t occlGetStats(occlComm_t comm, occlStats_t* out);
occlResult_t occlGetCollStats(occlComm_t comm, int collId, occlCollStats_t* out);
occlResult_t occlGetProbes(occlComm_t comm, occlProbes_t* out);
occlResult_t occlGetFootprint(occlComm_t comm, occlFootprint_t* out);

/* Device event trace of block `block` (cfg.traceCap > 0): the most recent
 * min(written, traceCap) records, oldest first, into the caller's out[0..cap);
 * *n = count copied.  occlTraceReset forgets everything recorded so far.
 * Errors: occlInvalidArgument (block out of range, out NULL with cap > 0),
 * occlInvalidUsage (reset while the daemon runs). */
occlResult_t occlGetTrace(occlComm_t comm, int block, occlTraceRec_t* out, size_t cap, size_t* n);
occlResult_t occlTraceReset(occlComm_t comm);

/* --- daemon lifecycle: voluntary quit and event-driven start (PAPER.md:406-416,
 *     §3.1.3), made explicit ---------------------------------------------------- */
/* Push an Exiting SQE: every block drains its task queue, then
 * exits.  A later submission restarts the daemon (event-driven start).
 * Errors: occlInvalidArgument, occlInvalidUsage (not connected). */
occlResult_t occlCommExit(occlComm_t comm);
/* Launch the daemon now if it is not running (what the supervisor does on an
 * SQE when autoLaunch = 1).  Refuses a grid that cannot be co-resident.
 * Errors: occlInvalidArgument, occlInvalidUsage, occlCudaError. */
occlResult_t occlCommLaunch(occlComm_t comm);
/* Enable / disable the supervisor's event-driven start.  While it is disabled the
 * daemon does not quit voluntarily either (nobody would restart it): launches
 * made with occlCommLaunch run until their Exiting SQE.  Errors: occlInvalidArgument. */
occlResult_t occlCommSetAutoLaunch(occlComm_t comm, int enable);
/* Wait until no daemon kernel of this communicator is running (timeoutNs < 0:
 * forever).  Errors: occlInvalidArgument, occlTimeout, occlCudaError. */
occlResult_t occlCommQuiesce(occlComm_t comm, int64_t timeoutNs);
/* The CUDA stream (cudaStream_t, owned by the communicator) the daemon kernel is
 * launched on.  Errors: occlInvalidArgument. */
occlResult_t occlCommGetStream(occlComm_t comm, void** stream);
/* Number of blocks (lanes) a collective of this shape uses -- the per-collective
 * grid size of PAPER.md:469, :488, identical on every rank; kind: 0 all-reduce,
 * 1 all-gather, 2 reduce-scatter, 3 broadcast, 4 reduce.  Errors: occlInvalidArgument. */
occlResult_t occlCollBlocks(occlComm_t comm, int kind, size_t count, occlDataType_t datatype,
                            int* nblocks);

#ifdef __cplusplus
}
#endif
#endif /* OCCL_H_ */
