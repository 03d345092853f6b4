// occl_daemon.cu -- the persistent, preemptible daemon kernel (sm_100a).
//
// One launch per rank; every block is an independent scheduler ("lane") with its
// own task queue in shared memory.  Per block:
//
//   loop:
//     thread 0 : fetch an SQE (policy-gated) or pick the task
//                queue entry at `pos`; decide voluntary quit
//     threads  : load the entry's context into the shared-memory cache if it is
//                not there (16 B per thread)
//     per slice:
//       thread 0 : wait for the recv connector to be readable / the send
//                  connector writable, counting failed polls; preempt when the
//                  count exceeds the spin threshold (two-phase blocking,
//                  PAPER.md:361-366)
//       all      : 128-bit coalesced recv / reduce / copy / send of the slice
//       thread 0 : fence + publish head (downstream) / credit (upstream);
//                  advance the dynamic context (loop, step, slice); raise the
//                  threshold (stickiness)
//     preempted : lazy save of the dynamic context, rotate
//     done      : completion counter; the last block posts the CQE
//
// Connectors (push model): rank r writes slices into rank r+1's connector
// memory and bumps r+1's `head`; r+1 returns `credit` into r's flags.  Both
// counters are monotonic per (collective, block) across submissions, so a
// preempted collective resumes exactly where it stopped.
// Connectors are dedicated per (collective, block).
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "occl_internal.h"

using namespace occl;

namespace {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint64_t ld_relaxed(const void* p, int sys) {
  uint64_t v;
  if (sys) asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else     asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const void* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(void* p, uint64_t v, int sys) {
  if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
  else     asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_volatile_u64(volatile uint64_t* p, uint64_t v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel(int sys) {
  if (sys) asm volatile("fence.acq_rel.sys;" ::: "memory");
  else     asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void fence_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ uint4 ld_cg(const uint4* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_v4(uint4* p, const uint4& v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_cg_v4(void* p, const uint4& v) {
  asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
template <typename T>
__device__ __forceinline__ T ld_cg_scalar(const T* p) {
  return *reinterpret_cast<const volatile T*>(p);
}

// ------------------------------------------------------------------ reduction (+)
// f32: IEEE add, round-to-nearest-even (no FMA contraction: plain __fadd_rn).
// i32: two's-complement wrap.  bf16: correctly rounded bf16 add (__hadd2).
template <int DT> __device__ __forceinline__ uint4 vadd(const uint4& a, const uint4& b);
template <> __device__ __forceinline__ uint4 vadd<kF32>(const uint4& a, const uint4& b) {
  uint4 r;
  r.x = __float_as_uint(__fadd_rn(__uint_as_float(a.x), __uint_as_float(b.x)));
  r.y = __float_as_uint(__fadd_rn(__uint_as_float(a.y), __uint_as_float(b.y)));
  r.z = __float_as_uint(__fadd_rn(__uint_as_float(a.z), __uint_as_float(b.z)));
  r.w = __float_as_uint(__fadd_rn(__uint_as_float(a.w), __uint_as_float(b.w)));
  return r;
}
template <> __device__ __forceinline__ uint4 vadd<kI32>(const uint4& a, const uint4& b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
__device__ __forceinline__ uint32_t add_bf16x2(uint32_t a, uint32_t b) {
  __nv_bfloat162 x = *reinterpret_cast<__nv_bfloat162*>(&a);
  __nv_bfloat162 y = *reinterpret_cast<__nv_bfloat162*>(&b);
  __nv_bfloat162 z = __hadd2(x, y);
  return *reinterpret_cast<uint32_t*>(&z);
}
template <> __device__ __forceinline__ uint4 vadd<kBF16>(const uint4& a, const uint4& b) {
  return make_uint4(add_bf16x2(a.x, b.x), add_bf16x2(a.y, b.y), add_bf16x2(a.z, b.z), add_bf16x2(a.w, b.w));
}

// ------------------------------------------------------------------ primitives
// Action bits of the fused primitives.
enum : int { A_RECV = 1, A_REDUCE = 2, A_COPY = 4, A_SEND = 8 };
enum : int {
  P_SEND = A_SEND,
  P_RECV = A_RECV | A_COPY,
  P_COPYSEND = A_COPY | A_SEND,
  P_RECVCOPYSEND = A_RECV | A_COPY | A_SEND,
  P_RECVREDUCESEND = A_RECV | A_REDUCE | A_SEND,
  P_RECVREDUCECOPY = A_RECV | A_REDUCE | A_COPY,
  P_RECVREDUCECOPYSEND = A_RECV | A_REDUCE | A_COPY | A_SEND,
  P_COPY = A_COPY,
};

struct SliceDesc {
  const char* src;     // send-buffer slice (reduce operand / data to send)
  const char* cin;     // recv connector slot
  char* dst;           // recv-buffer slice
  char* cout;          // downstream connector slot
  int64_t nelem;
  int prim;
  int dtype;
};

template <int DT> struct Elem;
template <> struct Elem<kF32> { typedef float T; };
template <> struct Elem<kI32> { typedef int32_t T; };
template <> struct Elem<kBF16> { typedef uint16_t T; };

template <int DT>
__device__ __forceinline__ typename Elem<DT>::T sadd(typename Elem<DT>::T a, typename Elem<DT>::T b);
template <> __device__ __forceinline__ float sadd<kF32>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ int32_t sadd<kI32>(int32_t a, int32_t b) {
  return (int32_t)((uint32_t)a + (uint32_t)b);
}
template <> __device__ __forceinline__ uint16_t sadd<kBF16>(uint16_t a, uint16_t b) {
  __nv_bfloat16 x = __ushort_as_bfloat16(a), y = __ushort_as_bfloat16(b);
  return __bfloat16_as_ushort(__hadd(x, y));
}

// Move one slice with all threads of the block: 128-bit vectors, U independent
// loads in flight per thread, then the stores.  The action
// bits are warp-uniform runtime flags; only the element type is a template.
template <int DT>
__device__ __forceinline__ void move_slice(const SliceDesc& d) {
  typedef typename Elem<DT>::T T;
  constexpr int A = 16 / sizeof(T);
  constexpr int U = 4;
  const int prim = d.prim;
  const bool recv = prim & A_RECV, reduce = prim & A_REDUCE, copy = prim & A_COPY, send = prim & A_SEND;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = (int)d.nelem;                     // <= sliceBytes / sizeof(T)
  if (n <= 0) return;
  const bool aligned = ((((uintptr_t)d.src) | ((uintptr_t)d.dst)) & 15) == 0;
  const int nvec = aligned ? n / A : 0;
  const uint4* vs = reinterpret_cast<const uint4*>(d.src);
  const uint4* vi = reinterpret_cast<const uint4*>(recv ? d.cin : d.src);
  uint4* vd = reinterpret_cast<uint4*>(d.dst);
  uint4* vo = reinterpret_cast<uint4*>(d.cout);
  for (int base = tid; base < nvec; base += U * nt) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nt;
      if (i < nvec) {
        a[u] = ld_cg(vi + i);
        if (reduce) b[u] = ld_cg(vs + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = base + u * nt;
      if (i < nvec) {
        uint4 v = a[u];
        if (reduce) v = vadd<DT>(a[u], b[u]);
        if (copy) st_v4(vd + i, v);
        if (send) st_cg_v4(vo + i, v);
      }
    }
  }
  // scalar tail (ragged segment ends) or the whole slice when misaligned
  const T* ss = reinterpret_cast<const T*>(d.src);
  const T* si = reinterpret_cast<const T*>(recv ? d.cin : d.src);
  T* sd = reinterpret_cast<T*>(d.dst);
  T* so = reinterpret_cast<T*>(d.cout);
  for (int e = nvec * A + tid; e < n; e += nt) {
    T v = ld_cg_scalar(si + e);
    if (reduce) v = sadd<DT>(v, ld_cg_scalar(ss + e));
    if (copy) sd[e] = v;
    if (send) so[e] = v;
  }
}

__device__ __forceinline__ void move_slice_any(const SliceDesc& d) {
  if (d.dtype == kBF16) move_slice<kBF16>(d);
  else if (d.dtype == kF32) move_slice<kF32>(d);
  else move_slice<kI32>(d);
}

// ------------------------------------------------------------------ ring sequences
// Per-rank primitive sequence of the Ring algorithm and
// the segment each step touches (reading R5).  Ring: r -> r+1.
__device__ __forceinline__ int md(int x, int n) { x %= n; return x < 0 ? x + n : x; }

__device__ __forceinline__ void step_prim(int kind, int n, int r, int root, int step, bool inplace,
                                          int& prim, int& seg) {
  if (n == 1) { prim = P_COPY; seg = 0; return; }
  switch (kind) {
    case kAllReduce:
      if (step == 0) { prim = P_SEND; seg = md(r - 1, n); }
      else if (step < n - 1) { prim = P_RECVREDUCESEND; seg = md(r - 1 - step, n); }
      else if (step == n - 1) { prim = P_RECVREDUCECOPYSEND; seg = r; }
      else if (step < 2 * n - 2) { prim = P_RECVCOPYSEND; seg = md(r - (step - n + 1), n); }
      else { prim = P_RECV; seg = md(r + 1, n); }
      return;
    case kReduceScatter:
      if (step == 0) { prim = P_SEND; seg = md(r - 1, n); }
      else if (step < n - 1) { prim = P_RECVREDUCESEND; seg = md(r - 1 - step, n); }
      else { prim = P_RECVREDUCECOPY; seg = r; }
      return;
    case kAllGather:
      if (step == 0) { prim = P_COPYSEND; seg = r; }
      else if (step < n - 1) { prim = P_RECVCOPYSEND; seg = md(r - step, n); }
      else { prim = P_RECV; seg = md(r + 1, n); }
      return;
    default: {  // broadcast: chain root -> root+1 -> ... -> root-1
      const int pos = md(r - root, n);
      seg = 0;
      if (pos == 0) prim = inplace ? P_SEND : P_COPYSEND;
      else if (pos == n - 1) prim = P_RECV;
      else prim = P_RECVCOPYSEND;
      return;
    }
  }
}

__device__ __forceinline__ int elem_size(int dt) { return dt == kBF16 ? 2 : 4; }

// Segment q's base offsets (elements) in the send / recv buffers and length.
__device__ __forceinline__ void seg_geom(int kind, int n, int r, uint64_t count, uint64_t segLen, int q,
                                         uint64_t& sendOff, uint64_t& recvOff, uint64_t& len) {
  if (n == 1 || kind == kBroadcast) { sendOff = 0; recvOff = 0; len = count; return; }
  switch (kind) {
    case kAllReduce: {
      const uint64_t lo = (uint64_t)q * segLen;
      sendOff = recvOff = lo;
      len = lo >= count ? 0 : (count - lo < segLen ? count - lo : segLen);
      return;
    }
    case kReduceScatter: sendOff = (uint64_t)q * count; recvOff = 0; len = count; return;
    default: sendOff = 0; recvOff = (uint64_t)q * count; len = count; return;  // all-gather
  }
}

// ------------------------------------------------------------------ shared control
enum : int { CMD_NONE = 0, CMD_RUN = 1, CMD_EXIT = 2 };
enum : int { RUN_PREEMPT = 0, RUN_GO = 1, RUN_DONE = 2 };

// Scheduler state of one block.  Lives in shared memory and is touched only by
// thread 0, so it costs the data-moving threads no registers.
struct Sched {
  uint64_t cursor, lastFetch, iter;
  uint64_t T, headSeen, creditSeen;
  uint32_t qlen, pos, exiting;
  int lastRun, curId;
  int cmd, way, needLoad, go;
  SliceDesc desc;
};

struct Smem {
  CtxSlot* cache;      // [W]  direct-mapped context cache
  int* cacheTag;       // [W]
  uint32_t* tq;        // [maxColl] task queue: id | stall << 16
};

__device__ __forceinline__ void save_dyn(CtxSlot* g, const CtxSlot& cx) {
  uint4* gd = reinterpret_cast<uint4*>(&g->d);
  const uint4* sd = reinterpret_cast<const uint4*>(&cx.d);
  st_cg_v4(gd, sd[0]);
  st_cg_v4(gd + 1, sd[1]);
}

// Admit an SQE into this block's task queue: write the static context and reset
// the dynamic cursor (keeping the connector sequence numbers).
__device__ __noinline__ void admit(const DaemonParams& p, Sched& sh, const Smem& m, const Sqe& e) {
  const int b = blockIdx.x, G = p.G, n = p.nranks, W = p.cacheWays;
  const int c = (int)e.collId;
  CtxSlot* g = &p.ctx[(size_t)c * G + b];
  const int isz = elem_size(e.dtype);
  const uint64_t A = 16 / isz;
  uint64_t segLen = e.count;
  if (n > 1 && e.kind == kAllReduce) {
    const uint64_t per = (e.count + n - 1) / n;
    segLen = (per + A - 1) / A * A;                 // segment-first owner map (R6)
  }
  uint64_t part = (segLen + e.nblocks - 1) / e.nblocks;
  part = (part + A - 1) / A * A;
  const uint64_t E = p.sliceBytes / isz;
  const uint64_t chunk = E * p.slicesPerChunk;
  uint64_t nloops = (part + chunk - 1) / chunk;
  if (nloops == 0) nloops = 1;
  int nsteps = 1;
  if (n > 1) nsteps = e.kind == kAllReduce ? 2 * n - 1 : (e.kind == kBroadcast ? 1 : n);
  const uint64_t nsent = g->d.nsent, nrecv = g->d.nrecv;
  uint4 w[kCtxBytes / 16];
  CtxSlot* ns = reinterpret_cast<CtxSlot*>(w);
  ns->s.sendbuff = e.sendbuff; ns->s.recvbuff = e.recvbuff; ns->s.subSeq = e.subSeq;
  ns->s.segLen = segLen; ns->s.part = part; ns->s.count = e.count;
  ns->d.loop = 0; ns->d.step = 0; ns->d.slc = 0; ns->d.nloops = (uint32_t)nloops;
  ns->d.kind = e.kind; ns->d.dtype = (uint8_t)e.dtype; ns->d.progressed = 0;
  ns->d.nsent = nsent; ns->d.nrecv = nrecv;
  ns->root = e.root; ns->nblocks = e.nblocks; ns->nsteps = (uint16_t)nsteps;
  uint4* dst = reinterpret_cast<uint4*>(g);
#pragma unroll
  for (int i = 0; i < kCtxBytes / 16; ++i) st_cg_v4(dst + i, w[i]);
  const int way = c % W;
  if (m.cacheTag[way] == c) m.cacheTag[way] = -1;
  if (p.orderPolicy == 0) {
    m.tq[sh.qlen++] = (uint32_t)c;                  // FIFO: tail
  } else {
    for (uint32_t i = sh.qlen; i > 0; --i) m.tq[i] = m.tq[i - 1];
    m.tq[0] = (uint32_t)c;                          // priority: front
    ++sh.qlen;
    if (sh.qlen > 1) sh.pos = (sh.pos + 1) % sh.qlen;
  }
  p.blkStats[b].fetched++;
}

// One scheduling round (thread 0): bookkeeping of the previous run, SQ fetch,
// entry selection, voluntary quit.  Sets sh.cmd.
__device__ __noinline__ void schedule(const DaemonParams& p, Sched& sh, const Smem& m) {
  const int b = blockIdx.x, G = p.G, W = p.cacheWays;
  int cmd = CMD_NONE;
  if (sh.lastRun >= 0) {
    CtxSlot& cx = m.cache[sh.way];
    const int id = sh.curId;
    CollStat& cs = p.collStats[(size_t)id * G + b];
    CtxSlot* g = &p.ctx[(size_t)id * G + b];
    if (sh.lastRun == RUN_DONE) {
      // completion counter; the block reaching the collective's grid size posts
      // the CQE.  CQ slot = collId with a single writer, so a
      // release store suffices (R9).
      cs.completions++;
      cx.d.progressed = 0;
      save_dyn(g, cx);
      fence_acq_rel(1);
      const uint32_t old = atom_add_acq_rel(&p.complCnt[id], 1u);
      if (old + 1 == cx.nblocks) {
        p.complCnt[id] = 0;
        fence_sys();
        st_volatile_u64(&p.cqDone[id], cx.s.subSeq);
        p.blkStats[b].cqes++;
      }
      for (uint32_t i = sh.pos; i + 1 < sh.qlen; ++i) m.tq[i] = m.tq[i + 1];
      --sh.qlen;
      if (sh.pos >= sh.qlen) sh.pos = 0;
    } else {
      // preempted: lazy save of a dynamic context that progressed
      if (cx.d.progressed) {
        cx.d.progressed = 0;
        save_dyn(g, cx);
        cs.ctxSaves++;
      }
      cs.preemptions++;
      uint32_t st = m.tq[sh.pos] >> 16;
      if (st < 0xffff) ++st;
      m.tq[sh.pos] = (m.tq[sh.pos] & 0xffffu) | (st << 16);
      sh.pos = (sh.pos + 1) % sh.qlen;
    }
    sh.lastRun = -1;
  }
  ++sh.iter;
  const uint64_t now = globaltimer();
  const uint32_t qlen = sh.qlen;
  bool allStalled = qlen > 0;
  for (uint32_t i = 0; i < qlen && allStalled; ++i) allStalled = (m.tq[i] >> 16) >= p.stallLimit;
  // -- fetch an SQE, gated by the order policy
  const bool canFetch = !sh.exiting && qlen < (uint32_t)p.maxColl &&
                        (qlen == 0 || (p.orderPolicy == 0 ? allStalled : (sh.iter % (uint64_t)p.priorityCadence) == 0));
  bool fetched = false;
  if (canFetch) {
    const Sqe* slot = p.sq + (sh.cursor % p.sqDepth);
    const uint64_t seq = ld_acquire_sys(&slot->seq);
    if (seq == sh.cursor + 1) {
      const volatile Sqe* vs = slot;
      Sqe e;
      e.subSeq = vs->subSeq; e.count = vs->count; e.sendbuff = vs->sendbuff; e.recvbuff = vs->recvbuff;
      e.collId = vs->collId; e.kind = vs->kind; e.dtype = vs->dtype; e.nblocks = vs->nblocks;
      e.root = vs->root;
      ++sh.cursor;
      p.blk[b].sqCursor = sh.cursor;
      fence_sys();                                   // SQE reads complete before the slot is freed
      st_volatile_u64(&p.sqCursorHost[b], sh.cursor);
      sh.lastFetch = now;
      fetched = true;
      if (e.kind == kExit) sh.exiting = 1;          // Exiting SQE
      else if (b < (int)e.nblocks) admit(p, sh, m, e);   // blockIdx < grid size (reading Q11)
    }
  }
  if (!fetched) {
    const bool stuck = qlen == 0 || allStalled;
    if (qlen == 0 && sh.exiting) {
      sh.exiting = 0;
      p.blkStats[b].exits++;
      cmd = CMD_EXIT;
    } else if (stuck && p.quitEnabled && now - sh.lastFetch > p.quitIdleNs) {
      p.blkStats[b].quits++;                         // voluntary quit
      cmd = CMD_EXIT;
    } else if (qlen > 0) {
      const int c = (int)(m.tq[sh.pos] & 0xffffu);
      const int way = c % W;
      sh.way = way;
      sh.needLoad = m.cacheTag[way] != c;
      if (sh.needLoad) {
        m.cacheTag[way] = c;
        p.collStats[(size_t)c * G + b].ctxLoads++;
      }
      sh.curId = c;
      // initial spin threshold from the queue position
      if (p.stickiness) {
        const uint64_t dec = (uint64_t)sh.pos * p.spinStep;
        uint64_t T = dec >= p.spinBase ? p.spinMin : p.spinBase - dec;
        sh.T = T < p.spinMin ? p.spinMin : T;
      } else {
        sh.T = p.spinBase;
      }
      sh.headSeen = 0;
      sh.creditSeen = 0;
      cmd = CMD_RUN;
    } else {
      p.blkStats[b].idlePolls++;
      if (p.idleSleepNs) __nanosleep(p.idleSleepNs);
    }
    if (cmd == CMD_EXIT) {                           // persist what survives the quit
      BlockState bs;
      bs.sqCursor = sh.cursor; bs.qlen = sh.qlen; bs.pos = sh.pos; bs.exiting = sh.exiting; bs.pad = 0;
      p.blk[b] = bs;
      for (uint32_t i = 0; i < sh.qlen; ++i) p.tqSave[(size_t)b * p.maxColl + i] = m.tq[i];
    }
  }
  sh.cmd = cmd;
}

// Thread 0: locate the current slice and wait for the connectors, counting
// failed polls (two-phase blocking).  Sets sh.go / sh.desc.
__device__ __noinline__ void prepare_wait(const DaemonParams& p, Sched& sh, const Smem& m) {
  const int b = blockIdx.x, G = p.G, K = p.K, n = p.nranks, sys = p.sysScope;
  CtxSlot& cx = m.cache[sh.way];
  DynCtx& d = cx.d;
  if (d.loop >= d.nloops) { sh.go = RUN_DONE; return; }
  const int c = sh.curId;
  int prim, seg;
  step_prim(d.kind, n, p.rank, cx.root, d.step, cx.s.sendbuff == cx.s.recvbuff, prim, seg);
  uint64_t sendOff, recvOff, len;
  seg_geom(d.kind, n, p.rank, cx.s.count, cx.s.segLen, seg, sendOff, recvOff, len);
  const int isz = elem_size(d.dtype);
  const uint64_t E = p.sliceBytes / isz;
  const uint64_t laneLo = (uint64_t)b * cx.s.part;
  uint64_t laneHi = laneLo + cx.s.part;
  if (laneHi > len) laneHi = len;
  const uint64_t lo = laneLo + ((uint64_t)d.loop * p.slicesPerChunk + d.slc) * E;
  uint64_t hi = lo + E;
  if (hi > laneHi) hi = laneHi;
  const size_t cb = (size_t)c * G + b;
  const bool needRecv = prim & A_RECV, needSend = prim & A_SEND;
  const char* fl = p.flagsLocal + cb * kFlagStride;
  uint64_t spins = 0;
  for (;;) {
    bool ok = true;
    if (needRecv && d.nrecv >= sh.headSeen) {
      sh.headSeen = ld_relaxed(fl, sys);
      ok = d.nrecv < sh.headSeen;
    }
    if (ok && needSend && d.nsent - sh.creditSeen >= (uint64_t)K) {
      sh.creditSeen = ld_relaxed(fl + 128, sys);
      ok = d.nsent - sh.creditSeen < (uint64_t)K;
    }
    if (ok) break;
    if (++spins > sh.T) { sh.go = RUN_PREEMPT; return; }
  }
  if (needRecv || needSend) fence_acq_rel(sys);      // acquire the peer's data / credit
  SliceDesc& sd = sh.desc;
  sd.src = reinterpret_cast<const char*>(cx.s.sendbuff) + (sendOff + lo) * isz;
  sd.dst = reinterpret_cast<char*>(cx.s.recvbuff) + (recvOff + lo) * isz;
  sd.cin = p.dataLocal + (cb * K + (d.nrecv % K)) * p.sliceBytes;
  sd.cout = p.dataNext + (cb * K + (d.nsent % K)) * p.sliceBytes;
  sd.nelem = hi > lo ? (int64_t)(hi - lo) : 0;
  sd.prim = prim;
  sd.dtype = d.dtype;
  sh.go = RUN_GO;
}

// Thread 0, after the block's barrier: publish the slice to the peers
// (commit visibility) and advance the dynamic context.
__device__ __noinline__ void commit(const DaemonParams& p, Sched& sh, const Smem& m) {
  const int b = blockIdx.x, sys = p.sysScope;
  CtxSlot& cx = m.cache[sh.way];
  DynCtx& d = cx.d;
  const int prim = sh.desc.prim;
  const size_t cb = (size_t)sh.curId * p.G + b;
  if (prim & (A_RECV | A_SEND)) fence_acq_rel(sys);
  if (prim & A_SEND) {
    d.nsent++;
    st_relaxed(p.flagsNext + cb * kFlagStride, d.nsent, sys);          // head of rank r+1
  }
  if (prim & A_RECV) {
    d.nrecv++;
    st_relaxed(p.flagsPrev + cb * kFlagStride + 128, d.nrecv, sys);    // credit of rank r-1
  }
  if (++d.slc == p.slicesPerChunk) {
    d.slc = 0;
    if (++d.step == cx.nsteps) { d.step = 0; d.loop++; }
  }
  d.progressed = 1;
  m.tq[sh.pos] &= 0xffffu;                          // progressed: no longer stalled
  if (p.stickiness) {                               // raise the threshold
    uint64_t T = sh.T * p.spinBoost;
    sh.T = T > p.spinCap ? p.spinCap : T;
  }
  p.collStats[cb].slices++;
}

}  // namespace

// =============================================================================
// The daemon kernel.  Launched with the largest grid/block of all collectives
// (PAPER.md:470): grid = G blocks, one scheduler per block.
// =============================================================================
__global__ void __launch_bounds__(512, 1) occl_daemon_kernel(const DaemonParams* __restrict__ pp) {
  const DaemonParams& p = *pp;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ Sched sh;
  const int W = p.cacheWays;
  Smem m;
  m.cache = reinterpret_cast<CtxSlot*>(smem);
  m.cacheTag = reinterpret_cast<int*>(m.cache + W);
  m.tq = reinterpret_cast<uint32_t*>(m.cacheTag + W);
  const int tid = threadIdx.x;
  const int b = blockIdx.x;

  if (tid == 0) {
    const BlockState bs = p.blk[b];
    sh.cursor = bs.sqCursor;
    sh.qlen = bs.qlen;
    sh.pos = bs.pos;
    sh.exiting = bs.exiting;
    sh.iter = 0;
    sh.lastRun = -1;
    sh.curId = -1;
    for (uint32_t i = 0; i < sh.qlen; ++i) m.tq[i] = p.tqSave[(size_t)b * p.maxColl + i];
    for (int w = 0; w < W; ++w) m.cacheTag[w] = -1;
    sh.lastFetch = globaltimer();
    p.blkStats[b].launches++;
  }
  __syncthreads();

  for (;;) {
    if (tid == 0) schedule(p, sh, m);
    __syncthreads();
    const int cmd = sh.cmd;
    if (cmd == CMD_EXIT) break;
    if (cmd == CMD_NONE) continue;

    // context load into the shared-memory cache, 16 B per thread
    const int way = sh.way;
    if (sh.needLoad) {
      if (tid < kCtxBytes / 16) {
        const uint4* g = reinterpret_cast<const uint4*>(&p.ctx[(size_t)m.cacheTag[way] * p.G + b]);
        reinterpret_cast<uint4*>(&m.cache[way])[tid] = ld_cg(g + tid);
      }
      __syncthreads();
    }

    // primitive execution, slice by slice, until preempted or done
    for (;;) {
      if (tid == 0) prepare_wait(p, sh, m);
      __syncthreads();
      const int go = sh.go;
      if (go != RUN_GO) {
        if (tid == 0) sh.lastRun = go;
        break;
      }
      {
        const SliceDesc sd = sh.desc;
        move_slice_any(sd);
      }
      __syncthreads();
      if (tid == 0) commit(p, sh, m);
    }
  }
}

extern "C" size_t occl_internal_daemon_smem(int maxColl, int cacheWays) {
  return (size_t)cacheWays * sizeof(CtxSlot) + (size_t)cacheWays * sizeof(int) + (size_t)(maxColl + 1) * 4 + 16;
}

// `pDev` points to a device-memory copy of the parameters (constant for the
// communicator's lifetime); `p` is the host copy.
extern "C" int occl_internal_launch_daemon(const DaemonParams* p, const DaemonParams* pDev, int blockThreads,
                                           void* stream) {
  const size_t smem = occl_internal_daemon_smem(p->maxColl, p->cacheWays);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(occl_daemon_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return (int)e;
  }
  occl_daemon_kernel<<<p->G, blockThreads, smem, (cudaStream_t)stream>>>(pDev);
  return (int)cudaGetLastError();
}
