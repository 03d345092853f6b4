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
#include <cuda_fp16.h>
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
__device__ __forceinline__ uint64_t ld_acquire(const void* p, int sys) {
  uint64_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  else     asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(void* p, uint64_t v, int sys) {
  if (sys) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
  else     asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
}
// Monotonic publication of a connector counter: slices are published by whichever
// data warp finishes last, so two publications may race; max keeps it monotonic.
__device__ __forceinline__ void red_max_relaxed(void* p, uint64_t v, int sys) {
  if (sys) asm volatile("red.relaxed.sys.global.max.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
  else     asm volatile("red.relaxed.gpu.global.max.u64 [%0], %1;" :: "l"(p), "l"(v) : "memory");
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

// ------------------------------------------------------------------ reducing function (+)
// The collective's reducing function, per element, bit-exact with
// the oracle (R7 / R22): sum / prod / max / min.
// f32: IEEE add / multiply round-to-nearest-even (__fadd_rn / __fmul_rn: no FMA
// contraction).  i32: two's-complement wrap, signed max / min.  bf16 / f16: the
// correctly rounded 16-bit result (__hadd2 / __hmul2 / __hmax2 / __hmin2).
enum : int { kSum = 0, kProd = 1, kMax = 2, kMin = 3 };

// max / min are IEEE 754-2019 maximum / minimum (reading R24): -0 < +0
// whatever the operand order, so a ring fold of signed zeros is order-free.  For
// two zeros the result's sign bit is the AND (max) / OR (min) of theirs.
template <int OP> __device__ __forceinline__ uint32_t op_f32(uint32_t a, uint32_t b) {
  const float x = __uint_as_float(a), y = __uint_as_float(b);
  if constexpr (OP == kSum) return __float_as_uint(__fadd_rn(x, y));
  else if constexpr (OP == kProd) return __float_as_uint(__fmul_rn(x, y));
  else if constexpr (OP == kMax) return ((a | b) << 1) == 0 ? (a & b) : __float_as_uint(fmaxf(x, y));
  else return ((a | b) << 1) == 0 ? (a | b) : __float_as_uint(fminf(x, y));
}
// signed-zero rule of max / min on the two 16-bit lanes of a packed word
template <int OP> __device__ __forceinline__ uint32_t zero_fix16(uint32_t r, uint32_t a, uint32_t b) {
  if constexpr (OP == kMax || OP == kMin) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t sh = 16u * h, ah = (a >> sh) & 0xffffu, bh = (b >> sh) & 0xffffu;
      if (((ah | bh) & 0x7fffu) == 0) {
        const uint32_t v = OP == kMax ? (ah & bh) : (ah | bh);
        r = (r & ~(0xffffu << sh)) | (v << sh);
      }
    }
  }
  return r;
}
template <int OP> __device__ __forceinline__ uint32_t op_i32(uint32_t a, uint32_t b) {
  if constexpr (OP == kSum) return a + b;
  else if constexpr (OP == kProd) return a * b;
  else if constexpr (OP == kMax) return (uint32_t)max((int32_t)a, (int32_t)b);
  else return (uint32_t)min((int32_t)a, (int32_t)b);
}
template <int OP> __device__ __forceinline__ uint32_t op_bf16x2(uint32_t a, uint32_t b) {
  const __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162 y = *reinterpret_cast<const __nv_bfloat162*>(&b);
  __nv_bfloat162 z;
  if constexpr (OP == kSum) z = __hadd2(x, y);
  else if constexpr (OP == kProd) z = __hmul2(x, y);
  else if constexpr (OP == kMax) z = __hmax2(x, y);
  else z = __hmin2(x, y);
  return zero_fix16<OP>(*reinterpret_cast<uint32_t*>(&z), a, b);
}
template <int OP> __device__ __forceinline__ uint32_t op_f16x2(uint32_t a, uint32_t b) {
  const __half2 x = *reinterpret_cast<const __half2*>(&a);
  const __half2 y = *reinterpret_cast<const __half2*>(&b);
  __half2 z;
  if constexpr (OP == kSum) z = __hadd2(x, y);
  else if constexpr (OP == kProd) z = __hmul2(x, y);
  else if constexpr (OP == kMax) z = __hmax2(x, y);
  else z = __hmin2(x, y);
  return zero_fix16<OP>(*reinterpret_cast<uint32_t*>(&z), a, b);
}
template <int OP> __device__ __forceinline__ uint64_t op_i64(uint64_t a, uint64_t b) {
  if constexpr (OP == kSum) return a + b;
  else if constexpr (OP == kProd) return a * b;
  else if constexpr (OP == kMax) return (uint64_t)max((long long)a, (long long)b);
  else return (uint64_t)min((long long)a, (long long)b);
}
template <int OP> __device__ __forceinline__ uint64_t op_f64(uint64_t a, uint64_t b) {
  const double x = __longlong_as_double((long long)a), y = __longlong_as_double((long long)b);
  double z;
  if constexpr (OP == kSum) z = __dadd_rn(x, y);
  else if constexpr (OP == kProd) z = __dmul_rn(x, y);
  else if constexpr (OP == kMax) { if (((a | b) << 1) == 0) return a & b; z = fmax(x, y); }
  else { if (((a | b) << 1) == 0) return a | b; z = fmin(x, y); }
  return (uint64_t)__double_as_longlong(z);
}
template <int DT, int OP> __device__ __forceinline__ uint64_t op_d(uint64_t a, uint64_t b) {
  if constexpr (DT == kI64) return op_i64<OP>(a, b);
  else return op_f64<OP>(a, b);
}
// one 32-bit lane of packed elements
template <int DT, int OP> __device__ __forceinline__ uint32_t op_w(uint32_t a, uint32_t b) {
  if constexpr (DT == kF32) return op_f32<OP>(a, b);
  else if constexpr (DT == kI32) return op_i32<OP>(a, b);
  else if constexpr (DT == kBF16) return op_bf16x2<OP>(a, b);
  else return op_f16x2<OP>(a, b);
}
template <int DT, int OP> __device__ __forceinline__ uint4 vop(const uint4& a, const uint4& b) {
  if constexpr (DT == kI64 || DT == kF64) {           // two 64-bit elements per vector
    const uint64_t lo = op_d<DT, OP>(((uint64_t)a.y << 32) | a.x, ((uint64_t)b.y << 32) | b.x);
    const uint64_t hi = op_d<DT, OP>(((uint64_t)a.w << 32) | a.z, ((uint64_t)b.w << 32) | b.z);
    return make_uint4((uint32_t)lo, (uint32_t)(lo >> 32), (uint32_t)hi, (uint32_t)(hi >> 32));
  } else {
    return make_uint4(op_w<DT, OP>(a.x, b.x), op_w<DT, OP>(a.y, b.y), op_w<DT, OP>(a.z, b.z),
                      op_w<DT, OP>(a.w, b.w));
  }
}

// ------------------------------------------------------------------ primitives
// Action bits of the fused primitives.
enum : int { A_RECV = 1, A_REDUCE = 2, A_COPY = 4, A_SEND = 8,
             A_DIN = 16,    // direct receive: the upstream wrote the data into our recv buffer
             A_DOUT = 32,   // direct send: write into the downstream's recv buffer, not its connector
             A_LL = 64,     // LL protocol: 16-B lines {data, flag, data, flag}, no release fence
             A_DREAD = 128,   // direct read: the input is the upstream's send buffer (no message)
             A_KEEPOUT = 256,   // direct send whose data the downstream re-reads next hop (L2 evict-last)
             A_LLRUN = 512 };   // LL run: the compute warps move every remaining slice themselves (Pipe::llr)
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
  char* headOut;       // downstream head flag (published = headVal) when prim sends
  char* creditOut;     // upstream credit flag (published = creditVal) when prim receives
  uint64_t headVal, creditVal;
  int64_t nelem;
  int prim;
  int dtype;
  int op;              // reducing function (kSum / kProd / kMax / kMin)
  uint32_t gen;        // LL speculation: the pipe's abort generation when the slice was issued
};

template <int DT> struct Elem;
template <> struct Elem<kF32> { typedef uint32_t T; };
template <> struct Elem<kI32> { typedef uint32_t T; };
template <> struct Elem<kBF16> { typedef uint16_t T; };
template <> struct Elem<kF16> { typedef uint16_t T; };
template <> struct Elem<kI64> { typedef uint64_t T; };
template <> struct Elem<kF64> { typedef uint64_t T; };

// one element (bit pattern) of the reducing function
template <int DT, int OP>
__device__ __forceinline__ typename Elem<DT>::T sop(typename Elem<DT>::T a, typename Elem<DT>::T b) {
  if constexpr (sizeof(typename Elem<DT>::T) == 8) {
    return op_d<DT, OP>(a, b);
  } else if constexpr (sizeof(typename Elem<DT>::T) == 4) {
    return op_w<DT, OP>(a, b);
  } else {
    return (typename Elem<DT>::T)(op_w<DT, OP>((uint32_t)a, (uint32_t)b) & 0xffffu);   // low half only
  }
}

// Move one slice with the data warps: 128-bit vectors, U independent loads in
// flight per thread (twice that for reduce), then the stores.
// Loads bypass L1 (ld.global.cg): connector slots are rewritten by peers and the
// persistent kernel must never see a stale line.  The action bits are
// warp-uniform runtime flags; only the element type is a template.
template <int DT, int OP>
__device__ __forceinline__ void move_slice(const int prim, const char* src, const char* cin, char* dst, char* cout,
                                           const int64_t nelem, const int tid, const int nt) {
  typedef typename Elem<DT>::T T;
  constexpr int A = 16 / sizeof(T);
  constexpr int U = 2;                            // slices here are < kTmaMinBytes: 2 x 16 B per thread covers them
  const bool recv = prim & (A_RECV | A_DREAD), reduce = prim & A_REDUCE, copy = prim & A_COPY, send = prim & A_SEND;
  const int n = (int)nelem;                       // <= sliceBytes / sizeof(T)
  if (n <= 0) return;
  const bool aligned = ((((uintptr_t)src) | ((uintptr_t)dst) | ((uintptr_t)cin) | ((uintptr_t)cout)) & 15) == 0;
  const int nvec = aligned ? n / A : 0;
  const uint4* vs = reinterpret_cast<const uint4*>(src);
  const uint4* vi = reinterpret_cast<const uint4*>(recv ? cin : src);
  uint4* vd = reinterpret_cast<uint4*>(dst);
  uint4* vo = reinterpret_cast<uint4*>(cout);
  int i = tid;
  // full tiles: U vectors per thread, no bounds checks
  for (; i + (U - 1) * nt < nvec; i += U * nt) {
    uint4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldcg(vi + i + u * nt);
    if (reduce) {
      uint4 c[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = __ldcg(vs + i + u * nt);
#pragma unroll
      for (int u = 0; u < U; ++u) a[u] = vop<DT, OP>(a[u], c[u]);
    }
    if (copy) {
#pragma unroll
      for (int u = 0; u < U; ++u) __stcg(vd + i + u * nt, a[u]);
    }
    if (send) {
#pragma unroll
      for (int u = 0; u < U; ++u) __stcg(vo + i + u * nt, a[u]);
    }
  }
  // remaining vectors, one per thread per iteration
  for (; i < nvec; i += nt) {
    uint4 v = __ldcg(vi + i);
    if (reduce) v = vop<DT, OP>(v, __ldcg(vs + i));
    if (copy) __stcg(vd + i, v);
    if (send) __stcg(vo + i, v);
  }
  // scalar tail (ragged segment ends) or the whole slice when misaligned
  const T* ss = reinterpret_cast<const T*>(src);
  const T* si = reinterpret_cast<const T*>(recv ? cin : src);
  T* sd = reinterpret_cast<T*>(dst);
  T* so = reinterpret_cast<T*>(cout);
  for (int e = nvec * A + tid; e < n; e += nt) {
    T v = ld_cg_scalar(si + e);
    if (reduce) v = sop<DT, OP>(v, ld_cg_scalar(ss + e));
    if (copy) sd[e] = v;
    if (send) so[e] = v;
  }
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
    case kReduce: {  // chain root+1 -> root+2 -> ... -> root (NCCL ring Reduce), one segment
      const int pos = md(r - root - 1, n);
      seg = 0;
      if (pos == 0) prim = P_SEND;
      else if (pos == n - 1) prim = P_RECVREDUCECOPY;
      else prim = P_RECVREDUCESEND;
      return;
    }
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

// Direct mode: data that is FINAL -- the all-gather phase of an
// all-reduce, every hop of an all-gather or broadcast -- goes straight into the
// downstream's recv buffer instead of its connector (when that buffer is
// addressable), and a direct receive finds it in place: RecvCopySend becomes a
// recv-buffer -> peer recv-buffer copy and the final Recv moves no data.  The
// head / credit protocol is unchanged (a direct message still takes a connector
// sequence number), so flow control and resume are exactly as before.
__device__ __forceinline__ int directify(int prim, int kind, int n, int step, bool dOut, bool dIn, bool dRead) {
  if (n == 1) return prim;
  // direct read: the first reduce step reads the upstream's send
  // buffer itself, so the upstream's step 0 (copying it into our connector) and
  // the message disappear on both ends of the edge
  if (dRead && (kind == kAllReduce || kind == kReduceScatter)) {
    if (step == 0 && dOut) return 0;                              // no-op: the downstream reads our buffer
    if (step == 1 && dIn) prim = (prim & ~A_RECV) | A_DREAD;
  }
  if (kind == kReduceScatter || kind == kReduce) return prim;   // partial sums are not final
  const bool agPhase = kind != kAllReduce || step >= n - 1;    // data on the wire is final
  if (dOut && agPhase && (prim & A_SEND)) prim |= A_DOUT;
  const bool finalIn = kind != kAllReduce || step >= n;          // received data is final
  if (dIn && finalIn && (prim & A_RECV)) prim = (prim | A_DIN) & ~A_COPY;  // already in place
  return prim;
}

// Does the downstream read (and forward) the data we direct-send at `step`?  Then
// it is worth keeping in L2 for one hop (l2Hints == 3).
__device__ __forceinline__ bool downstream_forwards(int kind, int n, int r, int root, int step) {
  switch (kind) {
    case kAllReduce: return step + 1 <= 2 * n - 3;
    case kAllGather: return step + 1 <= n - 2;
    case kBroadcast: return md(r - root, n) + 1 <= n - 2;
    default: return false;
  }
}

__device__ __forceinline__ int elem_size(int dt) {
  return (dt == kBF16 || dt == kF16) ? 2 : ((dt == kI64 || dt == kF64) ? 8 : 4);
}

// Segment q's base offsets (elements) in the send / recv buffers and length.
__device__ __forceinline__ void seg_geom(int kind, int n, int r, uint64_t count, uint64_t segLen, int q,
                                         uint64_t& sendOff, uint64_t& recvOff, uint64_t& len) {
  if (n == 1 || kind == kBroadcast || kind == kReduce) { sendOff = 0; recvOff = 0; len = count; return; }
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

// ------------------------------------------------------------------ mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" :: "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
               " selp.u32 %0, 1, 0, p;\n}" : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n LAB_WAIT_%=:\n"
               " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra LAB_WAIT_%=;\n}" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
               :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// 1-D bulk copy global -> shared through the TMA unit; completes on `bar`.
__device__ __forceinline__ void tma_load(void* smemDst, const void* gsrc, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(smemDst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// ------------------------------------------------------------------ event trace
// Record slots are claimed with a shared-memory counter (the control and the
// publisher lanes both trace); the timestamp is taken first so the claim does
// not skew it.  The publisher writes the block's running count back at exit.
struct TraceCtl {
  uint32_t base, idx;
};
__device__ __forceinline__ void trace_at_t(const DaemonParams& p, TraceCtl& tc, int b, uint32_t ev, int coll,
                                           uint32_t arg, uint64_t t) {
  if (!p.traceCap) return;
  const uint32_t k = tc.base + atomicAdd(&tc.idx, 1u);       // shared-memory atomic
  TraceRec* r = p.trace + (size_t)b * p.traceCap + (k % p.traceCap);
  const uint4 v = make_uint4((uint32_t)t, (uint32_t)(t >> 32), (ev << 24) | ((uint32_t)coll & 0xffffu), arg);
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" :: "l"(r), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  atomicMax(&p.traceCount[b], k + 1);                          // readable while the daemon runs
}
__device__ __forceinline__ void trace_at(const DaemonParams& p, TraceCtl& tc, int b, uint32_t ev, int coll,
                                         uint32_t arg) {
  if (!p.traceCap) return;
  trace_at_t(p, tc, b, ev, coll, arg, globaltimer());
}

// ------------------------------------------------------------------ shared control
enum : int { CMD_NONE = 0, CMD_RUN = 1, CMD_EXIT = 2 };
enum : int { RUN_PREEMPT = 0, RUN_GO = 1, RUN_DONE = 2 };
constexpr int P_EXIT = 0x100;          // descriptor telling the data warps to leave
constexpr int kMaxDepth = 8;           // max slices in flight between control and data warps
constexpr int kMaxBlockThreads = 608;  // control + TMA producer + publisher warps + up to 16 compute warps (104 registers)
constexpr int kRoleWarps = 3;          // warps 0..2: control, producer, publisher
constexpr int kTile = 16384;           // TMA staging tile (bytes per operand)
constexpr int kMaxStages = 6;          // staging ring depth: up to 6 x 2 x 16 KiB of loads in flight
constexpr int kTmaMinBytes = 16384;    // slices below this use register loads (latency-bound sizes)
constexpr uint32_t kQuitLatch = 0x80000000u;   // quitWord: every block of the launch voted to quit
constexpr uint64_t kSqPollNs = 2000;           // a blocked collective polls the SQ at most this often
constexpr int kSqBurst = 4;                    // host SQ slots read by one bulk copy
constexpr int kBoardOff = kDirectOff + 64;     // readiness board slot in the (collId, block 0) direct line
constexpr int kReadyScan = 64;                 // queue entries the priority scheduler checks for readiness

// Scheduler state of one block; touched only by the control thread.
struct Sched {
  uint64_t cursor, lastFetch, iter;
  uint64_t T;
  uint32_t qlen, pos, exiting;
  uint32_t rr;                 // priority policy: next non-front entry to visit
  uint32_t voted;              // this block voted for the launch's voluntary quit
  uint64_t lastProgress;       // %globaltimer of the last run that committed a slice
  uint64_t lastSqPoll;         // %globaltimer of this block's last SQ check while blocked (priority policy)
  uint32_t sqPhase;            // parity of the SQ staging mbarrier
  uint32_t needHostPoll;       // a blocked run yielded because the host SQ holds a new SQE
  uint32_t boostOk;            // the running entry may be boosted (stickiness, R10 / R29)
  int lastRun, curId;
  int way;
  unsigned long long cycRun, cycPoll, cycAcqFence, cycRelFence, nCommit;   // probes
  unsigned long long cycCtxLoad, nCtxLoad, cycCtxSave, nCtxSave;
  unsigned long long cycCqe, nCqe;
  unsigned long long idlePolls;
};

// LL run (llSpeculate == 2, DESIGN.md §LL runs): for a latency-bound (LL)
// collective the control lane hands the compute warps the whole remaining slice
// schedule at once; they walk it themselves -- per slice: geometry, credit,
// poll their lines, reduce / copy / store, one named barrier, the credit to the
// upstream -- and stop when the schedule is done or a slice has not completed
// within limitNs.  Wire-compatible with the per-slice LL path (same lines,
// sequence numbers and credits).  Written by the control lane before the run's
// descriptor is published; the out fields by compute thread 0 before its warp
// releases the descriptor (empty[]).
struct LLStep {                 // one ring step of an LL run: primitive and segment geometry
  uint64_t sendOff, recvOff, len;
  int prim, pad;
};
struct LLRun {
  uint64_t sendbuff, recvbuff, count, segLen, laneLo, part, E;
  const char* llIn;
  char* llOut;
  const char* creditIn;   // our credit, raised by the downstream
  char* creditOut;        // the upstream's credit, raised by us
  uint64_t llSlot, limitNs;
  uint64_t nsent, nrecv, creditSeen;
  uint32_t loop, step, slc, nloops;
  int kind, n, r, root, inplace, dtype, op, spc, nsteps, K, sys;
  // out
  uint64_t oNsent, oNrecv, oCreditSeen, tProg;
  uint32_t oLoop, oStep, oSlc, nDone;
  // in-run exchange between compute threads
  uint64_t credit;        // thread 0's credit poll, broadcast
  uint32_t abort[3];      // [0], [1] by slice parity: a thread's line poll timed out; [2] credit poll timed out
};

// Control -> data warp pipeline: slice descriptors in a ring of `depth` buffers.
// full[i] completes when the control thread published ring[i]; every compute
// warp arrives on sdone[i] when it finished its share of the slice; the
// publisher thread then makes the slice visible to the peers (ONE release fence
// for every slice finished so far + head / credit store) and completes empty[i].
// The fence -- an L2 round trip that waits for the SM's outstanding stores --
// thus never stalls a compute warp (a fenced compute warp would hold back the
// staging ring for the whole block).  Slices are published in order, so the
// connector counters stay monotonic.
struct Pipe {
  SliceDesc ring[kMaxDepth];
  uint64_t full[kMaxDepth];      // control -> producer / compute / publisher: descriptor valid
  uint64_t sdone[kMaxDepth];     // compute warps -> publisher: slice moved (count = compute warps)
  uint64_t empty[kMaxDepth];     // publisher + producer + compute -> control: slice published, descriptor read
  TraceCtl tr;                   // event-trace slot counter of this block
  // LL speculation (cfg.llSpeculate): the control thread raises abortGen to make
  // data warps give up slices whose lines have not arrived; a warp that gave up
  // sets fail[i] before its sdone arrive.  Only the control thread writes
  // abortGen and clears fail[i] (after empty[i], before reusing the slot).
  uint32_t abortGen;
  uint32_t fail[kMaxDepth];
  LLRun llr;                     // the LL run in flight (at most one: the control lane waits for it)
  LLStep llsteps[2 * kMaxRanks]; // its per-step table (built by the compute warps at the run's start)
};

struct Smem {
  TraceCtl* tr;        // event-trace slot counter (in the pipe)
  CtxSlot* cache;      // [W]  direct-mapped context cache
  int* cacheTag;       // [W]
  uint32_t* tq;        // [maxColl] task queue: id | stall << 16
  int32_t* prio;       // [maxColl] priority of each queued collective (by id)
  uint32_t* subLo;     // [maxColl] low 32 bits of each queued collective's submission number
  uint8_t* subOf;      // [maxColl] its ring (RingDesc index)
  uint8_t* ready;      // [maxColl] every member admitted it (readiness board, reading R29)
  SqeWire* sqbuf;      // [kSqBurst] host SQ slots read by one TMA bulk copy (sq_fetch)
  uint64_t* sqbar;     // its mbarrier
};

__device__ __forceinline__ void save_dyn(CtxSlot* g, const DynCtx& d) {
  uint4* gd = reinterpret_cast<uint4*>(&g->d);
  const uint4* sd = reinterpret_cast<const uint4*>(&d);
  st_cg_v4(gd, sd[0]);
  st_cg_v4(gd + 1, sd[1]);
}

// Admit an SQE into this block's task queue: write the static context and reset
// the dynamic cursor (keeping the connector sequence numbers).
__device__ __noinline__ void admit(const DaemonParams& p, int b, int lane, Sched& sh, const Smem& m, const Sqe& e) {
  const RingDesc& R = p.rings[e.sub];                 // (by reference: the struct holds 64 member pointers)
  const int G = p.G, n = R.nranks, W = p.cacheWays;
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
  // LL for collectives whose per-block part is small (latency-bound): identical
  // decision on every rank (same count, ring size, grid size and config)
  const uint32_t ll = (p.llMaxBytes && n > 1 && part * isz <= p.llMaxBytes) ? 1u : 0u;
  const uint64_t E = (ll ? p.llSliceBytes : p.sliceBytes) / isz;
  // a block whose part fits in fewer slices than a chunk sends no empty slices:
  // every message of the ring is a hop of latency (same on all ranks)
  uint64_t spc = (part + E - 1) / E;
  if (spc < 1) spc = 1;
  if (spc > (uint64_t)p.slicesPerChunk) spc = p.slicesPerChunk;
  const uint64_t chunk = E * spc;
  uint64_t nloops = (part + chunk - 1) / chunk;
  if (nloops == 0) nloops = 1;
  int nsteps = 1;
  if (n > 1) nsteps = e.kind == kAllReduce ? 2 * n - 1 : ((e.kind == kBroadcast || e.kind == kReduce) ? 1 : n);
  const uint64_t nsent = g->d.nsent, nrecv = g->d.nrecv;
  uint4 w[kCtxBytes / 16];
  CtxSlot* ns = reinterpret_cast<CtxSlot*>(w);
  ns->s.sendbuff = e.sendbuff; ns->s.recvbuff = e.recvbuff; ns->s.subSeq = e.subSeq;
  ns->s.segLen = segLen; ns->s.part = part; ns->s.count = e.count;
  ns->d.loop = 0; ns->d.step = 0; ns->d.slc = 0; ns->d.nloops = (uint32_t)nloops;
  ns->d.kind = e.kind; ns->d.dtype = (uint8_t)e.dtype; ns->d.progressed = 0;
  ns->d.nsent = nsent; ns->d.nrecv = nrecv;
  ns->root = e.root; ns->nblocks = e.nblocks; ns->nsteps = (uint16_t)nsteps; ns->priority = e.priority;
  ns->lane = (uint32_t)lane;
  ns->sub = e.sub;
  ns->op = e.op;
  ns->proto = ll;
  ns->spc = (uint32_t)spc;
  uint4* dst = reinterpret_cast<uint4*>(g);
#pragma unroll
  for (int i = 0; i < kCtxBytes / 16; ++i) st_cg_v4(dst + i, w[i]);
  if (p.directRead && R.directNext && n > 1 && !ll && (e.kind == kAllReduce || e.kind == kReduceScatter)) {
    // tell the downstream where this submission's send buffer is (direct read)
    char* f = R.flagsNext + ((size_t)c * G + b) * kFlagStride + kDirectOff + 16;
    st_relaxed(f, e.sendbuff, p.sysScope);
    if (p.sysScope) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(f + 8), "l"(e.subSeq) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(f + 8), "l"(e.subSeq) : "memory");
  }
  if (R.directPrev && n > 1 && e.kind != kReduceScatter && !ll) {
    // tell the upstream where this submission's final data goes (direct mode)
    char* f = R.flagsPrev + ((size_t)c * G + b) * kFlagStride + kDirectOff;
    st_relaxed(f, e.recvbuff, p.sysScope);
    if (p.sysScope) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(f + 8), "l"(e.subSeq) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(f + 8), "l"(e.subSeq) : "memory");
  }
  // install the fresh context in its cache way as well: the collective just
  // admitted usually runs next, and this saves its first context load (a global
  // round trip).  Every cached context is clean between runs (a run's end saves
  // it), so evicting the way's occupant loses nothing.
  const int way = c % W;
  {
    uint4* cw = reinterpret_cast<uint4*>(&m.cache[way]);
#pragma unroll
    for (int i = 0; i < kCtxBytes / 16; ++i) cw[i] = w[i];
    m.cacheTag[way] = c;
  }
  m.prio[c] = e.priority;
  m.subLo[c] = (uint32_t)e.subSeq;
  m.subOf[c] = (uint8_t)e.sub;
  m.ready[c] = (n == 1) ? 1 : 0;
  if (lane == 0 && p.orderPolicy == 1 && p.readyFirst) {
    // readiness board (reading R29): this rank admitted submission subSeq of c
    char* slot = p.flagsLocal + (size_t)c * G * kFlagStride + kBoardOff;
    if (p.sysScope) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(slot), "l"(e.subSeq) : "memory");
    else asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(slot), "l"(e.subSeq) : "memory");
  }
  if (p.orderPolicy == 0) {
    m.tq[sh.qlen++] = (uint32_t)c;                  // FIFO: tail
  } else {
    // priority order: the queue is kept sorted by the
    // user-defined priority (ties: arrival); a collective that outranks the
    // current front goes to the front and the traversal restarts there.  With a
    // globally agreed priority every rank's queue has the same order, so the
    // ranks converge on the same front (de-facto gang scheduling).
    uint32_t at = sh.qlen;
    while (at > 0 && m.prio[m.tq[at - 1] & 0xffffu] > e.priority) {
      m.tq[at] = m.tq[at - 1];
      --at;
    }
    m.tq[at] = (uint32_t)c;
    ++sh.qlen;
    sh.pos = 0;
  }
  p.blkStats[b].fetched++;
  trace_at(p, *m.tr, b, kEvFetch, c, (uint32_t)e.subSeq);
}

// SQ fetch through a device-memory mirror.  Every block consumes
// every SQE, but only the block holding `fetchLock` reads the
// host SQ over PCIe: it copies new SQEs into the mirror (as long as no block
// still needs the slot it overwrites), publishes the mirror tail, and tells the
// host which SQ slots are free.  The other blocks read the mirror from L2.  This
// replaces G PCIe reads per SQE (and per idle poll) with one.
__device__ __noinline__ bool sq_fetch(const DaemonParams& p, const Smem& m, Sched& sh, int b) {
  if (atomicCAS(p.fetchLock, 0u, 1u) != 0u) return true;       // another block is fetching
  trace_at(p, *m.tr, b, kEvMark, 0, 1);
  // any host poll restarts the rank's rate-limit clock for busy blocks (schedule())
  *reinterpret_cast<volatile unsigned long long*>(p.mirrorTail + 3) = (unsigned long long)globaltimer();
  uint64_t t = ld_relaxed(p.mirrorTail, 0);
  // the slowest block's cursor bounds which mirror slots may be overwritten; a
  // cached value is a safe lower bound (cursors only grow), so the G cursors are
  // re-read only when the mirror looks full -- in parallel, then one fence
  uint64_t minCur = ld_relaxed(p.mirrorTail + 2, 0);
  if (t - minCur >= p.sqDepth - 64) {
    uint64_t m = ~0ull;
    for (int bb = 0; bb < p.G; ++bb) {
      const uint64_t c = ld_relaxed(&p.blk[bb].sqCursor, 0);
      m = c < m ? c : m;
    }
    fence_acq_rel(0);                                          // acquire: slot reuse after their loads
    minCur = m;
    st_relaxed(p.mirrorTail + 2, m, 0);
  }
  const uint64_t t0 = t;
  constexpr int B = kSqBurst;
  for (;;) {
    // ONE PCIe round trip: up to B slots in one TMA bulk copy into shared memory
    // (a thread's k independent ld.relaxed.sys loads of host memory are served
    // one after another: 23.7 us for 20 x 16 B vs 1.3 us for one bulk copy,
    // scripts/micro/hostread.cu).  Every 16-B chunk carries the SQE's stamp
    // (SqeWire) and the host writes each chunk with one aligned 16-B store, so a
    // slot is valid iff its five stamps match -- no second trip is needed.
    uint64_t room = p.sqDepth - (t - minCur);
    if (room > 256 - (t - t0)) room = 256 - (t - t0);
    int nb = room < (uint64_t)B ? (int)room : B;         // (at most 256 SQEs per call)
    const uint32_t first = (uint32_t)(t % p.sqDepth);
    if ((uint32_t)nb > p.sqDepth - first) nb = (int)(p.sqDepth - first);   // no wrap inside one copy
    if (nb <= 0) break;
    mbar_expect_tx(m.sqbar, (uint32_t)nb * (uint32_t)sizeof(SqeWire));
    tma_load(m.sqbuf, p.sq + first, (uint32_t)nb * (uint32_t)sizeof(SqeWire), m.sqbar);
    mbar_wait(m.sqbar, sh.sqPhase);
    sh.sqPhase ^= 1u;
    int valid = 0;
    for (int i = 0; i < nb; ++i) {
      bool ok = valid == i;
      const uint32_t stamp = (uint32_t)(t + i + 1);
#pragma unroll
      for (int q = 0; q < kWireChunks; ++q) ok = ok && m.sqbuf[i].c[q][0] == stamp;
      if (ok) valid = i + 1;
    }
    trace_at(p, *m.tr, b, kEvMark, valid, 2);
    if (!valid) break;
    for (int i = 0; i < valid; ++i) {
      uint32_t words[15];
#pragma unroll
      for (int q = 0; q < kWireChunks; ++q) {
        words[3 * q] = m.sqbuf[i].c[q][1]; words[3 * q + 1] = m.sqbuf[i].c[q][2];
        words[3 * q + 2] = m.sqbuf[i].c[q][3];
      }
      Sqe e;
      sqe_from_words(words, t + i + 1, e);
      const uint4* src = reinterpret_cast<const uint4*>(&e);
      uint4* dst = reinterpret_cast<uint4*>(p.sqMirror + (t + i) % p.sqDepth);
#pragma unroll
      for (int q = 0; q < 4; ++q) st_cg_v4(dst + q, src[q]);
    }
    t += valid;
    trace_at(p, *m.tr, b, kEvMark, valid, 4);
    if (valid < nb) break;
  }
  if (t != t0) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(p.mirrorTail), "l"(t) : "memory");
    fence_sys();                                               // host SQE reads done before the slots are freed
    st_volatile_u64(&p.sqCursorHost[0], t);
    trace_at(p, *m.tr, b, kEvMark, 0, 5);
  }
  asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p.fetchLock), "r"(0u) : "memory");
  return false;
}

// Has every member of the collective's ring admitted submission `lo` of c?  One
// slot per rank on the readiness board (reading R29), read with independent
// relaxed loads -- a hint for the scheduler, not an ordering point.
__device__ __noinline__ bool coll_ready(const DaemonParams& p, const RingDesc& R, int c, uint32_t lo) {
  const int n = R.nranks;
  if (n <= 1) return true;
  const size_t off = (size_t)c * p.G * kFlagStride + kBoardOff;
  for (int q0 = 0; q0 < n; q0 += 8) {
    uint64_t v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = q0 + i < n ? ld_relaxed(R.flagsOf[q0 + i] + off, p.sysScope) : (uint64_t)lo;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if ((int32_t)((uint32_t)v[i] - lo) < 0) return false;
  }
  return true;
}

// The first of the first `lim` queue entries (priority order) that every member
// admitted, or -1.  Entries are checked two at a time: the board loads of
// a pair (up to 2 x 8 ranks) are issued together, so a scan costs one round trip
// per pair, not per entry; an entry once seen ready stays ready for its
// submission (m.ready).
__device__ __noinline__ int ready_scan(const DaemonParams& p, const Smem& m, uint32_t lim) {
  for (uint32_t i0 = 0; i0 < lim; i0 += 2) {
    int rdy[2];
    uint64_t v[2][8];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      rdy[j] = 0;
      const uint32_t i = i0 + j;
      if (i >= lim) continue;
      const int ci = (int)(m.tq[i] & 0xffffu);
      if (m.ready[ci]) { rdy[j] = 1; continue; }
      const RingDesc& R = p.rings[m.subOf[ci]];
      const int n = R.nranks;
      rdy[j] = n <= 8 ? 2 : 3;                       // 2: decide from v[j]; 3: more than 8 members
      const size_t off = (size_t)ci * p.G * kFlagStride + kBoardOff;
#pragma unroll
      for (int q = 0; q < 8; ++q) v[j][q] = q < n ? ld_relaxed(R.flagsOf[q] + off, p.sysScope) : ~0ull;
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const uint32_t i = i0 + j;
      if (i >= lim) break;
      const int ci = (int)(m.tq[i] & 0xffffu);
      if (rdy[j] == 2) {
        bool ok = true;
        const uint32_t lo = m.subLo[ci];
#pragma unroll
        for (int q = 0; q < 8; ++q) ok = ok && (v[j][q] == ~0ull || (int32_t)((uint32_t)v[j][q] - lo) >= 0);
        if (ok) { m.ready[ci] = 1; rdy[j] = 1; }
      } else if (rdy[j] == 3 && coll_ready(p, p.rings[m.subOf[ci]], ci, m.subLo[ci])) {
        m.ready[ci] = 1;
        rdy[j] = 1;
      }
      if (rdy[j] == 1) return (int)i;
    }
  }
  return -1;
}

// One scheduling round: bookkeeping of the previous run, SQ fetch, entry
// selection, voluntary quit.  Returns CMD_*.
__device__ __noinline__ int schedule(const DaemonParams& p, int b, Sched& sh, const Smem& m) {
  const int G = p.G, W = p.cacheWays;
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
      trace_at(p, *m.tr, b, kEvDone, id, 0);
      cx.d.progressed = 0;
      save_dyn(g, cx.d);
      // a one-block collective needs no completion counter: its own fence.sys
      // orders the data (its data warps' stores, acquired through the pipe's
      // mbarriers) before the CQE
      bool last = cx.nblocks == 1;
      if (!last) {
        fence_acq_rel(0);                             // gpu scope: the CQE writer's fence.sys is cumulative
        const uint32_t old = atom_add_acq_rel(&p.complCnt[id], 1u);
        last = old + 1 == cx.nblocks;
      }
      if (last) {
        const long long tq = clock64();
        if (cx.nblocks != 1) p.complCnt[id] = 0;
        fence_sys();                                  // the collective's data before its CQE
        if (p.cqMode == 0) {
          st_volatile_u64(&p.cqDone[id], cx.s.subSeq);  // id slot, single writer (reading R9)
        } else {
          const uint64_t slot = atomicAdd((unsigned long long*)p.cqReserve, 1ull);
          volatile uint64_t* e = p.cqRing + (slot % p.cqDepth);
          if (p.cqMode == 2) {
            // optimized ring: {stamp = slot + 1, id} in ONE 64-bit write; the
            // poller validates the stamp, so no fence and no tail update
            st_volatile_u64(e, ((slot + 1) << 32) | (uint32_t)id);
          } else {
            // vanilla ring: entry, fence, then the tail -- in slot order, so a
            // block waits (host-memory reads) for its predecessors' tail update
            st_volatile_u64(e, (uint64_t)(uint32_t)id);
            fence_sys();
            while (ld_acquire_sys((const void*)p.cqTail) != slot) {}
            asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(p.cqTail), "l"(slot + 1) : "memory");
          }
        }
        sh.cycCqe += clock64() - tq;
        ++sh.nCqe;
        p.blkStats[b].cqes++;
        trace_at(p, *m.tr, b, kEvCqe, id, (uint32_t)cx.s.subSeq);
      }
      for (uint32_t i = sh.pos; i + 1 < sh.qlen; ++i) m.tq[i] = m.tq[i + 1];
      --sh.qlen;
      if (sh.pos >= sh.qlen) sh.pos = 0;
    } else {
      // preempted: lazy save of a dynamic context that progressed
      if (cx.d.progressed) {
        cx.d.progressed = 0;
        const long long t0 = clock64();
        save_dyn(g, cx.d);                           // probe: the paper's 0.05 us save
        sh.cycCtxSave += clock64() - t0;
        ++sh.nCtxSave;
        cs.ctxSaves++;
      }
      cs.preemptions++;
      trace_at(p, *m.tr, b, kEvPreempt, id, sh.pos);
      uint32_t st = m.tq[sh.pos] >> 16;
      if (st < 0xffff) ++st;
      m.tq[sh.pos] = (m.tq[sh.pos] & 0xffffu) | (st << 16);
      if (p.orderPolicy == 1 && sh.qlen > 1) {
        // priority order (reading R10): the traversal interleaves the queue front
        // with the other entries (0, r1, 0, r2, ...) -- fair, but the highest-
        // priority collective is retried every other switch, so ranks re-converge
        // on the same front quickly after a straggler shows up
        if (sh.pos != 0) {
          sh.pos = 0;
        } else {
          if (sh.rr == 0 || sh.rr >= sh.qlen) sh.rr = 1;
          sh.pos = sh.rr++;
        }
      } else {
        sh.pos = (sh.pos + 1) % sh.qlen;
      }
    }
    sh.lastRun = -1;
  }
  ++sh.iter;
  const uint64_t now = globaltimer();
  const uint32_t qlen = sh.qlen;
  bool allStalled = qlen > 0;
  for (uint32_t i = 0; i < qlen && allStalled; ++i) allStalled = (m.tq[i] >> 16) >= p.stallLimit;
  // reading R3, time-based variant: "cannot progress for a long time" = no queued
  // entry committed a slice for stallNs (and the current front was preempted)
  if (!allStalled && qlen > 0 && p.stallNs && (m.tq[sh.pos] >> 16) > 0 && now - sh.lastProgress > p.stallNs)
    allStalled = true;
  // -- fetch an SQE, gated by the order policy
  const bool canFetch = !sh.exiting && qlen < (uint32_t)p.maxColl &&
                        (qlen == 0 || (p.orderPolicy == 0 ? allStalled : (sh.iter % (uint64_t)p.priorityCadence) == 0));
  if (canFetch) {
    // FIFO fetches one SQE; the priority policy drains what is
    // there ("checking the SQ more frequently") so that every rank
    // sorts the same set of collectives as early as possible
    const int burst = p.orderPolicy == 0 ? 1 : 32;
    bool fetched = false;
    uint64_t tail = ld_acquire(p.mirrorTail, 0);
    if (tail <= sh.cursor) {
      // The host SQ itself (a PCIe round trip under the rank's fetch lock) is
      // polled at once by an idle block, but by a block with queued work at most
      // once per sqYieldNs per rank: otherwise a block about to run a collective
      // it just admitted would first wait for a PCIe round trip.  (sqYieldNs = 0:
      // no rate limit.)  Liveness: some block of the rank polls within sqYieldNs.
      bool poll = qlen == 0 || p.sqYieldNs == 0 || sh.needHostPoll;
      if (!poll) {
        unsigned long long* lastHost = reinterpret_cast<unsigned long long*>(p.mirrorTail + 3);
        const unsigned long long lh = *reinterpret_cast<volatile unsigned long long*>(lastHost);
        poll = now - lh > p.sqYieldNs && atomicCAS(lastHost, lh, (unsigned long long)now) == lh;
      }
      if (poll) {
        sh.needHostPoll = 0;
        sq_fetch(p, m, sh, b);                           // one block at a time copies host SQEs to the mirror
        tail = ld_acquire(p.mirrorTail, 0);
      }
    }
    for (int k = 0; k < burst && !sh.exiting && sh.qlen < (uint32_t)p.maxColl && sh.cursor < tail; ++k) {
      // the SQE from the device-memory mirror (L2), 4 independent 16-B loads
      const uint4* src = reinterpret_cast<const uint4*>(p.sqMirror + (sh.cursor % p.sqDepth));
      uint4 w[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) w[q] = ld_cg(src + q);
      Sqe e;
      memcpy(&e, w, sizeof(Sqe));
      ++sh.cursor;
      // release: the mirror slot's loads are done before the fetcher may reuse it
      asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(&p.blk[b].sqCursor), "l"(sh.cursor) : "memory");
      sh.lastFetch = now;
      fetched = true;
      if (e.kind == kExit) {
        sh.exiting = 1;                              // Exiting SQE
      } else {
        // the collective's blocks start at lane 0 = block (collId mod G), so that
        // independent small collectives run on different SMs; participate iff
        // lane < grid size (reading Q11)
        const int lane = (b - (int)(e.collId % (uint32_t)p.G) + p.G) % p.G;
        if (lane < (int)e.nblocks) admit(p, b, lane, sh, m, e);
      }
    }
    if (fetched) return CMD_NONE;
  }
  // Readiness scan (reading R29, priority policy): the highest-priority entry
  // among the first kReadyScan that EVERY member rank admitted.  With
  // readyFirst = 2 and the whole queue inside the scan window, a queue with no
  // ready entry is not run at all -- none of its collectives can complete -- and
  // the block waits like an idle one (and counts as stuck for the quit vote);
  // with readyFirst = 1 its entries are visited for spinMin each.
  int readyPick = -1;
  bool waitReady = false;
  if (qlen > 0 && p.orderPolicy == 1 && p.readyFirst) {
    // (a round trip per pair of not-yet-ready entries; tried alternatives -- 8
    // entries, 8 every round + 64 every 4th -- completed the live workloads within
    // noise of this and preempted up to 36x more, profiles/r02/live_ab_scan_m20)
    const uint32_t lim = qlen < (uint32_t)kReadyScan ? qlen : (uint32_t)kReadyScan;
    readyPick = ready_scan(p, m, lim);
    waitReady = readyPick < 0 && p.readyFirst >= 2 && lim >= qlen;
  }
  const bool stuck = qlen == 0 || allStalled || waitReady;
  // Voluntary quit is decided for the whole launch: a block
  // that has been stuck or idle for quitIdleNs only VOTES; the launch quits once
  // every block voted (a block gone alone would strand the SQEs of its lanes --
  // and cap the SQ mirror with its stale cursor -- until its siblings quit too).
  // quitWord = votes | kQuitLatch; the latch is set by a CAS from exactly
  // quitTotal votes, and a vote is withdrawn only by a CAS that sees no latch,
  // so once latched every block leaves.  A block that consumed the Exiting SQE
  // keeps its vote.
  bool quitNow = false;
  if (p.quitEnabled && !(qlen == 0 && sh.exiting)) {
    const bool eligible = stuck && now - sh.lastFetch > p.quitIdleNs;
    if (eligible && !sh.voted) {
      atomicAdd(p.quitWord, 1u);
      sh.voted = 1;
    } else if (!eligible && sh.voted) {
      uint32_t w = *(volatile uint32_t*)p.quitWord;
      for (;;) {
        if (w & kQuitLatch) { quitNow = true; break; }
        const uint32_t o = atomicCAS(p.quitWord, w, w - 1);
        if (o == w) { sh.voted = 0; break; }
        w = o;
      }
    }
    if (sh.voted && !quitNow) {
      const uint32_t w = *(volatile uint32_t*)p.quitWord;
      quitNow = (w & kQuitLatch) ||
                (w == p.quitTotal && atomicCAS(p.quitWord, w, w | kQuitLatch) == w);
    }
  }
  if (qlen == 0 && sh.exiting) {
    sh.exiting = 0;
    if (!sh.voted && p.quitWord) atomicAdd(p.quitWord, 1u);
    sh.voted = 1;
    p.blkStats[b].exits++;
    trace_at(p, *m.tr, b, kEvExit, 0, 0);
    cmd = CMD_EXIT;
  } else if (quitNow) {
    p.blkStats[b].quits++;                           // voluntary quit
    trace_at(p, *m.tr, b, kEvQuit, 0, 0);
    cmd = CMD_EXIT;
  } else if (qlen > 0 && !waitReady) {
    // Priority policy with the readiness board (reading R29): the ready entry of
    // the scan runs, with the full (boostable) threshold -- all ranks converge on
    // it.  If none is ready, the traversal position of R10 is kept and the entry
    // waits at most spinMin: a collective some rank has not even admitted cannot
    // complete.
    bool ready = true;
    if (p.orderPolicy == 1 && p.readyFirst) {
      if (readyPick >= 0) sh.pos = (uint32_t)readyPick;
      else ready = false;
    }
    // only the front -- and with the board only a front every member admitted --
    // is boosted and gets the full threshold; any other pick waits at most spinMin
    // (a boosted non-front pick held its rank for up to spinCap while a higher-
    // priority collective became ready elsewhere: live runs 2-3x slower)
    sh.boostOk = p.orderPolicy == 1 ? (sh.pos == 0 && (!p.readyFirst || ready)) : 1;
    const int c = (int)(m.tq[sh.pos] & 0xffffu);
    const int way = c % W;
    sh.way = way;
    if (m.cacheTag[way] != c) {
      // context load into the shared-memory cache: 8 independent 16-B loads in
      // flight
      m.cacheTag[way] = c;
      const long long t0 = clock64();
      const uint4* gsrc = reinterpret_cast<const uint4*>(&p.ctx[(size_t)c * G + b]);
      uint4 v[kCtxBytes / 16];
#pragma unroll
      for (int i = 0; i < kCtxBytes / 16; ++i) v[i] = ld_cg(gsrc + i);
      uint4* dst = reinterpret_cast<uint4*>(&m.cache[way]);
#pragma unroll
      for (int i = 0; i < kCtxBytes / 16; ++i) dst[i] = v[i];
      sh.cycCtxLoad += clock64() - t0;                 // probe: the paper's 0.45 us load
      ++sh.nCtxLoad;
      p.collStats[(size_t)c * G + b].ctxLoads++;
    }
    sh.curId = c;
    // initial spin threshold from the queue position.  Under
    // the priority policy (reading R10) the front is where every rank converges;
    // a lower-priority entry is visited only for as long as it progresses
    // (spinMin of waiting), so a rank does not hold a peer-less entry while the
    // others arrive at the front
    if (p.stickiness && p.orderPolicy == 1 && !sh.boostOk) {
      sh.T = p.spinMin;
    } else if (p.stickiness && p.orderPolicy == 1) {
      sh.T = p.spinBase;                              // the front / the first ready entry
    } else if (p.stickiness) {
      const uint64_t dec = (uint64_t)sh.pos * p.spinStep;
      uint64_t T = dec >= p.spinBase ? p.spinMin : p.spinBase - dec;
      sh.T = T < p.spinMin ? p.spinMin : T;
    } else {
      sh.T = p.spinBase;
    }
    cmd = CMD_RUN;
  } else {
    ++sh.idlePolls;                                  // (a global ++ here cost an L2 round trip per idle round)
    if (p.idleSleepNs) __nanosleep(p.idleSleepNs);
  }
  if (cmd == CMD_EXIT) {                             // persist what survives the quit
    BlockState bs;
    bs.sqCursor = sh.cursor; bs.qlen = sh.qlen; bs.pos = sh.pos; bs.exiting = sh.exiting; bs.pad = 0;
    p.blk[b] = bs;
    for (uint32_t i = 0; i < sh.qlen; ++i) p.tqSave[(size_t)b * p.maxColl + i] = m.tq[i];
  }
  return cmd;
}


// Cursor of one collective on one block: (loop, step, slice) + connector counts.
struct Cursor {
  uint32_t loop, step, slc;
  uint64_t nsent, nrecv;
};

__device__ __forceinline__ void advance(Cursor& d, int prim, int slicesPerChunk, int nsteps) {
  if (prim & A_SEND) d.nsent++;
  if (prim & A_RECV) d.nrecv++;
  if (++d.slc == (uint32_t)slicesPerChunk) {
    d.slc = 0;
    if (++d.step == (uint32_t)nsteps) { d.step = 0; d.loop++; }
  }
}

// (defined after the data-warp roles: the LL-run code sits after every hot
// loop of the bandwidth path, whose layout it would otherwise shift)
__device__ __noinline__ int ll_run_control(const DaemonParams& p, int b, Sched& sh, const Smem& m, Pipe& pipe,
                                           uint32_t& issued, uint32_t& committed, Cursor& dc, uint64_t& T,
                                           unsigned long long& nSlices);

// Run the collective at the front of the scheduler until it is done or preempted.
// Everything hot lives in registers of the control thread: the static context,
// the issue cursor `di` (runs ahead) and the committed cursor `dc`.
//   issue : one poll of the connectors for the next slice (a failed poll is one
//           "spin"); polls are acquire loads, and a cached
//           head/credit value needs no new poll -- the acquire that observed it
//           already ordered the peer's data before us.
//   commit: all slices the data warps finished, in order, under ONE release
//           fence; then the head (downstream) / credit (upstream) counters are
//           published once (commit visibility).
__device__ __forceinline__ int run_collective(const DaemonParams& p, int b, Sched& sh, const Smem& m, Pipe& pipe,
                                              uint32_t& issued, uint32_t& committed) {
  const uint32_t D = (uint32_t)p.pipeDepth;
  CtxSlot& cx = m.cache[sh.way];
  const RingDesc& R = p.rings[cx.sub];                   // the collective's own ring
  const int n = R.nranks, r = R.rank, K = p.K, sys = p.sysScope, spc = (int)cx.spc;
  // ---- static context -> registers
  const uint64_t sendbuff = cx.s.sendbuff, recvbuff = cx.s.recvbuff, count = cx.s.count;
  const uint64_t segLen = cx.s.segLen, part = cx.s.part;
  const int kind = cx.d.kind, dtype = cx.d.dtype, root = cx.root, nsteps = cx.nsteps;
  const uint32_t nloops = cx.d.nloops;
  const bool inplace = sendbuff == recvbuff;
  const int isz = elem_size(dtype);
  const bool ll = cx.proto != 0;
  const uint64_t E = (ll ? p.llSliceBytes : p.sliceBytes) / isz;
  const size_t cb = (size_t)sh.curId * p.G + b;
  const uint64_t llSlot = 2ull * p.llSliceBytes;                  // bytes of one LL slot (16-B lines)
  const char* llIn = p.llLocal + cb * K * llSlot;
  char* llOut = R.llNext + cb * K * llSlot;
  const char* headIn = p.flagsLocal + cb * kFlagStride;
  const char* creditIn = headIn + 128;
  char* headOut = R.flagsNext + cb * kFlagStride;
  char* creditOut = R.flagsPrev + cb * kFlagStride + 128;
  char* connIn = p.dataLocal + cb * K * p.sliceBytes;
  char* connOut = R.dataNext + cb * K * p.sliceBytes;
  const char* directIn = p.flagsLocal + cb * kFlagStride + kDirectOff;   // {peer recvbuff, subSeq}
  const bool dOut = R.directNext != 0 && !ll, dIn = R.directPrev != 0 && !ll;
  // LL speculation: recv slices go to the data warps before their lines arrived
  // (the warps poll the lines themselves); a run whose oldest issued slice does
  // not complete within the spin threshold aborts its speculative slices
  const bool spec = ll && p.llSpeculate == 1;
  uint64_t specSince = 0;
  const bool dRead = p.directRead != 0;
  const bool keepOut = p.l2Hints >= 3;
  const char* srcIn = p.flagsLocal + cb * kFlagStride + kDirectOff + 16;  // {upstream sendbuff, subSeq}
  // Read-done acknowledgement of direct read (reduce-scatter).  An RS rank's own
  // completion does not depend on its downstream's progress: when its last
  // loop's sends fit in the connector ((n-2) * spc <= K) it could post its CQE
  // -- and its caller rewrite the send buffer or resubmit the id -- while the
  // downstream has not yet read that buffer.  So the downstream raises `ack` in
  // our flag line (+32) to the submission number once it committed its last
  // direct-read slice, and we hold RUN_DONE until then (a failed ack poll is a
  // spin: preemptible like any connector wait).  An all-reduce needs no ack:
  // its final Recv carries data the downstream produced after its direct read.
  // (the ack addresses are recomputed where used: keeping them live costs the
  // control thread registers it spills in its hot loop)
  const bool dreadUp = dRead && dOut && n > 1 && kind == kReduceScatter;     // downstream reads our buffer
  const bool dreadDown = dRead && dIn && n > 1 && kind == kReduceScatter;    // we read our upstream's
  uint64_t peerSrc = 0;                                   // upstream's send buffer (direct read)
  const uint64_t subSeq = cx.s.subSeq;
  uint64_t peerRecv = 0;                                  // downstream's recv buffer (direct sends)
  bool prepared = false;                                  // pipe.ring[issued % D] holds the next slice
  const char* llLast = nullptr;                           // LL: last line of the next slice's input
  int curPrim = 0;
  uint64_t doutOff = 0, dreadOff = 0;
  // ---- dynamic context -> registers
  Cursor dc{cx.d.loop, cx.d.step, cx.d.slc, cx.d.nsent, cx.d.nrecv};
  Cursor di = dc;
  const uint64_t laneLo = (uint64_t)cx.lane * part;
  uint64_t headSeen = 0, creditSeen = 0;
  // spins are counted in time: T x spinNs of failed polling (R1) --
  // an LL poll (a 16-B line in L2) and a cached head poll differ 10x in cost
  uint64_t T = sh.T, spinStart = 0;
  const uint64_t spinNs = p.spinNs;
  unsigned long long nSlices = 0, cPoll = 0;
  uint32_t nFailed = 0;
  const long long tRun = clock64();
  trace_at(p, *m.tr, b, kEvSwitchIn, sh.curId, sh.pos);
  // commit one slice the data warps finished (in order); the downstream side of
  // a reduce-scatter direct read acknowledges its last direct-read slice
  auto commit = [&](uint32_t slot) {
    const int cp = pipe.ring[slot].prim;
    if (dreadDown && (cp & A_DREAD) && dc.loop + 1 == nloops && dc.slc + 1 == (uint32_t)spc) {
      char* ackOut = p.rings[cx.sub].flagsPrev + cb * kFlagStride + kDirectOff + 32;
      if (sys) asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(ackOut), "l"(subSeq) : "memory");
      else asm volatile("st.release.gpu.global.u64 [%0], %1;" :: "l"(ackOut), "l"(subSeq) : "memory");
    }
    advance(dc, cp, spc, nsteps);
  };
  // drain the pipe before leaving the run: every issued slice completes (its
  // connectors were ready) -- except, with LL speculation, slices whose lines have
  // not come: the abort makes their warps give up, and only the prefix of slices
  // that completed before the first given-up one is committed
  auto drain = [&]() {
    if (spec) *reinterpret_cast<volatile uint32_t*>(&pipe.abortGen) = pipe.abortGen + 1;
    bool failed = false;
    while (committed != issued) {
      const uint32_t slot = committed % D;
      mbar_wait(&pipe.empty[slot], (committed / D) & 1);
      if (spec) {
        if (*reinterpret_cast<volatile uint32_t*>(&pipe.fail[slot])) failed = true;
        pipe.fail[slot] = 0;
      }
      if (!failed) {
        commit(slot);
        ++nSlices;
      }
      ++committed;
    }
  };
  int run;
  // LL runs for the latency-bound shape: one slice per ring step (a block whose
  // part is one LL slice -- the LL spread of occl_host.cc gives every small
  // collective that shape).  Longer LL schedules keep the per-slice path, whose
  // pipe overlaps the next slice's poll with the current slice's move (an LL
  // run moves its slices strictly one after another: 1 MiB AR 164 vs 126 us).
  if (ll && p.llSpeculate == 2 && spc == 1 && nloops == 1) {
    run = ll_run_control(p, b, sh, m, pipe, issued, committed, dc, T, nSlices);
  } else
  for (;;) {
    // ---- slices the data warps moved and published: advance the committed cursor
    if (committed != issued && mbar_test(&pipe.empty[committed % D], (committed / D) & 1)) {
      do {
        commit(committed % D);
        ++committed;
        ++nSlices;
      } while (committed != issued && mbar_test(&pipe.empty[committed % D], (committed / D) & 1));
      // raise the threshold.  Priority policy (reading R10): only
      // the queue front -- the collective every rank converges on -- is boosted;
      // a visit to a lower-priority entry keeps its short position threshold, so
      // progress a pair of neighbours makes on it (up to K slices) does not make
      // a rank stick to it for up to spinCap while the others wait at the front
      if (p.stickiness && sh.boostOk) {
        T *= p.spinBoost;
        if (T > p.spinCap) T = p.spinCap;
      }
      m.tq[sh.pos] &= 0xffffu;                            // progressed: not stalled
      specSince = 0;
    }
    if (spec && committed != issued) {                    // speculative slices outstanding
      const uint64_t now = globaltimer();
      if (specSince == 0) {
        specSince = now;
      } else if (now - specSince > T * spinNs) {          // the upstream is not there: preempt
        drain();
        run = RUN_PREEMPT;
        break;
      }
    }
    if (di.loop >= nloops) {                              // everything issued
      if (committed != issued) continue;
      if (!dreadUp || ld_acquire(p.flagsLocal + cb * kFlagStride + kDirectOff + 32, sys) == subSeq) {
        run = RUN_DONE;
        break;
      }
      // the downstream has not finished reading our send buffer: a failed poll
      const uint64_t now = globaltimer();
      if (spinStart == 0) spinStart = now;
      if (now - spinStart > T * spinNs) { run = RUN_PREEMPT; break; }   // pipe already drained
      continue;
    }
    if (issued - committed == D) continue;                // every buffer busy
    // ---- prepare the next slice's descriptor BEFORE its connectors are ready,
    // so that publishing it is a single mbarrier arrive once they are
    SliceDesc& sd = pipe.ring[issued % D];
    if (!prepared) {
      int seg;
      step_prim(kind, n, r, root, di.step, inplace, curPrim, seg);
      curPrim = directify(curPrim, kind, n, di.step, dOut, dIn, dRead);
      if (keepOut && (curPrim & A_DOUT) && downstream_forwards(kind, n, r, root, di.step)) curPrim |= A_KEEPOUT;
      uint64_t sendOff, recvOff, len;
      seg_geom(kind, n, r, count, segLen, seg, sendOff, recvOff, len);
      uint64_t laneHi = laneLo + part;
      if (laneHi > len) laneHi = len;
      const uint64_t lo = laneLo + ((uint64_t)di.loop * spc + di.slc) * E;
      uint64_t hi = lo + E;
      if (hi > laneHi) hi = laneHi;
      doutOff = (recvOff + lo) * isz;
      dreadOff = (sendOff + lo) * isz;
      sd.src = reinterpret_cast<const char*>(sendbuff) + (sendOff + lo) * isz;
      sd.dst = reinterpret_cast<char*>(recvbuff) + doutOff;
      sd.nelem = hi > lo ? (int64_t)(hi - lo) : 0;
      if (ll) {
        curPrim |= A_LL;
        sd.cin = llIn + (di.nrecv % K) * llSlot;
        sd.cout = llOut + (di.nsent % K) * llSlot;
        // the receiver polls the slice's last line (every message has >= 1 line)
        const uint64_t lines = ((uint64_t)sd.nelem * isz + 7) / 8;
        llLast = sd.cin + 16 * ((lines ? lines : 1) - 1);
      } else {
        sd.cin = (curPrim & A_DIN) ? sd.dst : connIn + (di.nrecv % K) * p.sliceBytes;
        sd.cout = connOut + (di.nsent % K) * p.sliceBytes;   // direct sends: set once the peer is known
      }
      sd.prim = curPrim;
      sd.dtype = dtype;
      sd.op = (int)cx.op;
      sd.headOut = headOut;
      sd.creditOut = creditOut;
      sd.headVal = di.nsent + 1;
      sd.creditVal = di.nrecv + 1;
      prepared = true;
    }
    const int prim = curPrim;
    // ---- issue it if its connectors are ready
    const bool needRecv = prim & A_RECV, needSend = prim & A_SEND;
    bool ok = true;
    const long long tp = clock64();
    if (needRecv && (prim & A_LL) && !spec) {
      // LL: the data carries its own flags -- the last line of the slice holds
      // the message sequence number once the upstream wrote it
      uint32_t f0, f1;
      asm volatile("{\n .reg .u32 a, c;\n ld.volatile.global.v4.u32 {a, %0, c, %1}, [%2];\n}"
                   : "=r"(f0), "=r"(f1) : "l"(llLast) : "memory");
      ok = f0 == (uint32_t)(di.nrecv + 1) && f1 == (uint32_t)(di.nrecv + 1);
    } else if (needRecv && di.nrecv >= headSeen) {
      headSeen = ld_acquire(headIn, sys);
      ok = di.nrecv < headSeen;
    }
    if (ok && needSend && di.nsent - creditSeen >= (uint64_t)K) {
      creditSeen = ld_acquire(creditIn, sys);
      ok = di.nsent - creditSeen < (uint64_t)K;
    }
    if (ok && (prim & A_DREAD) && peerSrc == 0) {         // the upstream admitted this submission?
      if (ld_acquire(srcIn + 8, sys) == subSeq) peerSrc = ld_relaxed(srcIn, sys);
      ok = peerSrc != 0;
    }
    if (ok && (prim & A_DOUT) && peerRecv == 0) {         // the downstream admitted this submission?
      if (ld_acquire(directIn + 8, sys) == subSeq) peerRecv = ld_relaxed(directIn, sys);
      ok = peerRecv != 0;
    }
    if (!ok) {
      cPoll += clock64() - tp;
      const uint64_t now = globaltimer();
      if (spinStart == 0) {
        spinStart = now;
        trace_at(p, *m.tr, b, kEvMark, sh.curId, 30);     // first failed poll of this slice
      }
      ++nFailed;
      // Priority policy, "checking the SQ more frequently": a
      // collective blocked for longer than the minimal threshold yields as soon
      // as new SQEs are there, so the scheduler admits and sorts them before any
      // entry runs again.  A blocked control thread looks at the device mirror
      // (an L2 read) every kSqPollNs; the host SQ itself is peeked (ONE 16-B
      // PCIe load: the stamp of the next unfetched slot) by at most one blocked
      // block of the rank per sqYieldNs -- otherwise no block of a rank whose
      // collectives all wait would see new SQEs.  The scheduler fetches them
      // after the yield.  No call here: a call in this loop makes the control
      // thread spill its live state around it (measured -27 % bench busbw).
      bool yieldSq = false;
      if (p.orderPolicy == 1 && p.sqYieldNs && now - spinStart > (uint64_t)p.spinMin * spinNs &&
          now - sh.lastSqPoll > kSqPollNs) {
        sh.lastSqPoll = now;
        const uint64_t tail = ld_acquire(p.mirrorTail, 0);
        if (tail > sh.cursor) {
          yieldSq = true;
        } else {
          unsigned long long* lastHost = reinterpret_cast<unsigned long long*>(p.mirrorTail + 3);
          const unsigned long long lh = *reinterpret_cast<volatile unsigned long long*>(lastHost);
          if (now - lh > p.sqYieldNs && atomicCAS(lastHost, lh, (unsigned long long)now) == lh) {
            uint32_t stamp;
            asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(stamp) : "l"(p.sq[tail % p.sqDepth].c[0])
                         : "memory");
            yieldSq = stamp == (uint32_t)(tail + 1);
            // the scheduler must fetch it now: its own host polls are rate
            // limited by the clock this peek just restarted
            if (yieldSq) sh.needHostPoll = 1;
          }
        }
      }
      if (yieldSq || now - spinStart > T * spinNs) {     // two-phase blocking: preempt
        drain();
        run = RUN_PREEMPT;                                // the prepared descriptor is dropped
        break;
      }
      continue;
    }
    if (nFailed) {
      trace_at(p, *m.tr, b, kEvMark, nFailed > 0xffff ? 0xffff : (int)nFailed, 31);   // failed polls of this slice
      nFailed = 0;
    }
    spinStart = 0;
    if (prim & A_DOUT) sd.cout = reinterpret_cast<char*>(peerRecv) + doutOff;
    if (prim & A_DREAD) sd.cin = reinterpret_cast<const char*>(peerSrc) + dreadOff;   // same layout as ours
    sd.gen = pipe.abortGen;
    mbar_arrive(&pipe.full[issued % D]);
    trace_at(p, *m.tr, b, kEvIssue, sh.curId,
          (uint32_t)(di.nsent & 0x3fff) | ((uint32_t)(di.nrecv & 0x3fff) << 14) | ((uint32_t)(prim & 0xf) << 28));
    ++issued;
    prepared = false;
    advance(di, prim, spc, nsteps);
  }
  // ---- registers -> dynamic context in the shared-memory cache
  if (nSlices) cx.d.progressed = 1;
  cx.d.loop = dc.loop; cx.d.step = (uint16_t)dc.step; cx.d.slc = (uint16_t)dc.slc;
  cx.d.nsent = dc.nsent; cx.d.nrecv = dc.nrecv;
  sh.T = T;
  if (nSlices) sh.lastProgress = globaltimer();
  sh.cycRun += clock64() - tRun;
  sh.cycPoll += cPoll;
  sh.nCommit += nSlices;
  p.collStats[cb].slices += nSlices;
  return run;
}

// The control thread (lane 0 of warp 0): scheduler + connector protocol.  Feeds
// slice descriptors to the data warps through the pipe, `pipeDepth` in flight.
__device__ __noinline__ void control_main(const DaemonParams& p, int b, Sched& sh, const Smem& m, Pipe& pipe) {
  const uint32_t D = (uint32_t)p.pipeDepth;
  uint32_t issued = 0, committed = 0;               // kernel-lifetime slice counters
  trace_at(p, *m.tr, b, kEvStart, 0, (uint32_t)sh.cursor);
  for (;;) {
    const int cmd = schedule(p, b, sh, m);
    if (cmd == CMD_NONE) continue;
    if (cmd == CMD_EXIT) break;
    sh.lastRun = run_collective(p, b, sh, m, pipe, issued, committed);
  }
  BlockStat& bst = p.blkStats[b];
  bst.cycRun += sh.cycRun;
  bst.cycPoll += sh.cycPoll;
  bst.cycAcqFence += sh.cycAcqFence;
  bst.nCommit += sh.nCommit;
  bst.cycCtxLoad += sh.cycCtxLoad;
  bst.nCtxLoad += sh.nCtxLoad;
  bst.cycCtxSave += sh.cycCtxSave;
  bst.nCtxSave += sh.nCtxSave;
  bst.cycCqe += sh.cycCqe;
  bst.nCqe += sh.nCqe;
  bst.idlePolls += sh.idlePolls;
  // release the data warps (the pipe is drained after every run)
  pipe.ring[issued % D].prim = P_EXIT;
  mbar_arrive(&pipe.full[issued % D]);
}

// ------------------------------------------------------------------ TMA staging
// Same with an L2 cache-eviction policy (user buffers are streamed exactly once:
// evict-first keeps the connector lines, which are re-read, resident in L2).
__device__ __forceinline__ void tma_load_hint(void* smemDst, const void* gsrc, uint32_t bytes, uint64_t* bar,
                                              uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               :: "r"(smem_u32(smemDst)), "l"(gsrc), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st_cg_hint(void* p, const uint4& v, uint64_t pol) {
  asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}
// Bulk (TMA) store shared -> global, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_store(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_store_hint(void* gdst, const void* ssrc, uint32_t bytes, uint64_t pol) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;"
               :: "l"(gdst), "r"(smem_u32(ssrc)), "r"(bytes), "l"(pol) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Invalidate a consumed connector line in L2 without writing it back: the slot
// is rewritten by the upstream before anyone reads it again (PTX `discard`
// behaves like a weak write, so the credit's release orders it before the
// upstream's next write into the slot).
__device__ __forceinline__ void discard_l2_line(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" :: "l"(p) : "memory");
}
// Demote a line the upstream stored evict-last (l2Hints == 3) once it is read:
// the final data stays cached only as long as the next hop needs it.
__device__ __forceinline__ void demote_l2_line(const void* p) {
  asm volatile("applypriority.global.L2::evict_normal [%0], 128;" :: "l"(p) : "memory");
}
__device__ __forceinline__ uint4 lds_v4(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// A slice goes through the TMA staging ring when its vector part is 16-B aligned
// (connector slots always are; user buffers almost always).  Otherwise the
// compute warps move it with register loads (move_slice).
__device__ __forceinline__ int tma_vec_bytes(int dtype, int64_t nelem, const char* src, const char* dst,
                                             const char* cout, const char* cin) {
  const int isz = elem_size(dtype);
  if (nelem <= 0) return 0;
  // cout / cin may be peer buffers (direct send / direct read)
  if ((((uintptr_t)src) | ((uintptr_t)dst) | ((uintptr_t)cout) | ((uintptr_t)cin)) & 15) return 0;
  const int vb = (int)((nelem * isz) & ~(int64_t)15);
  return vb >= kTmaMinBytes ? vb : 0;          // small slices: lower-latency register path
}

struct Stage {                 // one staging slot: the incoming operand and the local operand
  uint4 in[kTile / 16];
  uint4 loc[kTile / 16];
};

// Producer lane (warp 1 lane 0): streams every slice's operands into the staging
// ring with cp.async.bulk, p.stages tiles ahead of the compute warps.
__device__ __noinline__ void producer_main(const DaemonParams& p, Pipe& pipe, Stage* st, uint64_t* tfull,
                                           uint64_t* tempty) {
  const uint32_t D = (uint32_t)p.pipeDepth, S = (uint32_t)p.stages;
  const bool hints = p.l2Hints != 0;
  const uint64_t pol = policy_evict_first();
  uint32_t cs = 0, cph = 0;                          // staging slot and its phase parity
  for (uint32_t j = 0;; ++j) {
    mbar_wait(&pipe.full[j % D], (j / D) & 1);
    const SliceDesc sd = pipe.ring[j % D];
    if (sd.prim == P_EXIT) break;
    // the descriptor is copied: the control thread may reuse its buffer.  Slices
    // the producer does not stage (LL, register path, direct final receive) can
    // complete without it, so without this arrive the control thread could
    // rewrite ring[j % D] before this lane has read it
    mbar_arrive(&pipe.empty[j % D]);
    if (!(sd.prim & (A_COPY | A_SEND))) continue;     // direct final receive: data already in place
    if (sd.prim & A_LL) continue;                     // LL slices are moved by the compute warps alone
    const int vb = tma_vec_bytes(sd.dtype, sd.nelem, sd.src, sd.dst, sd.cout, sd.cin);
    if (vb == 0) continue;
    // order the acquire of the peer's head (generic proxy) before the bulk reads (async proxy)
    asm volatile("fence.proxy.async.global;" ::: "memory");
    const bool recv = sd.prim & (A_RECV | A_DREAD), reduce = sd.prim & A_REDUCE;
    const char* in = recv ? sd.cin : sd.src;
    for (int off = 0; off < vb; off += kTile) {
      const uint32_t s = cs;
      mbar_wait(&tempty[s], cph ^ 1);
      if (++cs == S) { cs = 0; cph ^= 1; }
      const uint32_t sz = (uint32_t)min(kTile, vb - off);
      mbar_expect_tx(&tfull[s], reduce ? 2 * sz : sz);
      if (recv || !hints) tma_load(st[s].in, in + off, sz, &tfull[s]);
      else tma_load_hint(st[s].in, in + off, sz, &tfull[s], pol);
      if (reduce) {
        if (hints) tma_load_hint(st[s].loc, sd.src + off, sz, &tfull[s], pol);
        else tma_load(st[s].loc, sd.src + off, sz, &tfull[s]);
      }
    }
  }
}

// Compute warps: reduce / copy the staged tiles into the recv buffer and the
// downstream connector with 128-bit stores.  L2 policies by l2Hints (l2):
//   own recv buffer (final data, not re-read)     : l2 >= 1 evict-first
//   downstream connector (read once, then discarded): l2 >= 2 evict-last, so the
//                                                     streamed user buffers leave L2 first
//   direct send into the downstream's recv buffer : l2 >= 3 evict-last when the
//     downstream forwards it at its next hop (A_KEEPOUT; it demotes the lines to
//     normal once read), evict-first on the last hop
template <int DT, int OP>
__device__ __forceinline__ void consume_tile(const int prim, char* dst, char* cout, const Stage& s, int sz, int tid,
                                             int nt, int l2, uint64_t polFirst, uint64_t polLast) {
  const bool reduce = prim & A_REDUCE, copy = prim & A_COPY, send = prim & A_SEND;
  // 0 plain, 1 evict-first, 2 evict-last
  const int sendPol = !(prim & A_DOUT) ? (l2 >= 2 ? 2 : 0) : (l2 >= 3 ? ((prim & A_KEEPOUT) ? 2 : 1) : 0);
  const uint64_t sp = sendPol == 2 ? polLast : polFirst;
  uint4* vd = reinterpret_cast<uint4*>(dst);
  uint4* vo = reinterpret_cast<uint4*>(cout);
  const int nv = sz >> 4;
  for (int i = tid; i < nv; i += nt) {
    uint4 v = lds_v4(&s.in[i]);
    if (reduce) v = vop<DT, OP>(v, lds_v4(&s.loc[i]));
    if (copy) {
      if (l2 >= 1) st_cg_hint(vd + i, v, polFirst);
      else __stcg(vd + i, v);
    }
    if (send) {
      if (sendPol) st_cg_hint(vo + i, v, sp);
      else __stcg(vo + i, v);
    }
  }
}

// LL slice (NCCL's low-latency protocol idea, re-done for the daemon): every
// 16-B line carries 8 B of payload and the message sequence number twice,
// written with one 16-B store, so the receiver needs no head flag and the
// sender no release fence -- a line is valid once both flags match.  Used for
// latency-bound collectives (small per-block parts).  Payload = the slice's
// elements packed 8 B per line; reduction per element as in the Simple path.
template <int DT, int OP>
__device__ __forceinline__ void ll_slice(const int prim, const char* src, const char* cin, char* dst, char* cout,
                                         const int64_t nelem, const uint32_t inSeq, const uint32_t outSeq,
                                         const int tid, const int nt, const volatile uint32_t* abortGen,
                                         const uint32_t gen, bool& ok, uint64_t* tLine) {
  // tLine (tracing only): [0] this thread's first line in, [1] its store of the
  // slice's last line
  typedef typename Elem<DT>::T T;
  constexpr int PER = 8 / sizeof(T);                 // elements per line
  const bool recv = prim & A_RECV, reduce = prim & A_REDUCE, copy = prim & A_COPY, send = prim & A_SEND;
  const int64_t lines = (nelem + PER - 1) / PER;
  const int64_t nl = lines ? lines : 1;              // an empty message still carries one token line
  const T* s = reinterpret_cast<const T*>(src);
  T* d = reinterpret_cast<T*>(dst);
  for (int64_t l = tid; l < nl; l += nt) {
    union { uint32_t w[2]; T e[PER]; } pay;
    pay.w[0] = pay.w[1] = 0;
    const int64_t e0 = l * PER;
    if (recv) {
      // the local operand is loaded BEFORE the line is polled: its L2 round trip
      // overlaps the wait instead of following it (one round trip less per hop)
      union { uint32_t w[2]; T e[PER]; } loc;
      loc.w[0] = loc.w[1] = 0;
      if (reduce) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
          if (e0 + k < nelem) loc.e[k] = ld_cg_scalar(s + e0 + k);
      }
      uint32_t x0, f0, x1, f1;
      for (uint32_t spin = 0;; ++spin) {
        asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(cin + 16 * l) : "memory");
        if (f0 == inSeq && f1 == inSeq) break;
        // speculative slice the control thread gave up on: leave it (redone later;
        // every line is idempotent to rewrite -- same data, same sequence number)
        if ((spin & 7) == 7 && *abortGen != gen) { ok = false; return; }
      }
      if (tLine && l == tid) tLine[0] = globaltimer();   // trace: first line in
      pay.w[0] = x0;
      pay.w[1] = x1;
      if (reduce) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
          if (e0 + k < nelem) pay.e[k] = sop<DT, OP>(pay.e[k], loc.e[k]);
      }
    } else {
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (e0 + k < nelem) pay.e[k] = ld_cg_scalar(s + e0 + k);
    }
    if (copy) {
#pragma unroll
      for (int k = 0; k < PER; ++k)
        if (e0 + k < nelem) d[e0 + k] = pay.e[k];
    }
    if (send)
      asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};"
                   :: "l"(cout + 16 * l), "r"(pay.w[0]), "r"(outSeq), "r"(pay.w[1]), "r"(outSeq) : "memory");
    if (tLine && l == nl - 1) tLine[1] = globaltimer();
  }
}

// Compute warps: every compute warp takes part in every slice, in order.  The
// descriptor is read field by field into registers (a struct copy would live in
// local memory and be re-read in the inner loop).
template <int DT, int OP>
__device__ __forceinline__ void reduce_tile_smem(Stage& st, int sz, int tid, int nt) {
  const int nv = sz >> 4;
  for (int i = tid; i < nv; i += nt) {
    const uint4 v = vop<DT, OP>(lds_v4(&st.in[i]), lds_v4(&st.loc[i]));
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" :: "r"(smem_u32(&st.in[i])), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w) : "memory");
  }
}

// ragged tail (< 16 B) of a TMA-path slice, straight from global memory
template <int DT, int OP>
__device__ __forceinline__ void tail_slice(const int prim, const char* src, const char* cin, char* dst, char* cout,
                                           int64_t e0, int64_t nelem, int tid, int nt) {
  typedef typename Elem<DT>::T T;
  const bool rv = prim & (A_RECV | A_DREAD), rd = prim & A_REDUCE;
  const T* si = reinterpret_cast<const T*>(rv ? cin : src);
  const T* ss = reinterpret_cast<const T*>(src);
  for (int64_t e = e0 + tid; e < nelem; e += nt) {
    T v = ld_cg_scalar(si + e);
    if (rd) v = sop<DT, OP>(v, ld_cg_scalar(ss + e));
    if (prim & A_COPY) reinterpret_cast<T*>(dst)[e] = v;
    if (prim & A_SEND) reinterpret_cast<T*>(cout)[e] = v;
  }
}

// Instantiate FN<dtype, op>(args...) for the slice's runtime (dtype, op); copy-only
// slices use the element size alone (op irrelevant).
#define OCCL_DISPATCH(dtype, op, FN, ...)                                          \
  do {                                                                             \
    switch ((dtype) * 4 + (op)) {                                                  \
      case kI32 * 4 + kSum: FN<kI32, kSum>(__VA_ARGS__); break;                    \
      case kI32 * 4 + kProd: FN<kI32, kProd>(__VA_ARGS__); break;                  \
      case kI32 * 4 + kMax: FN<kI32, kMax>(__VA_ARGS__); break;                    \
      case kI32 * 4 + kMin: FN<kI32, kMin>(__VA_ARGS__); break;                    \
      case kF32 * 4 + kSum: FN<kF32, kSum>(__VA_ARGS__); break;                    \
      case kF32 * 4 + kProd: FN<kF32, kProd>(__VA_ARGS__); break;                  \
      case kF32 * 4 + kMax: FN<kF32, kMax>(__VA_ARGS__); break;                    \
      case kF32 * 4 + kMin: FN<kF32, kMin>(__VA_ARGS__); break;                    \
      case kBF16 * 4 + kSum: FN<kBF16, kSum>(__VA_ARGS__); break;                  \
      case kBF16 * 4 + kProd: FN<kBF16, kProd>(__VA_ARGS__); break;                \
      case kBF16 * 4 + kMax: FN<kBF16, kMax>(__VA_ARGS__); break;                  \
      case kBF16 * 4 + kMin: FN<kBF16, kMin>(__VA_ARGS__); break;                  \
      case kF16 * 4 + kSum: FN<kF16, kSum>(__VA_ARGS__); break;                    \
      case kF16 * 4 + kProd: FN<kF16, kProd>(__VA_ARGS__); break;                  \
      case kF16 * 4 + kMax: FN<kF16, kMax>(__VA_ARGS__); break;                    \
      case kF16 * 4 + kMin: FN<kF16, kMin>(__VA_ARGS__); break;                    \
      case kI64 * 4 + kSum: FN<kI64, kSum>(__VA_ARGS__); break;                    \
      case kI64 * 4 + kProd: FN<kI64, kProd>(__VA_ARGS__); break;                  \
      case kI64 * 4 + kMax: FN<kI64, kMax>(__VA_ARGS__); break;                    \
      case kI64 * 4 + kMin: FN<kI64, kMin>(__VA_ARGS__); break;                    \
      case kF64 * 4 + kSum: FN<kF64, kSum>(__VA_ARGS__); break;                    \
      case kF64 * 4 + kProd: FN<kF64, kProd>(__VA_ARGS__); break;                  \
      case kF64 * 4 + kMax: FN<kF64, kMax>(__VA_ARGS__); break;                    \
      default: FN<kF64, kMin>(__VA_ARGS__); break;                                 \
    }                                                                              \
  } while (0)

// LL slices out of line: the 24 (dtype, op) instantiations of the abortable
// line loop would otherwise raise compute_main's register pressure into spills
// on the bandwidth (TMA) path.
__device__ __noinline__ bool ll_dispatch(int prim, int dtype, int op, const char* src, const char* cin, char* dst,
                                         char* cout, int64_t nelem, uint32_t inSeq, uint32_t outSeq, int ctid,
                                         int cnt, const volatile uint32_t* abortGen, uint32_t gen, uint64_t* tLine) {
  bool ok = true;
  OCCL_DISPATCH(dtype, op, ll_slice, prim, src, cin, dst, cout, nelem, inSeq, outSeq, ctid, cnt, abortGen, gen, ok,
                tLine);
  return ok;
}

// The data loop's position, kept across the returns compute_main makes for LL
// runs (see the kernel).
struct ComputeState {
  uint32_t j, cs, cph;                 // descriptors consumed; staging slot and its phase parity
  unsigned long long cWait, cData, nData;   // probes
};

// Returns the pipe slot of an LL-run descriptor (its run is entered by the
// caller; the descriptor is not yet released), or -1 at the daemon's exit.
__device__ __noinline__ int compute_main(const DaemonParams& p, int b, Pipe& pipe, Stage* stages, uint64_t* tfull,
                                         uint64_t* tempty, uint64_t* tred, const int ctid, const int cnt,
                                         ComputeState& st) {
  const uint32_t D = (uint32_t)p.pipeDepth, S = (uint32_t)p.stages;
  const bool bulk = p.bulkStores != 0;
  const int lane = ctid & 31;
  const bool discard = p.discardConsumed != 0;
  const int l2 = p.l2Hints;
  const uint64_t pol = policy_evict_first(), polKeep = policy_evict_last();
  const bool leader = ctid == 0;                       // probes
  unsigned long long cWait = st.cWait, cData = st.cData, nData = st.nData;
  uint32_t cs = st.cs, cph = st.cph;                   // staging slot and its phase parity
  for (uint32_t j = st.j;; ++j) {
    const uint32_t i = j % D;
    const long long t0 = clock64();
    mbar_wait(&pipe.full[i], (j / D) & 1);
    // lane 0 reads the descriptor and broadcasts it: the warp's only reader of
    // ring[i] is then the lane that hands it back on empty[i] (direct ordering)
    int prim = 0, dtype = 0, op = 0;
    uint32_t inSeq = 0, outSeq = 0, gen = 0;
    unsigned long long nel = 0, a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    if (lane == 0) {
      const SliceDesc* dp = &pipe.ring[i];
      prim = dp->prim; dtype = dp->dtype; op = dp->op;
      inSeq = (uint32_t)dp->creditVal; outSeq = (uint32_t)dp->headVal; gen = dp->gen;
      nel = (unsigned long long)dp->nelem;
      a0 = (uintptr_t)dp->src; a1 = (uintptr_t)dp->cin; a2 = (uintptr_t)dp->dst; a3 = (uintptr_t)dp->cout;
    }
    prim = __shfl_sync(0xffffffffu, prim, 0);
    if (prim == P_EXIT) break;
    if (prim & A_LLRUN) {                              // the caller runs it (ll_run_dispatch)
      st.j = j; st.cs = cs; st.cph = cph;
      st.cWait = cWait; st.cData = cData; st.nData = nData;
      return (int)i;
    }
    dtype = __shfl_sync(0xffffffffu, dtype, 0);
    op = __shfl_sync(0xffffffffu, op, 0);
    inSeq = __shfl_sync(0xffffffffu, inSeq, 0);
    outSeq = __shfl_sync(0xffffffffu, outSeq, 0);
    gen = __shfl_sync(0xffffffffu, gen, 0);
    const int64_t nelem = (int64_t)__shfl_sync(0xffffffffu, nel, 0);
    const char* src = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, a0, 0));
    const char* cin = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, a1, 0));
    char* dst = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, a2, 0));
    char* cout = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, a3, 0));
    const long long t1 = clock64();
    const int vb = tma_vec_bytes(dtype, nelem, src, dst, cout, cin);
    if (prim & A_LL) {
      // trace (thread 0 of the compute warps): woke with the descriptor / first
      // line in / slice stored -- the parts of an LL hop (scripts/trace_ll.py)
      // (and the thread that stores the slice's last line -- the one the
      // downstream's control lane polls: that store, 23, and its first line in, 24)
      uint64_t tLine[2] = {0, 0};
      const bool tr = p.traceCap != 0;
      if (tr && ctid == 0) trace_at(p, pipe.tr, b, kEvMark, (int)i, 20);
      const bool ok = ll_dispatch(prim, dtype, op, src, cin, dst, cout, nelem, inSeq, outSeq, ctid, cnt,
                                  &pipe.abortGen, gen, tr ? tLine : nullptr);
      if (tr && ctid == 0) {
        trace_at_t(p, pipe.tr, b, kEvMark, (int)i, 21, tLine[0]);
        trace_at(p, pipe.tr, b, kEvMark, (int)i, 22);
      }
      if (tr && tLine[1]) {
        trace_at_t(p, pipe.tr, b, kEvMark, (int)i, 23, tLine[1]);
        trace_at_t(p, pipe.tr, b, kEvMark, (int)i, 24, tLine[0]);
      }
      if (__any_sync(0xffffffffu, !ok) && lane == 0) atomicOr(&pipe.fail[i], 1u);   // before sdone's release
    } else if (!(prim & (A_COPY | A_SEND))) {
      // direct final receive: the data is already in place, nothing to move
    } else if (vb == 0) {                              // small or misaligned: register path
      OCCL_DISPATCH(dtype, op, move_slice, prim, src, cin, dst, cout, nelem, ctid, cnt);
    } else {
      const bool disc = discard && (prim & A_RECV) && !(prim & A_DIN) && !((uintptr_t)cin & 127);
      // l2Hints == 3: a direct receive we forward was stored evict-last by the upstream
      const bool demote = l2 >= 3 && (prim & A_DIN) && (prim & A_SEND) && !((uintptr_t)cin & 127);
      for (int off = 0; off < vb; off += kTile) {
        const uint32_t s = cs;
        mbar_wait(&tfull[s], cph);
        if (++cs == S) { cs = 0; cph ^= 1; }
        const int sz = min(kTile, vb - off);
        if (disc && ctid < (sz >> 7)) discard_l2_line(cin + off + ((size_t)ctid << 7));  // tile is in smem now
        if (demote && ctid < (sz >> 7)) demote_l2_line(cin + off + ((size_t)ctid << 7));   // kept by the upstream
        if (bulk) {
          // bulk-store mode: reduce in place in shared memory; the publisher lane
          // stores the tile with cp.async.bulk (copy tiles need no compute at all)
          if (prim & A_REDUCE) {
            OCCL_DISPATCH(dtype, op, reduce_tile_smem, stages[s], sz, ctid, cnt);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
          }
          // every tile (copy tiles too) completes one tred phase, so tred[s] stays
          // in step with the stage's phase
          __syncwarp();
          if (lane == 0) mbar_arrive(&tred[s]);
          continue;
        }
        if (prim & A_REDUCE) {
          OCCL_DISPATCH(dtype, op, consume_tile, prim, dst + off, cout + off, stages[s], sz, ctid, cnt, l2, pol, polKeep);
        } else {
          consume_tile<kI32, kSum>(prim, dst + off, cout + off, stages[s], sz, ctid, cnt, l2, pol, polKeep);   // copy only
        }
        // every lane releases its own reads of the tile to the producer's next TMA
        // load into it (direct ordering; measured free vs one elected lane)
        mbar_arrive(&tempty[s]);
      }
      // ragged tail (< 16 B) straight from global memory
      const int64_t e0 = vb / elem_size(dtype);
      if (e0 < nelem) OCCL_DISPATCH(dtype, op, tail_slice, prim, src, cin, dst, cout, e0, nelem, ctid, cnt);
    }
    // this warp's stores (ordered by __syncwarp) are released to the publisher,
    // which fences once and raises the peers' flags (publisher_main)
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&pipe.sdone[i]);
      mbar_arrive(&pipe.empty[i]);                   // this warp is done with ring[i] too
    }
    if (leader) {
      const long long t2 = clock64();
      cWait += t1 - t0;
      cData += t2 - t1;
      ++nData;
    }
  }
  if (leader) {
    atomicAdd(&p.blkStats[b].cycDataWait, cWait);
    atomicAdd(&p.blkStats[b].cycData, cData);
    atomicAdd(&p.blkStats[b].nData, nData);
  }
  return -1;
}

// Publisher lane (warp 2 lane 0): makes finished slices visible to the peers in
// order.  Every slice that is already finished when the publisher gets to it is
// covered by the same release fence; then the head of the downstream rank and
// the credit of the upstream rank are raised to the last slice's values
// (commit visibility).
__device__ __noinline__ void publisher_main(const DaemonParams& p, int b, Pipe& pipe, Stage* stages, uint64_t* tfull,
                                            uint64_t* tempty, uint64_t* tred) {
  const uint32_t D = (uint32_t)p.pipeDepth, S = (uint32_t)p.stages;
  unsigned long long cycFence = 0, nFence = 0;
  const int sys = p.sysScope;
  const bool bulk = p.bulkStores != 0, hints = p.l2Hints != 0;
  const uint64_t pol = policy_evict_first();
  uint32_t cs = 0, cph = 0;                         // bulk mode: staging slot / phase (same walk as the producer)
  uint32_t j = 0;
  bool poisoned = false;                            // LL speculation: abort generation not to publish
  uint32_t poisonGen = 0;
  for (;;) {
    const uint32_t i = j % D;
    mbar_wait(&pipe.full[i], (j / D) & 1);
    if (pipe.ring[i].prim == P_EXIT) {
      if (p.traceCap) p.traceCount[b] = pipe.tr.base + pipe.tr.idx;   // control traced its last record already
      atomicAdd(&p.blkStats[b].cycRelFence, cycFence);                // release-fence probe (publisher lane)
      atomicAdd(&p.blkStats[b].nFence, nFence);
      break;
    }
    bool bulkSlice = false;
    if (bulk) {
      // bulk-store mode: this lane stores every staged tile of a TMA-path slice
      // (cp.async.bulk, one group per tile), hands each stage back once its
      // store has read it, and publishes after the slice's writes completed --
      // the release fence then waits for no generic stores at all
      const SliceDesc& d = pipe.ring[i];
      const int vb = (d.prim & (A_COPY | A_SEND)) && !(d.prim & A_LL)
                         ? tma_vec_bytes(d.dtype, d.nelem, d.src, d.dst, d.cout, d.cin) : 0;
      if (vb > 0) {
        bulkSlice = true;
        const bool copy = d.prim & A_COPY, send = d.prim & A_SEND;
        int prev = -1;
        for (int off = 0; off < vb; off += kTile) {
          const uint32_t st = cs, ph = cph;
          if (++cs == S) { cs = 0; cph ^= 1; }
          const uint32_t sz = (uint32_t)min(kTile, vb - off);
          mbar_wait(&tred[st], ph);                   // tile staged (and reduced in place)
          if (copy) {
            if (hints) bulk_store_hint(d.dst + off, stages[st].in, sz, pol);
            else bulk_store(d.dst + off, stages[st].in, sz);
          }
          if (send) bulk_store(d.cout + off, stages[st].in, sz);
          bulk_commit();
          if (prev >= 0) {
            bulk_wait_read1();                       // the previous tile's stores have read their stage
            mbar_arrive(&tempty[prev]);
          }
          prev = (int)st;
        }
        bulk_wait_read0();
        mbar_arrive(&tempty[prev]);
      }
    }
    mbar_wait(&pipe.sdone[i], (j / D) & 1);
    if (bulkSlice) bulk_wait_all();                  // the slice's bulk writes are complete
    {
      // LL speculation: a slice a data warp gave up on -- and every later slice of
      // the same abort generation -- is not published; the control thread redoes it
      const uint32_t g = pipe.ring[i].gen;
      if (*reinterpret_cast<volatile uint32_t*>(&pipe.fail[i])) { poisoned = true; poisonGen = g; }
      if (poisoned && g == poisonGen) {
        mbar_arrive(&pipe.empty[i]);
        ++j;
        continue;
      }
    }
    bool send = false, recv = false, needFence = false;
    uint64_t hv = 0, cv = 0;
    char* ho = nullptr;
    char* co = nullptr;
    uint32_t k = j;
    for (;;) {
      const SliceDesc& d = pipe.ring[k % D];
      if (d.prim & A_SEND) { send = true; hv = d.headVal; ho = d.headOut; }
      if (d.prim & A_RECV) { recv = true; cv = d.creditVal; co = d.creditOut; }
      // LL data needs no release (its lines carry their own flags); LL credits
      // follow loads that already returned their values
      if ((d.prim & (A_SEND | A_RECV)) && !(d.prim & A_LL)) needFence = true;
      const uint32_t k1 = k + 1;
      if (bulk) break;                              // bulk mode publishes slice by slice
      if (!mbar_test(&pipe.full[k1 % D], (k1 / D) & 1)) break;
      const SliceDesc& d1 = pipe.ring[k1 % D];
      if (d1.prim == P_EXIT) break;
      if ((d1.prim & A_SEND) && ho && d1.headOut != ho) break;
      if ((d1.prim & A_RECV) && co && d1.creditOut != co) break;
      if (!mbar_test(&pipe.sdone[k1 % D], (k1 / D) & 1)) break;
      if (*reinterpret_cast<volatile uint32_t*>(&pipe.fail[k1 % D])) break;   // handled on its own
      k = k1;
    }
    trace_at(p, pipe.tr, b, kEvSdone, k - j + 1, (uint32_t)(hv & 0xffff) | ((uint32_t)(cv & 0xffff) << 16));
    if (needFence) {                            // LL data carries its own flags: no release needed
      const long long tf = clock64();
      fence_acq_rel(sys);
      cycFence += clock64() - tf;
      ++nFence;
    }
    if (send) red_max_relaxed(ho, hv, sys);     // head of rank r+1
    if (recv) red_max_relaxed(co, cv, sys);     // credit of rank r-1
    trace_at(p, pipe.tr, b, kEvPublish, k - j + 1, (uint32_t)(hv & 0xffff) | ((uint32_t)(cv & 0xffff) << 16));
    for (uint32_t q = j; q <= k; ++q) mbar_arrive(&pipe.empty[q % D]);
    j = k + 1;
  }
}

// Named barrier of the compute warps (id 1; barrier 0 is the launch's
// __syncthreads).  Non-aligned form: lanes leave the line loop divergently.
__device__ __forceinline__ void bar_sync_compute(int cnt) {
  asm volatile("barrier.sync 1, %0;" :: "r"(cnt) : "memory");
}

// Compute warps: one LL run (LLRun).  Every compute thread walks the same slice
// schedule (the geometry is recomputed per thread -- no broadcast needed); thread
// ctid moves lines ctid, ctid + cnt, ... of each slice.  A slice ends with one
// named barrier; then thread 0 raises the upstream's credit.  A line not there
// within limitNs of its slice's start aborts the run: every thread leaves after
// the slice's barrier, so the reported cursor is the first incomplete slice (its
// partly sent lines are rewritten identically when it is redone).
// The step table of an LL run: step t's primitive and segment geometry (PAPER.md
// ring schedule, step_prim / seg_geom), built once per run by compute thread t
// -- per slice only a table lookup and the slice's offset remain on the chain
// between two hops (computing the geometry per slice took ~1.2 us of it).
__device__ __noinline__ void ll_steps(const LLRun& L, LLStep* tab, int ctid, int cnt) {
  for (int t = ctid; t < L.nsteps; t += cnt) {
    int prim, seg;
    step_prim(L.kind, L.n, L.r, L.root, t, L.inplace != 0, prim, seg);
    uint64_t sendOff, recvOff, len;
    seg_geom(L.kind, L.n, L.r, L.count, L.segLen, seg, sendOff, recvOff, len);
    tab[t].sendOff = sendOff;
    tab[t].recvOff = recvOff;
    tab[t].len = len;
    tab[t].prim = prim;
  }
}

template <int DT, int OP>
__device__ __forceinline__ void ll_run(const DaemonParams& p, LLRun& L, Pipe& pipe, int b, const int ctid,
                                       int cnt) {
  typedef typename Elem<DT>::T T;
  constexpr int PER = 8 / sizeof(T);                 // elements per line
  const uint64_t limitNs = L.limitNs;
  const int K = L.K, spc = L.spc, nsteps = L.nsteps, sys = L.sys;
  const uint32_t nloops = L.nloops;
  const uint64_t laneLo = L.laneLo, part = L.part, E = L.E, llSlot = L.llSlot;
  const T* sendbuff = reinterpret_cast<const T*>(L.sendbuff);
  T* recvbuff = reinterpret_cast<T*>(L.recvbuff);
  const char* llIn = L.llIn;
  char* llOut = L.llOut;
  Cursor c{L.loop, L.step, L.slc, L.nsent, L.nrecv};
  uint32_t slotIn = (uint32_t)(c.nrecv % (uint64_t)K), slotOut = (uint32_t)(c.nsent % (uint64_t)K);
  uint64_t creditSeen = L.creditSeen;
  volatile uint32_t* abortf = L.abort;                // [0], [1]: line timeouts by slice parity; [2]: credit timeout
  uint32_t nDone = 0;
  const bool tr = p.traceCap != 0 && ctid == 0;
  const LLStep* tab = pipe.llsteps;
  // only the warps a slice has lines for take part (a 4 KiB all-reduce at 8
  // ranks: 64 lines, 2 of 16 warps): the others leave at once, and the per-slice
  // barrier waits for fewer warps
  {
    const uint64_t maxElem = part < E ? part : E;
    int nw = (int)(((maxElem * sizeof(T) + 7) / 8 + 31) / 32);
    if (nw < 1) nw = 1;
    if (nw * 32 < cnt) cnt = nw * 32;
    if (ctid >= cnt) return;
  }
  ll_steps(L, pipe.llsteps, ctid, cnt);
  bar_sync_compute(cnt);
  while (c.loop < nloops) {
    const uint32_t par = nDone & 1;
    if (ctid == 0) abortf[par ^ 1] = 0;              // the next slice's flag (this one's is clear: we got here)
    const uint64_t t0 = globaltimer();
    if (tr) trace_at_t(p, pipe.tr, b, kEvMark, (int)c.step, 40, t0);
    const LLStep& S = tab[c.step];
    const int prim = S.prim;
    uint64_t laneHi = laneLo + part;
    if (laneHi > S.len) laneHi = S.len;
    const uint64_t lo = laneLo + ((uint64_t)c.loop * spc + c.slc) * E;
    uint64_t hi = lo + E;
    if (hi > laneHi) hi = laneHi;
    const int64_t nelem = hi > lo ? (int64_t)(hi - lo) : 0;
    const T* src = sendbuff + (S.sendOff + lo);
    T* dst = recvbuff + (S.recvOff + lo);
    const char* cin = llIn + slotIn * llSlot;
    char* cout = llOut + slotOut * llSlot;
    const bool recv = prim & A_RECV, reduce = prim & A_REDUCE, copy = prim & A_COPY, send = prim & A_SEND;
    if (tr) trace_at(p, pipe.tr, b, kEvMark, (int)c.step, 42);
    if (send && c.nsent - creditSeen >= (uint64_t)K) {
      // flow control: thread 0 polls the downstream's credit, the barrier broadcasts it
      if (ctid == 0) {
        uint64_t cr;
        for (;;) {
          cr = ld_acquire(L.creditIn, sys);
          if (c.nsent - cr < (uint64_t)K) break;
          if (globaltimer() - t0 > limitNs) { abortf[2] = 1; break; }
        }
        *reinterpret_cast<volatile uint64_t*>(&L.credit) = cr;
      }
      bar_sync_compute(cnt);
      if (tr) trace_at(p, pipe.tr, b, kEvMark, (int)c.step, 43);
      if (abortf[2]) break;                            // sticky for the run: every thread sees it
      const uint64_t cr = *reinterpret_cast<volatile uint64_t*>(&L.credit);
      if (cr > creditSeen) creditSeen = cr;
    }
    // thread 0 reads the downstream's credit once per sending slice, early (the
    // load is in flight while the lines are polled) and hands it to every thread
    // through the slice's barrier: the blocking credit wait above becomes rare
    uint64_t crEarly = 0;
    if (send && ctid == 0) crEarly = ld_relaxed(L.creditIn, sys);
    const uint32_t inSeq = (uint32_t)(c.nrecv + 1), outSeq = (uint32_t)(c.nsent + 1);
    const int64_t lines = (nelem + PER - 1) / PER;
    const int64_t nl = lines ? lines : 1;              // an empty message still carries one token line
    for (int64_t l = ctid; l < nl; l += cnt) {
      union { uint32_t w[2]; T e[PER]; } pay, loc;
      pay.w[0] = pay.w[1] = 0;
      const int64_t e0 = l * PER;
      if (recv) {
        // the local operand is loaded before the line is polled (its round trip
        // overlaps the wait)
        loc.w[0] = loc.w[1] = 0;
        if (reduce) {
#pragma unroll
          for (int k = 0; k < PER; ++k)
            if (e0 + k < nelem) loc.e[k] = ld_cg_scalar(src + e0 + k);
        }
        uint32_t x0, f0, x1, f1;
        bool got = true;
        uint32_t spin = 0;
        for (;; ++spin) {
          asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(x0), "=r"(f0), "=r"(x1), "=r"(f1) : "l"(cin + 16 * l) : "memory");
          if (f0 == inSeq && f1 == inSeq) break;
          if ((spin & 7) == 7 && (abortf[par] || globaltimer() - t0 > limitNs)) {
            abortf[par] = 1;
            got = false;
            break;
          }
        }
        if (!got) break;
        if (tr && l == ctid) trace_at(p, pipe.tr, b, kEvMark, (int)spin, 44);
        pay.w[0] = x0;
        pay.w[1] = x1;
        if (reduce) {
#pragma unroll
          for (int k = 0; k < PER; ++k)
            if (e0 + k < nelem) pay.e[k] = sop<DT, OP>(pay.e[k], loc.e[k]);
        }
      } else {
#pragma unroll
        for (int k = 0; k < PER; ++k)
          if (e0 + k < nelem) pay.e[k] = ld_cg_scalar(src + e0 + k);
      }
      if (copy) {
#pragma unroll
        for (int k = 0; k < PER; ++k)
          if (e0 + k < nelem) dst[e0 + k] = pay.e[k];
      }
      if (send)
        asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};"
                     :: "l"(cout + 16 * l), "r"(pay.w[0]), "r"(outSeq), "r"(pay.w[1]), "r"(outSeq) : "memory");
    }
    if (tr) trace_at(p, pipe.tr, b, kEvMark, (int)c.step, 45);
    if (send && ctid == 0) *reinterpret_cast<volatile uint64_t*>(&L.credit) = crEarly;
    bar_sync_compute(cnt);
    if (abortf[par]) break;
    if (send) {                                        // credits are monotonic: a later value is as good
      const uint64_t cr = *reinterpret_cast<volatile uint64_t*>(&L.credit);
      if (cr > creditSeen) creditSeen = cr;
    }
    if (ctid == 0) {
      // LL credits follow loads that already returned their values: no fence
      if (recv) red_max_relaxed(L.creditOut, c.nrecv + 1, sys);
      L.tProg = globaltimer();
      if (tr) trace_at(p, pipe.tr, b, kEvMark, (int)c.step, 41);
    }
    if (recv && ++slotIn == (uint32_t)K) slotIn = 0;
    if (send && ++slotOut == (uint32_t)K) slotOut = 0;
    advance(c, prim, spc, nsteps);
    ++nDone;
  }
  if (ctid == 0) {
    L.oLoop = c.loop; L.oStep = c.step; L.oSlc = c.slc;
    L.oNsent = c.nsent; L.oNrecv = c.nrecv; L.oCreditSeen = creditSeen;
    L.nDone = nDone;
  }
}


// Entered from the kernel's top level, not from compute_main: as a callee of the
// data loop its registers made compute_main spill (176 B) and slowed every
// Simple-protocol slice (1 MiB AR 165 vs 121 us).
__device__ __noinline__ void ll_run_dispatch(const DaemonParams& p, Pipe& pipe, int b, int ctid, int cnt) {
  LLRun& L = pipe.llr;
  OCCL_DISPATCH(L.dtype, L.op, ll_run, p, L, pipe, b, ctid, cnt);
}

// Control lane side of an LL run (LLRun; llSpeculate == 2).  One descriptor
// hands the compute warps the collective's remaining slices; the lane waits for
// the run, takes over the cursor it reports and decides as the per-slice path
// does: done, or -- no slice completed for T spins -- preempted.  Under the
// priority policy a run gives up after spinMin spins at most, so that the lane
// can look at the SQ (yield to new SQEs) and re-issue the run
// when nothing new is there.  Returns RUN_DONE / RUN_PREEMPT.
__device__ __noinline__ int ll_run_control(const DaemonParams& p, int b, Sched& sh, const Smem& m, Pipe& pipe,
                                           uint32_t& issued, uint32_t& committed, Cursor& dc, uint64_t& T,
                                           unsigned long long& nSlices) {
  const uint32_t D = (uint32_t)p.pipeDepth;
  CtxSlot& cx = m.cache[sh.way];
  const RingDesc& R = p.rings[cx.sub];
  const size_t cb = (size_t)sh.curId * p.G + b;
  const int K = p.K;
  const uint64_t llSlot = 2ull * p.llSliceBytes;
  LLRun& L = pipe.llr;
  // the downstream's credit as it stands (relaxed; its latency overlaps the stores
  // below): without it the run's first send would wait for a credit poll
  const uint64_t cr0 = ld_relaxed(p.flagsLocal + cb * kFlagStride + 128, p.sysScope);
  L.sendbuff = cx.s.sendbuff; L.recvbuff = cx.s.recvbuff; L.count = cx.s.count; L.segLen = cx.s.segLen;
  L.part = cx.s.part;
  L.laneLo = (uint64_t)cx.lane * cx.s.part;
  L.E = p.llSliceBytes / elem_size(cx.d.dtype);
  L.llIn = p.llLocal + cb * K * llSlot;
  L.llOut = R.llNext + cb * K * llSlot;
  L.creditIn = p.flagsLocal + cb * kFlagStride + 128;
  L.creditOut = R.flagsPrev + cb * kFlagStride + 128;
  L.llSlot = llSlot;
  L.nloops = cx.d.nloops;
  L.kind = cx.d.kind; L.n = R.nranks; L.r = R.rank; L.root = cx.root;
  L.inplace = cx.s.sendbuff == cx.s.recvbuff; L.dtype = cx.d.dtype; L.op = (int)cx.op; L.spc = (int)cx.spc;
  L.nsteps = cx.nsteps; L.K = K; L.sys = p.sysScope;
  L.creditSeen = cr0;
  const uint64_t spinNs = p.spinNs;
  const bool yieldable = p.orderPolicy == 1 && p.sqYieldNs != 0;
  uint64_t tProg = globaltimer();                      // last progress (or the run's start)
  for (;;) {
    const uint64_t hard = T * spinNs;
    uint64_t lim = hard;
    if (yieldable && (uint64_t)p.spinMin * spinNs < lim) lim = (uint64_t)p.spinMin * spinNs;
    L.limitNs = lim;
    L.loop = dc.loop; L.step = dc.step; L.slc = dc.slc; L.nsent = dc.nsent; L.nrecv = dc.nrecv;
    L.abort[0] = L.abort[1] = L.abort[2] = 0;
    L.nDone = 0;
    L.tProg = 0;
    SliceDesc& sd = pipe.ring[issued % D];
    sd.prim = A_LL | A_LLRUN;
    sd.dtype = cx.d.dtype; sd.op = (int)cx.op; sd.nelem = 0;
    sd.src = nullptr; sd.cin = nullptr; sd.dst = nullptr; sd.cout = nullptr;
    sd.gen = pipe.abortGen;
    mbar_arrive(&pipe.full[issued % D]);             // committed == issued: the slot is free
    trace_at(p, *m.tr, b, kEvIssue, sh.curId, 0xfff00000u);
    ++issued;
    mbar_wait(&pipe.empty[committed % D], (committed / D) & 1);
    ++committed;
    const uint32_t nd = L.nDone;
    dc.loop = L.oLoop; dc.step = L.oStep; dc.slc = L.oSlc; dc.nsent = L.oNsent; dc.nrecv = L.oNrecv;
    L.creditSeen = L.oCreditSeen;
    if (nd) {
      nSlices += nd;
      tProg = L.tProg;
      if (p.stickiness && sh.boostOk) {               // raise the threshold, once per run
        T *= p.spinBoost;
        if (T > p.spinCap) T = p.spinCap;
      }
      m.tq[sh.pos] &= 0xffffu;                        // progressed: not stalled
    }
    if (dc.loop >= cx.d.nloops) return RUN_DONE;
    const uint64_t now = globaltimer();
    if (now - tProg > T * spinNs) return RUN_PREEMPT;  // two-phase blocking: preempt
    if (yieldable) {
      // the run gave up after spinMin spins: new SQEs? (as in the per-slice path)
      const uint64_t tail = ld_acquire(p.mirrorTail, 0);
      if (tail > sh.cursor) return RUN_PREEMPT;
      unsigned long long* lastHost = reinterpret_cast<unsigned long long*>(p.mirrorTail + 3);
      const unsigned long long lh = *reinterpret_cast<volatile unsigned long long*>(lastHost);
      if (now - lh > p.sqYieldNs && atomicCAS(lastHost, lh, (unsigned long long)now) == lh) {
        uint32_t stamp;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(stamp) : "l"(p.sq[tail % p.sqDepth].c[0])
                     : "memory");
        if (stamp == (uint32_t)(tail + 1)) {
          sh.needHostPoll = 1;
          return RUN_PREEMPT;
        }
      }
    }
  }
}

}  // namespace

// =============================================================================
// The daemon kernel.  Launched with the largest grid/block of all collectives
// (PAPER.md:470): G blocks per rank, one scheduler per block.  One launch may
// serve several ranks that live on the same device (virtual ranks): blocks
// [i*G, (i+1)*G) run rank pp[i]'s daemon with its own SQ, CQ, contexts and
// connectors -- the per-rank daemons are then co-resident by construction.
//
// Warp roles: warp 0 lane 0 is the control thread (scheduler, SQ/CQ, connector
// flags, context switches); warp 1 lane 0 is the TMA producer streaming slice
// operands into a shared-memory staging ring (cp.async.bulk); warps 2.. are
// compute warps that reduce/copy staged tiles and store them.  Control and the
// data warps communicate through a descriptor pipe with mbarriers; the last
// compute warp to finish a slice publishes it to the peers.
// =============================================================================
template <int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB) occl_daemon_kernel(const DaemonParams* __restrict__ pp, int G) {
  const int lr = blockIdx.x / G;
  // The parameters live in shared memory for the launch (uploaded only while no
  // daemon runs): a field read in a hot loop is then an LDS, not a global load
  // that misses L1 after every gpu-scope acquire (CCTL.IVALL invalidates the SM's
  // L1) -- the control lane's idle LL poll iteration read 4-6 fields that way
  // and took ~1 us (scripts/trace_ll.py, profiles/r02/)
  __shared__ __align__(16) DaemonParams sp;
  static_assert(sizeof(DaemonParams) % 8 == 0, "DaemonParams copy granularity");
  {
    const uint2* src = reinterpret_cast<const uint2*>(&pp[lr]);
    uint2* dst = reinterpret_cast<uint2*>(&sp);
    for (int i = threadIdx.x; i < (int)(sizeof(DaemonParams) / 8); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  const DaemonParams& p = sp;
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ Sched sh;
  __shared__ Pipe pipe;
  __shared__ uint64_t tfull[kMaxStages], tempty[kMaxStages], tred[kMaxStages];
  __shared__ __align__(128) SqeWire sqbuf[kSqBurst];
  __shared__ __align__(8) uint64_t sqbar;
  const int W = p.cacheWays;
  Stage* stages = reinterpret_cast<Stage*>(smem);                       // 128-B aligned
  Smem m;
  m.cache = reinterpret_cast<CtxSlot*>(smem + p.stages * sizeof(Stage));
  m.cacheTag = reinterpret_cast<int*>(m.cache + W);
  m.tq = reinterpret_cast<uint32_t*>(m.cacheTag + W);
  m.prio = reinterpret_cast<int32_t*>(m.tq + p.maxColl);
  m.subLo = reinterpret_cast<uint32_t*>(m.prio + p.maxColl);
  m.subOf = reinterpret_cast<uint8_t*>(m.subLo + p.maxColl);
  m.ready = m.subOf + p.maxColl;
  m.tr = &pipe.tr;
  m.sqbuf = sqbuf;
  m.sqbar = &sqbar;
  const int tid = threadIdx.x;
  const int b = blockIdx.x - lr * G;
  const int nComputeWarps = (int)(blockDim.x >> 5) - kRoleWarps;
  const uint32_t D = (uint32_t)p.pipeDepth;

  if (tid == 0) {
    const BlockState bs = p.blk[b];
    sh.cursor = bs.sqCursor;
    sh.qlen = bs.qlen;
    sh.pos = bs.pos;
    sh.exiting = bs.exiting;
    sh.iter = 0;
    sh.rr = 1;
    sh.voted = 0;
    sh.lastProgress = 0;
    sh.lastSqPoll = 0;
    sh.sqPhase = 0;
    sh.needHostPoll = 0;
    sh.boostOk = 1;
    mbar_init(&sqbar, 1);
    sh.lastRun = -1;
    sh.curId = -1;
    sh.cycRun = sh.cycPoll = sh.cycAcqFence = sh.cycRelFence = sh.nCommit = 0;
    sh.cycCtxLoad = sh.nCtxLoad = sh.cycCtxSave = sh.nCtxSave = 0;
    sh.cycCqe = sh.nCqe = 0;
    sh.idlePolls = 0;
    for (uint32_t i = 0; i < sh.qlen; ++i) {
      m.tq[i] = p.tqSave[(size_t)b * p.maxColl + i];
      const int c = (int)(m.tq[i] & 0xffffu);
      m.prio[c] = p.ctx[(size_t)c * G + b].priority;
      m.subLo[c] = (uint32_t)p.ctx[(size_t)c * G + b].s.subSeq;
      m.subOf[c] = (uint8_t)p.ctx[(size_t)c * G + b].sub;
      m.ready[c] = 0;
    }
    for (int w = 0; w < W; ++w) m.cacheTag[w] = -1;
    pipe.tr.base = p.traceCap ? p.traceCount[b] : 0;
    pipe.tr.idx = 0;
    pipe.abortGen = 0;
    for (int i = 0; i < kMaxDepth; ++i) pipe.fail[i] = 0;
    sh.lastFetch = globaltimer();
    for (uint32_t i = 0; i < D; ++i) {
      mbar_init(&pipe.full[i], 1);
      mbar_init(&pipe.sdone[i], nComputeWarps);
      // publisher (slice published) + producer + compute warps (descriptor read):
      // every reader of ring[i] releases it directly to the control thread
      mbar_init(&pipe.empty[i], 2 + nComputeWarps);
    }
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(&tfull[i], 1);
      // every compute lane frees a stage; bulk mode: the storing lane does
      mbar_init(&tempty[i], p.bulkStores ? 1 : 32 * nComputeWarps);
      mbar_init(&tred[i], nComputeWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    p.blkStats[b].launches++;
  }
  __syncthreads();

  if (tid < 32 * kRoleWarps) {
    if (tid == 0) control_main(p, b, sh, m, pipe);
    else if (tid == 32) producer_main(p, pipe, stages, tfull, tempty);
    else if (tid == 64) publisher_main(p, b, pipe, stages, tfull, tempty, tred);
    return;
  }
  // compute warps: the data loop, left for each LL run (entered here, at the top
  // level, so that the run's registers do not constrain the data loop's)
  ComputeState cst{0, 0, 0, 0, 0, 0};
  const int ctid = tid - 32 * kRoleWarps, cnt = nComputeWarps * 32;
  for (;;) {
    const int i = compute_main(p, b, pipe, stages, tfull, tempty, tred, ctid, cnt, cst);
    if (i < 0) break;
    ll_run_dispatch(p, pipe, b, ctid, cnt);
    __syncwarp();
    if ((ctid & 31) == 0) {
      mbar_arrive(&pipe.sdone[i]);
      mbar_arrive(&pipe.empty[i]);                     // this warp is done with ring[i] too
    }
    ++cst.j;
  }
}

extern "C" size_t occl_internal_daemon_smem(int maxColl, int cacheWays, int stages) {
  return (size_t)stages * sizeof(Stage) + (size_t)cacheWays * sizeof(CtxSlot) + (size_t)cacheWays * sizeof(int) +
         (size_t)(maxColl + 1) * 4 + (size_t)maxColl * 4 + (size_t)maxColl * (4 + 1 + 1) + 16;
}

// Two builds of the daemon: one block per SM (up to 640 threads) or two blocks
// per SM (up to 384 threads each, 80 registers) -- two independent schedulers
// per SM hide each other's ring latency.
typedef void (*DaemonFn)(const DaemonParams*, int);
static DaemonFn daemon_fn(int blocksPerSM) {
  return blocksPerSM >= 2 ? occl_daemon_kernel<384, 2> : occl_daemon_kernel<kMaxBlockThreads, 1>;
}

// `pDev` points to a device-memory array of `nranks` parameter blocks (one per
// rank served by this launch, constant for the communicators' lifetime); `p` is
// the host copy of the first (all share G, maxColl and cacheWays).  The daemon is
// persistent: every block must be resident at once, otherwise blocks that never
// start would deadlock the ring -- checked against the occupancy calculator.
extern "C" int occl_internal_launch_daemon(const DaemonParams* p, const DaemonParams* pDev, int nranks,
                                           int blockThreads, void* stream) {
  const size_t smem = occl_internal_daemon_smem(p->maxColl, p->cacheWays, p->stages);
  DaemonFn fn = daemon_fn(p->blocksPerSM);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  int dev = 0, sms = 0, per = 0;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return (int)e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return (int)e;
  if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fn, blockThreads, smem)) != cudaSuccess) return (int)e;
  if ((long long)per * sms < (long long)p->G * nranks) return (int)cudaErrorCooperativeLaunchTooLarge;
  fn<<<p->G * nranks, blockThreads, smem, (cudaStream_t)stream>>>(pDev, p->G);
  return (int)cudaGetLastError();
}
