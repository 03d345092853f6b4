// Raw data-path ceiling of one daemon block for the 8-rank ring all-reduce mix,
// WITHOUT the ring's synchronisation: every CTA moves the same slices the daemon
// moves per step (per loop: Send, 6 x RecvReduceSend, RecvReduceCopySend,
// 6 x RecvCopySend, Recv; 2 slices per step) with connector slots that stay
// L2-resident and user buffers streamed from DRAM.
// Variants: TMA staging S x 16 KiB per operand (the daemon's mover), a unified
// pool (copy slices use both halves), register loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 ringmix.cu -o ringmix
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra W_%=;\n}" ::"r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void tma_load(void* s, const void* g, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(s)), "l"(g), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_ef(void* s, const void* g, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
               ::"r"(smem_u32(s)), "l"(g), "r"(bytes), "r"(smem_u32(bar)), "l"(pol) : "memory");
}
__device__ __forceinline__ uint4 lds(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ uint4 fadd4(uint4 a, uint4 b) {
  return make_uint4(__float_as_uint(__uint_as_float(a.x) + __uint_as_float(b.x)),
                    __float_as_uint(__uint_as_float(a.y) + __uint_as_float(b.y)),
                    __float_as_uint(__uint_as_float(a.z) + __uint_as_float(b.z)),
                    __float_as_uint(__uint_as_float(a.w) + __uint_as_float(b.w)));
}
enum { RECV = 1, RED = 2, COPY = 4, SEND = 8 };
__device__ __forceinline__ int prim_of(int step, int n) {
  if (step == 0) return SEND;
  if (step < n - 1) return RECV | RED | SEND;
  if (step == n - 1) return RECV | RED | COPY | SEND;
  if (step < 2 * n - 2) return RECV | COPY | SEND;
  return RECV | COPY;
}

constexpr int kTile = 16384;
constexpr int kSlots = 4;

// Per CTA: src / dst are this CTA's DRAM streams; cin / cout its connector slots.
// POOL: tiles of 16 KiB in a ring of NT tiles; a reduce tile takes 2 consecutive.
template <int NT, bool HINT>
__global__ void __launch_bounds__(576, 1) tma_ring(const char* src0, char* dst0, char* conn0, size_t perCta,
                                                   int slice, int nloops, int n) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t full[NT], empty[NT];
  const int nw = blockDim.x / 32 - 2;
  const char* src = src0 + perCta * blockIdx.x;
  char* dst = dst0 + perCta * blockIdx.x;
  // ring of n ranks x G blocks: block b of rank r writes the connector that block b
  // of rank r+1 reads (total connector footprint n x G x kSlots x slice)
  const int G = gridDim.x / n, r = blockIdx.x / G, b = blockIdx.x % G;
  char* cin = conn0 + (size_t)blockIdx.x * kSlots * slice;
  char* cout = conn0 + (size_t)(((r + 1) % n) * G + b) * kSlots * slice;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NT; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], nw); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tid = threadIdx.x;
  const int tilesPerSlice = slice / kTile;
  if (tid == 32) return;
  // walk the same sequence in producer and consumers
  const bool producer = tid == 0;
  const int ct = tid - 64, nct = nw * 32, lane = tid & 31;
  if (!producer && tid < 64) return;
  uint32_t t = 0;          // tile slot counter (pool position)
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint64_t nsend = 0, nrecv = 0;
  for (int l = 0; l < nloops; ++l)
    for (int step = 0; step < 2 * n - 1; ++step)
      for (int sl = 0; sl < 2; ++sl) {
        const int prim = prim_of(step, n);
        const int seg = (step * 7 + l) % n;   // segment offsets: just spread over the stream
        const size_t off = ((size_t)l * 2 + sl) * slice + (size_t)seg * ((size_t)nloops * 2 * slice);
        const char* in = (prim & RECV) ? cin + (nrecv % kSlots) * slice : src + off;
        char* o = cout + (nsend % kSlots) * slice;
        for (int k = 0; k < tilesPerSlice; ++k) {
          const int need = (prim & RED) ? 2 : 1;
          const uint32_t s0 = t % NT, s1 = (t + 1) % NT;
          const uint32_t p0 = (t / NT) & 1, p1 = ((t + 1) / NT) & 1;
          if (producer) {
            mbar_wait(&empty[s0], p0 ^ 1);
            mbar_expect_tx(&full[s0], kTile);
            if (HINT && !(prim & RECV)) tma_load_ef(sm + (size_t)s0 * kTile, in + (size_t)k * kTile, kTile, &full[s0], pol);
            else tma_load(sm + (size_t)s0 * kTile, in + (size_t)k * kTile, kTile, &full[s0]);
            if (need == 2) {
              mbar_wait(&empty[s1], p1 ^ 1);
              mbar_expect_tx(&full[s1], kTile);
              if (HINT) tma_load_ef(sm + (size_t)s1 * kTile, src + off + (size_t)k * kTile, kTile, &full[s1], pol);
              else tma_load(sm + (size_t)s1 * kTile, src + off + (size_t)k * kTile, kTile, &full[s1]);
            }
          } else {
            mbar_wait(&full[s0], p0);
            if (need == 2) mbar_wait(&full[s1], p1);
            if (HINT && (prim & RECV) && ct < kTile / 128)
              asm volatile("discard.global.L2 [%0], 128;" ::"l"(in + (size_t)k * kTile + ct * 128) : "memory");
            const uint4* vi = reinterpret_cast<const uint4*>(sm + (size_t)s0 * kTile);
            const uint4* vl = reinterpret_cast<const uint4*>(sm + (size_t)s1 * kTile);
            uint4* vd = reinterpret_cast<uint4*>(dst + off + (size_t)k * kTile);
            uint4* vo = reinterpret_cast<uint4*>(o + (size_t)k * kTile);
            for (int i = ct; i < kTile / 16; i += nct) {
              uint4 v = lds(vi + i);
              if (prim & RED) v = fadd4(v, lds(vl + i));
              if (prim & COPY) {
                if (HINT) asm volatile("st.global.cg.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(vd + i),
                                       "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
                else __stcg(vd + i, v);
              }
              if (prim & SEND) __stcg(vo + i, v);
            }
            __syncwarp();
            if (lane == 0) {
              mbar_arrive(&empty[s0]);
              if (need == 2) mbar_arrive(&empty[s1]);
            }
          }
          t += need;
        }
        if (prim & SEND) ++nsend;
        if (prim & RECV) ++nrecv;
      }
}

template <int NT, bool HINT>
float run(int g, const char* src, char* dst, char* conn, size_t perCta, int slice, int nloops, int n) {
  const size_t smem = (size_t)NT * kTile;
  cudaFuncSetAttribute(tma_ring<NT, HINT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0);
    tma_ring<NT, HINT><<<g, 576, smem>>>(src, dst, conn, perCta, slice, nloops, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("err %s\n", cudaGetErrorString(e));
  return best;
}

int main(int argc, char** argv) {
  const int n = 8, g = 144, slice = (argc > 1 ? atoi(argv[1]) : 128) << 10;
  const int nloops = 7 * (128 << 10) / slice;            // ~1.78 MiB per segment per block
  const size_t perCta = (size_t)n * nloops * 2 * slice;  // this CTA's share of the rank buffer
  char *src, *dst, *conn;
  cudaMalloc(&src, perCta * g);
  cudaMalloc(&dst, perCta * g);
  cudaMalloc(&conn, (size_t)g * kSlots * slice);
  cudaMemset(src, 0, perCta * g);
  const double slicesPerCta = (double)nloops * (2 * n - 1) * 2;
  auto pr = [&](const char* nm, float ms) {
    printf("slice %dK %-22s %.3f ms  per-slice %.2f us\n", slice >> 10, nm, ms, ms * 1e3 / slicesPerCta);
  };
  pr("pool 12x16K", run<12, false>(g, src, dst, conn, perCta, slice, nloops, n));
  pr("pool 12x16K hints", run<12, true>(g, src, dst, conn, perCta, slice, nloops, n));
  pr("pool 8x16K hints", run<8, true>(g, src, dst, conn, perCta, slice, nloops, n));
  return 0;
}
