// Data-mover microbenchmark: how a daemon block should move a slice on sm_100a.
// One CTA per SM, each CTA owns a contiguous range (like a daemon lane).
//   reg   : 128-bit register loads/stores, U in flight per thread
//   tlds  : TMA (cp.async.bulk) loads into an S-stage smem ring, 16 compute warps
//           read smem and st.global.cg (the daemon's current data path)
//   tbulk : TMA loads + TMA bulk stores (cp.async.bulk.global.shared::cta), no
//           compute warps touch the data (copy primitives)
//   *add  : same with two operands and an fp32 add (reduce primitives)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mover.cu -o mover
#include <cstdio>
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
__device__ __forceinline__ void tma_store(void* g, const void* s, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(g), "r"(smem_u32(s)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ uint4 lds(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void sts(void* p, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(p)), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
}
__device__ __forceinline__ uint4 fadd4(uint4 a, uint4 b) {
  return make_uint4(__float_as_uint(__uint_as_float(a.x) + __uint_as_float(b.x)),
                    __float_as_uint(__uint_as_float(a.y) + __uint_as_float(b.y)),
                    __float_as_uint(__uint_as_float(a.z) + __uint_as_float(b.z)),
                    __float_as_uint(__uint_as_float(a.w) + __uint_as_float(b.w)));
}

template <int U, bool ADD>
__global__ void __launch_bounds__(512, 1) reg_k(const uint4* a, const uint4* b, uint4* c, size_t n) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t lo = per * blockIdx.x, hi = min(n, lo + per);
  const int nt = blockDim.x;
  for (size_t i = lo + threadIdx.x; i + (U - 1) * nt < hi; i += U * nt) {
    uint4 v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(a + i + u * nt);
    if (ADD) {
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = __ldcg(b + i + u * nt);
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = fadd4(v[u], w[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(c + i + u * nt, v[u]);
  }
}

// TMA ring of S stages x T bytes (per operand).  Warp 0 lane 0 produces; in
// BULK mode warp 1 lane 0 issues the bulk stores; warps 2.. compute.
template <int T, int S, bool ADD, bool BULK, int FX = 0>
__global__ void __launch_bounds__(576, 1) tma_k(const char* a, const char* b, char* c, size_t bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  char* in = reinterpret_cast<char*>(sm);                 // [S][T]
  char* loc = in + (size_t)S * T;                          // [S][T] (ADD)
  __shared__ uint64_t full[S], empty[S], red[S];
  const int nw = blockDim.x / 32 - 2;
  const size_t per = (bytes / gridDim.x) & ~(size_t)(T - 1);
  const size_t lo = per * blockIdx.x;
  const int ntile = (int)(per / T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], BULK ? 1 : nw);
      mbar_init(&red[s], nw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int t = 0; t < ntile; ++t) {
      const int s = t % S, u = t / S;
      if ((FX & 1) && (t % 4) == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
      mbar_wait(&empty[s], (u & 1) ^ 1);
      mbar_expect_tx(&full[s], ADD ? 2 * T : T);
      tma_load(in + (size_t)s * T, a + lo + (size_t)t * T, T, &full[s]);
      if (ADD) tma_load(loc + (size_t)s * T, b + lo + (size_t)t * T, T, &full[s]);
    }
    return;
  }
  if (tid == 32 && (FX & 8) && !BULK) {
    // fence-latency probe while the data warps stream stores
    long long tot = 0; int cnt = 0;
    const long long t_end = clock64() + 2000000;
    while (clock64() < t_end) {
      const long long t0 = clock64();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      tot += clock64() - t0; ++cnt;
    }
    if (blockIdx.x == 0) printf("fence probe (generic stores): %d fences, avg %lld cycles\n", cnt, tot / (cnt ? cnt : 1));
    return;
  }
  if (tid == 32) {
    if (!BULK) return;
    // bulk-store issuer: stage s is released once its store has READ the smem
    for (int t = 0; t < ntile; ++t) {
      const int s = t % S, u = t / S;
      if (ADD) mbar_wait(&red[s], u & 1);
      else mbar_wait(&full[s], u & 1);
      tma_store(c + lo + (size_t)t * T, in + (size_t)s * T, T);
      bulk_commit();
      if (t >= 2) {
        bulk_wait_read<2>();
        mbar_arrive(&empty[(t - 2) % S]);
      }
    }
    bulk_wait_read<0>();
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    return;
  }
  if (tid == 33 && (FX & 8) && BULK) {
    long long tot = 0; int cnt = 0;
    const long long t_end = clock64() + 2000000;
    while (clock64() < t_end) {
      const long long t0 = clock64();
      asm volatile("fence.acq_rel.gpu;" ::: "memory");
      tot += clock64() - t0; ++cnt;
    }
    if (blockIdx.x == 0) printf("fence probe (bulk stores): %d fences, avg %lld cycles\n", cnt, tot / (cnt ? cnt : 1));
    return;
  }
  if (tid < 64) return;
  if (BULK && !ADD) return;
  const int ct = tid - 64, nct = nw * 32, lane = tid & 31;
  for (int t = 0; t < ntile; ++t) {
    const int s = t % S, u = t / S;
    mbar_wait(&full[s], u & 1);
    const uint4* vi = reinterpret_cast<const uint4*>(in + (size_t)s * T);
    const uint4* vl = reinterpret_cast<const uint4*>(loc + (size_t)s * T);
    uint4* vo = reinterpret_cast<uint4*>(c + lo + (size_t)t * T);
    for (int i = ct; i < T / 16; i += nct) {
      uint4 v = lds(vi + i);
      if (ADD) v = fadd4(v, lds(vl + i));
      if (BULK) sts((void*)(vi + i), v);
      else __stcg(vo + i, v);
    }
    if (BULK) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(BULK ? &red[s] : &empty[s]);
    if ((FX & 2) && (t % 4) == 3 && lane == 0) {
      __shared__ uint32_t done;
      uint32_t old;
      asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&done)) : "memory");
      if (old == 1000000) done = 0;
    }
    if ((FX & 4) && (t % 4) == 3 && lane == 0) asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
}

typedef void (*TmaFn)(const char*, const char*, char*, size_t);

template <int T, int S, bool ADD, bool BULK, int FX = 0>
float run_tma(int g, const char* a, const char* b, char* c, size_t bytes) {
  const size_t smem = (size_t)S * T * (ADD ? 2 : 1);
  cudaFuncSetAttribute(tma_k<T, S, ADD, BULK, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    tma_k<T, S, ADD, BULK, FX><<<g, 576, smem>>>(a, b, c, bytes);
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

template <int U, bool ADD>
float run_reg(int g, const char* a, const char* b, char* c, size_t bytes) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    reg_k<U, ADD><<<g, 512>>>((const uint4*)a, (const uint4*)b, (uint4*)c, bytes / 16);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  const size_t bytes = 512ull << 20;
  char *a, *b, *c;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaMalloc(&c, bytes);
  cudaMemset(a, 1, bytes);
  cudaMemset(b, 2, bytes);
  int grids[] = {144, 18};
  for (int g : grids) {
    printf("grid %d\n", g);
    run_tma<16384, 6, false, false, 8>(g, a, b, c, bytes);
    run_tma<16384, 12, false, true, 8>(g, a, b, c, bytes);
    run_tma<16384, 6, true, false, 8>(g, a, b, c, bytes);
    run_tma<16384, 6, true, true, 8>(g, a, b, c, bytes);
  }
  return 0;
}
