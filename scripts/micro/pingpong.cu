// One-way flag latency between two SMs (scripts/micro): block 0 and block `peer`
// (one thread each) bounce a counter N times through global memory; one-way =
// elapsed / (2N).  Variants: the load/store flavours the daemon uses for LL lines
// and connector heads, and a poll loop that also reads %globaltimer.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong pingpong.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gtimer() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint32_t smid() { uint32_t s; asm volatile("mov.u32 %0, %smid;" : "=r"(s)); return s; }

template <int V>
__device__ __forceinline__ uint32_t ld_flag(const uint32_t* p) {
  uint32_t v, a, b, c;
  if (V == 0) asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 1) asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 2) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  if (V == 3) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(v), "=r"(b), "=r"(c) : "l"(p) : "memory");
  if (V == 5) asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v), "=r"(a), "=r"(b), "=r"(c) : "l"(p) : "memory");
  if (V == 4) asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int V>
__device__ __forceinline__ void st_flag(uint32_t* p, uint32_t v) {
  if (V == 0 || V == 5) asm volatile("st.volatile.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  if (V == 1) asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  if (V == 2) asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
  if (V == 3) asm volatile("st.volatile.global.v4.u32 [%0], {%1,%1,%1,%1};" :: "l"(p), "r"(v) : "memory");
  if (V == 4) asm volatile("st.relaxed.sys.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}

template <int V, bool TIMER>
__global__ void pp(uint32_t* flags, int peer, int N, unsigned long long* out, uint32_t* sms) {
  if (threadIdx.x != 0) return;
  const int b = blockIdx.x;
  if (b != 0 && b != peer) return;
  uint32_t* mine = flags + (b == 0 ? 0 : 32);     // separate 128-B lines
  uint32_t* other = flags + (b == 0 ? 32 : 0);
  if (b == 0) sms[0] = smid(); else sms[1] = smid();
  unsigned long long t0 = gtimer(), dummy = 0;
  for (int i = 1; i <= N; ++i) {
    if (b == 0) {
      st_flag<V>(other, 2 * i - 1);
      while (ld_flag<V>(mine) != 2 * i) { if (TIMER) dummy += gtimer(); }
    } else {
      while (ld_flag<V>(mine) != 2 * i - 1) { if (TIMER) dummy += gtimer(); }
      st_flag<V>(other, 2 * i);
    }
  }
  if (b == 0) out[0] = gtimer() - t0 + (dummy == 1);
}

__global__ void timer_cost(unsigned long long* out) {
  if (threadIdx.x) return;
  long long c0 = clock64();
  unsigned long long s = 0;
  for (int i = 0; i < 1000; ++i) s += gtimer();
  out[1] = clock64() - c0 + (s == 1);
}

template <int V, bool T>
double run(uint32_t* flags, int peer, unsigned long long* out, uint32_t* sms, int N) {
  cudaMemset(flags, 0, 1024);
  pp<V, T><<<148, 32>>>(flags, peer, N, out, sms);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  return h / (2.0 * N);
}

int main() {
  uint32_t* flags; unsigned long long* out; uint32_t* sms;
  cudaMalloc(&flags, 1024); cudaMalloc(&out, 64); cudaMalloc(&sms, 8);
  const int N = 2000;
  const char* names[] = {"volatile.u32", "relaxed.gpu", "release/acquire.gpu", "volatile.v4 (LL line)", "relaxed.sys",
                         "st.volatile.u32 / ld.volatile.v4"};
  printf("{\"one_way_ns\": {");
  for (int peer : {1, 37, 74, 111, 147}) {
    double r[6], rt;
    r[0] = run<0, false>(flags, peer, out, sms, N);
    r[1] = run<1, false>(flags, peer, out, sms, N);
    r[2] = run<2, false>(flags, peer, out, sms, N);
    r[3] = run<3, false>(flags, peer, out, sms, N);
    r[4] = run<4, false>(flags, peer, out, sms, N);
    r[5] = run<5, false>(flags, peer, out, sms, N);
    rt = run<0, true>(flags, peer, out, sms, N);
    uint32_t s[2];
    cudaMemcpy(s, sms, 8, cudaMemcpyDeviceToHost);
    printf("%s\"peer%d_sm%u_%u\": {", peer == 1 ? "" : ", ", peer, s[0], s[1]);
    for (int v = 0; v < 6; ++v) printf("\"%s\": %.1f, ", names[v], r[v]);
    printf("\"volatile.u32 + globaltimer in poll loop\": %.1f}", rt);
  }
  timer_cost<<<1, 32>>>(out);
  cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("}, \"globaltimer_read_cycles\": %.1f}\n", h[1] / 1000.0);
  return 0;
}
