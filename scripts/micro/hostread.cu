// Host-memory read latency microbenchmark (the daemon's SQ fetch):
// how long does ONE thread take to read k x 16 B of pinned, mapped host memory?
//   relaxed_sys : k independent ld.relaxed.sys.global.v4 (the daemon's sq_fetch)
//   volatile    : k independent ld.volatile.global.v4
//   weak_cv     : k independent ld.global.cv.v4 (weak, "don't cache")
//   warp        : the k chunks read by k lanes of one warp (one coalesced load)
//   bulk        : one cp.async.bulk of k x 16 B into shared memory (TMA), mbarrier wait
//   dev_l2      : relaxed_sys on device memory (reference: an L2 round trip)
// Each variant: 200 repetitions (host rewrites nothing; the data is constant), the
// median of %globaltimer deltas in ns, for k = 1, 4, 20.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 hostread.cu -o hostread
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t gt() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

constexpr int REPS = 200;
constexpr int KMAX = 32;

template <int MODE>
__global__ void kread(const uint4* src, int k, uint64_t* out, uint32_t* sink) {
  __shared__ __align__(128) uint4 buf[KMAX];
  __shared__ __align__(8) uint64_t bar;
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t acc = 0, phase = 0;
  for (int rep = 0; rep < REPS; ++rep) {
    __syncwarp();
    const uint64_t t0 = gt();
    if (MODE == 3) {                                     // warp: lane i reads chunk i
      if (lane < k) {
        uint4 v;
        asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + lane) : "memory");
        acc += v.x + v.w;
      }
      __syncwarp();
    } else if (lane == 0) {
      if (MODE == 4) {                                   // bulk copy into smem
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;"
                     ::"r"(smem_u32(&bar)), "r"(k * 16) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(smem_u32(buf)), "l"(src), "r"(k * 16), "r"(smem_u32(&bar)) : "memory");
        asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
                     " @!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
        phase ^= 1;
        acc += buf[k - 1].x;
      } else {
        uint4 v[KMAX];
#pragma unroll
        for (int i = 0; i < KMAX; ++i) {
          if (i < k) {
            if (MODE == 0 || MODE == 5)
              asm volatile("ld.relaxed.sys.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "l"(src + i) : "memory");
            else if (MODE == 1)
              asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "l"(src + i) : "memory");
            else
              asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                           : "=r"(v[i].x), "=r"(v[i].y), "=r"(v[i].z), "=r"(v[i].w) : "l"(src + i) : "memory");
          }
        }
#pragma unroll
        for (int i = 0; i < KMAX; ++i)
          if (i < k) acc += v[i].x ^ v[i].w;
      }
    }
    __syncwarp();
    const uint64_t t1 = gt();
    if (lane == 0) out[rep] = t1 - t0;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}

template <int MODE>
static double run(const uint4* src, int k, uint64_t* dout, uint32_t* sink) {
  kread<MODE><<<1, 32>>>(src, k, dout, sink);
  cudaDeviceSynchronize();
  std::vector<uint64_t> h(REPS);
  cudaMemcpy(h.data(), dout, REPS * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  std::sort(h.begin() + 10, h.end());               // first 10: warm-up
  return (double)h[10 + (REPS - 10) / 2];
}

int main() {
  uint4* host;
  cudaHostAlloc(&host, KMAX * 16, cudaHostAllocMapped);
  for (int i = 0; i < KMAX; ++i) host[i] = make_uint4(i, i + 1, i + 2, i + 3);
  uint4* hdev;
  cudaHostGetDevicePointer(&hdev, host, 0);
  uint4* dev;
  cudaMalloc(&dev, KMAX * 16);
  cudaMemcpy(dev, host, KMAX * 16, cudaMemcpyHostToDevice);
  uint64_t* dout;
  uint32_t* sink;
  cudaMalloc(&dout, REPS * sizeof(uint64_t));
  cudaMalloc(&sink, 4);
  printf("{");
  const int ks[] = {1, 4, 20};
  bool first = true;
  for (int k : ks) {
    const double r[6] = {run<0>(hdev, k, dout, sink), run<1>(hdev, k, dout, sink), run<2>(hdev, k, dout, sink),
                         run<3>(hdev, k, dout, sink), run<4>(hdev, k, dout, sink), run<5>(dev, k, dout, sink)};
    const char* names[6] = {"relaxed_sys", "volatile", "weak_cv", "warp", "bulk", "dev_l2"};
    for (int m = 0; m < 6; ++m) {
      printf("%s\"%s_k%d_ns\": %.0f", first ? "" : ", ", names[m], k, r[m]);
      first = false;
    }
  }
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
