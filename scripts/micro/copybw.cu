// Per-SM bandwidth calibration: plain grid-stride copy / add kernels with 1 CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

template <int U>
__global__ void __launch_bounds__(512, 1) copy_k(const uint4* __restrict__ a, uint4* __restrict__ c, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(a + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(c + i + u * stride, v[u]);
  }
  for (; i < n; i += stride) __stcg(c + i, __ldcg(a + i));
}

// contiguous-chunk variant: each CTA owns a contiguous range (like a daemon lane)
template <int U>
__global__ void __launch_bounds__(512, 1) copy_chunk_k(const uint4* __restrict__ a, uint4* __restrict__ c, size_t n) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t lo = per * blockIdx.x, hi = min(n, lo + per);
  const int nt = blockDim.x;
  size_t i = lo + threadIdx.x;
  for (; i + (U - 1) * nt < hi; i += U * nt) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(a + i + u * nt);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(c + i + u * nt, v[u]);
  }
  for (; i < hi; i += nt) __stcg(c + i, __ldcg(a + i));
}

template <int U>
__global__ void __launch_bounds__(512, 1) add_chunk_k(const uint4* __restrict__ a, const uint4* __restrict__ b,
                                                      uint4* __restrict__ c, size_t n) {
  const size_t per = (n + gridDim.x - 1) / gridDim.x;
  const size_t lo = per * blockIdx.x, hi = min(n, lo + per);
  const int nt = blockDim.x;
  size_t i = lo + threadIdx.x;
  for (; i + (U - 1) * nt < hi; i += U * nt) {
    uint4 v[U], w[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { v[u] = __ldcg(a + i + u * nt); w[u] = __ldcg(b + i + u * nt); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      float4 x = *reinterpret_cast<float4*>(&v[u]), y = *reinterpret_cast<float4*>(&w[u]);
      x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
      __stcg(c + i + u * nt, *reinterpret_cast<uint4*>(&x));
    }
  }
}

int main() {
  const size_t bytes = 256ull << 20, n = bytes / 16;
  uint4 *a, *b, *c;
  cudaMalloc(&a, bytes); cudaMalloc(&b, bytes); cudaMalloc(&c, bytes);
  cudaMemset(a, 1, bytes); cudaMemset(b, 2, bytes);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int grids[] = {18, 36, 72, 144, 148, 296, 592};
  for (int kind = 0; kind < 4; ++kind) {
    for (int g : grids) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        if (kind == 0) copy_k<8><<<g, 512>>>(a, c, n);
        else if (kind == 1) copy_chunk_k<8><<<g, 512>>>(a, c, n);
        else if (kind == 2) add_chunk_k<8><<<g, 512>>>(a, b, c, n);
        else copy_chunk_k<4><<<g, 512>>>(a, c, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
      }
      double traffic = (kind == 2 ? 3.0 : 2.0) * bytes;
      printf("%-12s grid %4d: %.3f ms  traffic %.0f GB/s  per-CTA %.1f GB/s\n",
             kind == 0 ? "copy-stride" : kind == 1 ? "copy-chunk" : kind == 2 ? "add-chunk" : "copy-chunkU4", g, best,
             traffic / best / 1e6, traffic / best / 1e6 / g);
    }
  }
  return 0;
}
