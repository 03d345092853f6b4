// testgen.cu -- GPU implementation of the seeded counter-based input generator
// of inputs/hashgen.py (SURVEY.md §8(c) "Inputs").  TEST/BENCH SUPPORT ONLY: it
// is built into its own library (libocclgen.so), holds none of the collective
// method's arithmetic, and is never called by the product path.
//
//   u = splitmix64(seed ^ (coll << 40) ^ (rank << 32) ^ i)
//   f32 : (int(u >> 40) - 2^23) * 2^(-23 - ((u >> 32) & 7))
//   bf16: (int(u >> 56) - 128)  * 2^(-7  - ((u >> 32) & 7))   (exact, top 16 bits)
//   f16 : (int(u >> 53) - 1024) * 2^(-10 - ((u >> 32) & 7))  (exact in binary16)
//   i32 : low 32 bits of u
//   i64 : all 64 bits of u
//   f64 : (int(u >> 11) - 2^52) * 2^(-52 - ((u >> 32) & 7))   (exact in binary64)
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <stdint.h>

namespace {
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(void* dst, uint64_t count, int dtype, uint64_t base, uint64_t offset) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t u = splitmix64(base ^ (offset + i));
    const int e = (int)((u >> 32) & 7);
    if (dtype == 0) {
      reinterpret_cast<uint32_t*>(dst)[i] = (uint32_t)(u & 0xFFFFFFFFull);
    } else if (dtype == 1) {
      const int m = (int)(u >> 40) - (1 << 23);
      reinterpret_cast<float*>(dst)[i] = ldexpf((float)m, -23 - e);
    } else if (dtype == 2) {
      const int m = (int)(u >> 56) - 128;
      const float f = ldexpf((float)m, -7 - e);
      reinterpret_cast<uint16_t*>(dst)[i] = (uint16_t)(__float_as_uint(f) >> 16);
    } else if (dtype == 3) {
      const int m = (int)(u >> 53) - 1024;
      reinterpret_cast<__half*>(dst)[i] = __float2half_rn(ldexpf((float)m, -10 - e));   // exact
    } else if (dtype == 4) {
      reinterpret_cast<uint64_t*>(dst)[i] = u;
    } else {
      const long long m = (long long)(u >> 11) - (1ll << 52);
      reinterpret_cast<double*>(dst)[i] = ldexp((double)m, -52 - e);                      // exact
    }
  }
}
}  // namespace

extern "C" int occlTestFill(void* dst, uint64_t count, int dtype, uint64_t seed, uint32_t coll, uint32_t rank,
                            uint64_t offset, void* stream) {
  if (count == 0) return 0;
  const uint64_t base = seed ^ ((uint64_t)coll << 40) ^ ((uint64_t)rank << 32);
  int blocks = (int)((count + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(dst, count, dtype, base, offset);
  return (int)cudaGetLastError();
}
