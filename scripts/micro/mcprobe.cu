// NVLS feasibility probe in C (scripts/micro): can this lease create a multicast
// object (cuMulticastCreate) with one device, bind memory and run multimem
// instructions on it?  Prints one JSON line with each step's CUresult.
// nvcc -gencode arch=compute_100a,code=sm_100a -o mcprobe mcprobe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>

__global__ void mm_kernel(float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i * 4 >= n) return;
  float4 v;
  asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(mc + 4 * i) : "memory");
  reinterpret_cast<float4*>(out)[i] = v;
}

int main() {
  CUresult r;
  cuInit(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUcontext ctx; cuDevicePrimaryCtxRetain(&ctx, dev); cuCtxSetCurrent(ctx);
  int mcs = -1; cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("{\"multicast_supported\": %d", mcs);
  const CUmemAllocationHandleType types[] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                             CU_MEM_HANDLE_TYPE_FABRIC};
  const char* names[] = {"none", "posix_fd", "fabric"};
  for (int t = 0; t < 3; ++t) {
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.handleTypes = types[t];
    prop.flags = 0;
    size_t gran = 0;
    r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    prop.size = gran ? gran : (2 << 20);
    CUmemGenericAllocationHandle mc = 0;
    CUresult rc = cuMulticastCreate(&mc, &prop);
    printf(", \"%s\": {\"granularity\": [%d, %zu], \"create\": %d", names[t], (int)r, gran, (int)rc);
    if (rc == CUDA_SUCCESS) {
      CUresult ra = cuMulticastAddDevice(mc, dev);
      CUmemAllocationProp ap = {};
      ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
      ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      ap.location.id = 0;
      ap.requestedHandleTypes = types[t];
      CUmemGenericAllocationHandle mh = 0;
      CUresult rm = cuMemCreate(&mh, prop.size, &ap, 0);
      CUresult rb = rm == CUDA_SUCCESS ? cuMulticastBindMem(mc, 0, mh, 0, prop.size, 0) : rm;
      CUdeviceptr va = 0;
      CUresult rr = cuMemAddressReserve(&va, prop.size, 0, 0, 0);
      CUresult rmap = rr == CUDA_SUCCESS ? cuMemMap(va, prop.size, 0, mc, 0) : rr;
      CUmemAccessDesc ad = {};
      ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
      CUresult racc = rmap == CUDA_SUCCESS ? cuMemSetAccess(va, prop.size, &ad, 1) : rmap;
      printf(", \"add_device\": %d, \"mem_create\": %d, \"bind\": %d, \"map\": %d, \"access\": %d", (int)ra, (int)rm,
             (int)rb, (int)rmap, (int)racc);
      if (racc == CUDA_SUCCESS) {
        float* out; cudaMalloc(&out, 4096 * sizeof(float));
        mm_kernel<<<4, 256>>>((float*)va, out, 4096);
        cudaError_t ke = cudaDeviceSynchronize();
        printf(", \"multimem_kernel\": %d", (int)ke);
      }
    }
    printf("}");
  }
  printf("}\n");
  return 0;
}
