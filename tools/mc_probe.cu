// Probe: NVLink SHARP / multicast (NVLS) support and a multimem.st round trip
// between the visible GPUs (single process).  nvcc -arch=sm_100a mc_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
__global__ void mcstore(float* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.global.f32 [%0], %1;" :: "l"(mc + i), "f"(float(i)) : "memory");
}
int main() {
  CK(cuInit(0));
  int n = 0; cudaGetDeviceCount(&n);
  for (int d = 0; d < n; ++d) {
    CUdevice dev; CK(cuDeviceGet(&dev, d)); int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("device %d multicast %d\n", d, mc);
  }
  CUmulticastObjectProp prop = {}; prop.numDevices = n; prop.handleTypes = CU_MEM_HANDLE_TYPE_NONE; size_t gran = 0;
  prop.size = 2 << 20;
  CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  prop.size = ((32 << 20) + gran - 1) / gran * gran;
  printf("granularity %zu size %zu\n", gran, prop.size);
  CUmemGenericAllocationHandle mch; CK(cuMulticastCreate(&mch, &prop));
  std::vector<CUdeviceptr> ptr(n); std::vector<CUmemGenericAllocationHandle> mem(n);
  for (int d = 0; d < n; ++d) { CUdevice dev; CK(cuDeviceGet(&dev, d)); CK(cuMulticastAddDevice(mch, dev)); }
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d);
    CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = d;
    CK(cuMemCreate(&mem[d], prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mem[d], 0, prop.size, 0));
    CK(cuMemAddressReserve(&ptr[d], prop.size, gran, 0, 0));
    CK(cuMemMap(ptr[d], prop.size, 0, mem[d], 0));
    CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = d; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(ptr[d], prop.size, &ad, 1));
  }
  CUdeviceptr mcptr; cudaSetDevice(0);
  CK(cuMemAddressReserve(&mcptr, prop.size, gran, 0, 0));
  CK(cuMemMap(mcptr, prop.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(mcptr, prop.size, &ad, 1));
  const int N = prop.size / 4;
  mcstore<<<(N + 255) / 256, 256>>>((float*)mcptr, N);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a); for (int k = 0; k < 20; ++k) mcstore<<<(N + 255) / 256, 256>>>((float*)mcptr, N); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
  printf("multimem.st %zu MiB to %d GPUs: %.3f ms = %.0f GB/s egress-equivalent per destination\n", prop.size >> 20, n, ms, prop.size / ms / 1e6);
  for (int d = 0; d < n; ++d) {
    cudaSetDevice(d); std::vector<float> h(4); cudaMemcpy(h.data(), (void*)(ptr[d] + 4 * 1000), 16, cudaMemcpyDeviceToHost);
    printf("device %d sees %.0f %.0f %.0f %.0f\n", d, h[0], h[1], h[2], h[3]);
  }
  return 0;
}
