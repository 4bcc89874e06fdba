// Probe: NVLink bandwidth per SM for register stores (st.global.v4), TMA bulk
// stores (cp.async.bulk.global.shared::cta) and TMA bulk loads from a peer,
// with K CTAs (one per SM).  Single process, GPU0 -> GPU1 memory.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#define RT(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
constexpr int CHUNK = 32 * 1024;
__device__ __forceinline__ uint32_t sptr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void st_kernel(uint4* dst, size_t n_vec_per_cta) {
  uint4* d = dst + blockIdx.x * n_vec_per_cta;
  uint4 v = make_uint4(blockIdx.x, 1, 2, 3);
  for (size_t i = threadIdx.x; i < n_vec_per_cta; i += blockDim.x) d[i] = v;
}

__global__ void bulk_store_kernel(char* dst, size_t bytes_per_cta, int inflight) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < CHUNK * 4 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  char* d = dst + blockIdx.x * bytes_per_cta;
  int k = 0;
  for (size_t off = 0; off < bytes_per_cta; off += CHUNK, ++k) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(d + off), "r"(sptr(sm + (k % 4) * CHUNK)), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (inflight == 2) asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory");
    else if (inflight == 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 32;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void bulk_load_kernel(const char* src, size_t bytes_per_cta, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int s = 0; s < 4; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sptr(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const char* s0 = src + blockIdx.x * bytes_per_cta;
  const int n = static_cast<int>(bytes_per_cta / CHUNK);
  for (int k = 0; k < n; ++k) {
    const int s = k % 4;
    if (k >= 4) {  // wait for the stage's previous load
      const uint32_t parity = ((k / 4) - 1) & 1;
      uint32_t ok = 0;
      while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sptr(&bar[s])), "r"(parity) : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sptr(&bar[s])), "r"(CHUNK) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" :: "r"(sptr(sm + s * CHUNK)), "l"(s0 + static_cast<size_t>(k) * CHUNK), "r"(CHUNK), "r"(sptr(&bar[s])) : "memory");
  }
  for (int k = n; k < n + 4; ++k) {  // drain
    const int s = k % 4;
    const uint32_t parity = ((k / 4) - 1) & 1;
    uint32_t ok = 0;
    while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(ok) : "r"(sptr(&bar[s])), "r"(parity) : "memory");
  }
  sink[blockIdx.x] = sm[7];
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const size_t total = 512ull << 20;
  char *remote, *local; unsigned long long* sink;
  RT(cudaSetDevice(1)); RT(cudaMalloc(&remote, total)); RT(cudaDeviceEnablePeerAccess(0, 0));
  RT(cudaSetDevice(0)); RT(cudaMalloc(&local, total)); RT(cudaMalloc(&sink, 148 * 8)); RT(cudaDeviceEnablePeerAccess(1, 0));
  RT(cudaFuncSetAttribute(bulk_store_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * CHUNK));
  RT(cudaFuncSetAttribute(bulk_load_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * CHUNK));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int ks[] = {1, 2, 4, 8, 16, 32, 64, 148};
  for (int K : ks) {
    const size_t per = (total / K) / CHUNK * CHUNK;
    float ms[4];
    for (int mode = 0; mode < 4; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) st_kernel<<<K, 512>>>(reinterpret_cast<uint4*>(remote), per / 16);
        if (mode == 1) bulk_store_kernel<<<K, 128, 4 * CHUNK>>>(remote, per, 2);
        if (mode == 2) bulk_store_kernel<<<K, 128, 4 * CHUNK>>>(remote, per, 32);
        if (mode == 3) bulk_load_kernel<<<K, 32, 4 * CHUNK>>>(remote, per, sink);
        cudaEventRecord(b); RT(cudaEventSynchronize(b));
        cudaEventElapsedTime(&ms[mode], a, b);
      }
    }
    const double gb = double(per) * K / 1e9;
    printf("K=%3d  st.global %6.1f GB/s (%5.1f/SM) | bulk store 2-deep %6.1f (%5.1f/SM) | 32-deep %6.1f (%5.1f/SM) | bulk load from peer %6.1f (%5.1f/SM)\n", K,
           gb / ms[0] * 1e3, gb / ms[0] * 1e3 / K, gb / ms[1] * 1e3, gb / ms[1] * 1e3 / K, gb / ms[2] * 1e3, gb / ms[2] * 1e3 / K,
           gb / ms[3] * 1e3, gb / ms[3] * 1e3 / K);
  }
  return 0;
}
