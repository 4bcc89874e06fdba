// HBM write ceiling on B200: pure writes (16-byte st.global, st.global.cs,
// cp.async.bulk shared->global) and a 1:4 read:write fan-out, to bound
// write-heavy plans (cfg1A writes 4 bytes per byte read).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_write_probe tools/hbm_write_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st_plain(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void st_cs(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) __stcs(p + i, v);
}
// each CTA owns contiguous 32 KiB chunks; one thread issues bulk stores of its smem buffer
__global__ void st_bulk(char* p, size_t chunks) {
  extern __shared__ __align__(128) char buf[];
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(buf));
    int inflight = 0;
    for (size_t c = blockIdx.x; c < chunks; c += gridDim.x) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 32768;" ::"l"(p + c * 32768), "r"(s) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++inflight > 6) asm volatile("cp.async.bulk.wait_group.read 6;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void fan4(const uint4* __restrict__ src, uint4* d0, uint4* d1, uint4* d2, uint4* d3, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldcs(src + i);
    __stcs(d0 + i, v); __stcs(d1 + i, v); __stcs(d2 + i, v); __stcs(d3 + i, v);
  }
}

// 4 independent 16-byte loads in flight per thread before the 16 stores
__global__ void fan4_u4(const uint4* __restrict__ src, uint4* d0, uint4* d1, uint4* d2, uint4* d3, size_t n) {
  const size_t step = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += 4 * step) {
    uint4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) if (i + k * step < n) v[k] = __ldcs(src + i + k * step);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k * step < n) {
        __stcs(d0 + i + k * step, v[k]); __stcs(d1 + i + k * step, v[k]);
        __stcs(d2 + i + k * step, v[k]); __stcs(d3 + i + k * step, v[k]);
      }
  }
}

template <class F>
float time_ms(F f) {
  for (int i = 0; i < 3; ++i) f();
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  const int it = 20;
  for (int i = 0; i < it; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / it;
}

int main() {
  const size_t bytes = size_t(1) << 30;
  char* p;
  cudaMalloc(&p, bytes * 2);
  const size_t n = bytes / 16;
  cudaFuncSetAttribute(st_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  printf("{");
  for (int per_sm : {4, 8, 16}) {
    const int g = 148 * per_sm;
    float t = time_ms([&] { st_plain<<<g, 256>>>(reinterpret_cast<uint4*>(p), n); });
    printf("\"st_plain_%d\": %.0f, ", per_sm, bytes / (t * 1e-3) / 1e9);
    t = time_ms([&] { st_cs<<<g, 256>>>(reinterpret_cast<uint4*>(p), n); });
    printf("\"st_cs_%d\": %.0f, ", per_sm, bytes / (t * 1e-3) / 1e9);
  }
  for (int per_sm : {1, 2, 4}) {
    const float t = time_ms([&] { st_bulk<<<148 * per_sm, 128, 32768>>>(p, bytes / 32768); });
    printf("\"st_bulk_%d\": %.0f, ", per_sm, bytes / (t * 1e-3) / 1e9);
  }
  {  // 1:4 fan-out: 256 MiB read (beyond L2), 1 GiB written
    const size_t m = bytes / 4 / 16;
    uint4* s = reinterpret_cast<uint4*>(p + bytes);
    uint4* d = reinterpret_cast<uint4*>(p);
    const float t = time_ms([&] { fan4<<<148 * 8, 256>>>(s, d, d + m, d + 2 * m, d + 3 * m, m); });
    printf("\"fan4_total\": %.0f, \"fan4_write\": %.0f", 1.25 * bytes / (t * 1e-3) / 1e9, bytes / (t * 1e-3) / 1e9);
    for (int per_sm : {4, 16}) {
      const float u = time_ms([&] { fan4_u4<<<148 * per_sm, 256>>>(s, d, d + m, d + 2 * m, d + 3 * m, m); });
      printf(", \"fan4_u4_%d_total\": %.0f", per_sm, 1.25 * bytes / (u * 1e-3) / 1e9);
    }
  }
  printf("}\n");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { fprintf(stderr, "%s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
