// HBM read-heavy ceilings on B200, to bound read-dominated plans (cfg2e's
// fused program reads 4 bytes per byte written): pure streaming reads, and a
// k:1 read:write reduction (k input streams summed into one output), with
// plain register loads (several vectors in flight per thread) at a range of
// grid sizes.  Prints GB/s (read + write bytes / time, best of 10).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/hbm_read_probe tools/hbm_read_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

// pure reads: every thread folds U vectors per iteration into a register sum
template <int U>
__global__ void rd_only(const uint4* __restrict__ p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n ? __ldcs(p + i + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;  // keeps the loads alive
}

// k-term bf16x2 sums in fp32 (the cfg2e phase shape), one output stream
template <int K>
__global__ void rd_k_wr_1(const uint4* const* __restrict__ in, uint4* __restrict__ out, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint4 v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __ldcs(in[k] + i);
    uint4 r = v[0];
#pragma unroll
    for (int k = 1; k < K; ++k) {
      r.x += v[k].x;  // integer adds: the probe measures bytes, not arithmetic
      r.y += v[k].y;
      r.z += v[k].z;
      r.w += v[k].w;
    }
    __stcs(out + i, r);
  }
}

template <class F>
float best_ms(F&& launch) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t bytes = size_t{1} << 30;  // 1 GiB per stream (>> 126 MB L2)
  const size_t n = bytes / 16;
  uint4* buf[7];
  for (auto& b : buf) {
    cudaMalloc(&b, bytes);
    cudaMemset(b, 1, bytes);
  }
  unsigned* sink;
  cudaMalloc(&sink, 4);
  const uint4** ins;
  cudaMalloc(&ins, 6 * sizeof(void*));
  cudaMemcpy(ins, buf, 6 * sizeof(void*), cudaMemcpyHostToDevice);
  printf("{\"sms\": %d", sms);
  for (int per_sm : {4, 8, 16}) {
    const int grid = sms * per_sm;
    float ms = best_ms([&] { rd_only<4><<<grid, 256>>>(buf[0], n, sink); });
    printf(", \"read_only_u4_g%d\": %.0f", per_sm, bytes / (ms * 1e-3) / 1e9);
    ms = best_ms([&] { rd_k_wr_1<4><<<grid, 256>>>(ins, buf[6], n); });
    printf(", \"read4_write1_g%d\": %.0f", per_sm, 5.0 * bytes / (ms * 1e-3) / 1e9);
    ms = best_ms([&] { rd_k_wr_1<6><<<grid, 256>>>(ins, buf[6], n); });
    printf(", \"read6_write1_g%d\": %.0f", per_sm, 7.0 * bytes / (ms * 1e-3) / 1e9);
    ms = best_ms([&] { rd_k_wr_1<1><<<grid, 256>>>(ins, buf[6], n); });
    printf(", \"copy_g%d\": %.0f", per_sm, 2.0 * bytes / (ms * 1e-3) / 1e9);
  }
  printf("}\n");
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
