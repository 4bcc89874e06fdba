// Probe: stream wait-value / write-value across two GPUs (single process).
// GPU0 kernel sets a local flag; GPU0 copy stream waits for it (wait-value),
// copies 8 MiB to GPU1 and sets GPU1's flag (write-value on peer memory);
// GPU1 stream waits on its flag, then a kernel checks the data.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define RT(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
#define DR(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)
__global__ void setflag(unsigned* f, unsigned v) { __threadfence_system(); asm volatile("red.release.sys.global.add.u32 [%0], %1;" :: "l"(f), "r"(v) : "memory"); }
__global__ void fill(int* p, int n) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = i; }
__global__ void check(const int* p, int n, int* bad) { for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) if (p[i] != i) atomicAdd(bad, 1); }
int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  DR(cuInit(0));
  int can = 0; RT(cudaDeviceCanAccessPeer(&can, 0, 1)); printf("peer %d\n", can);
  CUdevice d0; DR(cuDeviceGet(&d0, 0)); int memops = -1; DR(cuDeviceGetAttribute(&memops, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, d0)); printf("stream mem ops v1 attr %d\n", memops);
  const int n = 2 << 20;
  int *a, *b, *bad; unsigned *f0, *f1;
  RT(cudaSetDevice(1)); RT(cudaMalloc(&b, n * 4)); RT(cudaMalloc(&f1, 4)); RT(cudaMemset(f1, 0, 4)); RT(cudaMalloc(&bad, 4)); RT(cudaMemset(bad, 0, 4));
  RT(cudaDeviceEnablePeerAccess(0, 0));
  RT(cudaSetDevice(0)); RT(cudaMalloc(&a, n * 4)); RT(cudaMalloc(&f0, 4)); RT(cudaMemset(f0, 0, 4));
  RT(cudaDeviceEnablePeerAccess(1, 0));
  cudaStream_t s0, c0, s1;
  RT(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking)); RT(cudaStreamCreateWithFlags(&c0, cudaStreamNonBlocking));
  void* pw = nullptr; void* pv = nullptr; cudaDriverEntryPointQueryResult q;
  RT(cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &pw, 12000, cudaEnableDefault, &q)); printf("ByVersion(12000) wait entry %p q=%d (direct %p)\n", pw, (int)q, (void*)&cuStreamWaitValue32);
  RT(cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &pv, 12000, cudaEnableDefault, &q)); printf("ByVersion(12000) write entry %p q=%d (direct %p)\n", pv, (int)q, (void*)&cuStreamWriteValue32);
  auto waitv = &cuStreamWaitValue32;   // cuda.h maps these to the _v2 entry points
  auto writev = &cuStreamWriteValue32;
  for (unsigned epoch = 1; epoch <= 3; ++epoch) {
    RT(cudaSetDevice(0));
    printf("epoch %u: enqueue wait on c0\n", epoch);
    DR(waitv((CUstream)c0, (CUdeviceptr)f0, epoch, CU_STREAM_WAIT_VALUE_GEQ));
    RT(cudaMemcpyAsync(b, a, n * 4, cudaMemcpyDeviceToDevice, c0));
    DR(writev((CUstream)c0, (CUdeviceptr)f1, epoch, CU_STREAM_WRITE_VALUE_DEFAULT));
    fill<<<148, 256, 0, s0>>>(a, n);
    setflag<<<1, 1, 0, s0>>>(f0, 1);
    RT(cudaStreamSynchronize(s0));
    unsigned hf = 0; RT(cudaMemcpy(&hf, f0, 4, cudaMemcpyDeviceToHost)); printf("  flag0 = %u (kernel done)\n", hf);
    printf("  c0 query: %d\n", (int)cudaStreamQuery(c0));
    RT(cudaSetDevice(1));
    if (epoch == 1) RT(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
    DR(waitv((CUstream)s1, (CUdeviceptr)f1, epoch, CU_STREAM_WAIT_VALUE_GEQ));
    printf("  enqueued wait on s1\n");
    check<<<148, 256, 0, s1>>>(b, n, bad);
    RT(cudaStreamSynchronize(s1));
    int h = -1; RT(cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost));
    printf("epoch %u ok, bad=%d\n", epoch, h);
  }
  return 0;
}
