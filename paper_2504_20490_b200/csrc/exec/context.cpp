// hshard-b200 executor: per-GPU context (symmetric arena, peer mapping, barriers).
//
// One process per GPU.  Every rank allocates an arena of the same size and
// carves shards out of it with the same sequence of bump allocations, so an
// (rank, offset) pair names a buffer on any GPU.  Peers' arenas are mapped
// once through CUDA IPC (cudaIpcOpenMemHandle with lazy peer access), after
// which a kernel on this GPU can load any peer's shard directly over NVLink.
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <string>

#include "nccl_dyn.hpp"
#include "program.hpp"

namespace hshard::exec {

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

Context::Context(int rank, int world, int gpu, size_t arena_bytes)
    : rank_(rank), world_(world), gpu_(gpu) {
  if (world < 1 || rank < 0 || rank >= world) fail(Errc::UnknownDevice, "bad rank/world");
  cuda_check(cudaSetDevice(gpu), "cudaSetDevice");
  cuda_check(cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, gpu), "SM count");
  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  arena_bytes_ = arena_bytes;
  if (arena_bytes_ > 0) cuda_check(cudaMalloc(&arena_, arena_bytes_), "cudaMalloc(arena)");
  cuda_check(cudaMalloc(&flags_, 256 * sizeof(unsigned int)), "cudaMalloc(flags)");
  cuda_check(cudaMemset(flags_, 0, 256 * sizeof(unsigned int)), "cudaMemset(flags)");
  cuda_check(cudaMalloc(&barrier_error_, sizeof(int)), "cudaMalloc(err)");
  cuda_check(cudaMemset(barrier_error_, 0, sizeof(int)), "cudaMemset(err)");
  cuda_check(cudaMalloc(&counter_, sizeof(unsigned long long)), "cudaMalloc(counter)");
  cuda_check(cudaMalloc(&d_peer_flags_, world * sizeof(unsigned int*)), "cudaMalloc(peers)");
  peer_arena_.assign(world, nullptr);
  peer_flags_.assign(world, nullptr);
  peer_arena_[rank] = arena_;
  peer_flags_[rank] = flags_;
  cuda_check(cudaMemcpy(d_peer_flags_, peer_flags_.data(), world * sizeof(unsigned int*),
                        cudaMemcpyHostToDevice),
             "cudaMemcpy(peers)");
  const char* pool_mb = std::getenv("HS_TABLE_POOL_MB");
  pool_ = std::make_shared<TablePool>(gpu, static_cast<size_t>(pool_mb ? std::atoll(pool_mb) : 1024) << 20);
  cuda_check(cudaDeviceSynchronize(), "context init");
}

TablePool::TablePool(int gpu, size_t bytes) : gpu_(gpu) {
  if (bytes && cudaMalloc(&base_, bytes) == cudaSuccess) {
    bytes_ = bytes;
    free_[0] = bytes;
  } else {
    cudaGetLastError();  // no pool: every table block is a cudaMalloc
    base_ = nullptr;
  }
}

TablePool::~TablePool() {
  if (base_) {
    cudaSetDevice(gpu_);
    cudaFree(base_);
  }
}

void* TablePool::alloc(size_t bytes) {
  bytes = (std::max<size_t>(bytes, 1) + 255) & ~size_t{255};
  {
    std::lock_guard<std::mutex> lock(mu_);
    for (auto it = free_.begin(); it != free_.end(); ++it)
      if (it->second >= bytes) {
        const size_t off = it->first, left = it->second - bytes;
        free_.erase(it);
        if (left) free_[off + bytes] = left;
        used_[off] = bytes;
        return base_ + off;
      }
  }
  void* p = nullptr;
  cuda_check(cudaMalloc(&p, bytes), "cudaMalloc(tables)");
  return p;
}

void TablePool::free(void* p) {
  char* c = static_cast<char*>(p);
  if (!base_ || c < base_ || c >= base_ + bytes_) {
    cudaFree(p);
    return;
  }
  std::lock_guard<std::mutex> lock(mu_);
  const size_t off = static_cast<size_t>(c - base_);
  auto u = used_.find(off);
  if (u == used_.end()) return;
  size_t start = off, len = u->second;
  used_.erase(u);
  auto next = free_.lower_bound(start);
  if (next != free_.end() && next->first == start + len) {
    len += next->second;
    next = free_.erase(next);
  }
  if (next != free_.begin()) {
    auto prev = std::prev(next);
    if (prev->first + prev->second == start) {
      start = prev->first;
      len += prev->second;
      free_.erase(prev);
    }
  }
  free_[start] = len;
}

Context::Context(AnalysisTag, int rank, int world) : rank_(rank), world_(world), gpu_(-1) {
  if (world < 1 || rank < 0 || rank >= world) fail(Errc::UnknownDevice, "bad rank/world");
  analysis_ = true;
  arena_bytes_ = size_t{1} << 44;
  peer_arena_.resize(world);
  for (int r = 0; r < world; ++r)  // disjoint, 4 KiB-aligned virtual bases
    peer_arena_[r] = reinterpret_cast<char*>((uintptr_t{1} << 46) * static_cast<uintptr_t>(r + 1));
  arena_ = peer_arena_[rank];
  peers_open_ = true;
}

std::unique_ptr<Context> Context::analysis(int rank, int world) {
  return std::unique_ptr<Context>(new Context(AnalysisTag{}, rank, world));
}

Context::~Context() {
  if (analysis_) return;
  cudaSetDevice(gpu_);
  cudaDeviceSynchronize();
  if (nccl_comm_) nccl::api().CommDestroy(static_cast<ncclComm_t>(nccl_comm_));
  for (auto& [key, p] : imported_) cudaIpcCloseMemHandle(p);
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    if (peer_arena_[r]) cudaIpcCloseMemHandle(peer_arena_[r]);
    if (peer_flags_[r]) cudaIpcCloseMemHandle(peer_flags_[r]);
  }
  pool_.reset();  // the device block goes with the last program still holding it
  cudaFree(d_peer_flags_);
  cudaFree(counter_);
  cudaFree(barrier_error_);
  cudaFree(flags_);
  if (arena_) cudaFree(arena_);
  if (stream_) cudaStreamDestroy(stream_);
}

char* Context::arena_of(int r) const {
  if (r < 0 || r >= world_) fail(Errc::UnknownDevice, "rank " + std::to_string(r) + " out of range");
  if (!peer_arena_[r]) fail(Errc::CommError, "peer arena " + std::to_string(r) + " not mapped");
  return peer_arena_[r];
}

void Context::ipc_handles(unsigned char out[128]) const {
  cudaIpcMemHandle_t a{}, f{};
  if (arena_) cuda_check(cudaIpcGetMemHandle(&a, arena_), "cudaIpcGetMemHandle(arena)");
  cuda_check(cudaIpcGetMemHandle(&f, flags_), "cudaIpcGetMemHandle(flags)");
  std::memcpy(out, &a, 64);
  std::memcpy(out + 64, &f, 64);
}

void Context::open_peers(const unsigned char* all) {
  if (peers_open_) return;
  cuda_check(cudaSetDevice(gpu_), "cudaSetDevice");
  for (int r = 0; r < world_; ++r) {
    if (r == rank_) continue;
    cudaIpcMemHandle_t a, f;
    std::memcpy(&a, all + 128 * r, 64);
    std::memcpy(&f, all + 128 * r + 64, 64);
    void* pa = nullptr;
    void* pf = nullptr;
    cuda_check(cudaIpcOpenMemHandle(&pa, a, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle(arena)");
    cuda_check(cudaIpcOpenMemHandle(&pf, f, cudaIpcMemLazyEnablePeerAccess),
               "cudaIpcOpenMemHandle(flags)");
    peer_arena_[r] = static_cast<char*>(pa);
    peer_flags_[r] = static_cast<unsigned int*>(pf);
  }
  cuda_check(cudaMemcpy(d_peer_flags_, peer_flags_.data(), world_ * sizeof(unsigned int*),
                        cudaMemcpyHostToDevice),
             "cudaMemcpy(peers)");
  peers_open_ = true;
}

size_t Context::alloc(size_t bytes) {
  const size_t off = (cursor_ + 255) & ~size_t{255};
  if (off + bytes > arena_bytes_)
    fail(Errc::CudaError, "arena exhausted: need " + std::to_string(off + bytes) + " of " +
                              std::to_string(arena_bytes_) + " bytes");
  cursor_ = off + bytes;
  return off;
}

void Context::reset_alloc(size_t offset) {
  if (offset > arena_bytes_) fail(Errc::CudaError, "reset beyond arena");
  cursor_ = offset;
}

void Context::barrier(cudaStream_t s) {
  if (world_ == 1) return;
  if (!peers_open_) fail(Errc::CommError, "barrier before open_peers");
  ++epoch_;
  cuda_check(launch_barrier(d_peer_flags_, world_, rank_, epoch_, 20ull * 1000 * 1000 * 1000,
                            barrier_error_, s),
             "barrier launch");
}

void Context::nccl_init(const unsigned char id[128]) {
  if (nccl_comm_) return;
  ncclUniqueId uid;
  static_assert(sizeof(uid) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(&uid, id, sizeof(uid));
  cuda_check(cudaSetDevice(gpu_), "cudaSetDevice");
  ncclComm_t comm;
  nccl::check(nccl::api().CommInitRank(&comm, world_, uid, rank_), "ncclCommInitRank");
  nccl_comm_ = comm;
}

void Context::check_barrier_error() {
  int err = 0;
  cuda_check(cudaMemcpy(&err, barrier_error_, sizeof(int), cudaMemcpyDeviceToHost), "barrier err");
  if (err) fail(Errc::DeadlockDetected, "cross-rank barrier timed out (a peer never arrived)");
}

// cuMemGetAddressRange through the runtime's driver entry point (no link
// against libcuda): the base and size of the allocation holding `ptr`.
namespace {
using GetRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
GetRangeFn get_range() {
  static GetRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<GetRangeFn>(f);
  }();
  return fn;
}
}  // namespace

void Context::ipc_export(const void* ptr, unsigned char out[80]) const {
  GetRangeFn range = get_range();
  if (!range) fail(Errc::CudaError, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, reinterpret_cast<unsigned long long>(ptr)) != 0)
    fail(Errc::CudaError, "ipc_export: not a device allocation");
  cudaIpcMemHandle_t h{};
  cuda_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle(buffer)");
  const uint64_t off = reinterpret_cast<uint64_t>(ptr) - base, sz = size;
  std::memcpy(out, &h, 64);
  std::memcpy(out + 64, &off, 8);
  std::memcpy(out + 72, &sz, 8);
}

char* Context::ipc_import(const unsigned char in[80]) {
  uint64_t off = 0;
  std::memcpy(&off, in + 64, 8);
  const std::string key(reinterpret_cast<const char*>(in), 64);
  auto it = imported_.find(key);
  if (it == imported_.end()) {
    cudaIpcMemHandle_t h{};
    std::memcpy(&h, in, 64);
    void* p = nullptr;
    cuda_check(cudaSetDevice(gpu_), "cudaSetDevice");
    cuda_check(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle(buffer)");
    it = imported_.emplace(key, static_cast<char*>(p)).first;
  }
  return it->second + off;
}

void Context::clear_error() {
  if (analysis_) return;
  cuda_check(cudaDeviceSynchronize(), "clear_error sync");
  cuda_check(cudaMemset(barrier_error_, 0, sizeof(int)), "clear_error");
}

}  // namespace hshard::exec
