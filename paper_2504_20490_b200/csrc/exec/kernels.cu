// hshard-b200 executor kernels (sm_100a).
//
// box_phase_kernel: one persistent launch per plan phase.  Each CTA walks
// work items (grid-stride); an item is a run of rows of one task's box.
// Per 16-byte vector a thread issues one streaming load per term (local HBM
// or a peer GPU's HBM over NVLink), accumulates in the dtype's accumulator in
// term order, rounds once and issues one streaming store.  Loads of UNROLL
// vectors are in flight per thread per term, so a 2048-thread SM keeps
// ~128 KB of reads outstanding -- enough to saturate HBM3e (and NVLink for
// peer terms) without TMA: the boxes are already row-contiguous, there is no
// transpose to stage through shared memory, and every byte is touched once.
#include <cstdint>

#include "kernels.cuh"

namespace hshard::exec {

namespace {

constexpr int kBlock = 512;
constexpr int kUnroll = 4;        // vectors in flight per thread (copy)
constexpr int kUnrollReduce = 2;  // per term (reduce: accumulators live in registers)

// ---------------------------------------------------------------- arithmetic
template <class T>
struct Arith;

template <>
struct Arith<uint16_t> {  // bf16 stored as raw bits
  using A = float;
  __device__ static A widen(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
  __device__ static uint16_t narrow(A f) {
    const uint32_t u = __float_as_uint(f);
    return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
  }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
};

template <>
struct Arith<float> {
  using A = float;
  __device__ static A widen(float v) { return v; }
  __device__ static float narrow(A v) { return v; }
  __device__ static A add(A a, A b) { return __fadd_rn(a, b); }
};

template <>
struct Arith<double> {
  using A = double;
  __device__ static A widen(double v) { return v; }
  __device__ static double narrow(A v) { return v; }
  __device__ static A add(A a, A b) { return __dadd_rn(a, b); }
};

template <>
struct Arith<int32_t> {  // wrapping adds, as two's complement
  using A = uint32_t;
  __device__ static A widen(int32_t v) { return static_cast<uint32_t>(v); }
  __device__ static int32_t narrow(A v) { return static_cast<int32_t>(v); }
  __device__ static A add(A a, A b) { return a + b; }
};

template <>
struct Arith<int64_t> {
  using A = unsigned long long;
  __device__ static A widen(int64_t v) { return static_cast<A>(v); }
  __device__ static int64_t narrow(A v) { return static_cast<int64_t>(v); }
  __device__ static A add(A a, A b) { return a + b; }
};

// ---------------------------------------------------------------- vectors
template <int VB>
struct Raw;
template <>
struct Raw<16> { using type = uint4; };
template <>
struct Raw<8> { using type = uint2; };
template <>
struct Raw<4> { using type = uint32_t; };
template <>
struct Raw<2> { using type = uint16_t; };
template <>
struct Raw<1> { using type = uint8_t; };

template <int VB>
__device__ __forceinline__ typename Raw<VB>::type ld_stream(const char* p) {
  using R = typename Raw<VB>::type;
  if constexpr (VB == 16) {
    return __ldcs(reinterpret_cast<const uint4*>(p));
  } else if constexpr (VB == 8) {
    return __ldcs(reinterpret_cast<const uint2*>(p));
  } else if constexpr (VB == 4) {
    return __ldcs(reinterpret_cast<const unsigned int*>(p));
  } else {
    return *reinterpret_cast<const volatile R*>(p);
  }
}

template <int VB>
__device__ __forceinline__ void st_stream(char* p, typename Raw<VB>::type v) {
  if constexpr (VB == 16) {
    __stcs(reinterpret_cast<uint4*>(p), v);
  } else if constexpr (VB == 8) {
    __stcs(reinterpret_cast<uint2*>(p), v);
  } else if constexpr (VB == 4) {
    __stcs(reinterpret_cast<unsigned int*>(p), v);
  } else {
    *reinterpret_cast<typename Raw<VB>::type*>(p) = v;
  }
}

template <class T, int VB>
union Lanes {
  typename Raw<VB>::type raw;
  T e[VB / sizeof(T)];
};

struct ItemCtx {
  char* dst_row0;       // first vector of the item in dst
  int64_t dst_row_step; // bytes between rows
  int32_t nvcol;
  int32_t nvec;
  int32_t nterms;
};

// Shared per-item term bases (computed once per item by the first threads).
struct SharedTerms {
  const char* row0[kMaxTerms];
  int64_t row_step[kMaxTerms];
};

template <class T, int VB>
__device__ __noinline__ void run_copy(const ItemCtx c, const char* src_row0, int64_t src_step) {
  using R = typename Raw<VB>::type;
  for (int base = threadIdx.x; base < c.nvec; base += kBlock * kUnroll) {
    R v[kUnroll];
    char* d[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int idx = base + u * kBlock;
      d[u] = nullptr;
      if (idx < c.nvec) {
        const int r = idx / c.nvcol;
        const int col = idx - r * c.nvcol;
        v[u] = ld_stream<VB>(src_row0 + r * src_step + static_cast<int64_t>(col) * VB);
        d[u] = c.dst_row0 + r * c.dst_row_step + static_cast<int64_t>(col) * VB;
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (d[u]) st_stream<VB>(d[u], v[u]);
  }
}

template <int VB>
__device__ __noinline__ void run_zero(const ItemCtx c) {
  using R = typename Raw<VB>::type;
  R z;
  memset(&z, 0, sizeof(R));
  for (int idx = threadIdx.x; idx < c.nvec; idx += kBlock) {
    const int r = idx / c.nvcol;
    const int col = idx - r * c.nvcol;
    st_stream<VB>(c.dst_row0 + r * c.dst_row_step + static_cast<int64_t>(col) * VB, z);
  }
}

template <class T, int VB>
__device__ __noinline__ void run_reduce(const ItemCtx c, const SharedTerms& st) {
  using Ar = Arith<T>;
  using A = typename Ar::A;
  constexpr int E = VB / sizeof(T);
  constexpr int kUnroll = kUnrollReduce;
  for (int base = threadIdx.x; base < c.nvec; base += kBlock * kUnroll) {
    A acc[kUnroll][E];
    int r[kUnroll], col[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int idx = base + u * kBlock;
      r[u] = idx / c.nvcol;
      col[u] = idx - r[u] * c.nvcol;
    }
    // term 0 initialises the accumulator (no +0.0, keeps -0.0 exact)
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * kBlock < c.nvec) {
        Lanes<T, VB> x;
        x.raw = ld_stream<VB>(st.row0[0] + r[u] * st.row_step[0] + static_cast<int64_t>(col[u]) * VB);
#pragma unroll
        for (int e = 0; e < E; ++e) acc[u][e] = Ar::widen(x.e[e]);
      }
    }
    for (int k = 1; k < c.nterms; ++k) {
      const char* b = st.row0[k];
      const int64_t rs = st.row_step[k];
      Lanes<T, VB> x[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (base + u * kBlock < c.nvec)
          x[u].raw = ld_stream<VB>(b + r[u] * rs + static_cast<int64_t>(col[u]) * VB);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (base + u * kBlock < c.nvec) {
#pragma unroll
          for (int e = 0; e < E; ++e) acc[u][e] = Ar::add(acc[u][e], Ar::widen(x[u].e[e]));
        }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * kBlock < c.nvec) {
        Lanes<T, VB> y;
#pragma unroll
        for (int e = 0; e < E; ++e) y.e[e] = Ar::narrow(acc[u][e]);
        st_stream<VB>(c.dst_row0 + r[u] * c.dst_row_step + static_cast<int64_t>(col[u]) * VB, y.raw);
      }
    }
  }
}

template <class T, int VB>
__device__ __forceinline__ void run_item(const TaskDesc& task, const WorkItem& w, const TermDesc* terms,
                         SharedTerms& st) {
  const int64_t es = sizeof(T);
  const int32_t i2 = w.plane % task.n[2];
  const int32_t i3 = w.plane / task.n[2];
  ItemCtx c;
  c.dst_row_step = task.dst_stride[0] * es;
  c.dst_row0 = task.dst + es * (w.row0 * task.dst_stride[0] + i2 * task.dst_stride[1] +
                                i3 * task.dst_stride[2]) +
               static_cast<int64_t>(w.vcol0) * VB;
  c.nvcol = w.nvcol;
  c.nvec = w.nrow * w.nvcol;
  c.nterms = task.nterms;
  if (task.nterms == 0) {
    run_zero<VB>(c);
    return;
  }
  auto term_row0 = [&](const TermDesc& t) {
    return t.base + es * (w.row0 * t.stride[0] + i2 * t.stride[1] + i3 * t.stride[2]) +
           static_cast<int64_t>(w.vcol0) * VB;
  };
  if (task.nterms == 1) {
    const TermDesc t = terms[task.term0];
    run_copy<T, VB>(c, term_row0(t), t.stride[0] * es);
    return;
  }
  __syncthreads();  // previous item's readers are done with st
  if (threadIdx.x < task.nterms) {
    const TermDesc t = terms[task.term0 + threadIdx.x];
    st.row0[threadIdx.x] = term_row0(t);
    st.row_step[threadIdx.x] = t.stride[0] * es;
  }
  __syncthreads();
  run_reduce<T, VB>(c, st);
}

template <class T, int VB>
__global__ void __launch_bounds__(kBlock, 2) box_phase_kernel(PhaseTables t) {
  __shared__ SharedTerms st;
  for (int it = blockIdx.x; it < t.n_items; it += gridDim.x) {
    const WorkItem w = t.items[it];
    const TaskDesc task = t.tasks[w.task];
    run_item<T, VB>(task, w, t.terms, st);
  }
}

// ---------------------------------------------------------------- datagen
__device__ __forceinline__ uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

__device__ __forceinline__ uint32_t hash3(uint32_t seed, uint32_t key, uint64_t lin) {
  uint32_t h = mix32(seed * 0x9E3779B1U + key * 0x85EBCA77U + 0x165667B1U);
  h = mix32(h ^ static_cast<uint32_t>(lin));
  return mix32(h ^ static_cast<uint32_t>(lin >> 32) ^ 0x27D4EB2FU);
}

__device__ __forceinline__ uint32_t piece_key(int tid, int level, int g, int p) {
  return static_cast<uint32_t>(tid) * 1000003U + static_cast<uint32_t>(level) * 7919U +
         static_cast<uint32_t>(g) * 131U + static_cast<uint32_t>(p);
}

__device__ __forceinline__ int64_t gv(uint32_t h) { return static_cast<int64_t>((h >> 8) % 8) - 4; }

__device__ int64_t logical_grid(const FillDesc& f, uint64_t lin) {
  return gv(hash3(f.seed, piece_key(f.tensor_id, 0, 0, 0), lin));
}

__device__ int64_t piece_grid(const FillDesc& f, uint64_t lin) {
  const int64_t x = logical_grid(f, lin);
  int64_t t = x;
  if (f.tg >= 0) {
    if (f.tg < f.hsize - 1) {
      t = gv(hash3(f.seed, piece_key(f.tensor_id, 1, f.tg, 0), lin));
    } else {
      int64_t s = 0;
      for (int k = 0; k < f.hsize - 1; ++k) s += gv(hash3(f.seed, piece_key(f.tensor_id, 1, k, 0), lin));
      t = x - s;
    }
  }
  if (f.P == 1) return t;
  if (f.p < f.P - 1) return gv(hash3(f.seed, piece_key(f.tensor_id, 2, f.g, f.p), lin));
  int64_t s = 0;
  for (int k = 0; k < f.P - 1; ++k) s += gv(hash3(f.seed, piece_key(f.tensor_id, 2, f.g, k), lin));
  return t - s;
}

__device__ float piece_real(const FillDesc& f, uint64_t lin) {
  const uint32_t h = hash3(f.seed, piece_key(f.tensor_id, 3, f.tg + 1, f.p), lin);
  return static_cast<float>(static_cast<double>(h >> 8) * 0x1p-23 - 1.0);
}

template <class T>
__device__ T encode_int(int64_t v);
template <>
__device__ uint16_t encode_int<uint16_t>(int64_t v) {
  return Arith<uint16_t>::narrow(static_cast<float>(v));
}
template <>
__device__ float encode_int<float>(int64_t v) { return static_cast<float>(v); }
template <>
__device__ double encode_int<double>(int64_t v) { return static_cast<double>(v); }
template <>
__device__ int32_t encode_int<int32_t>(int64_t v) { return static_cast<int32_t>(v); }
template <>
__device__ int64_t encode_int<int64_t>(int64_t v) { return v; }

template <class T>
__device__ T encode_real(float v) {
  if constexpr (sizeof(T) == 2) return Arith<uint16_t>::narrow(v);
  else return static_cast<T>(v);
}

template <class T>
__device__ double decode(T v) {
  if constexpr (sizeof(T) == 2) return static_cast<double>(Arith<uint16_t>::widen(v));
  else return static_cast<double>(v);
}

// Box cell c (row-major over ext) -> logical linear index.
__device__ __forceinline__ uint64_t cell_lin(const FillDesc& f, int64_t c) {
  int64_t idx[4];
  for (int d = f.ndim - 1; d >= 0; --d) {
    idx[d] = c % f.ext[d];
    c /= f.ext[d];
  }
  uint64_t lin = 0;
  for (int d = 0; d < f.ndim; ++d) lin = lin * f.shape[d] + (f.lo[d] + idx[d]);
  return lin;
}

template <class T>
__global__ void fill_kernel(FillDesc f, int64_t cells) {
  T* out = reinterpret_cast<T*>(f.dst);
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t lin = cell_lin(f, c);
    if (f.mode == 0 || std::is_integral_v<T> && sizeof(T) != 2)
      out[c] = encode_int<T>(piece_grid(f, lin));
    else
      out[c] = encode_real<T>(piece_real(f, lin));
  }
}

template <class T>
__global__ void verify_kernel(FillDesc f, int64_t cells, unsigned long long* bad) {
  const T* in = reinterpret_cast<const T*>(f.dst);
  unsigned long long mine = 0;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double want = static_cast<double>(logical_grid(f, cell_lin(f, c)));
    mine += decode<T>(in[c]) != want;
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(bad, mine);
}

// ---------------------------------------------------------------- barrier
__global__ void barrier_kernel(unsigned int* const* peer_flags, int world, int rank,
                               unsigned int epoch, unsigned long long timeout_ns, int* error) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int p = 0; p < world; ++p) {
    unsigned int* slot = peer_flags[p] + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
  }
  unsigned int* mine = peer_flags[rank];
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int p = 0; p < world; ++p) {
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + p) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (now - t0 > timeout_ns) {
        *error = 1;
        return;
      }
    }
  }
  __threadfence_system();
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g > 148 * 8) g = 148 * 8;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <template <class> class K, class... Args>
cudaError_t by_dtype(int dtype, dim3 grid, dim3 block, cudaStream_t s, Args... args) {
  switch (dtype) {
    case 0: K<float>::launch(grid, block, s, args...); break;
    case 1: K<double>::launch(grid, block, s, args...); break;
    case 2: K<int32_t>::launch(grid, block, s, args...); break;
    case 3: K<int64_t>::launch(grid, block, s, args...); break;
    case 4: K<uint16_t>::launch(grid, block, s, args...); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

template <class T>
struct PhaseK {
  static void launch(dim3 g, dim3 b, cudaStream_t s, PhaseTables t, int vb) {
    switch (vb) {
      case 16: box_phase_kernel<T, 16><<<g, b, 0, s>>>(t); break;
      case 8:
        if constexpr (sizeof(T) <= 8) box_phase_kernel<T, 8><<<g, b, 0, s>>>(t);
        break;
      case 4:
        if constexpr (sizeof(T) <= 4) box_phase_kernel<T, 4><<<g, b, 0, s>>>(t);
        break;
      case 2:
        if constexpr (sizeof(T) <= 2) box_phase_kernel<T, 2><<<g, b, 0, s>>>(t);
        break;
    }
  }
};
template <class T>
struct FillK {
  static void launch(dim3 g, dim3 b, cudaStream_t s, FillDesc f, int64_t cells) {
    fill_kernel<T><<<g, b, 0, s>>>(f, cells);
  }
};
template <class T>
struct VerifyK {
  static void launch(dim3 g, dim3 b, cudaStream_t s, FillDesc f, int64_t cells,
                     unsigned long long* bad) {
    verify_kernel<T><<<g, b, 0, s>>>(f, cells, bad);
  }
};

}  // namespace

cudaError_t launch_phase(const PhaseTables& t, int dtype, int vec_bytes, int grid, cudaStream_t s) {
  if (t.n_items == 0) return cudaSuccess;
  return by_dtype<PhaseK>(dtype, dim3(grid), dim3(kBlock), s, t, vec_bytes);
}

cudaError_t launch_fill(const FillDesc& f, int dtype, cudaStream_t s) {
  int64_t cells = 1;
  for (int d = 0; d < f.ndim; ++d) cells *= f.ext[d];
  if (cells == 0) return cudaSuccess;
  return by_dtype<FillK>(dtype, dim3(grid_for(cells, 256 * 8)), dim3(256), s, f, cells);
}

cudaError_t launch_verify(const FillDesc& f, int dtype, unsigned long long* bad, cudaStream_t s) {
  int64_t cells = 1;
  for (int d = 0; d < f.ndim; ++d) cells *= f.ext[d];
  if (cells == 0) return cudaSuccess;
  return by_dtype<VerifyK>(dtype, dim3(grid_for(cells, 256 * 8)), dim3(256), s, f, cells, bad);
}

cudaError_t launch_barrier(unsigned int* const* peer_flags, int world, int rank,
                           unsigned int epoch, unsigned long long timeout_ns, int* error,
                           cudaStream_t s) {
  barrier_kernel<<<1, 32, 0, s>>>(peer_flags, world, rank, epoch, timeout_ns, error);
  return cudaGetLastError();
}

}  // namespace hshard::exec
