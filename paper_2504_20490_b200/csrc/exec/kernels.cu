// hshard-b200 executor kernels (sm_100a).
//
// TMA pipeline (16-byte-aligned items, the hot path): one persistent CTA per
//   SM, warp-specialised.  Warp 0 is the producer: for each work item it arms
//   a stage's mbarrier with the item's byte count and its lanes issue one
//   cp.async.bulk (TMA bulk copy, global -> shared) per (term, row) segment.
//   16 consumer warps wait for the stage, read every term from shared memory,
//   form the grouped ordered sum in the dtype's accumulator (packed f32x2 /
//   bf16x2 where the dtype allows) and store the result (st.global.cs, or TMA
//   bulk stores for copies under HS_PROG_BULK_STORE) to every output.  Four
//   48 KB stages keep ~144 KB per SM in flight independently of register
//   pressure, which is what an HBM3e stream needs.  Three schedulers:
//     box_phase_tma_static_kernel  items dealt round-robin (N=1, uniform local launches)
//     box_phase_tma_tail_kernel    15/16 static, the tail dynamic (unstreamed N>1)
//     box_phase_tma_kernel         two dynamic queues, ready flags, signaller warp (streamed N>1)
//   Each can open with the phase's cross-rank barrier (folded_barrier).
// box_phase_kernel (any vector width): the register path, used for boxes
//   whose pointers / strides / row lengths are not 16-byte aligned.
#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

namespace hshard::exec {

namespace {

constexpr int kBlock = 512;     // register path
constexpr int kConsumerWarps = 16;                   // 512 consumer threads
constexpr int kTmaThreads = 32 * (kConsumerWarps + 1);  // + 1 producer warp
constexpr int kDynThreads = kTmaThreads + 32;           // multi-GPU kernel: + 1 signaller warp
constexpr int kSigRing = 64;                            // signaller queue slots

// ---------------------------------------------------------------- arithmetic
template <class T>
struct Arith;

template <>
struct Arith<uint16_t> {  // bf16 stored as raw bits
  using A = float;
  __device__ static A widen(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }
  __device__ static uint16_t narrow(A f) {  // round to nearest even: one F2FP instruction
    uint16_t r;
    asm("cvt.rn.bf16.f32 %0, %1;" : "=h"(r) : "f"(f));
    return r;
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

// Grouped ordered sum of `nterms` vectors fetched by `get(k)`:
//   round(sum_g round_g(sum_{k in g} widen(term_k)))   (round_g only if |g| > 1)
template <class T, int VB, class Get>
__device__ __forceinline__ typename Raw<VB>::type grouped_sum(int nterms, int ngroups,
                                                              const uint8_t* gsize, Get get) {
  using Ar = Arith<T>;
  using A = typename Ar::A;
  constexpr int E = VB / sizeof(T);
  A outer[E];
  int k = 0;
  const int ng = ngroups ? ngroups : nterms;
  for (int g = 0; g < ng; ++g) {
    const int sz = ngroups ? gsize[g] : 1;
    Lanes<T, VB> x;
    x.raw = get(k++);
    A inner[E];
#pragma unroll
    for (int e = 0; e < E; ++e) inner[e] = Ar::widen(x.e[e]);
    for (int j = 1; j < sz; ++j) {
      x.raw = get(k++);
#pragma unroll
      for (int e = 0; e < E; ++e) inner[e] = Ar::add(inner[e], Ar::widen(x.e[e]));
    }
    if (sz > 1) {
#pragma unroll
      for (int e = 0; e < E; ++e) inner[e] = Ar::widen(Ar::narrow(inner[e]));
    }
    if (g == 0) {
#pragma unroll
      for (int e = 0; e < E; ++e) outer[e] = inner[e];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e) outer[e] = Ar::add(outer[e], inner[e]);
    }
  }
  Lanes<T, VB> y;
#pragma unroll
  for (int e = 0; e < E; ++e) y.e[e] = Ar::narrow(outer[e]);
  return y.raw;
}

// Row-0 byte address and row step of an operand for a work item.
// Packed form for the 16-byte TMA consumers: fp32 pairs in 64-bit registers
// (FADD2: two IEEE round-to-nearest adds per instruction, the same per-lane
// result as __fadd_rn), bf16 pairs narrowed by one F2FP.  Same order of
// additions and roundings as grouped_sum, so bit-identical.
__device__ __forceinline__ unsigned long long add_f32x2(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}

template <class T>
struct Pack2;
template <>
struct Pack2<uint16_t> {  // one 32-bit word = 2 bf16 -> 2 fp32 lanes
  static constexpr int kWordsPerPair = 1;
  __device__ static unsigned long long widen(const uint32_t* w) {
    return (static_cast<unsigned long long>(w[0] & 0xffff0000u) << 32) | (w[0] << 16);
  }
  __device__ static void narrow(unsigned long long v, uint32_t* w) {
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;"
        : "=r"(w[0])
        : "f"(__uint_as_float(static_cast<uint32_t>(v >> 32))), "f"(__uint_as_float(static_cast<uint32_t>(v))));
  }
};
template <>
struct Pack2<float> {  // two 32-bit words = 2 fp32 lanes
  static constexpr int kWordsPerPair = 2;
  __device__ static unsigned long long widen(const uint32_t* w) {
    return (static_cast<unsigned long long>(w[1]) << 32) | w[0];
  }
  __device__ static void narrow(unsigned long long v, uint32_t* w) {
    w[0] = static_cast<uint32_t>(v);
    w[1] = static_cast<uint32_t>(v >> 32);
  }
};

template <class T, class Get>
__device__ __forceinline__ uint4 grouped_sum_packed(int nterms, int ngroups, const uint8_t* gsize, Get get) {
  constexpr int P = 4 / Pack2<T>::kWordsPerPair;  // pairs per 16-byte vector
  constexpr int WP = Pack2<T>::kWordsPerPair;
  unsigned long long outer[P], inner[P];
  int k = 0;
  const int ng = ngroups ? ngroups : nterms;
  for (int g = 0; g < ng; ++g) {
    const int sz = ngroups ? gsize[g] : 1;
    uint4 x = get(k++);
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
    for (int i = 0; i < P; ++i) inner[i] = Pack2<T>::widen(xw + i * WP);
    for (int j = 1; j < sz; ++j) {
      x = get(k++);
#pragma unroll
      for (int i = 0; i < P; ++i) inner[i] = add_f32x2(inner[i], Pack2<T>::widen(xw + i * WP));
    }
    if (sz > 1) {  // the group rounds to the storage type before joining the outer sum
#pragma unroll
      for (int i = 0; i < P; ++i) {
        uint32_t w[WP];
        Pack2<T>::narrow(inner[i], w);
        inner[i] = Pack2<T>::widen(w);
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i) outer[i] = g == 0 ? inner[i] : add_f32x2(outer[i], inner[i]);
  }
  uint4 y;
  uint32_t* yw = reinterpret_cast<uint32_t*>(&y);
#pragma unroll
  for (int i = 0; i < P; ++i) Pack2<T>::narrow(outer[i], yw + i * WP);
  return y;
}

// The 16-byte consumers' reduction: packed for bf16 / fp32, generic otherwise.
template <class T, class Get>
__device__ __forceinline__ uint4 grouped_sum16(int nterms, int ngroups, const uint8_t* gsize, Get get) {
  if constexpr (std::is_same_v<T, uint16_t> || std::is_same_v<T, float>)
    return grouped_sum_packed<T>(nterms, ngroups, gsize, get);
  else
    return grouped_sum<T, 16>(nterms, ngroups, gsize, get);
}

struct RowPtr {
  char* row0;
  int64_t step;
};

__device__ __forceinline__ RowPtr row_ptr(const TermDesc& t, const WorkItem& w, const TaskDesc& task,
                                          int64_t es, int vb) {
  const int32_t i2 = w.plane % task.n[2];
  const int32_t i3 = w.plane / task.n[2];
  RowPtr p;
  p.row0 = const_cast<char*>(t.base) +
           es * (w.row0 * t.stride[0] + i2 * t.stride[1] + i3 * t.stride[2]) +
           static_cast<int64_t>(w.vcol0) * vb;
  p.step = t.stride[0] * es;
  return p;
}

// ---------------------------------------------------------------- register path
// Programmatic dependent launch (PhaseTables::pdl): every phase kernel lets
// the next launch on its stream be scheduled at once (its CTAs take SMs as
// this grid's CTAs retire and run their prologue), and waits -- before its
// first access to memory an earlier kernel may write, and before announcing
// a folded cross-rank barrier -- until every earlier grid on the stream has
// completed with its memory visible (griddepcontrol.wait).  Without the
// launch attribute both are no-ops.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

template <class T, int VB, bool kReduce>
__global__ void __launch_bounds__(kBlock, kReduce ? 1 : 2) box_phase_kernel(PhaseTables t) {
  __shared__ RowPtr ops[kMaxTerms + kMaxOuts];
  __shared__ TaskDesc task_s;
  using R = typename Raw<VB>::type;
  pdl_begin();
  for (int it = blockIdx.x; it < t.n_items; it += gridDim.x) {
    const WorkItem w = t.items[it];
    __syncthreads();  // previous item done with ops / task_s
    if (threadIdx.x == 0) task_s = t.tasks[w.task];
    __syncthreads();
    const int nt = task_s.nterms, no = task_s.nout;
    if (threadIdx.x < nt)
      ops[threadIdx.x] = row_ptr(t.terms[task_s.term0 + threadIdx.x], w, task_s, sizeof(T), VB);
    else if (threadIdx.x < nt + no)
      ops[threadIdx.x] = row_ptr(t.terms[task_s.out0 + threadIdx.x - nt], w, task_s, sizeof(T), VB);
    __syncthreads();
    const int nvcol = w.nvcol, nvec = w.nrow * w.nvcol;
    if constexpr (!kReduce) {
      // copy / zero: kCopyUnroll independent 16-byte loads in flight per thread
      constexpr int U = 4;
      for (int base = threadIdx.x; base < nvec; base += kBlock * U) {
        R val[U];
        int r[U];
        int64_t cb[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int v = base + u * kBlock;
          r[u] = v / nvcol;
          cb[u] = static_cast<int64_t>(v - r[u] * nvcol) * VB;
          if (nt == 0)
            memset(&val[u], 0, sizeof(R));
          else if (v < nvec)
            val[u] = ld_stream<VB>(ops[0].row0 + r[u] * ops[0].step + cb[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (base + u * kBlock < nvec)
            for (int o = 0; o < no; ++o)
              st_stream<VB>(ops[nt + o].row0 + r[u] * ops[nt + o].step + cb[u], val[u]);
      }
    } else {
    // grouped ordered sum, U vectors in lock-step so U loads per term are in flight
    using Ar = Arith<T>;
    using A = typename Ar::A;
    constexpr int E = VB / sizeof(T);
    constexpr int U = 2;
    const int ng = task_s.ngroups ? task_s.ngroups : nt;
    for (int base = threadIdx.x; base < nvec; base += kBlock * U) {
      int r[U];
      int64_t cb[U];
      bool on[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int v = base + u * kBlock;
        on[u] = v < nvec;
        r[u] = v / nvcol;
        cb[u] = static_cast<int64_t>(v - r[u] * nvcol) * VB;
      }
      A outer[U][E], inner[U][E];
      int k = 0;
      for (int g = 0; g < ng; ++g) {
        const int sz = task_s.ngroups ? task_s.gsize[g] : 1;
        for (int j = 0; j < sz; ++j, ++k) {
          Lanes<T, VB> x[U];
#pragma unroll
          for (int u = 0; u < U; ++u)
            if (on[u]) x[u].raw = ld_stream<VB>(ops[k].row0 + r[u] * ops[k].step + cb[u]);
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int e = 0; e < E; ++e)
              inner[u][e] = j == 0 ? Ar::widen(x[u].e[e]) : Ar::add(inner[u][e], Ar::widen(x[u].e[e]));
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const A v = sz > 1 ? Ar::widen(Ar::narrow(inner[u][e])) : inner[u][e];
            outer[u][e] = g == 0 ? v : Ar::add(outer[u][e], v);
          }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!on[u]) continue;
        Lanes<T, VB> y;
#pragma unroll
        for (int e = 0; e < E; ++e) y.e[e] = Ar::narrow(outer[u][e]);
        for (int o = 0; o < no; ++o) st_stream<VB>(ops[nt + o].row0 + r[u] * ops[nt + o].step + cb[u], y.raw);
      }
    }
    }
  }
}

// ---------------------------------------------------------------- TMA path
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Waits for the barrier phase; traps (kernel error, never a hang) after ~10 s.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  if (mbar_try_wait(bar, parity)) return;
  const unsigned long long t0 = global_ns();
  while (!mbar_try_wait(bar, parity)) {
    if (global_ns() - t0 > 10ull * 1000 * 1000 * 1000) asm volatile("trap;");
  }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA bulk store shared -> global, tracked by the issuing thread's bulk groups.
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src_smem),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// the shared-memory source of every committed group has been read
__device__ __forceinline__ void bulk_wait_read_all() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// ... of every committed group but the most recent one
__device__ __forceinline__ void bulk_wait_read_but_last() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// HS_PROG_BULK_STORE, consumer side of a copy item (nterms == 1) in stage s.
// The staged rows of the first min(nout, bulk_outs) outputs leave through TMA
// bulk stores, one (output, row) per lane of consumer warp 1; all consumer
// warps store the remaining outputs from registers, so fan-out copies keep
// both store paths busy and the TMA unit is not monopolised by stores while it
// must also feed the stages.  Warp 1 releases a stage one copy later, once
// the stores have read it (`held`), so the store queue never drains between
// items; outputs may be peer addresses.
__device__ __forceinline__ void bulk_copy_item(const TmaRecHead* h, const TmaOperand* outs,
                                               const unsigned char* in, int bulk_outs, uint64_t* empty,
                                               int s, int& held) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ctid = threadIdx.x - 32;
  constexpr int nct = kTmaThreads - 32;
  const int nvcol = h->nvcol, nvec = h->nrow * h->nvcol, no = h->nout;
  const int nb = min(no, bulk_outs);
  if (warp == 1) {
    const int nrow = h->nrow;
    const uint32_t row_bytes = static_cast<uint32_t>(nvcol) * 16;
    for (int j = lane; j < nb * nrow; j += 32) {
      const int o = j / nrow, r = j - o * nrow;
      bulk_s2g(outs[o].row0 + r * outs[o].step, smem_u32(in) + r * row_bytes, row_bytes);
    }
    bulk_commit();
  }
  if (no > nb)
    for (int v = ctid; v < nvec; v += nct) {
      const int r = v / nvcol;
      const int64_t cb = static_cast<int64_t>(v - r * nvcol) * 16;
      const uint4 val = *reinterpret_cast<const uint4*>(in + static_cast<size_t>(v) * 16);
      for (int o = nb; o < no; ++o) __stcs(reinterpret_cast<uint4*>(outs[o].row0 + r * outs[o].step + cb), val);
    }
  if (warp == 1) {
    if (held >= 0) {
      bulk_wait_read_but_last();
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[held]);
    }
    held = s;
  } else {
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// Before a non-copy item: warp 1 releases the stage its bulk stores held.
__device__ __forceinline__ void bulk_release_held(uint64_t* empty, int& held) {
  if ((threadIdx.x >> 5) != 1 || held < 0) return;
  bulk_wait_read_all();
  __syncwarp();
  if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[held]);
  held = -1;
}

// Streamed launches, signalling side.  A system-scope fence in an SM that is
// streaming costs microseconds (it waits for the SM's outstanding memory
// traffic), so consumer warps never issue one: each consumer warp of an item
// of a signalling task orders its stores with fence.cta and counts itself in
// shared memory; the item's last warp queues the task's SigDesc index in a
// shared ring.  A dedicated signaller warp drains the ring in batches: one
// fence.sc.sys per batch (cumulative over every queued item's stores, which
// it acquired through the ring), then per entry one add to the task's item
// counter and -- when that add completes the task's run -- red.release.sys
// on every consumer flag.
struct SigRing {
  unsigned int cnt[kTmaStages];  // consumer warps done with the stage's item
  unsigned int slot[kSigRing];   // SigDesc index + 1; 0 = empty
  unsigned int tail;             // next slot to fill
  unsigned int consumers_done;   // consumer warps that have exited
};

__device__ __forceinline__ void tma_count(SigRing* ring, int s, int sig, int lane) {
  __threadfence_block();
  __syncwarp();
  if (lane == 0 && atomicAdd(&ring->cnt[s], 1u) == kConsumerWarps - 1) {
    ring->cnt[s] = 0;
    const unsigned int k = atomicAdd(&ring->tail, 1u) % kSigRing;
    volatile unsigned int* v = ring->slot + k;
    while (*v != 0) __nanosleep(64);  // ring full: the signaller is a batch behind
    __threadfence_block();
    *v = static_cast<unsigned int>(sig) + 1;
  }
  __syncwarp();
}

__device__ void tma_signaller(const PhaseTables& t, SigRing* ring, int lane) {
  unsigned int head = 0;
  while (true) {
    volatile unsigned int* v = ring->slot + (head + lane) % kSigRing;
    const unsigned int e = *v;
    // consecutive ready entries from head
    const unsigned int ready = __ballot_sync(0xffffffffu, e != 0);
    const int n = __ffs(~ready) - 1 < 0 ? 32 : __ffs(~ready) - 1;
    if (n == 0) {
      // consumer warps queue every item before they exit, so once all have
      // exited an empty head slot means the ring is drained
      if (*reinterpret_cast<volatile unsigned int*>(&ring->consumers_done) == kConsumerWarps) {
        __threadfence_block();
        if (__ballot_sync(0xffffffffu, *v != 0) == 0) return;
      } else {
        __nanosleep(128);
      }
      continue;
    }
    __threadfence_system();
    if (lane < n) {
      *v = 0;
      const SigDesc d = t.sigs[e - 1];
      const unsigned long long old = atomicAdd(&t.done[d.done], 1ull);
      if ((old + 1) % d.expected == 0)
        for (uint32_t k = 0; k < d.ntargets; ++k)
          asm volatile("red.release.sys.global.add.u32 [%0], 1;" ::"l"(t.targets[d.target0 + k]) : "memory");
    }
    head += n;
    __syncwarp();
  }
}

// TMA item record of item `i`, decoded from the task descriptors (every lane
// returns its 16-byte word of the record: lanes 0-2 the TmaRecHead, lane 3 + k
// operand k).  `cur` is the warp's cursor into the task table: consecutive
// items are usually in the current task or the next; otherwise a binary
// search over TmaTask::item0 finds it.
// Used by expand_records_kernel, once per compiled program: the phase kernels
// keep reading one prefetched record word per lane (a dependent decode in the
// producer warp measured 6-40% slower: it stalls the warp that issues the TMA).
__device__ __forceinline__ int tma_find(const PhaseTables& t, int i, int cur) {
  const TmaTask* tt = t.ttasks;
  if (cur >= t.n_ttasks || __ldg(&tt[cur].item0) > i) cur = 0;
  if (__ldg(&tt[cur + 1].item0) > i) return cur;
  int lo = cur + 1, hi = t.n_ttasks - 1;  // largest k with item0 <= i
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(&tt[mid].item0) <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int kEs>
__device__ __forceinline__ uint4 tma_record(const PhaseTables& t, int i, int lane, int& cur) {
  cur = tma_find(t, i, cur);
  const TmaTask* tk = t.ttasks + cur;
  const int4 w0 = __ldg(reinterpret_cast<const int4*>(tk));      // item0, nterms, nout, ngroups
  const int4 w1 = __ldg(reinterpret_cast<const int4*>(tk) + 1);  // wait, sig, need, mode
  const int4 w2 = __ldg(reinterpret_cast<const int4*>(tk) + 2);  // n1, n2, row_vecs, per
  const int4 w3 = __ldg(reinterpret_cast<const int4*>(tk) + 3);  // cpr, term0, out0, pad
  const int j = i - w0.x;
  const int n1 = w2.x, row_vecs = w2.z, per = w2.w, cpr = w3.x;
  int pl, r, c, nrow, nvcol;
  if (w1.w == 0) {  // row chunks
    const int per_plane = n1 * cpr;
    pl = j / per_plane;
    const int rem = j - pl * per_plane;
    r = rem / cpr;
    c = (rem - r * cpr) * per;
    nvcol = min(per, row_vecs - c);
    nrow = 1;
  } else {  // row runs
    pl = j / cpr;
    r = (j - pl * cpr) * per;
    nrow = min(per, n1 - r);
    c = 0;
    nvcol = row_vecs;
  }
  if (lane == 0) return make_uint4(w0.y, w0.z, w0.w, nrow);
  if (lane == 1) return make_uint4(nvcol, w1.x, w1.y, w1.z);
  if (lane == 2) return __ldg(reinterpret_cast<const uint4*>(tk) + 4);  // gsize
  const int k = lane - kTmaHeadWords, nterms = w0.y;
  if (k >= nterms + w0.z) return make_uint4(0, 0, 0, 0);
  const TermDesc* td = t.terms + (k < nterms ? w3.y + k : w3.z + (k - nterms));
  const char* base = reinterpret_cast<const char*>(__ldg(reinterpret_cast<const unsigned long long*>(&td->base)));
  const int64_t s0 = __ldg(&td->stride[0]), s1 = __ldg(&td->stride[1]), s2 = __ldg(&td->stride[2]);
  const int n2 = w2.y;
  const int i2 = pl % n2, i3 = pl / n2;
  const unsigned long long row0 = reinterpret_cast<unsigned long long>(
      base + kEs * (static_cast<int64_t>(r) * s0 + i2 * s1 + i3 * s2) + static_cast<int64_t>(c) * 16);
  const unsigned long long step = static_cast<unsigned long long>(s0 * kEs);
  return make_uint4(static_cast<unsigned>(row0), static_cast<unsigned>(row0 >> 32), static_cast<unsigned>(step),
                    static_cast<unsigned>(step >> 32));
}

// Expands a launch's records from its task descriptors on the device, one
// warp per item (grid-stride): what the host used to build item by item.
// `na` in (0, n_items): items [0, na) (tasks with NVLink operands) and
// [na, n_items) (local-only tasks) are interleaved evenly in launch order --
// the k-th of the first class goes to slot ceil((k+1) n / na) - 1, the k-th of
// the second to floor(k n / (n - na)), a partition of [0, n) -- so the CTAs
// keep NVLink and HBM busy together instead of one class after the other.
template <int kEs>
__global__ void __launch_bounds__(256) expand_records_kernel(PhaseTables t, uint4* recs, int W, int na) {
  const int lane = threadIdx.x & 31;
  const int warps = static_cast<int>(gridDim.x * blockDim.x) >> 5;
  const int64_t n = t.n_items;
  int cur = 0;
  for (int i = static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5); i < t.n_items; i += warps) {
    const uint4 w = tma_record<kEs>(t, i, lane, cur);
    int64_t slot = i;
    if (na > 0 && na < n)
      slot = i < na ? ((static_cast<int64_t>(i) + 1) * n + na - 1) / na - 1
                    : ((static_cast<int64_t>(i) - na) * n) / (n - na);
    if (lane < W) recs[static_cast<size_t>(slot) * W + lane] = w;
  }
}

// Dynamic-schedule kernels: a CTA leaving the launch counts itself out; the
// last one resets the scheduler words for the program's next run.
__device__ __forceinline__ void sched_retire(const PhaseTables& t) {
  if (atomicAdd(&t.sched[1], 1) == static_cast<int>(gridDim.x) - 1) {
    t.sched[0] = 0;
    t.sched[1] = 0;
    t.sched[2] = 0;
  }
}

// Streamed launches: the producer warp's lane 0 waits until a consumer
// piece's producers have all signalled this run; bounded by ~10 s, after
// which it records DeadlockDetected and proceeds (never a hang).
// Folded barrier, thread 0 of every CTA: CTA 0 announces this rank (stream
// order: everything enqueued before this kernel has completed), then each CTA
// waits until every rank has announced -- launch_barrier's protocol without
// its launch.  False on timeout (error recorded; the CTA then does no work).
__device__ __noinline__ bool folded_barrier(unsigned int* const* flags, int world, int rank,
                                            unsigned int epoch, int* error) {
  if (blockIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < world; ++p)
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flags[p] + rank), "r"(epoch) : "memory");
  }
  const unsigned int* mine = flags[rank];
  const unsigned long long t0 = global_ns();
  for (int p = 0; p < world; ++p) {
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + p) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (global_ns() - t0 > 20ull * 1000 * 1000 * 1000) {
        *error = 1;
        return false;
      }
    }
  }
  // the TMA (async proxy) loads that follow read what peers wrote
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return true;
}

__device__ __forceinline__ void tma_wait(const PhaseTables& t, int flag, int need) {
  const unsigned int want = t.epoch * static_cast<unsigned int>(need);
  const unsigned int* f = t.wait_flags + flag;
  unsigned long long t0 = 0;
  const unsigned long long tw0 = t.trace ? global_ns() : 0;
  while (true) {
    unsigned int v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (static_cast<int>(v - want) >= 0) break;
    if (t0 == 0) t0 = global_ns();
    if (*reinterpret_cast<volatile int*>(t.error)) break;  // an earlier wait already gave up
    if (global_ns() - t0 > 10ull * 1000 * 1000 * 1000) {
      *t.error = 1;
      break;
    }
  }
  // the TMA (async proxy) loads that follow read what peers stored
  asm volatile("fence.proxy.async.global;" ::: "memory");
  if (t.trace) {  // debug timeline: total and count of waits that spun
    unsigned long long* tr = t.trace + blockIdx.x * 8;
    tr[3] += global_ns() - tw0;
    tr[4] += t0 != 0;
  }
}

// One consumer-warp pass over pipeline stage `iter`: wait for it, form every
// output vector of the item from shared memory, release the stage.  Returns
// false on the producer's end marker.
template <class T>
__device__ __forceinline__ bool tma_consume(const unsigned char* stage, const uint4* meta,
                                            uint64_t* full, uint64_t* empty, SigRing* ring, int iter,
                                            int lane) {
  const int ctid = threadIdx.x - 32;
  constexpr int nct = 32 * kConsumerWarps;
  const int s = iter % kTmaStages;
  mbar_wait(&full[s], (iter / kTmaStages) & 1);
  const uint4* m = meta + s * 32;
  const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
  const int nt = h->nterms;
  if (nt < 0) return false;
  const int nvcol = h->nvcol, nvec = h->nrow * h->nvcol, no = h->nout;
  const int ng = h->ngroups;
  const TmaOperand* outs = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords) + nt;
  const unsigned char* in = stage + s * kStageBytes;
  for (int v = ctid; v < nvec; v += nct) {
    const int r = v / nvcol;
    const int64_t cb = static_cast<int64_t>(v - r * nvcol) * 16;
    uint4 val;
    if (nt == 0) {
      val = make_uint4(0, 0, 0, 0);
    } else if (nt == 1) {
      val = *reinterpret_cast<const uint4*>(in + static_cast<size_t>(v) * 16);
    } else {
      val = grouped_sum16<T>(nt, ng, h->gsize, [&](int k) {
        return *reinterpret_cast<const uint4*>(in + (static_cast<size_t>(k) * nvec + v) * 16);
      });
    }
    for (int o = 0; o < no; ++o) __stcs(reinterpret_cast<uint4*>(outs[o].row0 + r * outs[o].step + cb), val);
  }
  const int sig = h->sig;  // read before the stage is released
  __syncwarp();
  if (sig >= 0) tma_count(ring, s, sig, lane);
  if (lane == 0) mbar_arrive(&empty[s]);
  return true;
}

template <class T>
__global__ void __launch_bounds__(kDynThreads, 1) box_phase_tma_kernel(PhaseTables t) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;
  uint4* meta = reinterpret_cast<uint4*>(smem + kTmaStages * kStageBytes);  // 32 words per stage
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kTmaStages * 32);
  uint64_t* empty = full + kTmaStages;
  SigRing* ring = reinterpret_cast<SigRing*>(empty + kTmaStages);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
      ring->cnt[s] = 0;
    }
    for (int k = 0; k < kSigRing; ++k) ring->slot[k] = 0;
    ring->tail = 0;
    ring->consumers_done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_begin();
  if (t.bar_flags) {  // folded cross-rank barrier (replaces a barrier launch)
    volatile int* ok = reinterpret_cast<volatile int*>(meta);  // unused until the first item
    if (threadIdx.x == 0) *ok = folded_barrier(t.bar_flags, t.bar_world, t.bar_rank, t.bar_epoch, t.error);
    __syncthreads();
    const int good = *ok;
    __syncthreads();  // every thread has read it before the producer reuses meta
    if (!good) {  // timed out (error recorded): still retire from the scheduler
      if (threadIdx.x == 0) sched_retire(t);
      return;
    }
  }
  const int W = t.rec_words;

  if (warp == kConsumerWarps + 1) {  // ---- signaller warp
    if (t.sigs) tma_signaller(t, ring, lane);
    return;
  }

  if (warp == 0) {
    // ---- producer warp: the item record is prefetched one item ahead (one
    // 16-byte word per lane); lane k then streams term k's rows.
    // Items [0, n_static) are dealt round-robin (no dependency: the record is
    // prefetched one item ahead); the rest are handed out dynamically (one
    // atomic per item) from two queues (PhaseTables::n_first / first_ctas).
    const unsigned full_mask = 0xffffffffu;
    const bool first_role = static_cast<int>(blockIdx.x) < t.first_ctas;
    unsigned long long* tr = t.trace ? t.trace + blockIdx.x * 8 : nullptr;
    if (tr && lane == 0) {
      tr[0] = global_ns();
      tr[2] = 0; tr[3] = 0; tr[4] = 0; tr[5] = 0; tr[6] = 0;  // [6] unused
      tr[7] = first_role;
    }
    // Tickets: lane 0 takes item i+2's index (an atomic) while item i is
    // issued and resolves it one iteration later, so neither the atomic nor
    // the record load that depends on it sits on the critical path.  A
    // first-queue ticket that comes back past n_first is exchanged for a
    // second-queue one (so a CTA never takes a first-queue item after a
    // second-queue one).
    bool first_open = first_role;
    int k_static = 0;
    auto issue = [&]() -> int {  // lane 0 only; encoded: >= 0 final, < 0 first-queue ticket
      const int st = blockIdx.x + k_static * static_cast<int>(gridDim.x);
      if (st < t.n_static) {
        ++k_static;
        return st;
      }
      if (first_open) return -1 - (t.n_static + atomicAdd(&t.sched[0], 1));
      return t.n_first + atomicAdd(&t.sched[2], 1);
    };
    auto resolve = [&](int ticket) -> int {  // all lanes
      int d = ticket;
      if (lane == 0 && d < 0) {
        d = -1 - d;
        if (d >= t.n_first) {
          first_open = false;
          d = t.n_first + atomicAdd(&t.sched[2], 1);
          if (tr && tr[5] == 0) tr[5] = global_ns();
        }
      }
      return __shfl_sync(full_mask, d, 0);
    };
    int it = resolve(lane == 0 ? issue() : 0);
    uint4 next = make_uint4(0, 0, 0, 0);
    int pend = 0;
    if (it < t.n_items) {
      if (lane < W) next = t.recs[static_cast<size_t>(it) * W + lane];
      if (lane == 0) pend = issue();
    }
    for (int iter = 0;; ++iter) {
      const int cur_it = it;
      const uint4 cur = next;
      if (cur_it < t.n_items) {
        it = resolve(pend);
        if (it < t.n_items) {
          if (lane < W) next = t.recs[static_cast<size_t>(it) * W + lane];
          if (lane == 0) pend = issue();
        }
      }
      const int s = iter % kTmaStages;
      if (iter >= kTmaStages) mbar_wait(&empty[s], ((iter / kTmaStages) + 1) & 1);
      uint4* m = meta + s * 32;
      if (cur_it >= t.n_items) {  // end marker for the consumers
        if (tr && lane == 0) { tr[1] = global_ns(); tr[2] = iter; }
        if (lane == 0) {
          reinterpret_cast<TmaRecHead*>(m)->nterms = -1;
          mbar_arrive_expect_tx(&full[s], 0);
          // the last CTA out resets the scheduler for the next launch
          if (atomicAdd(&t.sched[1], 1) == static_cast<int>(gridDim.x) - 1) {
            t.sched[0] = 0;
            t.sched[1] = 0;
            t.sched[2] = 0;
          }
        }
        return;
      }
      if (lane < W) m[lane] = cur;
      __syncwarp();
      const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
      if (h->wait >= 0) {
        if (lane == 0) tma_wait(t, h->wait, h->need);
        __syncwarp();
      }
      const int nt = h->nterms, nrow = h->nrow;
      const uint32_t row_bytes = static_cast<uint32_t>(h->nvcol) * 16;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], row_bytes * nrow * nt);  // release: meta
      __syncwarp();
      if (lane < nt) {
        const TmaOperand op = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords)[lane];
        unsigned char* dst = stage + s * kStageBytes + static_cast<size_t>(lane) * nrow * row_bytes;
        for (int r = 0; r < nrow; ++r) bulk_g2s(dst + r * row_bytes, op.row0 + r * op.step, row_bytes, &full[s]);
      }
    }
  }

  // ---- consumers (until the producer's end marker)
  for (int iter = 0;; ++iter)
    if (!tma_consume<T>(stage, meta, full, empty, ring, iter, lane)) break;
  __threadfence_block();
  if (lane == 0) atomicAdd(&ring->consumers_done, 1u);
}

// ---- multi-GPU launches without ready flags: static round-robin for ~15/16
// of the items, then one atomic per item (the kernel measured before the
// streamed variant existed; kept verbatim -- the streamed kernel's extra warp
// and ticket logic cost ~5% on copy-heavy plans).
// One consumer-warp pass over pipeline stage `iter`: wait for it, form every
// output vector of the item from shared memory, release the stage.  Returns
// false on the producer's end marker.
template <class T, bool kBulk>
__device__ __forceinline__ bool tma_consume_tail(const unsigned char* stage, const uint4* meta,
                                            uint64_t* full, uint64_t* empty, int iter, int lane,
                                            int bulk_outs, int& held) {
  const int ctid = threadIdx.x - 32;
  constexpr int nct = kTmaThreads - 32;
  const int s = iter % kTmaStages;
  mbar_wait(&full[s], (iter / kTmaStages) & 1);
  const uint4* m = meta + s * 32;
  const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
  const int nt = h->nterms;
  if (nt < 0) return false;
  const int nvcol = h->nvcol, nvec = h->nrow * h->nvcol, no = h->nout;
  const int ng = h->ngroups;
  const TmaOperand* outs = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords) + nt;
  const unsigned char* in = stage + s * kStageBytes;
  if constexpr (kBulk) {
    if (nt == 1) {  // outputs may be peer addresses (pushed copies)
      bulk_copy_item(h, outs, in, bulk_outs, empty, s, held);
      return true;
    }
    bulk_release_held(empty, held);
  }
  for (int v = ctid; v < nvec; v += nct) {
    const int r = v / nvcol;
    const int64_t cb = static_cast<int64_t>(v - r * nvcol) * 16;
    uint4 val;
    if (nt == 0) {
      val = make_uint4(0, 0, 0, 0);
    } else if (nt == 1) {
      val = *reinterpret_cast<const uint4*>(in + static_cast<size_t>(v) * 16);
    } else {
      val = grouped_sum16<T>(nt, ng, h->gsize, [&](int k) {
        return *reinterpret_cast<const uint4*>(in + (static_cast<size_t>(k) * nvec + v) * 16);
      });
    }
    for (int o = 0; o < no; ++o) __stcs(reinterpret_cast<uint4*>(outs[o].row0 + r * outs[o].step + cb), val);
  }
  __syncwarp();
  if (lane == 0) mbar_arrive(&empty[s]);
  return true;
}

template <class T, bool kBulk>
__global__ void __launch_bounds__(kTmaThreads, 1) box_phase_tma_tail_kernel(PhaseTables t) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;
  uint4* meta = reinterpret_cast<uint4*>(smem + kTmaStages * kStageBytes);  // 32 words per stage
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kTmaStages * 32);
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_begin();
  if (t.bar_flags) {  // folded cross-rank barrier (replaces a barrier launch)
    volatile int* ok = reinterpret_cast<volatile int*>(meta);  // unused until the first item
    if (threadIdx.x == 0) *ok = folded_barrier(t.bar_flags, t.bar_world, t.bar_rank, t.bar_epoch, t.error);
    __syncthreads();
    const int good = *ok;
    __syncthreads();  // every thread has read it before the producer reuses meta
    if (!good) {  // timed out (error recorded): still retire from the scheduler
      if (threadIdx.x == 0) sched_retire(t);
      return;
    }
  }
  const int W = t.rec_words;

  if (warp == 0) {
    // ---- producer warp: the item record is prefetched one item ahead (one
    // 16-byte word per lane); lane k then streams term k's rows.
    // Items [0, n_static) are dealt round-robin (no dependency: the record is
    // prefetched one item ahead); the tail is handed out dynamically (one
    // atomic per item) so CTAs that drew cheap items keep pulling work.
    const unsigned full_mask = 0xffffffffu;
    auto next_item = [&](int prev, int iter_next) {
      const int st = blockIdx.x + iter_next * static_cast<int>(gridDim.x);
      if (st < t.n_static) return st;
      int d = lane == 0 ? atomicAdd(&t.sched[0], 1) : 0;
      return t.n_static + __shfl_sync(full_mask, d, 0);
    };
    int it = next_item(-1, 0);
    uint4 next = make_uint4(0, 0, 0, 0);
    if (it < t.n_items) if (lane < W) next = t.recs[static_cast<size_t>(it) * W + lane];
    for (int iter = 0;; ++iter) {
      const int cur_it = it;
      const uint4 cur = next;
      if (cur_it < t.n_items) {
        const int nxt = next_item(cur_it, iter + 1);
        it = nxt;
        if (nxt < t.n_items && lane < W) next = t.recs[static_cast<size_t>(nxt) * W + lane];
      }
      const int s = iter % kTmaStages;
      if (iter >= kTmaStages) mbar_wait(&empty[s], ((iter / kTmaStages) + 1) & 1);
      uint4* m = meta + s * 32;
      if (cur_it >= t.n_items) {  // end marker for the consumers
        if (lane == 0) {
          reinterpret_cast<TmaRecHead*>(m)->nterms = -1;
          mbar_arrive_expect_tx(&full[s], 0);
          // the last CTA out resets the scheduler for the next launch
          if (atomicAdd(&t.sched[1], 1) == static_cast<int>(gridDim.x) - 1) {
            t.sched[0] = 0;
            t.sched[1] = 0;
          }
        }
        return;
      }
      if (lane < W) m[lane] = cur;
      __syncwarp();
      const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
      const int nt = h->nterms, nrow = h->nrow;
      const uint32_t row_bytes = static_cast<uint32_t>(h->nvcol) * 16;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], row_bytes * nrow * nt);  // release: meta
      __syncwarp();
      if (lane < nt) {
        const TmaOperand op = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords)[lane];
        unsigned char* dst = stage + s * kStageBytes + static_cast<size_t>(lane) * nrow * row_bytes;
        for (int r = 0; r < nrow; ++r) bulk_g2s(dst + r * row_bytes, op.row0 + r * op.step, row_bytes, &full[s]);
      }
    }
  }

  // ---- consumers (until the producer's end marker)
  int held = -1;  // kBulk, warp 1: the stage its last bulk stores may still be reading
  for (int iter = 0;; ++iter)
    if (!tma_consume_tail<T, kBulk>(stage, meta, full, empty, iter, lane, t.bulk_store, held)) break;
  if (kBulk && (threadIdx.x >> 5) == 1) bulk_wait_all();  // stores complete before the CTA retires
}

// Single-GPU variant (items dealt round-robin, no scheduler state): the
// kernel measured at 93% of HBM peak on cfg2e; kept verbatim because the
// dynamic-schedule kernel's extra per-item work costs ~8% there.
// kBulk (HS_PROG_BULK_STORE): copies leave through TMA bulk stores.  A template
// parameter, so the default instantiation's reduce path compiles exactly as
// before (a runtime branch here cost cfg2b/cfg2d 13-17%).
template <class T, bool kBulk>
__global__ void __launch_bounds__(kTmaThreads, 1) box_phase_tma_static_kernel(PhaseTables t) {
  extern __shared__ __align__(1024) unsigned char smem[];
  unsigned char* stage = smem;
  uint4* meta = reinterpret_cast<uint4*>(smem + kTmaStages * kStageBytes);  // 32 words per stage
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + kTmaStages * 32);
  uint64_t* empty = full + kTmaStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  pdl_begin();
  if (t.bar_flags) {  // folded cross-rank barrier (replaces a barrier launch)
    volatile int* ok = reinterpret_cast<volatile int*>(meta);  // unused until the first item
    if (threadIdx.x == 0) *ok = folded_barrier(t.bar_flags, t.bar_world, t.bar_rank, t.bar_epoch, t.error);
    __syncthreads();
    const int good = *ok;
    __syncthreads();  // every thread has read it before the producer reuses meta
    if (!good) return;
  }
  const int W = t.rec_words;

  if (warp == 0) {
    // ---- producer warp: the item record is prefetched one item ahead (one
    // 16-byte word per lane); lane k then streams term k's rows.
    int iter = 0;
    int it = blockIdx.x;
    uint4 next = make_uint4(0, 0, 0, 0);
    if (it < t.n_items) if (lane < W) next = t.recs[static_cast<size_t>(it) * W + lane];
    for (; it < t.n_items; it += gridDim.x, ++iter) {
      const uint4 cur = next;
      const int nit = it + gridDim.x;
      if (nit < t.n_items && lane < W) next = t.recs[static_cast<size_t>(nit) * W + lane];
      const int s = iter % kTmaStages;
      if (iter >= kTmaStages) mbar_wait(&empty[s], ((iter / kTmaStages) + 1) & 1);
      uint4* m = meta + s * 32;
      if (lane < W) m[lane] = cur;
      __syncwarp();
      const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
      const int nt = h->nterms, nrow = h->nrow;
      const uint32_t row_bytes = static_cast<uint32_t>(h->nvcol) * 16;
      if (lane == 0) mbar_arrive_expect_tx(&full[s], row_bytes * nrow * nt);  // release: meta
      __syncwarp();
      if (lane < nt) {
        const TmaOperand op = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords)[lane];
        unsigned char* dst = stage + s * kStageBytes + static_cast<size_t>(lane) * nrow * row_bytes;
        for (int r = 0; r < nrow; ++r) bulk_g2s(dst + r * row_bytes, op.row0 + r * op.step, row_bytes, &full[s]);
      }
    }
    return;
  }

  // ---- consumers
  const int ctid = threadIdx.x - 32;
  constexpr int nct = kTmaThreads - 32;
  int iter = 0;
  int held = -1;  // warp 1: the stage its last bulk stores may still be reading
  for (int it = blockIdx.x; it < t.n_items; it += gridDim.x, ++iter) {
    const int s = iter % kTmaStages;
    mbar_wait(&full[s], (iter / kTmaStages) & 1);
    const uint4* m = meta + s * 32;
    const TmaRecHead* h = reinterpret_cast<const TmaRecHead*>(m);
    const int nvcol = h->nvcol, nvec = h->nrow * h->nvcol, nt = h->nterms, no = h->nout;
    const int ng = h->ngroups;
    const TmaOperand* outs = reinterpret_cast<const TmaOperand*>(m + kTmaHeadWords) + nt;
    const unsigned char* in = stage + s * kStageBytes;
    if (kBulk && nt == 1) {
      bulk_copy_item(h, outs, in, t.bulk_store, empty, s, held);
      continue;
    }
    if (kBulk) bulk_release_held(empty, held);
    for (int v = ctid; v < nvec; v += nct) {
      const int r = v / nvcol;
      const int64_t cb = static_cast<int64_t>(v - r * nvcol) * 16;
      uint4 val;
      if (nt == 0) {
        val = make_uint4(0, 0, 0, 0);
      } else if (nt == 1) {
        val = *reinterpret_cast<const uint4*>(in + static_cast<size_t>(v) * 16);
      } else {
        val = grouped_sum16<T>(nt, ng, h->gsize, [&](int k) {
          return *reinterpret_cast<const uint4*>(in + (static_cast<size_t>(k) * nvec + v) * 16);
        });
      }
      for (int o = 0; o < no; ++o) __stcs(reinterpret_cast<uint4*>(outs[o].row0 + r * outs[o].step + cb), val);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (kBulk && warp == 1) bulk_wait_all();  // stores complete before the CTA retires
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
__device__ T encode_int(int64_t v) {
  if constexpr (std::is_same_v<T, uint16_t>) return Arith<uint16_t>::narrow(static_cast<float>(v));
  else return static_cast<T>(v);
}

template <class T>
__device__ T encode_real(float v) {
  if constexpr (std::is_same_v<T, uint16_t>) return Arith<uint16_t>::narrow(v);
  else return static_cast<T>(v);
}

template <class T>
__device__ double decode(T v) {
  if constexpr (std::is_same_v<T, uint16_t>) return static_cast<double>(Arith<uint16_t>::widen(v));
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
  constexpr bool kIntegral = std::is_integral_v<T> && !std::is_same_v<T, uint16_t>;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cells;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t lin = cell_lin(f, c);
    if (f.mode == 0 || kIntegral)
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
  const unsigned long long t0 = global_ns();
  for (int p = 0; p < world; ++p) {
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine + p) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (global_ns() - t0 > timeout_ns) {
        *error = 1;
        return;
      }
    }
  }
  __threadfence_system();
}

__global__ void signal_kernel(unsigned int* const* targets, int n, unsigned int epoch) {
  // stream order: the copies before this kernel have completed
  __threadfence_system();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(targets[i]), "r"(epoch) : "memory");
}

__global__ void wait_flags_kernel(const unsigned int* const* flags, int n, unsigned int epoch,
                                  unsigned long long timeout_ns, int* error) {
  const unsigned long long t0 = global_ns();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags[i]) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (*reinterpret_cast<volatile int*>(error) || global_ns() - t0 > timeout_ns) {
        *error = 1;
        break;
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

constexpr size_t kTmaSmem = kTmaStages * kStageBytes + kTmaStages * 32 * sizeof(uint4) +
                            2 * kTmaStages * sizeof(uint64_t);
constexpr size_t kDynSmem = kTmaSmem + sizeof(SigRing);

// Phase kernels launch with the programmatic-stream-serialization attribute
// when the program asks for it (see pdl_begin).
inline void launch_k(void (*k)(PhaseTables), dim3 g, dim3 b, size_t smem, cudaStream_t s, const PhaseTables& t) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = g;
  cfg.blockDim = b;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = t.pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, t);
}

template <class T>
struct PhaseK {
  template <bool R>
  static void reg(dim3 g, dim3 b, cudaStream_t s, PhaseTables t, int vb) {
    switch (vb) {
      case 16: launch_k(box_phase_kernel<T, 16, R>, g, b, 0, s, t); break;
      case 8:
        if constexpr (sizeof(T) <= 8) launch_k(box_phase_kernel<T, 8, R>, g, b, 0, s, t);
        break;
      case 4:
        if constexpr (sizeof(T) <= 4) launch_k(box_phase_kernel<T, 4, R>, g, b, 0, s, t);
        break;
      case 2:
        if constexpr (sizeof(T) <= 2) launch_k(box_phase_kernel<T, 2, R>, g, b, 0, s, t);
        break;
    }
  }
  static void launch(dim3 g, dim3 b, cudaStream_t s, PhaseTables t, int vb, bool tma, bool reduce) {
    if (tma) {
      static bool configured = [] {
        cudaFuncSetAttribute(box_phase_tma_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kDynSmem));
        cudaFuncSetAttribute(box_phase_tma_static_kernel<T, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
        cudaFuncSetAttribute(box_phase_tma_static_kernel<T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
        cudaFuncSetAttribute(box_phase_tma_tail_kernel<T, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
        cudaFuncSetAttribute(box_phase_tma_tail_kernel<T, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kTmaSmem));
        return true;
      }();
      (void)configured;
      if (t.sigs)  // streamed: ready flags, two queues, signaller warp
        launch_k(box_phase_tma_kernel<T>, g, dim3(kDynThreads), kDynSmem, s, t);
      else if (t.n_static >= t.n_items)
        if (t.bulk_store)
          launch_k(box_phase_tma_static_kernel<T, true>, g, dim3(kTmaThreads), kTmaSmem, s, t);
        else
          launch_k(box_phase_tma_static_kernel<T, false>, g, dim3(kTmaThreads), kTmaSmem, s, t);
      else if (t.bulk_store)
        launch_k(box_phase_tma_tail_kernel<T, true>, g, dim3(kTmaThreads), kTmaSmem, s, t);
      else
        launch_k(box_phase_tma_tail_kernel<T, false>, g, dim3(kTmaThreads), kTmaSmem, s, t);
      return;
    }
    if (reduce)
      reg<true>(g, b, s, t, vb);
    else
      reg<false>(g, b, s, t, vb);
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

int tma_grid(int sm_count) { return sm_count; }

cudaError_t launch_expand_records(const PhaseTables& t, int dtype, uint4* recs, int rec_words, int sm_count,
                                  int interleave, cudaStream_t s) {
  if (t.n_items == 0) return cudaSuccess;
  const int blocks = std::max(1, std::min(sm_count * 8, (t.n_items + 7) / 8));
  switch (dtype) {
    case 0: case 2: expand_records_kernel<4><<<blocks, 256, 0, s>>>(t, recs, rec_words, interleave); break;
    case 1: case 3: expand_records_kernel<8><<<blocks, 256, 0, s>>>(t, recs, rec_words, interleave); break;
    case 4: expand_records_kernel<2><<<blocks, 256, 0, s>>>(t, recs, rec_words, interleave); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_phase(const PhaseTables& t, int dtype, int vec_bytes, bool tma, bool reduce,
                         int grid, cudaStream_t s) {
  if (t.n_items == 0) return cudaSuccess;
  return by_dtype<PhaseK>(dtype, dim3(grid), dim3(kBlock), s, t, vec_bytes, tma, reduce);
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

cudaError_t launch_signal(unsigned int* const* targets, int n, unsigned int epoch, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  signal_kernel<<<1, 32, 0, s>>>(targets, n, epoch);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const unsigned int* const* flags, int n, unsigned int epoch,
                              unsigned long long timeout_ns, int* error, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  wait_flags_kernel<<<1, 32, 0, s>>>(flags, n, epoch, timeout_ns, error);
  return cudaGetLastError();
}

cudaError_t launch_barrier(unsigned int* const* peer_flags, int world, int rank,
                           unsigned int epoch, unsigned long long timeout_ns, int* error,
                           cudaStream_t s) {
  barrier_kernel<<<1, 32, 0, s>>>(peer_flags, world, rank, epoch, timeout_ns, error);
  return cudaGetLastError();
}

}  // namespace hshard::exec
