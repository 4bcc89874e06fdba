// hshard-b200 executor: device-side descriptor tables and kernel entry points.
//
// A compiled program is, per plan phase, a flat table of box TASKS
//   dst_box := zero | copy(term0) | term0 + term1 + ... (fixed order, one rounding)
// each over a <=4-D strided box (innermost dim contiguous), and a table of
// WORK ITEMS that cut tasks into ~32-64 KB pieces so one persistent launch
// load-balances every box of every step of the phase across all 148 SMs.
// Terms may point into peer GPUs' arenas (NVLink loads): the same kernel is
// the intra-GPU box copy, the cross-GPU pull and the fused reduce-unpack.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace hshard::exec {

inline constexpr int kMaxTerms = 16;

struct TermDesc {
  const char* base;   // byte address of the box origin (may be a peer address)
  int64_t stride[3];  // element strides of outer dims 1..3
};

struct TaskDesc {
  char* dst;              // byte address of the box origin
  int64_t dst_stride[3];  // element strides of outer dims 1..3
  int32_t n[4];           // extents; n[0] innermost (contiguous) in elements
  int32_t term0;          // first term in the term table
  int32_t nterms;         // 0 = zero-fill, 1 = copy, >1 = ordered sum
  int32_t vec_bytes;      // 16/8/4/2/1: widest vector legal for every pointer and stride
  int32_t pad;
};

// A run of `nrow` consecutive rows of one (dim2, dim3) plane of a task,
// restricted to vectors [vcol0, vcol0 + nvcol) of each row.
struct WorkItem {
  int32_t task;
  int32_t row0;   // first dim-1 index
  int32_t nrow;
  int32_t plane;  // dim2 + n[2] * dim3
  int32_t vcol0;
  int32_t nvcol;
};

struct PhaseTables {
  const TaskDesc* tasks;
  const TermDesc* terms;
  const WorkItem* items;
  int32_t n_items;
};

// dtype codes follow hshard::DType (F32, F64, I32, I64, BF16).
// All items of one launch share the vector width `vec_bytes` (the kernel is
// specialised on it); a phase is split into at most one launch per width.
cudaError_t launch_phase(const PhaseTables& t, int dtype, int vec_bytes, int grid, cudaStream_t s);

// Counter-hash payload generator (mirror of oracle/datagen.py).
struct FillDesc {
  char* dst;
  int32_t ndim;
  int64_t shape[4];   // logical tensor
  int64_t lo[4];      // box origin (logical)
  int64_t ext[4];     // box extents
  uint32_t seed;
  int32_t tensor_id;
  int32_t hsize;
  int32_t tg;         // top partial piece (-1: none)
  int32_t g;          // subgroup
  int32_t p, P;       // bottom partial ordinal / count
  int32_t mode;       // 0 grid, 1 real
};
cudaError_t launch_fill(const FillDesc& f, int dtype, cudaStream_t s);
// Counts cells != logical grid value into *mismatches (device pointer).
cudaError_t launch_verify(const FillDesc& f, int dtype, unsigned long long* mismatches,
                          cudaStream_t s);

// Cross-rank barrier over peer-mapped flag words: every rank writes `epoch`
// into slot[rank] of every peer's flag array, then waits until its own array
// holds >= epoch in every slot.  Bounded spin: gives up after ~`timeout_ns`
// and records 1 in *error.
cudaError_t launch_barrier(unsigned int* const* peer_flags, int world, int rank,
                           unsigned int epoch, unsigned long long timeout_ns, int* error,
                           cudaStream_t s);

}  // namespace hshard::exec
