// hshard-b200 executor: device-side descriptor tables and kernel entry points.
//
// A compiled program is, per plan phase, a flat table of box TASKS
//   out_0 = out_1 = ... := zero | round(sum_g round_g(sum_{t in g} term_t))
// each over a <=4-D strided box whose innermost dim is contiguous.  Terms are
// summed in table order inside a group and groups in table order; a group of
// size > 1 is rounded to the storage dtype before it joins the outer sum, so a
// fused two-phase plan (phase-1 sums feeding phase-2 sums through the
// intermediate "mid" annotation) rounds exactly where the unfused plan does.
// A table of WORK ITEMS cuts tasks into pieces (a run of rows of one plane of
// the box) so one persistent launch load-balances every box of a phase.
// Terms may be peer-GPU addresses (NVLink loads); outputs are local.
#pragma once

#include <cstdint>

#include <cuda_runtime.h>

namespace hshard::exec {

inline constexpr int kMaxTerms = 16;
inline constexpr int kMaxOuts = 8;

struct TermDesc {
  const char* base;   // byte address of the box origin (may be a peer address)
  int64_t stride[3];  // element strides of outer dims 1..3
};

struct TaskDesc {
  int32_t n[4];       // extents; n[0] innermost (contiguous) in elements
  int32_t out0;       // first output in the term table (base = write address)
  int32_t nout;       // >= 1 outputs receive the same value
  int32_t term0;      // first input term
  int32_t nterms;     // 0 = zero-fill, 1 = copy, >1 = grouped ordered sum
  int32_t ngroups;    // 0 = flat (every term its own group)
  int32_t vec_bytes;  // widest vector legal for every pointer and stride
  uint8_t gsize[16];  // group sizes when ngroups > 0
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

// TMA-path item record, one fixed-size slot per item so the producer warp
// fetches one 16-byte word per lane, prefetched an item ahead (no dependent
// descriptor loads on its critical path): TmaRecHead, then (nterms + nout)
// TmaOperand (terms first, then outputs).  The host builds only one TmaTask
// per box task (TMA tasks own contiguous item ranges, TmaTask::item0); the
// records are expanded from them on the device at compile time
// (launch_expand_records) -- a cfg4 switch uploads 1034 descriptors instead of
// building 445k records on the host.
struct TmaRecHead {
  int32_t nterms, nout, ngroups, nrow;
  int32_t nvcol;
  int32_t wait;  // streamed launches: flag index this item waits on (-1: none)
  int32_t sig;   // streamed launches: SigDesc index signalled when its task is done (-1: none)
  int32_t need;  // producer pieces the waited-on flag counts per run
  uint8_t gsize[16];
};
struct TmaOperand {
  char* row0;    // address of the item's first row (may be a peer address for terms)
  int64_t step;  // bytes between rows
};
inline constexpr int kTmaHeadWords = sizeof(TmaRecHead) / 16;                 // 3

// A TMA box task: the item geometry and the record fields that do not vary
// by item.  Items [item0, next task's item0) cut the task's (plane, row) space
// into either row chunks (mode 0: one row, `per` vectors per item, `cpr`
// items per row) or row runs (mode 1: `per` whole rows per item, `cpr` items
// per plane); planes are (dim2, dim3) pairs, dim2 of extent n2.
struct TmaTask {
  int32_t item0;               // first item of the task in launch order
  int32_t nterms, nout, ngroups;
  int32_t wait, sig, need;     // as TmaRecHead
  int32_t mode;                // 0 row chunks, 1 row runs
  int32_t n1, n2;              // rows per plane, dim-2 extent
  int32_t row_vecs;            // 16-byte vectors per row
  int32_t per;                 // mode 0: vectors per item; mode 1: rows per item
  int32_t cpr;                 // mode 0: items per row; mode 1: items per plane
  int32_t term0, out0;         // operands in PhaseTables::terms
  int32_t pad;
  uint8_t gsize[16];
};
static_assert(sizeof(TmaTask) == 80, "TmaTask layout");
inline constexpr int kTmaMaxWords = kTmaHeadWords + kMaxTerms + kMaxOuts;    // 27 <= 32 lanes

// Streamed launches (both plan phases in one launch, no barrier between):
// a producer task's last finished item adds 1 (red.release.sys) to the flag
// of every consumer piece that reads its output, on the consumer's rank; a
// consumer item's producer warp waits (ld.acquire.sys) until its flag reaches
// epoch * need before loading.
struct SigDesc {
  uint32_t done;      // index of this task's item counter in PhaseTables::done
  uint32_t expected;  // TMA items of the task per run
  uint32_t target0;   // first flag pointer in PhaseTables::targets
  uint32_t ntargets;
};

struct PhaseTables {
  const TaskDesc* tasks;
  const TermDesc* terms;
  const WorkItem* items;  // register path
  const uint4* recs;      // TMA path: n_items slots of rec_words 16-byte words
  const TmaTask* ttasks;  // TMA path: n_ttasks descriptors in item order (+ sentinel); the
  int32_t n_ttasks;       // source launch_expand_records expands `recs` from
  int* sched;             // TMA path: {next first-queue item, finished CTAs, next second-queue
                          // item, pad}; zero between launches
  int32_t n_items;
  int32_t rec_words;      // TMA path: 16-byte words of the widest record of the launch
  int32_t n_static;       // TMA path: items [0, n_static) are dealt round-robin
  // TMA path queues: items [0, n_first) never wait; [n_first, n_items) may.
  // CTAs [0, first_ctas) drain the first queue, then the second; the others
  // take only the second, so no item that signals is ever queued behind a wait.
  int32_t n_first;
  int32_t first_ctas;
  uint32_t epoch;                    // run number (streamed launches)
  const SigDesc* sigs;
  unsigned int* const* targets;      // flag addresses, possibly on peers
  unsigned long long* done;          // per signalling task: items finished, all runs
  const unsigned int* wait_flags;    // this rank's flags
  int* error;                        // set when a wait times out (DeadlockDetected)
  unsigned long long* trace;         // debug (HS_TRACE): 8 globaltimer words per CTA, or null
  int32_t bulk_store;                // static TMA kernel: a copy's first bulk_store outputs leave
                                     // through TMA bulk stores (0: all from registers)
  // Folded cross-rank barrier (TMA kernels): when bar_flags is
  // set the kernel opens with launch_barrier's protocol for bar_epoch instead
  // of a separate barrier launch in front of it.
  unsigned int* const* bar_flags;    // every rank's flag array (peer-mapped), or null
  int32_t bar_world, bar_rank;
  uint32_t bar_epoch;
  int32_t pdl;                       // launch with programmatic stream serialization (pdl_begin)
};

// Shared-memory staging of the TMA kernel: kStages ring buffers of
// kStageBytes; the host sizes 16-byte-vector items so that
// nterms * nrow * nvcol * 16 <= kStageBytes.
#ifndef HS_TMA_STAGES  // exploration builds override these (tools/stage_sweep.sh)
#define HS_TMA_STAGES 4
#endif
#ifndef HS_STAGE_KB
#define HS_STAGE_KB 48
#endif
inline constexpr int kTmaStages = HS_TMA_STAGES;
inline constexpr int kStageBytes = HS_STAGE_KB * 1024;

// dtype codes follow hshard::DType (F32, F64, I32, I64, BF16).
// `tma`: items were sized for the TMA pipeline (16-byte vectors only).
// `reduce`: register-path items of tasks with >= 2 terms (a separate, higher
// register-budget instantiation from the copy/zero one).
cudaError_t launch_phase(const PhaseTables& t, int dtype, int vec_bytes, bool tma, bool reduce,
                         int grid, cudaStream_t s);
int tma_grid(int sm_count);
// Writes the launch's TMA item records (t.recs, t.rec_words words each) from
// its task descriptors (t.ttasks), on the device.  interleave in (0, n_items):
// the first `interleave` items and the rest are merged evenly in launch order.
cudaError_t launch_expand_records(const PhaseTables& t, int dtype, uint4* recs, int rec_words, int sm_count,
                                  int interleave, cudaStream_t s);

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

// Copy-engine relays: after the copies of a chunk, the sender's copy stream
// stores `epoch` (st.release.sys) into each receiver's flag word; the
// receiver's compute stream spins (ld.acquire.sys, bounded) until all its
// senders' words reach `epoch`.  Both are one-warp kernels.
cudaError_t launch_signal(unsigned int* const* targets, int n, unsigned int epoch, cudaStream_t s);
cudaError_t launch_wait_flags(const unsigned int* const* flags, int n, unsigned int epoch,
                              unsigned long long timeout_ns, int* error, cudaStream_t s);

}  // namespace hshard::exec
