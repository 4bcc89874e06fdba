// hshard-b200 executor: host-side context and plan compiler.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "hshard/resolve.hpp"
#include "hshard_c.h"
#include "hshard/switch.hpp"
#include "kernels.cuh"

namespace hshard::exec {

// HS_COMPILE_TRACE=1: per-stage compile times on stderr (cold-switch analysis).
struct StageClock {
  bool on = std::getenv("HS_COMPILE_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[compile] %-18s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

void cuda_check(cudaError_t e, const char* what);

// Device memory for program tables: first-fit in a block reserved with the
// context (HS_TABLE_POOL_MB, default 1024), so compiling a program does not
// pay cudaMalloc (3-16 ms measured for a cfg4 switch's 35 MB of records);
// beyond the block, cudaMalloc.  Owned jointly by the context and its
// programs: freed when the last of them goes.
class TablePool {
 public:
  TablePool(int gpu, size_t bytes);
  ~TablePool();
  void* alloc(size_t bytes);
  void free(void* p);

 private:
  std::mutex mu_;
  int gpu_;
  char* base_ = nullptr;
  size_t bytes_ = 0;
  std::map<size_t, size_t> free_;  // offset -> bytes (coalesced)
  std::map<size_t, size_t> used_;  // offset -> bytes
};

// Per-GPU context: one per process ("rank").  Owns the symmetric arena, the
// barrier flag block and (after open_peers) every peer's mapped arena.
class Context {
 public:
  Context(int rank, int world, int gpu, size_t arena_bytes);
  ~Context();
  // CUDA-free context for plan analysis (hs_analyze): virtual arenas, no
  // device memory; programs compiled against it build no device tables.
  static std::unique_ptr<Context> analysis(int rank, int world);
  bool is_analysis() const { return analysis_; }

  int rank() const { return rank_; }
  int world() const { return world_; }
  int gpu() const { return gpu_; }
  char* arena() const { return arena_; }
  size_t arena_bytes() const { return arena_bytes_; }
  cudaStream_t stream() const { return stream_; }
  char* arena_of(int r) const;  // this or a peer's arena base (mapped)
  bool peers_open() const { return world_ == 1 || peers_open_; }
  int sm_count() const { return sm_count_; }

  void ipc_handles(unsigned char out[128]) const;
  void open_peers(const unsigned char* all);  // world x 128 bytes, rank-major

  size_t alloc(size_t bytes);  // 256-byte aligned bump allocation
  void reset_alloc(size_t offset);
  size_t alloc_cursor() const { return cursor_; }

  // Cross-rank barrier on `s` (no-op when world == 1).
  void barrier(cudaStream_t s);
  // The same barrier folded into the prologue of the kernel launched next:
  // consumes an epoch; the kernel signals and waits (PhaseTables::bar_*).
  unsigned int next_epoch() { return ++epoch_; }
  unsigned int* const* peer_flag_table() const { return d_peer_flags_; }
  void check_barrier_error();
  // Clears a recorded DeadlockDetected (after the caller has drained every
  // rank), so the context can run again.
  void clear_error();

  unsigned long long* scratch_counter() const { return counter_; }
  int* error_flag() const { return barrier_error_; }

  // Caller-owned buffers across processes: export the allocation holding a
  // local device pointer (IPC handle + offset), import a peer's export
  // (mapped once per allocation; closed with the context).
  void ipc_export(const void* ptr, unsigned char out[80]) const;
  char* ipc_import(const unsigned char in[80]);

  // Device memory for program tables (TablePool, shared with the programs so
  // that a program destroyed after its context still frees correctly).
  const std::shared_ptr<TablePool>& tables() const { return pool_; }

  // NCCL communicator over the same ranks (HS_PROG_NCCL baseline transport).
  void nccl_init(const unsigned char id[128]);
  void* nccl_comm() const { return nccl_comm_; }

 private:
  int rank_, world_, gpu_;
  int sm_count_ = 148;
  char* arena_ = nullptr;
  size_t arena_bytes_ = 0;
  size_t cursor_ = 0;
  unsigned int* flags_ = nullptr;  // world slots, written by peers
  int* barrier_error_ = nullptr;
  unsigned long long* counter_ = nullptr;
  unsigned int** d_peer_flags_ = nullptr;
  std::vector<char*> peer_arena_;
  std::vector<unsigned int*> peer_flags_;
  std::map<std::string, char*> imported_;  // IPC handle bytes -> mapped base
  std::shared_ptr<TablePool> pool_;
  unsigned int epoch_ = 0;
  bool peers_open_ = false;
  cudaStream_t stream_ = nullptr;
  void* nccl_comm_ = nullptr;  // ncclComm_t
  bool analysis_ = false;
  struct AnalysisTag {};
  Context(AnalysisTag, int rank, int world);
};

// Where one tensor's shard for one virtual device lives in one layout state.
struct ShardLoc {
  SliceRegion region;
  int rank = -1;
  size_t offset = SIZE_MAX;  // arena byte offset on `rank`
  char* ptr = nullptr;       // caller-owned buffer (hs_prog_compile_ptrs): address in this process
  int subgroup = 0;          // annotation subgroup of the device
  int eff_hdim = -1;         // effective hdim of the annotation
};

// A shard in a layout state: (state, virtual device); the tensor is the task's.
struct Operand {
  int state = 0;
  DeviceId dev = -1;
  bool operator==(const Operand&) const = default;
  bool operator<(const Operand& o) const { return state != o.state ? state < o.state : dev < o.dev; }
};

// One box task in logical coordinates:
//   every dst := zero | round(sum_g round_g(sum_{t in g} term_t))
struct BoxTask {
  int phase = 0;
  StepKind kind = StepKind::Identity;
  int tensor = 0;
  int rank = 0;                 // executing rank (its kernels run this task)
  SliceRegion box;              // logical coordinates (bounds only)
  std::vector<Operand> dsts;    // >= 1; relay outputs may be on other ranks
  std::vector<Operand> terms;   // summation order; empty = zero-fill
  std::vector<int> groups;      // sizes; empty = flat (each term its own group)
  // streamed programs (one launch for both plan phases):
  int wait = -1;                // this consumer piece's flag index on its rank (-1: none)
  int need = 0;                 // producer pieces that signal that flag per run
  std::vector<std::pair<int, int>> targets;  // (rank, flag) signalled when this task is done
};

struct ProgramStats {
  int phases = 0;            // launched phases after fusion
  int plan_phases = 0;       // phases of the plan
  int64_t tasks = 0, items = 0, terms = 0, outputs = 0;
  int64_t copy_tasks = 0, reduce_tasks = 0, zero_tasks = 0, tma_items = 0;
  int64_t fused_tasks = 0;   // phase-2 tasks that read phase-1 inputs directly
  int64_t relay_outputs = 0; // phase-1 outputs stored into a consumer rank's relay buffer
  int64_t replica_swaps = 0; // remote terms re-sourced from a bit-identical replica
  int64_t shared_chunks = 0; // per-rank chunks of tasks shared across ranks
  int64_t pushed_copies = 0; // copies executed on the source's rank (remote stores)
  double model_ms[2] = {0, 0};  // relay variants' modelled time (keep-local, fuse-local)
  // Algorithmic bytes per run for THIS rank:
  int64_t hbm_read = 0;      // bytes of terms read from this GPU's HBM
  int64_t hbm_write = 0;     // bytes written to this GPU's HBM
  int64_t nvlink_in = 0;     // bytes of terms pulled from peers
  int64_t nvlink_out = 0;    // bytes peers pull from this GPU
  int64_t dst_bytes = 0;     // destination-resident bytes on this rank
  int64_t src_bytes = 0;     // source-resident bytes on this rank
  int64_t h2d_bytes = 0;     // host-buffer path: source bytes copied in per run (shards some task reads)
  int kernels_per_run = 0;   // phase kernels + barrier kernels
  bool streamed = false;     // both plan phases in one launch (ready flags)
  bool ce_relay = false;     // relays moved by the copy engines
  size_t trace_off = 0;      // EXPERIMENT
  int trace_ctas = 0;
  std::vector<int64_t> phase_items;
  // per launched phase, this rank: {local HBM read, HBM write, NVLink in}
  std::vector<std::array<int64_t, 3>> phase_bytes;
};

class Program {
 public:
  // Plan kinds: a CommPlan (one tensor) or a fused switch plan (many tensors).
  // Shards live in the arenas (src_off / dst_off: per (tensor slot, virtual
  // device) arena offsets on the owning rank) or in caller-owned buffers
  // (src_ptr / dst_ptr: addresses valid in THIS process -- local allocations,
  // or peers' buffers mapped with hs_ipc_import; null = absent).
  Program(Context& ctx, const CommPlan* comm, const SwitchPlan* sw, const std::vector<int>& v_to_rank,
          const size_t* src_off, const size_t* dst_off, int flags, const void* const* src_ptr = nullptr,
          const void* const* dst_ptr = nullptr);
  ~Program();

  void run(cudaStream_t s);
  void run_host(const void* const* src_host, void* const* dst_host);
  void run_host_async(const void* const* src_host, void* const* dst_host, cudaStream_t h2d, cudaStream_t compute,
                      cudaStream_t d2h);
  // Profiling: when enabled, run() brackets each phase's launches with CUDA
  // events on the launching stream; phase_ms() sums the elapsed times of all
  // runs since enabling (synchronises) and returns the run count.
  void set_profiling(bool on);
  int phase_ms(double* out, int n);
  int phases() const { return n_phases_; }
  const ProgramStats& stats() const { return stats_; }
  std::string stats_json() const;
  // Analysis contexts only: this rank's tasks after every rewrite.
  std::string tasks_json() const;
  int dtype() const { return dtype_; }

 private:
  struct Launch {
    PhaseTables tables{};
    int vec_bytes = 16;
    bool tma = false;
    bool reduce = false;
    int grid = 1;
  };
  struct DevicePhase {
    std::vector<Launch> launches;  // TMA launch + one per vector width present
    bool fold_barrier = false;     // the opening barrier runs in launches[0]'s prologue
  };

  void lower(const CommPlan* comm, const SwitchPlan* sw);
  // None: world 1 fusion.  KeepLocal / FuseLocal: remote mid reads become
  // relays (producers store into the consumer's HBM).  Pull: remote mid
  // reads pull the producer's materialised mid box (local groups fused).
  enum class RelayMode { None, KeepLocal, FuseLocal, Pull, Split };
  std::vector<BoxTask> fuse_phases(std::vector<BoxTask> tasks, RelayMode mode);
  double estimate_seconds(const std::vector<BoxTask>& tasks, int phases);
  void stage_for_nccl(std::vector<BoxTask>& tasks);
  void choose_replicas(std::vector<BoxTask>& tasks);
  std::vector<BoxTask> spread_shared(std::vector<BoxTask> tasks);
  static std::vector<BoxTask> merge_outputs(std::vector<BoxTask> tasks);
  std::vector<BoxTask> stream_phases(const std::vector<BoxTask>& tasks);
  std::vector<BoxTask> ce_relay(std::vector<BoxTask> tasks);
  std::vector<BoxTask> fanout_once(std::vector<BoxTask> tasks);
  void ce_geometry();  // copy geometry once offsets are assigned
  void ce_build();     // device-side signal / wait pointer tables
  void ce_run_phase_post(int p, cudaStream_t s);
  struct Flat;
  Flat flatten(const BoxTask& bt);
  bool tma_capable(const BoxTask& bt);
  bool tma_capable(const BoxTask& bt, const Flat& f);
  void build_tables(const std::vector<BoxTask>& tasks);
  ShardLoc& loc(int state, int tensor, DeviceId d);
  char* addr_of(const ShardLoc& L) const { return L.ptr ? L.ptr : ctx_.arena_of(L.rank) + L.offset; }
  static bool present(const ShardLoc& L) { return L.ptr || L.offset != SIZE_MAX; }

  Context& ctx_;
  int flags_ = 0;
  int dtype_ = 0;
  int es_ = 4;
  int n_virt_ = 0;
  int n_tensors_ = 1;
  int mid_state_ = -1;  // layout state index of the plan's mid annotation
  size_t final_state_ = 0;  // layout state index of the destination
  std::vector<int> v_to_rank_;
  std::vector<Shape> shapes_;
  // layout states: 0 = src, 1 = mid (CommPlan with mid) / dst, 2 = dst
  std::vector<std::map<std::pair<int, DeviceId>, ShardLoc>> states_;
  // loc() cache: per state, [tensor * n_virt + dev] -> map node (map nodes
  // never move and are never erased), filled on first lookup
  std::vector<std::vector<ShardLoc*>> dense_;
  int n_phases_ = 0;
  std::vector<DevicePhase> dphases_;
  void* dev_block_ = nullptr;
  std::shared_ptr<TablePool> pool_;  // dev_block_'s owner
  bool profiling_ = false;
  bool remote_final_writes_ = false;  // last phase stores into peers' shards
  bool streamed_ = false;             // both plan phases in one launch (ready flags)
  // HS_PROG_CE_RELAY: phases [0, K) produce row chunk k (exported), K = other
  // phase-1 work, K+1+k consume chunk k, 2K+1 = other phase-2 work.
  struct CeCopy {
    int chunk, sender, receiver;
    size_t src_off, dst_off;       // arena byte offsets (sender's mid, receiver's relay)
    size_t width, height, pitch;   // 2-D geometry (bytes, rows, bytes between rows)
    size_t planes, plane_stride;   // outer dim of a 3-D box
  };
  bool ce_mode_ = false;
  int ce_chunks_ = 4;
  size_t ce_flag_off_ = 0;                  // symmetric world x K flag words
  std::vector<CeCopy> ce_copies_;           // every rank's
  std::vector<SliceRegion> ce_boxes_;       // the logical box of each copy
  std::vector<DeviceId> ce_mid_dev_, ce_relay_dev_;
  std::vector<unsigned int**> ce_targets_;  // per chunk: device array of receivers' flag words
  std::vector<int> ce_ntargets_;
  std::vector<const unsigned int**> ce_waits_;  // per chunk: device array of my senders' flag words
  std::vector<int> ce_nwaits_;
  void* ce_dev_ = nullptr;
  cudaStream_t ce_stream_ = nullptr;
  std::vector<cudaEvent_t> ce_events_;
  size_t flag_off_ = 0;               // arena offset of the symmetric ready-flag array
  uint32_t runs_ = 0;                 // run counter = flag epoch
  // HS_PROG_NCCL baseline: per plan phase, this rank's grouped send/recv list
  struct Exchange {
    int peer;
    bool send;
    size_t offset;  // arena offset of the message
    size_t bytes;
  };
  bool nccl_mode_ = false;
  int staging_state_ = 1 << 30;
  std::vector<std::vector<Exchange>> exchanges_;
  std::vector<cudaEvent_t> events_;  // 2 per phase per profiled run
  cudaEvent_t host_ev_[3] = {nullptr, nullptr, nullptr};  // run_host_async: inputs landed / run done / read
  size_t events_used_ = 0;
  ProgramStats stats_;
  StageClock clock_;
  std::vector<BoxTask> analysed_;  // analysis contexts: this rank's final tasks
  // host-buffer path: (virtual device, tensor) -> (device address, bytes) on this rank
  std::vector<std::tuple<DeviceId, int, char*, size_t>> host_src_, host_dst_;
};

}  // namespace hshard::exec
