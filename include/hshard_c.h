/* hshard-b200 C ABI — the drop-in boundary of the HSPMD resharding path.
 *
 * The reference (Hetu v2 hshard, /root/reference/proj) is a C++20 library with
 * no FFI; its path is the C++ API in include/hshard (which this library
 * also exports, unchanged).  This header is the thin C layer any host
 * language binds (ctypes / cgo / JNI — see INTEGRATION.md):
 *   - plain pointers, sizes and NUL-terminated strings only;
 *   - annotations cross the boundary in the reference's own text form,
 *     HetAnnotation::str() (reference annotation.cpp:146-170), e.g.
 *       "hsize=2 hdim=0 [(0,1){-1:2}; (2,3){-1:2}] ratios=3/4,1/4";
 *   - every call returns 0 on success or 1 + hshard::Errc on failure
 *     (reference common.hpp:34-70 order; executor codes appended), with a
 *     thread-local message in hs_last_error();
 *   - strings returned through `char**` are malloc'd; release with hs_free.
 *
 * Each entry point names the reference interface it replaces. */
#ifndef HSHARD_C_H_
#define HSHARD_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes = hshard::DType ordinals (reference common.hpp:28 + BF16). */
enum { HS_F32 = 0, HS_F64 = 1, HS_I32 = 2, HS_I64 = 3, HS_BF16 = 4 };

const char* hs_last_error(void);
const char* hs_errc_name(int errc);           /* reference errc_name, common.cpp:50 */
void hs_free(void* p);
int hs_version(void);

/* ---------------------------------------------------------------- planner */
typedef struct hs_plan hs_plan; /* a CommPlan, or a fused switch BsrPlan */

/* classify(src, dst, shape, dtype, bandwidth)          reference resolve.hpp:95-97
 * bw: "u" (Bandwidth::uniform()) or "d=<w>;a-b=<w>;..." (Bandwidth::set). */
int hs_classify(const char* src, const char* dst, const int64_t* shape, int ndim, int dtype,
                const char* bw, hs_plan** out);

/* plan_switch(diff, shapes, bandwidth): build_table per changed tensor, then
 * fuse()                                   SPEC.md:419-427; reference bsr.hpp:50,96
 * shapes_flat holds ndims[i] extents per tensor, concatenated. */
int hs_plan_switch(int n, const int* tensor_ids, const char* const* src, const char* const* dst,
                   const int64_t* shapes_flat, const int* ndims, int dtype, const char* bw,
                   hs_plan** out);

/* Canonical JSON of the plan (byte-identical to oracle/ref_tool's dump of the
 * reference planner's CommPlan / BsrPlan). */
int hs_plan_dump(const hs_plan* plan, char** json);
void hs_plan_destroy(hs_plan* plan);

/* volume_report(plan, node_of)                     reference bsr.hpp:107-108
 * Per-sender intra-/inter-node transfer bytes (the paper's Table 3 shape) of a
 * switch's fused BsrPlan (or of every Bsr step of a CommPlan); node_of is
 * devices[i] -> nodes[i] for i < n.  -> JSON {"device": [intra, inter], ...}
 * with every device of node_of present; UnknownDevice for a transfer end
 * outside it. */
int hs_volume_report(const hs_plan* plan, int n, const int* devices, const int* nodes, char** json);
/* build_table(...) dump                                reference bsr.hpp:50-51 */
int hs_build_table(const char* src, const char* dst, const int64_t* shape, int ndim,
                   int tensor_id, int elem_bytes, char** json);
/* make_plan / make_plan_naive over build_table          reference bsr.hpp:92,100 */
int hs_make_plan(const char* src, const char* dst, const int64_t* shape, int ndim,
                 int elem_bytes, const char* bw, int naive, char** json);

/* placement(anno, shape, device)                  reference annotation.hpp:131
 * lo/hi receive ndim bounds; ord receives {partial_index, partial_count,
 * replica_index, replica_count}. */
int hs_placement(const char* anno, const int64_t* shape, int ndim, int device, int64_t* lo,
                 int64_t* hi, int* ord);
/* convert_hsize                                    reference annotation.hpp:133 */
int hs_convert_hsize(const char* anno, int target, char** out);
/* annotations_equal -> *eq                          reference annotation.hpp:134 */
int hs_annotations_equal(const char* a, const char* b, int* eq);
/* validate -> JSON list of Errc names              reference annotation.hpp:124 */
int hs_validate(const char* anno, const int64_t* shape, int ndim, char** json);
/* align_shard_specs -> JSON [[key_a,key_b,count],...] or null
 *                                                  reference annotation.hpp:143 */
int hs_align_shard_specs(const char* a, const char* b, char** json);

/* ---------------------------------------------------------------- strategy source
 * CompGraph + deduce_graph (reference graph.hpp:105-141, deduction.hpp:29-31)
 * and diff_strategies(graph, a, b).  `graph` is the line
 * form parsed by hshard::parse_graph (include/hshard/graph.hpp).
 * hs_graph_deduce deduces every strategy independently -> JSON
 *   {"tensors":[{"id","name","kind","shape","dtype","producer"}...],
 *    "topo":[node ids], "symbols":[...],
 *    "strategies":[{"ok":1,"slots":[anno or null...]} | {"ok":0,"error":Errc,"message":...}]}
 * hs_graph_diff deduces strategies a and b, binds symbols from `bindings`
 * ("B=8,S=2048"; NULL = none) -> JSON [{"tensor","name","src","dst","shape"}...]. */
int hs_graph_deduce(const char* graph, char** json);
int hs_graph_diff(const char* graph, int a, int b, const char* bindings, char** json);
/* Executable-graph specialization (reference specialize.hpp:27-85): deduce
 * `strategy`, then -> JSON {"phases": {node: "prologue"|"body"|"epilogue"},
 *   "exec_graphs": [{"device", "nodes": [{"node", "comm", "phase", "plan": CommPlan JSON | null}]}],
 *   "pipelines": [[[stage devices]...]...]}  (construct_pipelines' error, if any,
 * is reported as "pipelines_error" instead). */
int hs_graph_specialize(const char* graph, int strategy, const char* bindings, char** json);

/* ---------------------------------------------------------------- executor
 * The reference declares execute_plan (sim.hpp:77-79) but never defines it;
 * this is its B200 implementation.  One hs_ctx per process; one process per
 * GPU ("rank").  Virtual device v of a plan lives on rank v_to_rank[v]. */
typedef struct hs_ctx hs_ctx;
typedef struct hs_prog hs_prog;

/* Creates the per-GPU context: binds `gpu`, allocates a symmetric arena of
 * `arena_bytes` of HBM (all shards, intermediates and staging live in it) and
 * a flag block for cross-rank barriers.  Every rank must pass the same
 * arena_bytes: an (rank, offset) pair names the same buffer everywhere only
 * within the smallest arena (a rank sizing its arena from its own free memory
 * must agree on the minimum with its peers first). */
int hs_ctx_create(int rank, int world, int gpu, size_t arena_bytes, hs_ctx** out);
void hs_ctx_destroy(hs_ctx* ctx);
/* Base device pointer of this rank's arena. */
int hs_ctx_arena(hs_ctx* ctx, void** base, size_t* bytes);
/* IPC handles of this rank's arena/flags (2 x 64 bytes) for peers to open. */
int hs_ctx_ipc_handle(hs_ctx* ctx, unsigned char* out128);
/* Map every peer's arena (handles gathered by the host, rank-major,
 * world x 128 bytes).  Enables peer access.  Call once, after create. */
int hs_ctx_open_peers(hs_ctx* ctx, const unsigned char* all_handles);

/* NCCL communicator over the same ranks, for the HS_PROG_NCCL baseline
 * transport: rank 0 creates the id, the host broadcasts it, every rank inits. */
int hs_nccl_unique_id(unsigned char* out128);
int hs_ctx_nccl_init(hs_ctx* ctx, const unsigned char* id128);

/* Bump allocator inside the arena: offsets are identical on every rank when
 * every rank performs the same sequence of allocations (symmetric heap). */
int hs_ctx_alloc(hs_ctx* ctx, size_t bytes, size_t* offset);
int hs_ctx_reset_alloc(hs_ctx* ctx, size_t offset);

/* Compile a plan for this rank.  v_to_rank maps virtual device id -> rank for
 * ids [0, n_virt).  src_off / dst_off give, per virtual device id, the arena
 * offset of that device's shard on its rank (row-major over its placement
 * box; SIZE_MAX = not present).  Intermediate (mid) shards are allocated
 * from the arena by the compiler (symmetrically). flags: HS_PROG_* bits. */
enum {
  HS_PROG_FUSE_PHASES = 1, /* fuse phase-1 sums into phase-2 tasks (default when world == 1) */
  HS_PROG_NO_FUSE = 2,     /* never fuse (materialise the mid annotation) */
  HS_PROG_NO_TMA = 4,      /* register path only (A/B measurements) */
  HS_PROG_NO_MERGE = 8,    /* one task per destination shard (no multi-output tasks) */
  HS_PROG_NO_TMA_PEER = 16, /* peer-GPU (NVLink) terms use the register path, not TMA */
  HS_PROG_NO_RELAY = 32,    /* world > 1: phase 2 pulls remote mid boxes (no relay stores) */
  HS_PROG_NO_REPLICA = 64,  /* world > 1: read every term from the device the plan names */
  HS_PROG_NO_SHARE = 128,   /* world > 1: identical tasks on several ranks are not chunked */
  HS_PROG_PULL_COPIES = 256, /* world > 1: copies run on the destination's rank (pull) */
  HS_PROG_RELAY_KEEP_LOCAL = 512, /* world > 1: relay-waiting tasks keep local groups in phase 1 */
  HS_PROG_PUSH_ALL = 1024,        /* world > 1: every copy runs on its input's rank */
  HS_PROG_NCCL = 2048             /* world > 1: baseline transport -- remote inputs are packed,
                                     exchanged with grouped ncclSend/ncclRecv, and read locally
                                     (no peer-memory access, no device barriers) */,
  HS_PROG_NO_STREAM = 4096,       /* world > 1: two-phase programs keep a barrier between the
                                     phases instead of one launch with per-chunk ready flags */
  HS_PROG_PULL_MID = 8192,        /* world > 1: phase 2 pulls remote mid boxes from the
                                     producer's HBM (local groups still fused) instead of
                                     relay stores into the consumer's HBM */
  HS_PROG_CE_RELAY = 16384,       /* world > 1: relays move on the copy engines -- producers
                                     write their HBM in K row chunks, each chunk is copied to
                                     its consumers by DMA while the SMs continue, consumers of a
                                     chunk wait for it (implies NO_SHARE | PULL_COPIES) */
  HS_PROG_FANOUT_ONCE = 32768,    /* world > 1: a result stored to several destination shards on
                                     one remote GPU crosses NVLink once; that GPU copies it to
                                     the others in a following phase */
  HS_PROG_STATIC_LOCAL = 1 << 24, /* world > 1: launches of local-only items of one task shape
                                     use the fully static TMA kernel (bits 16..23 hold
                                     HS_PROG_STREAM_SHARE) */
  HS_PROG_BULK_STORE = 1 << 25,   /* the static TMA kernel stores the first two outputs of a copy
                                     with TMA bulk stores out of the staging buffer (the rest from
                                     registers); faster on some plans, slower on others -- the
                                     autotuner times it */
  HS_PROG_SEPARATE_BARRIERS = 1 << 26, /* world > 1: every cross-rank barrier is its own launch
                                     (default: folded into the prologue of the phase's first
                                     launch when that is a TMA kernel) */
  HS_PROG_SMALL_ITEMS = 1 << 27,  /* 16 KB TMA work items instead of 32 KB: plan-dependent (faster
                                     for two-output copies, slower for long single-output ones) --
                                     the autotuner times it */
  HS_PROG_NO_PDL = 1 << 28,       /* launch phase kernels without programmatic dependent launch
                                     (default: each launch is scheduled while the previous one on
                                     the stream drains and waits for it on the device) */
  HS_PROG_INTERLEAVE = 1 << 29,   /* world > 1, unstreamed launches: items of tasks with NVLink
                                     operands and of local-only tasks are merged evenly in launch
                                     order (default: task order) -- the autotuner times it */
  HS_PROG_SPLIT_RELAY = 1 << 30    /* world > 1, two-phase plans: a consumer's remote mid rows are
                                     split in two bands -- the producers push the first band into
                                     the consumer's relay buffer before the barrier, the consumer
                                     pulls the second after it -- so the NVLink transfer is spread
                                     over both phases; the autotuner times it */
};
/* Streamed programs: bits 16..23 of the flags = the share of CTAs that take
 * non-waiting work first, in 1/64 (0 = modelled from the phases' bytes). */
#define HS_PROG_STREAM_SHARE(sixty_fourths) (((sixty_fourths) & 0xff) << 16)
int hs_prog_compile(hs_ctx* ctx, const hs_plan* plan, const int* v_to_rank, int n_virt,
                    const size_t* src_off, const size_t* dst_off, int flags, hs_prog** out);
/* The same over CALLER-OWNED device buffers (the reference's functional
 * execute_plan takes shards as values, sim.hpp:77-79; a shard is
 * {device, gpu_ptr, box}): src_ptrs / dst_ptrs[slot * n_virt + v] is the
 * address of that shard, row-major over its placement box, valid in THIS
 * process -- any cudaMalloc / framework-allocator pointer on this GPU, or a
 * peer's buffer mapped with hs_ipc_import (N > 1).  NULL = absent (only the
 * shards this rank's tasks touch are required).  Buffers are not copied: the
 * program reshards the framework's tensors in place of a copy through the
 * arena.  HS_PROG_CE_RELAY is not available in this mode. */
int hs_prog_compile_ptrs(hs_ctx* ctx, const hs_plan* plan, const int* v_to_rank, int n_virt,
                         void* const* src_ptrs, void* const* dst_ptrs, int flags, hs_prog** out);
/* Multi-process buffers: export the allocation holding a local device pointer
 * (80 bytes: IPC handle, offset, allocation size) for the host to exchange;
 * import a peer's export into this process (mapped once per allocation,
 * closed with the context). */
int hs_ipc_export(hs_ctx* ctx, const void* ptr, unsigned char* out80);
int hs_ipc_import(hs_ctx* ctx, const unsigned char* in80, void** ptr);
void hs_prog_destroy(hs_prog* prog);
/* Run on `stream` (cudaStream_t, NULL = the ctx stream).  Multi-rank programs
 * include device-side barriers; every rank must call run. */
int hs_prog_run(hs_prog* prog, void* stream);
/* Host-buffer execution (reference-facing e2e path): H2D of this rank's
 * source shards from host pointers (indexed by virtual id; NULL = skip),
 * run, D2H of destination shards.  Synchronous. */
int hs_prog_run_host(hs_prog* prog, const void* const* src_host, void* const* dst_host);
/* The same, enqueued without synchronising: H2D on `h2d` (cudaStream_t),
 * the run on `compute` after it, D2H on `d2h` after the run (events order the
 * three streams).  A caller double-buffers steps with two programs over two
 * shard layouts sharing one compute stream (runs, and their barriers, stay in
 * order) so step k+1's H2D overlaps step k's run and D2H on a full-duplex
 * link.  Completion: synchronise `d2h`. */
int hs_prog_run_host_async(hs_prog* prog, const void* const* src_host, void* const* dst_host, void* h2d,
                           void* compute, void* d2h);
/* Per-phase kernel timing with CUDA events on the launching stream (bench /
 * roofline evidence).  hs_prog_profile(1) resets and enables; every run then
 * records 2 events per phase; hs_prog_phase_ms sums elapsed ms per phase over
 * the profiled runs (synchronising) and reports the run count. */
int hs_prog_profile(hs_prog* prog, int enable);
int hs_prog_phase_ms(hs_prog* prog, double* out, int n, int* runs);
/* JSON statistics: kernels per run, bytes (HBM read/write, NVLink in/out) per
 * run for this rank, task counts. */
int hs_prog_stats(const hs_prog* prog, char** json);

/* CPU-only dry run: compile `plan` for `rank` of `world` (virtual arenas, no
 * CUDA) and return the program statistics and this rank's final task list
 * as JSON (box, outputs, inputs, groups) -- how the multi-GPU partitioning is
 * tested without GPUs. */
int hs_analyze(const hs_plan* plan, int rank, int world, const int* v_to_rank, int n_virt, int flags,
               char** stats_json, char** tasks_json);

/* Deterministic counter-hash payload, written
 * into this rank's shard of virtual device `dev` for annotation `anno`. */
int hs_fill_shard(hs_ctx* ctx, const char* anno, const int64_t* shape, int ndim, int dtype,
                  int device, size_t offset, uint32_t seed, int tensor_id, int mode,
                  void* stream);
/* Count cells of the shard at `offset` that differ from the logical
 * counter-hash tensor (grid mode; non-Partial annotations only). */
int hs_verify_shard(hs_ctx* ctx, const char* anno, const int64_t* shape, int ndim, int dtype,
                    int device, size_t offset, uint32_t seed, int tensor_id,
                    unsigned long long* mismatches, void* stream);
/* Copy `bytes` at arena `offset` to/from host (synchronous). */
int hs_ctx_read(hs_ctx* ctx, size_t offset, void* host, size_t bytes);
int hs_ctx_write(hs_ctx* ctx, size_t offset, const void* host, size_t bytes);
int hs_ctx_sync(hs_ctx* ctx);
/* Enqueue a device-side cross-rank barrier on `stream` (NULL = the context's
 * stream): after it, every rank's work enqueued before its own barrier call
 * is complete and visible (the barrier each program run opens with).  Every
 * rank must call it; a rank that never arrives is reported as
 * DeadlockDetected by hs_ctx_sync.  No-op at world 1. */
int hs_ctx_barrier(hs_ctx* ctx, void* stream);
/* Clear a recorded DeadlockDetected (a timed-out barrier or ready-flag wait)
 * once every rank has drained, so the context can run again.  Kernels that
 * gave up still retire from their scheduler, so programs stay reusable. */
int hs_ctx_clear_error(hs_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* HSHARD_C_H_ */
