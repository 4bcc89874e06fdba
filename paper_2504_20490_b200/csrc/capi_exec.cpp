// hshard-b200 C ABI: executor entry points (include/hshard_c.h).
#include <cstring>
#include <memory>

#include "capi_common.hpp"
#include "exec/nccl_dyn.hpp"
#include "exec/program.hpp"

using namespace hshard;
using namespace hshard::capi;

struct hs_ctx {
  std::unique_ptr<exec::Context> c;
};
struct hs_prog {
  std::unique_ptr<exec::Program> p;
};

namespace {

exec::FillDesc fill_desc(hs_ctx* ctx, const char* anno, const int64_t* shape, int ndim, int dtype,
                         int device, size_t offset, uint32_t seed, int tensor_id, int mode) {
  const HetAnnotation a = parse_annotation(anno);
  const Shape sh = to_shape(shape, ndim);
  if (ndim > 4) fail(Errc::UnsupportedOp, "fill supports up to 4-d tensors");
  const SliceRegion r = placement(a, sh, device);
  const int64_t bytes = r.cells() * dtype_width(to_dtype(dtype));
  if (offset + bytes > ctx->c->arena_bytes()) fail(Errc::ShapeMismatch, "shard exceeds arena");
  exec::FillDesc f{};
  f.dst = ctx->c->arena() + offset;
  f.ndim = ndim;
  for (int d = 0; d < ndim; ++d) {
    f.shape[d] = sh[d];
    f.lo[d] = r.bounds[d][0];
    f.ext[d] = r.bounds[d][1] - r.bounds[d][0];
  }
  f.seed = seed;
  f.tensor_id = tensor_id;
  f.hsize = a.hsize;
  const int g = a.subgroup_of(device);
  f.g = g;
  f.tg = a.effective_hdim() == kPartial ? g : -1;
  f.p = r.partial_index;
  f.P = r.partial_count;
  f.mode = mode;
  return f;
}

}  // namespace

extern "C" {

int hs_ctx_create(int rank, int world, int gpu, size_t arena_bytes, hs_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<hs_ctx>();
    c->c = std::make_unique<exec::Context>(rank, world, gpu, arena_bytes);
    *out = c.release();
  });
}

void hs_ctx_destroy(hs_ctx* ctx) { delete ctx; }

int hs_ctx_arena(hs_ctx* ctx, void** base, size_t* bytes) {
  return guarded([&] {
    *base = ctx->c->arena();
    *bytes = ctx->c->arena_bytes();
  });
}

int hs_ctx_ipc_handle(hs_ctx* ctx, unsigned char* out128) {
  return guarded([&] { ctx->c->ipc_handles(out128); });
}

int hs_ctx_open_peers(hs_ctx* ctx, const unsigned char* all) {
  return guarded([&] { ctx->c->open_peers(all); });
}

int hs_nccl_unique_id(unsigned char* out128) {
  return guarded([&] {
    ncclUniqueId uid;
    exec::nccl::check(exec::nccl::api().GetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(out128, &uid, sizeof(uid));
  });
}

int hs_ctx_nccl_init(hs_ctx* ctx, const unsigned char* id128) {
  return guarded([&] { ctx->c->nccl_init(id128); });
}

int hs_ctx_alloc(hs_ctx* ctx, size_t bytes, size_t* offset) {
  return guarded([&] { *offset = ctx->c->alloc(bytes); });
}

int hs_ctx_reset_alloc(hs_ctx* ctx, size_t offset) {
  return guarded([&] { ctx->c->reset_alloc(offset); });
}

int hs_prog_compile(hs_ctx* ctx, const hs_plan* plan, const int* v_to_rank, int n_virt,
                    const size_t* src_off, const size_t* dst_off, int flags, hs_prog** out) {
  return guarded([&] {
    exec::cuda_check(cudaSetDevice(ctx->c->gpu()), "cudaSetDevice");
    std::vector<int> map(v_to_rank, v_to_rank + n_virt);
    auto p = std::make_unique<hs_prog>();
    p->p = std::make_unique<exec::Program>(*ctx->c, plan->comm ? &*plan->comm : nullptr,
                                           plan->sw ? &*plan->sw : nullptr, map, src_off, dst_off,
                                           flags);
    *out = p.release();
  });
}

int hs_prog_compile_ptrs(hs_ctx* ctx, const hs_plan* plan, const int* v_to_rank, int n_virt,
                         void* const* src_ptrs, void* const* dst_ptrs, int flags, hs_prog** out) {
  return guarded([&] {
    exec::cuda_check(cudaSetDevice(ctx->c->gpu()), "cudaSetDevice");
    std::vector<int> map(v_to_rank, v_to_rank + n_virt);
    auto p = std::make_unique<hs_prog>();
    p->p = std::make_unique<exec::Program>(*ctx->c, plan->comm ? &*plan->comm : nullptr,
                                           plan->sw ? &*plan->sw : nullptr, map, nullptr, nullptr, flags,
                                           src_ptrs, dst_ptrs);
    *out = p.release();
  });
}

int hs_ipc_export(hs_ctx* ctx, const void* ptr, unsigned char* out80) {
  return guarded([&] { ctx->c->ipc_export(ptr, out80); });
}

int hs_ipc_import(hs_ctx* ctx, const unsigned char* in80, void** ptr) {
  return guarded([&] { *ptr = ctx->c->ipc_import(in80); });
}

void hs_prog_destroy(hs_prog* prog) { delete prog; }

int hs_prog_run(hs_prog* prog, void* stream) {
  return guarded([&] { prog->p->run(static_cast<cudaStream_t>(stream)); });
}

int hs_prog_run_host_async(hs_prog* prog, const void* const* src_host, void* const* dst_host, void* h2d,
                           void* compute, void* d2h) {
  return guarded([&] {
    prog->p->run_host_async(src_host, dst_host, static_cast<cudaStream_t>(h2d), static_cast<cudaStream_t>(compute),
                            static_cast<cudaStream_t>(d2h));
  });
}

int hs_prog_run_host(hs_prog* prog, const void* const* src_host, void* const* dst_host) {
  return guarded([&] { prog->p->run_host(src_host, dst_host); });
}

int hs_prog_profile(hs_prog* prog, int enable) {
  return guarded([&] { prog->p->set_profiling(enable != 0); });
}

int hs_prog_phase_ms(hs_prog* prog, double* out, int n, int* runs) {
  return guarded([&] { *runs = prog->p->phase_ms(out, n); });
}

int hs_prog_stats(const hs_prog* prog, char** json) {
  return guarded([&] { *json = dup_string(prog->p->stats_json()); });
}

int hs_analyze(const hs_plan* plan, int rank, int world, const int* v_to_rank, int n_virt, int flags,
               char** stats_json, char** tasks_json) {
  return guarded([&] {
    auto ctx = exec::Context::analysis(rank, world);
    // every shard gets a distinct 256-byte-aligned virtual offset on its rank
    const auto& comm = plan->comm;
    std::vector<std::pair<const HetAnnotation*, const HetAnnotation*>> annos;
    std::vector<Shape> shapes;
    if (comm) {
      annos.emplace_back(&comm->src, &comm->dst);
      shapes.push_back(comm->shape);
    } else {
      for (const SwitchEntry& e : plan->sw->diff) {
        annos.emplace_back(&e.src, &e.dst);
        shapes.push_back(e.shape);
      }
    }
    const size_t n = annos.size() * static_cast<size_t>(n_virt);
    std::vector<size_t> src_off(n, SIZE_MAX), dst_off(n, SIZE_MAX);
    size_t next = 0;
    const int es = dtype_width(comm ? comm->dtype : plan->sw->dtype);
    for (size_t t = 0; t < annos.size(); ++t)
      for (int side = 0; side < 2; ++side)
        for (const auto& [d, r] : placements(side ? *annos[t].second : *annos[t].first, shapes[t])) {
          if (d < 0 || d >= n_virt) fail(Errc::UnknownDevice, "device without rank mapping");
          (side ? dst_off : src_off)[t * n_virt + d] = next;
          next += ((static_cast<size_t>(r.cells()) * es + 255) / 256) * 256;
        }
    ctx->alloc(next);
    std::vector<int> map(v_to_rank, v_to_rank + n_virt);
    exec::Program prog(*ctx, comm ? &*comm : nullptr, plan->sw ? &*plan->sw : nullptr, map,
                       src_off.data(), dst_off.data(), flags);
    *stats_json = dup_string(prog.stats_json());
    *tasks_json = dup_string(prog.tasks_json());
  });
}

int hs_fill_shard(hs_ctx* ctx, const char* anno, const int64_t* shape, int ndim, int dtype,
                  int device, size_t offset, uint32_t seed, int tensor_id, int mode, void* stream) {
  return guarded([&] {
    const exec::FillDesc f =
        fill_desc(ctx, anno, shape, ndim, dtype, device, offset, seed, tensor_id, mode);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->c->stream();
    exec::cuda_check(exec::launch_fill(f, dtype, s), "fill launch");
  });
}

int hs_verify_shard(hs_ctx* ctx, const char* anno, const int64_t* shape, int ndim, int dtype,
                    int device, size_t offset, uint32_t seed, int tensor_id,
                    unsigned long long* mismatches, void* stream) {
  return guarded([&] {
    const exec::FillDesc f = fill_desc(ctx, anno, shape, ndim, dtype, device, offset, seed, tensor_id, 0);
    cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->c->stream();
    unsigned long long* d = ctx->c->scratch_counter();
    exec::cuda_check(cudaMemsetAsync(d, 0, sizeof(*d), s), "memset");
    exec::cuda_check(exec::launch_verify(f, dtype, d, s), "verify launch");
    exec::cuda_check(cudaMemcpyAsync(mismatches, d, sizeof(*d), cudaMemcpyDeviceToHost, s), "D2H");
    exec::cuda_check(cudaStreamSynchronize(s), "verify sync");
  });
}

int hs_ctx_read(hs_ctx* ctx, size_t offset, void* host, size_t bytes) {
  return guarded([&] {
    if (offset + bytes > ctx->c->arena_bytes()) fail(Errc::ShapeMismatch, "read beyond arena");
    exec::cuda_check(cudaStreamSynchronize(ctx->c->stream()), "sync");
    exec::cuda_check(cudaMemcpy(host, ctx->c->arena() + offset, bytes, cudaMemcpyDeviceToHost), "D2H");
  });
}

int hs_ctx_write(hs_ctx* ctx, size_t offset, const void* host, size_t bytes) {
  return guarded([&] {
    if (offset + bytes > ctx->c->arena_bytes()) fail(Errc::ShapeMismatch, "write beyond arena");
    exec::cuda_check(cudaStreamSynchronize(ctx->c->stream()), "sync");
    exec::cuda_check(cudaMemcpy(ctx->c->arena() + offset, host, bytes, cudaMemcpyHostToDevice), "H2D");
  });
}

int hs_ctx_sync(hs_ctx* ctx) {
  return guarded([&] {
    exec::cuda_check(cudaStreamSynchronize(ctx->c->stream()), "sync");
    exec::cuda_check(cudaDeviceSynchronize(), "device sync");
    ctx->c->check_barrier_error();
  });
}

int hs_ctx_barrier(hs_ctx* ctx, void* stream) {
  return guarded([&] { ctx->c->barrier(stream ? static_cast<cudaStream_t>(stream) : ctx->c->stream()); });
}

int hs_ctx_clear_error(hs_ctx* ctx) {
  return guarded([&] { ctx->c->clear_error(); });
}

}  // extern "C"
