// hshard-b200: execute_plan / apply_switch with host Tensors (sim.hpp).
//
// The reference declares execute_plan (sim.hpp:77-79) but never defines it;
// this definition runs the plan on the B200: every virtual device's shard is
// placed in one GPU's arena, converted to the plan dtype, executed by the
// compiled program (the same kernels as the device-resident C ABI path) and
// read back.  Device: $HSHARD_GPU (default 0).  The context, placements and
// compiled program of a plan are cached (up to 8 plans, least recently used
// evicted): repeated calls with the same plan only upload, run and download.
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>

#include "hshard/sim.hpp"
#include "program.hpp"

namespace hshard {

namespace {

int host_gpu() {
  const char* e = std::getenv("HSHARD_GPU");
  return e ? std::atoi(e) : 0;
}

uint16_t to_bf16(double v) {
  const float f = static_cast<float>(v);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFFu + ((u >> 16) & 1u)) >> 16);
}

double from_bf16(uint16_t b) {
  const uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

std::vector<unsigned char> encode(const Tensor& t, DType dt) {
  const size_t n = t.data.size();
  std::vector<unsigned char> out(n * dtype_width(dt));
  for (size_t i = 0; i < n; ++i) {
    const double v = t.data[i];
    switch (dt) {
      case DType::F32: {
        const float x = static_cast<float>(v);
        std::memcpy(&out[i * 4], &x, 4);
        break;
      }
      case DType::F64: std::memcpy(&out[i * 8], &v, 8); break;
      case DType::I32: {
        const int32_t x = static_cast<int32_t>(v);
        std::memcpy(&out[i * 4], &x, 4);
        break;
      }
      case DType::I64: {
        const int64_t x = static_cast<int64_t>(v);
        std::memcpy(&out[i * 8], &x, 8);
        break;
      }
      case DType::BF16: {
        const uint16_t x = to_bf16(v);
        std::memcpy(&out[i * 2], &x, 2);
        break;
      }
    }
  }
  return out;
}

Tensor decode(const unsigned char* p, const Shape& shape, DType dt) {
  Tensor t(shape, dt);
  for (size_t i = 0; i < t.data.size(); ++i) {
    switch (dt) {
      case DType::F32: {
        float x;
        std::memcpy(&x, p + i * 4, 4);
        t.data[i] = x;
        break;
      }
      case DType::F64: std::memcpy(&t.data[i], p + i * 8, 8); break;
      case DType::I32: {
        int32_t x;
        std::memcpy(&x, p + i * 4, 4);
        t.data[i] = x;
        break;
      }
      case DType::I64: {
        int64_t x;
        std::memcpy(&x, p + i * 8, 8);
        t.data[i] = static_cast<double>(x);
        break;
      }
      case DType::BF16: {
        uint16_t x;
        std::memcpy(&x, p + i * 2, 2);
        t.data[i] = from_bf16(x);
        break;
      }
    }
  }
  return t;
}

// One compiled plan with its own context (arena sized for the plan's shards):
// placements, offsets and the program are built on the first call and reused
// by every later call with the same plan (plans and programs are
// cached, not rebuilt per call).
struct CachedRun {
  std::unique_ptr<exec::Context> ctx;
  std::unique_ptr<exec::Program> prog;
  std::vector<std::map<DeviceId, SliceRegion>> src_pl;
  std::map<std::pair<int, DeviceId>, size_t> src_off;                          // (slot, dev) -> offset
  std::map<std::pair<int, DeviceId>, std::pair<SliceRegion, size_t>> out;      // (slot, dev) -> dst
  uint64_t last_use = 0;
};

constexpr size_t kMaxCachedRuns = 8;
std::mutex g_cache_mu;
std::map<std::string, CachedRun> g_cache;
uint64_t g_clock = 0;

std::string cache_key(const CommPlan* comm, const SwitchPlan* sw, int gpu) {
  std::string k = "gpu=" + std::to_string(gpu) + "|";
  if (comm) return k + "comm|" + dump_plan(*comm);
  k += "switch|" + std::string(dtype_name(sw->dtype)) + "|";
  for (const SwitchEntry& e : sw->diff)
    k += std::to_string(e.tensor_id) + ":" + e.src.str() + ">" + e.dst.str() + "@" + join_ints(e.shape) + ";";
  return k + dump_bsr(sw->plan);
}

CachedRun& compiled(const CommPlan* comm, const SwitchPlan* sw, DType dt,
                    const std::vector<std::tuple<const HetAnnotation*, const HetAnnotation*, Shape>>& slots) {
  const int gpu = host_gpu();
  const std::string key = cache_key(comm, sw, gpu);
  auto it = g_cache.find(key);
  if (it != g_cache.end()) {
    it->second.last_use = ++g_clock;
    return it->second;
  }
  if (g_cache.size() >= kMaxCachedRuns) {  // evict the least recently used plan
    auto lru = g_cache.begin();
    for (auto i = g_cache.begin(); i != g_cache.end(); ++i)
      if (i->second.last_use < lru->second.last_use) lru = i;
    g_cache.erase(lru);
  }
  const int es = dtype_width(dt);
  int n_virt = 0;
  size_t bytes = 1 << 20;
  CachedRun run;
  std::vector<std::map<DeviceId, SliceRegion>> dst_pl;
  for (const auto& [s, d, shape] : slots) {
    run.src_pl.push_back(placements(*s, shape));
    dst_pl.push_back(placements(*d, shape));
    for (const auto& m : {&run.src_pl.back(), &dst_pl.back()})
      for (const auto& [dev, r] : *m) {
        n_virt = std::max(n_virt, dev + 1);
        bytes += static_cast<size_t>(r.cells()) * es + 256;
      }
  }
  if (comm && comm->mid)
    for (const auto& [dev, r] : placements(*comm->mid, comm->shape)) bytes += r.cells() * es + 256;
  run.ctx = std::make_unique<exec::Context>(0, 1, gpu, bytes);
  const size_t n = slots.size() * static_cast<size_t>(n_virt);
  std::vector<size_t> src_off(n, SIZE_MAX), dst_off(n, SIZE_MAX);
  for (size_t t = 0; t < slots.size(); ++t) {
    for (const auto& [dev, r] : run.src_pl[t]) {
      const size_t off = run.ctx->alloc(static_cast<size_t>(r.cells()) * es);
      src_off[t * n_virt + dev] = off;
      run.src_off[{static_cast<int>(t), dev}] = off;
    }
    for (const auto& [dev, r] : dst_pl[t]) {
      const size_t off = run.ctx->alloc(static_cast<size_t>(r.cells()) * es);
      dst_off[t * n_virt + dev] = off;
      run.out[{static_cast<int>(t), dev}] = {r, off};
    }
  }
  std::vector<int> v_to_rank(n_virt, 0);
  run.prog = std::make_unique<exec::Program>(*run.ctx, comm, sw, v_to_rank, src_off.data(), dst_off.data(), 0);
  run.last_use = ++g_clock;
  return g_cache.emplace(key, std::move(run)).first->second;
}

// Shared driver: annotations per tensor slot, host shards keyed by
// (slot, device) in, host shards keyed by (slot, device) out.
std::map<std::pair<int, DeviceId>, Tensor> run_on_gpu(
    const CommPlan* comm, const SwitchPlan* sw, DType dt,
    const std::vector<std::tuple<const HetAnnotation*, const HetAnnotation*, Shape>>& slots,
    const std::map<std::pair<int, DeviceId>, const Tensor*>& src) {
  const int es = dtype_width(dt);
  // validate the inputs before anything is compiled or uploaded
  for (size_t t = 0; t < slots.size(); ++t) {
    const auto& [s, d, shape] = slots[t];
    for (const auto& [dev, r] : placements(*s, shape)) {
      auto it = src.find({static_cast<int>(t), dev});
      if (it == src.end())
        fail(Errc::MissingShard, "no source shard for device " + std::to_string(dev));
      if (it->second->shape != r.extents())
        fail(sw ? Errc::MissingShard : Errc::ShapeMismatch, "device " + std::to_string(dev) + " shard [" +
                                      join_ints(it->second->shape) + "] vs placement " + r.str());
    }
  }
  std::lock_guard<std::mutex> lock(g_cache_mu);
  CachedRun& run = compiled(comm, sw, dt, slots);
  exec::Context& ctx = *run.ctx;
  for (const auto& [key, off] : run.src_off) {
    const auto raw = encode(*src.at(key), dt);
    exec::cuda_check(cudaMemcpy(ctx.arena() + off, raw.data(), raw.size(), cudaMemcpyHostToDevice),
                     "upload shard");
  }
  run.prog->run(ctx.stream());
  exec::cuda_check(cudaStreamSynchronize(ctx.stream()), "execute_plan");
  std::map<std::pair<int, DeviceId>, Tensor> result;
  std::vector<unsigned char> buf;
  for (const auto& [key, ro] : run.out) {
    buf.resize(static_cast<size_t>(ro.first.cells()) * es);
    exec::cuda_check(cudaMemcpy(buf.data(), ctx.arena() + ro.second, buf.size(), cudaMemcpyDeviceToHost),
                     "download shard");
    result.emplace(key, decode(buf.data(), ro.first.extents(), dt));
  }
  return result;
}

}  // namespace

std::map<DeviceId, Tensor> execute_plan(const CommPlan& plan,
                                        const std::map<DeviceId, Tensor>& src_shards,
                                        TrafficLog* traffic) {
  std::map<std::pair<int, DeviceId>, const Tensor*> src;
  for (const auto& [d, t] : src_shards) src[{0, d}] = &t;
  auto out = run_on_gpu(&plan, nullptr, plan.dtype, {{&plan.src, &plan.dst, plan.shape}}, src);
  std::map<DeviceId, Tensor> result;
  for (auto& [key, t] : out) result.emplace(key.second, std::move(t));
  if (traffic)
    for (const auto& [pair, b] : plan_traffic(plan).bytes) traffic->add(pair.first, pair.second, b);
  return result;
}

std::map<ShardKey, Tensor> apply_switch(const SwitchPlan& plan, const std::map<ShardKey, Tensor>& shards,
                                        TrafficLog* traffic) {
  std::vector<std::tuple<const HetAnnotation*, const HetAnnotation*, Shape>> slots;
  std::map<std::pair<int, DeviceId>, const Tensor*> src;
  for (size_t t = 0; t < plan.diff.size(); ++t) {
    const SwitchEntry& e = plan.diff[t];
    slots.emplace_back(&e.src, &e.dst, e.shape);
    for (const auto& [key, tensor] : shards)
      if (key.first == e.tensor_id) src[{static_cast<int>(t), key.second}] = &tensor;
  }
  auto out = run_on_gpu(nullptr, &plan, plan.dtype, slots, src);
  std::map<ShardKey, Tensor> result;
  for (auto& [key, t] : out) result.emplace(ShardKey{plan.diff[key.first].tensor_id, key.second}, std::move(t));
  // parameters the switch does not touch keep their shards
  std::set<int> moved;
  for (const SwitchEntry& e : plan.diff) moved.insert(e.tensor_id);
  for (const auto& [key, t] : shards)
    if (!moved.count(key.first)) result.emplace(key, t);
  if (traffic)
    for (const auto& [pair, b] : plan_traffic(plan).bytes) traffic->add(pair.first, pair.second, b);
  return result;
}

SimState apply_switch(const SimState& state, const SwitchPlan& plan) {
  // state holds every source placement of the moved
  // parameters (else MissingShard -- so applying a plan twice fails); the
  // result holds exactly the destination placements, old shards released.
  std::map<ShardKey, Tensor> shards;
  for (const SwitchEntry& e : plan.diff)
    for (const auto& [dev, r] : placements(e.src, e.shape)) {
      auto d = state.devices.find(dev);
      const auto* slot = d == state.devices.end() ? nullptr : [&]() -> const std::pair<SliceRegion, Tensor>* {
        auto it = d->second.store.find(e.tensor_id);
        return it == d->second.store.end() ? nullptr : &it->second;
      }();
      if (!slot || !slot->first.same_bounds(r) || slot->first.partial_index != r.partial_index ||
          slot->first.replica_index != r.replica_index)
        fail(Errc::MissingShard, "tensor " + std::to_string(e.tensor_id) + " has no source shard " + r.str() +
                                     " on device " + std::to_string(dev));
      shards.emplace(ShardKey{e.tensor_id, dev}, slot->second);
    }
  TrafficLog log;
  auto moved = apply_switch(plan, shards, &log);
  SimState out = state;
  for (const SwitchEntry& e : plan.diff)
    for (auto& [dev, ds] : out.devices) ds.store.erase(e.tensor_id);
  for (const SwitchEntry& e : plan.diff)
    for (const auto& [dev, r] : placements(e.dst, e.shape))
      out.devices[dev].store[e.tensor_id] = {r, std::move(moved.at({e.tensor_id, dev}))};
  for (const auto& [pair, b] : log.bytes) out.traffic.add(pair.first, pair.second, b);
  return out;
}

}  // namespace hshard
