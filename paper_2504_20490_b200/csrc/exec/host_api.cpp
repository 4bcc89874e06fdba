// hshard-b200: execute_plan / apply_switch with host Tensors (sim.hpp).
//
// The reference declares execute_plan (sim.hpp:77-79) but never defines it;
// this definition runs the plan on the B200: every virtual device's shard is
// placed in one GPU's arena, converted to the plan dtype, executed by the
// compiled program (the same kernels as the device-resident C ABI path) and
// read back.  Device: $HSHARD_GPU (default 0).
#include <cstdlib>
#include <cstring>

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

struct Side {
  // (slot, device) -> (placement, arena offset)
  std::map<std::pair<int, DeviceId>, std::pair<SliceRegion, size_t>> at;
};

// Shared driver: annotations per tensor slot, host shards keyed by
// (slot, device) in, host shards keyed by (slot, device) out.
std::map<std::pair<int, DeviceId>, Tensor> run_on_gpu(
    const CommPlan* comm, const SwitchPlan* sw, DType dt,
    const std::vector<std::tuple<const HetAnnotation*, const HetAnnotation*, Shape>>& slots,
    const std::map<std::pair<int, DeviceId>, const Tensor*>& src) {
  const int es = dtype_width(dt);
  int n_virt = 0;
  size_t bytes = 1 << 20;
  Side in, out;
  std::vector<std::map<DeviceId, SliceRegion>> src_pl, dst_pl;
  for (const auto& [s, d, shape] : slots) {
    src_pl.push_back(placements(*s, shape));
    dst_pl.push_back(placements(*d, shape));
    for (const auto& m : {&src_pl.back(), &dst_pl.back()})
      for (const auto& [dev, r] : *m) {
        n_virt = std::max(n_virt, dev + 1);
        bytes += static_cast<size_t>(r.cells()) * es + 256;
      }
  }
  if (comm && comm->mid)
    for (const auto& [dev, r] : placements(*comm->mid, comm->shape)) bytes += r.cells() * es + 256;

  exec::Context ctx(0, 1, host_gpu(), bytes);
  const size_t n = slots.size() * static_cast<size_t>(n_virt);
  std::vector<size_t> src_off(n, SIZE_MAX), dst_off(n, SIZE_MAX);
  for (size_t t = 0; t < slots.size(); ++t) {
    for (const auto& [dev, r] : src_pl[t]) {
      auto it = src.find({static_cast<int>(t), dev});
      if (it == src.end())
        fail(Errc::MissingShard, "no source shard for device " + std::to_string(dev));
      if (it->second->shape != r.extents())
        fail(sw ? Errc::MissingShard : Errc::ShapeMismatch, "device " + std::to_string(dev) + " shard [" +
                                      join_ints(it->second->shape) + "] vs placement " + r.str());
      const size_t off = ctx.alloc(static_cast<size_t>(r.cells()) * es);
      src_off[t * n_virt + dev] = off;
      const auto raw = encode(*it->second, dt);
      exec::cuda_check(cudaMemcpy(ctx.arena() + off, raw.data(), raw.size(), cudaMemcpyHostToDevice),
                       "upload shard");
    }
    for (const auto& [dev, r] : dst_pl[t]) {
      const size_t off = ctx.alloc(static_cast<size_t>(r.cells()) * es);
      dst_off[t * n_virt + dev] = off;
      out.at[{static_cast<int>(t), dev}] = {r, off};
    }
  }
  std::vector<int> v_to_rank(n_virt, 0);
  exec::Program prog(ctx, comm, sw, v_to_rank, src_off.data(), dst_off.data(), 0);
  prog.run(ctx.stream());
  exec::cuda_check(cudaStreamSynchronize(ctx.stream()), "execute_plan");
  std::map<std::pair<int, DeviceId>, Tensor> result;
  std::vector<unsigned char> buf;
  for (const auto& [key, ro] : out.at) {
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

}  // namespace hshard
