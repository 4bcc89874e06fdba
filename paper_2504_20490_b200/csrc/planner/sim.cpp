// hshard-b200: host halves of sim.hpp -- cluster model, traffic accounting,
// scatter / reassemble (SPEC.md:476-489 semantics).  execute_plan and
// apply_switch live in exec/host_api.cpp (they run on the GPU).
#include <algorithm>
#include <cmath>

#include "hshard/sim.hpp"

namespace hshard {

int VirtualCluster::width(DType t) const {
  auto it = widths.find(t);
  return it == widths.end() ? dtype_width(t) : it->second;
}

VirtualCluster VirtualCluster::single_node(int n_devices, double bw) {
  VirtualCluster c;
  for (int d = 0; d < n_devices; ++d) {
    c.devices.push_back(d);
    c.node_of[d] = 0;
  }
  c.bandwidth = Bandwidth::uniform(bw);
  return c;
}

VirtualCluster VirtualCluster::two_tier(const std::vector<std::vector<DeviceId>>& nodes,
                                        double intra, double inter) {
  VirtualCluster c;
  for (size_t n = 0; n < nodes.size(); ++n)
    for (DeviceId d : nodes[n]) {
      c.devices.push_back(d);
      c.node_of[d] = static_cast<int>(n);
    }
  c.bandwidth = Bandwidth::two_tier(c.node_of, intra, inter);
  return c;
}

std::map<DeviceId, VolumeEntry> volume_report(const BsrPlan& plan, const VirtualCluster& cluster) {
  return volume_report(plan, cluster.node_of);
}

void TrafficLog::add(DeviceId sender, DeviceId receiver, int64_t n) {
  if (sender != receiver && n > 0) bytes[{sender, receiver}] += n;
}

int64_t TrafficLog::total() const {
  int64_t t = 0;
  for (const auto& kv : bytes) t += kv.second;
  return t;
}

int64_t TrafficLog::sent_by(DeviceId d) const {
  int64_t t = 0;
  for (const auto& [pair, n] : bytes)
    if (pair.first == d) t += n;
  return t;
}

// ---------------------------------------------------------------- scatter / reassemble
std::map<DeviceId, Tensor> scatter(const HetAnnotation& anno, const Tensor& logical) {
  std::map<DeviceId, Tensor> out;
  const bool top_partial = anno.effective_hdim() == kPartial;
  for (const auto& [d, r] : placements(anno, logical.shape)) {
    const bool carries = r.partial_index == 0 && (!top_partial || anno.subgroup_of(d) == 0);
    SliceRegion box;
    box.bounds = r.bounds;
    out.emplace(d, carries ? logical.slice(box) : Tensor(r.extents(), logical.dtype));
  }
  return out;
}

Tensor reassemble(const HetAnnotation& anno, const std::map<DeviceId, Tensor>& shards,
                  const Shape& shape, double replica_tol) {
  // Y[(g, q)]: what subgroup g's replica q reconstructs on its top-tier box.
  std::map<std::pair<int, int>, Tensor> copies;
  DType dt = DType::F64;
  for (const auto& [d, r] : placements(anno, shape)) {
    auto it = shards.find(d);
    if (it == shards.end()) fail(Errc::MissingShard, "no shard for device " + std::to_string(d));
    if (it->second.shape != r.extents())
      fail(Errc::ShapeMismatch, "device " + std::to_string(d) + " shard shape [" +
                                    join_ints(it->second.shape) + "] vs placement " + r.str());
    dt = it->second.dtype;
    const std::pair<int, int> key{anno.subgroup_of(d), r.replica_index};
    auto [slot, fresh] = copies.try_emplace(key, Tensor(shape, dt));
    SliceRegion box;
    box.bounds = r.bounds;
    if (r.cells() > 0) slot->second.add_slice(box, it->second);
  }
  auto diverge = [replica_tol](const Tensor& a, const Tensor& b) {
    return replica_tol == 0.0 ? !a.bit_equal(b) : a.max_rel_diff(b) > replica_tol;
  };
  for (const auto& [key, t] : copies)
    if (key.second != 0 && diverge(t, copies.at({key.first, 0})))
      fail(Errc::ReplicaDivergence, "replica " + std::to_string(key.second) + " of subgroup " +
                                        std::to_string(key.first) + " differs");
  if (anno.effective_hdim() == kDuplicate) {
    for (const auto& [key, t] : copies)
      if (key.second == 0 && key.first != 0 && diverge(t, copies.at({0, 0})))
        fail(Errc::ReplicaDivergence, "subgroup " + std::to_string(key.first) + " differs");
    Tensor out = copies.at({0, 0});
    out.dtype = dt;
    return out;
  }
  Tensor out(shape, dt);
  for (const auto& [key, t] : copies)
    if (key.second == 0) out += t;
  return out;
}

// ---------------------------------------------------------------- traffic
namespace {

int64_t box_bytes(const SliceRegion& r, DType dt) { return r.cells() * dtype_width(dt); }

void step_traffic(const CommStep& step, const HetAnnotation& from, const HetAnnotation& to,
                  const Shape& shape, DType dt, TrafficLog& log) {
  switch (step.kind) {
    case StepKind::Identity:
      break;
    case StepKind::SendRecv:
      for (const auto& [s, r] : step.pairs) log.add(s, r, box_bytes(placement(from, shape, s), dt));
      break;
    case StepKind::AllReduce:
    case StepKind::ReduceScatter:
      for (const auto& grp : step.groups)
        for (DeviceId d : grp)
          for (DeviceId m : grp) log.add(m, d, box_bytes(placement(to, shape, d), dt));
      break;
    case StepKind::AllGather:
      for (const auto& grp : step.groups)
        for (DeviceId d : grp)
          for (DeviceId m : grp)
            if (auto x = intersect(placement(from, shape, m), placement(to, shape, d)))
              log.add(m, d, box_bytes(*x, dt));
      break;
    case StepKind::SplitAllReduce:
    case StepKind::SplitReduceScatter:
    case StepKind::SplitAllGather:
      for (const SliceCollective& sc : step.slices)
        for (DeviceId r : sc.receivers) {
          const SliceRegion rr = placement(to, shape, r);
          for (DeviceId c : sc.contributors)
            if (placement(from, shape, c).partial_index % rr.partial_count == rr.partial_index)
              log.add(c, r, box_bytes(sc.region, dt));
        }
      break;
    case StepKind::Bsr:
      for (const Transfer& t : step.bsr->transfers) log.add(t.sender, t.receiver, t.bytes);
      break;
  }
}

}  // namespace

TrafficLog plan_traffic(const CommPlan& plan) {
  TrafficLog log;
  const HetAnnotation& bottom_to = plan.bottom_target();
  for (const CommStep& s : plan.bottom_phase)
    step_traffic(s, plan.src, bottom_to, plan.shape, plan.dtype, log);
  const HetAnnotation& top_from = plan.mid ? *plan.mid : plan.src;
  for (const CommStep& s : plan.top_phase) step_traffic(s, top_from, plan.dst, plan.shape, plan.dtype, log);
  return log;
}

TrafficLog plan_traffic(const SwitchPlan& plan) {
  TrafficLog log;
  for (const Transfer& t : plan.plan.transfers) log.add(t.sender, t.receiver, t.bytes);
  return log;
}

}  // namespace hshard
