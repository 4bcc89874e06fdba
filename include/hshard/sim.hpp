// hshard-b200: the executor half of the reference's hshard/sim.hpp.
//
// The reference DECLARES these (sim.hpp:26-91) but defines none of them; here
// execute_plan / apply_switch run on the B200 (libhshard_b200.so kernels),
// with host Tensors in and out -- the reference-facing, host-buffer entry
// points.  Device-resident execution (shards already in HBM, several GPUs)
// is the C ABI in hshard_c.h (hs_ctx_* / hs_prog_*).
//
// Not provided: run() and oracle_run(), which execute whole computation
// graphs (CompGraph / ExecGraph) -- outside the resharding path.
// DeviceState / SimState (sim.hpp:51-60) are declared as in the reference and
// drive the SPEC's state-to-state apply_switch.
#pragma once

#include <set>

#include "hshard/resolve.hpp"
#include "hshard/switch.hpp"
#include "hshard/tensor.hpp"

namespace hshard {

// Deterministic virtual cluster (sim.hpp:26-38); bandwidth influences BSR
// sender choice only, never results.
struct VirtualCluster {
  std::vector<DeviceId> devices;
  std::map<DeviceId, int> node_of;
  Bandwidth bandwidth;
  std::map<DType, int> widths;

  int width(DType t) const;
  bool has_device(DeviceId d) const { return node_of.count(d) > 0; }

  static VirtualCluster single_node(int n_devices, double bw = 1.0);
  static VirtualCluster two_tier(const std::vector<std::vector<DeviceId>>& nodes, double intra,
                                 double inter);
};

std::map<DeviceId, VolumeEntry> volume_report(const BsrPlan& plan, const VirtualCluster& cluster);

// Directed (sender, receiver) -> bytes of every payload a plan moves between
// distinct virtual devices (self-pairs and local copies are not traffic).
struct TrafficLog {
  std::map<std::pair<DeviceId, DeviceId>, int64_t> bytes;

  void add(DeviceId sender, DeviceId receiver, int64_t n);
  int64_t total() const;
  int64_t sent_by(DeviceId d) const;
};

// Per-device simulator state (reference sim.hpp:51-60): tensor id ->
// (region, payload); regions match placement() of the tensor's current
// annotation.
struct DeviceState {
  std::map<int, std::pair<SliceRegion, Tensor>> store;
};

struct SimState {
  std::map<DeviceId, DeviceState> devices;
  TrafficLog traffic;
};

// Inverse of placement: concatenate Splits, sum Partials, require Duplicate
// replicas (and hdim -1 subgroups) to agree within replica_tol.
// Errors: MissingShard, ShapeMismatch, ReplicaDivergence.
Tensor reassemble(const HetAnnotation& anno, const std::map<DeviceId, Tensor>& shards,
                  const Shape& shape, double replica_tol = 0.0);

// Forward decomposition: Split slices, Duplicate copies, the full value on
// partial ordinal 0 (and top-tier Partial subgroup 0), zeros elsewhere.
std::map<DeviceId, Tensor> scatter(const HetAnnotation& anno, const Tensor& logical);

// Executes a CommPlan on the GPU (all virtual devices resident in one HBM).
// Values are converted to the plan's dtype on upload (bf16: round to
// nearest even); reductions accumulate in fp32 (bf16/f32) / f64 / wrapping
// integers in ascending device-id order and round once per plan phase.
std::map<DeviceId, Tensor> execute_plan(const CommPlan& plan,
                                        const std::map<DeviceId, Tensor>& src_shards,
                                        TrafficLog* traffic = nullptr);

// (tensor id, device) -> shard.
using ShardKey = std::pair<int, DeviceId>;

// moves every changed parameter to its destination
// placement with one fused batched send/recv; returns the new shards (the
// caller releases the old ones).  Errors: MissingShard.
std::map<ShardKey, Tensor> apply_switch(const SwitchPlan& plan,
                                        const std::map<ShardKey, Tensor>& shards,
                                        TrafficLog* traffic = nullptr);

// SPEC.md:428-433 apply_switch(simulator state, plan) -> new state: the
// moved parameters' source placements (MissingShard if any is absent, e.g. a
// plan applied twice) are replaced by their destination placements; the
// plan's traffic is added to state.traffic.  Runs on the GPU as above.
SimState apply_switch(const SimState& state, const SwitchPlan& plan);

// Traffic a plan implies (what execute_plan / apply_switch log).
TrafficLog plan_traffic(const CommPlan& plan);
TrafficLog plan_traffic(const SwitchPlan& plan);

}  // namespace hshard
