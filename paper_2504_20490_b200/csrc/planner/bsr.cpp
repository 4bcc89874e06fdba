// PORT NOTICE: this file is a port of the reference planner's src/bsr.cpp
// (hshard, Copyright 2026 The hshard Authors, Apache License 2.0 -- see
// NOTICE): the same algorithm statement for statement, with renamed
// identifiers, so that plans are byte-identical to the reference's.
//
// hshard-b200 planner: BSR tables, heuristic sender selection, fusion.
//
// Follows the reference bsr.cpp: finest-slice grid over the scope
// (:56-91, :95-135), row scan with heuristics I/II/III and lowest-id
// tie-break against a plan-global cumulative load (:172-203), per
// (sender, receiver) fusion groups (:163-170), fuse ordering by
// (tensor id, region bounds) (:205-242) and the volume report (:244-261).
#include <algorithm>
#include <set>
#include <unordered_map>

#include "hshard/bsr.hpp"
#include "planner_internal.hpp"

namespace hshard {

// ---------------------------------------------------------------- bandwidth
double Bandwidth::get(DeviceId a, DeviceId b) const {
  const auto it = links.find(std::minmax(a, b));
  return it != links.end() ? it->second : default_bw;
}

void Bandwidth::set(DeviceId a, DeviceId b, double bw) { links[std::minmax(a, b)] = bw; }

Bandwidth Bandwidth::uniform(double bw) {
  Bandwidth out;
  out.default_bw = bw;
  return out;
}

Bandwidth Bandwidth::two_tier(const std::map<DeviceId, int>& node_of, double intra,
                              double inter) {
  Bandwidth out = uniform(inter);
  for (auto a = node_of.begin(); a != node_of.end(); ++a)
    for (auto b = std::next(a); b != node_of.end(); ++b)
      if (a->second == b->second) out.set(a->first, b->first, intra);
  return out;
}

// ---------------------------------------------------------------- grid
namespace detail {

void for_each_grid_cell(const Cuts& cuts, const std::function<void(const SliceRegion&)>& fn) {
  const size_t rank = cuts.size();
  for (const auto& c : cuts)
    if (c.size() < 2) return;  // empty extent: no cells
  std::vector<size_t> at(rank, 0);
  SliceRegion cell;
  cell.bounds.resize(rank);
  while (true) {
    for (size_t d = 0; d < rank; ++d) cell.bounds[d] = {cuts[d][at[d]], cuts[d][at[d] + 1]};
    fn(cell);
    size_t d = rank;
    for (;;) {
      if (d == 0) return;
      --d;
      if (++at[d] + 1 < cuts[d].size()) break;
      at[d] = 0;
    }
  }
}

}  // namespace detail

namespace {

detail::Cuts scoped_cuts(const SliceRegion& scope, const std::vector<const SliceRegion*>& boxes) {
  detail::Cuts cuts(scope.bounds.size());
  for (size_t d = 0; d < cuts.size(); ++d) {
    const int64_t lo = scope.bounds[d][0], hi = scope.bounds[d][1];
    std::set<int64_t> s{lo, hi};
    for (const SliceRegion* r : boxes)
      for (int64_t v : r->bounds[d])
        if (lo < v && v < hi) s.insert(v);
    cuts[d].assign(s.begin(), s.end());
  }
  return cuts;
}

void reject_partial(const HetAnnotation& a, const char* side) {
  if (a.has_partial())
    fail(Errc::PartialUnderBsr,
         std::string("batched send-receive cannot move Partial values (") + side + " " + a.str() +
             ")");
}

}  // namespace

BsrTable build_table_scoped(const HetAnnotation& src, const HetAnnotation& dst,
                            const Shape& shape, int tensor_id, int elem_bytes,
                            const SliceRegion& scope, const std::vector<DeviceId>& devices) {
  const auto src_all = placements(src, shape);
  const auto dst_all = placements(dst, shape);

  std::map<DeviceId, SliceRegion> have, want;
  std::vector<const SliceRegion*> boxes;
  for (DeviceId d : devices) {
    if (auto it = src_all.find(d); it != src_all.end()) have.emplace(d, it->second);
    if (auto it = dst_all.find(d); it != dst_all.end()) want.emplace(d, it->second);
  }
  for (DeviceId d : devices) {
    if (auto it = have.find(d); it != have.end()) boxes.push_back(&it->second);
    if (auto it = want.find(d); it != want.end()) boxes.push_back(&it->second);
  }
  for (const SliceRegion* r : boxes)
    if (r->partial_count > 1)
      fail(Errc::PartialUnderBsr, "batched send-receive cannot move Partial values");

  BsrTable table;
  detail::for_each_grid_cell(scoped_cuts(scope, boxes), [&](const SliceRegion& cell) {
    BsrRow row;
    row.tensor_id = tensor_id;
    row.region = cell;
    row.bytes = cell.cells() * elem_bytes;
    for (const auto& [d, r] : have)
      if (r.covers(cell)) row.owners.push_back(d);
    for (const auto& [d, r] : want)
      if (r.covers(cell)) row.requesters.push_back(d);
    table.rows.push_back(std::move(row));
  });
  return table;
}

BsrTable build_table(const HetAnnotation& src, const HetAnnotation& dst, const Shape& shape,
                     int tensor_id, int elem_bytes) {
  reject_partial(src, "src");
  reject_partial(dst, "dst");
  std::set<DeviceId> devs;
  for (const HetAnnotation* a : {&src, &dst})
    for (DeviceId d : a->all_devices()) devs.insert(d);
  return build_table_scoped(src, dst, shape, tensor_id, elem_bytes, SliceRegion::whole(shape),
                            std::vector<DeviceId>(devs.begin(), devs.end()));
}

// ---------------------------------------------------------------- plans
int64_t BsrPlan::total_bytes() const {
  int64_t n = 0;
  for (const Transfer& t : transfers) n += t.bytes;
  return n;
}

std::map<DeviceId, int64_t> BsrPlan::send_load() const {
  std::map<DeviceId, int64_t> m;
  for (const Transfer& t : transfers) m[t.sender] += t.bytes;
  return m;
}

namespace {

// One pass over rows in the given order.  `bw == nullptr` selects the naive
// lowest-id-owner policy.
BsrPlan plan_rows(const std::vector<const BsrRow*>& rows, const Bandwidth* bw) {
  BsrPlan plan;
  std::unordered_map<DeviceId, int64_t> sent;
  auto sent_by = [&sent](DeviceId d) {
    auto it = sent.find(d);
    return it == sent.end() ? int64_t{0} : it->second;
  };
  for (const BsrRow* row : rows) {
    if (row->owners.empty()) {
      if (!row->requesters.empty())
        fail(Errc::NoOwner, "slice " + row->region.str() + " of tensor " +
                                std::to_string(row->tensor_id) + " has no owner");
      continue;
    }
    std::vector<DeviceId> owners = row->owners, wanting = row->requesters;
    std::sort(owners.begin(), owners.end());
    std::sort(wanting.begin(), wanting.end());
    for (DeviceId r : wanting) {
      if (std::binary_search(owners.begin(), owners.end(), r)) {  // heuristic I
        plan.local_copies.push_back({r, row->tensor_id, row->region});
        continue;
      }
      DeviceId pick = owners.front();
      if (bw) {
        double pick_bw = bw->get(pick, r);
        for (DeviceId o : owners) {
          const double o_bw = bw->get(o, r);
          const bool better = o_bw > pick_bw || (o_bw == pick_bw && sent_by(o) < sent_by(pick));
          if (better) {  // heuristic II, then III; ascending scan keeps lowest id
            pick = o;
            pick_bw = o_bw;
          }
        }
      }
      plan.transfers.push_back({row->tensor_id, row->region, pick, r, row->bytes});
      sent[pick] += row->bytes;
    }
  }
  std::map<std::pair<DeviceId, DeviceId>, std::vector<int>> by_pair;
  for (size_t i = 0; i < plan.transfers.size(); ++i)
    by_pair[{plan.transfers[i].sender, plan.transfers[i].receiver}].push_back(static_cast<int>(i));
  for (auto& [pair, idx] : by_pair) plan.fusion_groups.push_back({pair.first, pair.second, idx});
  return plan;
}

std::vector<const BsrRow*> row_ptrs(const BsrTable& t) {
  std::vector<const BsrRow*> v;
  v.reserve(t.rows.size());
  for (const BsrRow& r : t.rows) v.push_back(&r);
  return v;
}

}  // namespace

BsrPlan make_plan(const BsrTable& table, const Bandwidth& bandwidth) {
  return plan_rows(row_ptrs(table), &bandwidth);
}

BsrPlan make_plan_naive(const BsrTable& table) { return plan_rows(row_ptrs(table), nullptr); }

BsrPlan fuse(const std::vector<BsrTable>& tables, const Bandwidth& bandwidth) {
  std::set<int> all_ids;
  size_t listed = 0;
  std::vector<const BsrRow*> rows;
  for (const BsrTable& t : tables) {
    std::set<int> ids;
    for (const BsrRow& r : t.rows) {
      ids.insert(r.tensor_id);
      rows.push_back(&r);
    }
    listed += ids.size();
    all_ids.insert(ids.begin(), ids.end());
  }
  if (listed != all_ids.size()) fail(Errc::ParseError, "fused tables must cover disjoint tensor ids");
  std::stable_sort(rows.begin(), rows.end(), [](const BsrRow* a, const BsrRow* b) {
    return a->tensor_id != b->tensor_id ? a->tensor_id < b->tensor_id
                                        : a->region.bounds < b->region.bounds;
  });
  return plan_rows(rows, &bandwidth);
}

std::map<DeviceId, VolumeEntry> volume_report(const BsrPlan& plan,
                                              const std::map<DeviceId, int>& node_of) {
  std::map<DeviceId, VolumeEntry> out;
  for (const auto& kv : node_of) out[kv.first] = VolumeEntry{};
  auto node = [&node_of](DeviceId d, const char* role) {
    auto it = node_of.find(d);
    if (it == node_of.end())
      fail(Errc::UnknownDevice, std::string(role) + " " + std::to_string(d) + " not in cluster");
    return it->second;
  };
  for (const Transfer& t : plan.transfers) {
    const int ns = node(t.sender, "sender");
    const int nr = node(t.receiver, "receiver");
    (ns == nr ? out[t.sender].intra_bytes : out[t.sender].inter_bytes) += t.bytes;
  }
  return out;
}

}  // namespace hshard
