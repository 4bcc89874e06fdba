// hshard-b200 planner: batched send-receive (BSR) tables, sender choice, fusion.
//
// Behaviour is the reference planner's (bsr.cpp:22-261; planner notice in
// NOTICE) and is pinned byte for byte by tests/golden/plans.jsonl: the finest
// grid of every involved box within the scope, one row per cell in row-major
// order; per row and ascending receiver, heuristic I (the receiver owns the
// cell: local copy), else II (highest link bandwidth), III (least bytes sent so
// far, counted across the whole plan) and the lowest id; fusion groups per
// (sender, receiver); `fuse` orders rows by (tensor id, region bounds).
//
// Organisation: rows come from one detail::CoverGrid walk (owners and
// requesters read off each cell's cover set instead of testing every box);
// the heuristics live in a SenderChooser holding the running send ledger.
#include <algorithm>
#include <numeric>
#include <set>
#include <unordered_map>

#include "hshard/bsr.hpp"
#include "planner_internal.hpp"

namespace hshard {

// ---------------------------------------------------------------- bandwidth
namespace {
std::pair<DeviceId, DeviceId> link_key(DeviceId a, DeviceId b) { return a < b ? std::pair{a, b} : std::pair{b, a}; }
}  // namespace

double Bandwidth::get(DeviceId a, DeviceId b) const {
  const auto it = links.find(link_key(a, b));
  return it == links.end() ? default_bw : it->second;
}

void Bandwidth::set(DeviceId a, DeviceId b, double bw) { links[link_key(a, b)] = bw; }

Bandwidth Bandwidth::uniform(double bw) {
  Bandwidth out;
  out.default_bw = bw;
  return out;
}

Bandwidth Bandwidth::two_tier(const std::map<DeviceId, int>& node_of, double intra, double inter) {
  Bandwidth out = uniform(inter);
  std::map<int, std::vector<DeviceId>> members;  // node -> devices
  for (const auto& [d, n] : node_of) members[n].push_back(d);
  for (const auto& [n, devs] : members)
    for (size_t i = 0; i < devs.size(); ++i)
      for (size_t j = i + 1; j < devs.size(); ++j) out.set(devs[i], devs[j], intra);
  return out;
}

// ---------------------------------------------------------------- tables
BsrTable build_table_scoped(const HetAnnotation& src, const HetAnnotation& dst, const Shape& shape,
                            int tensor_id, int elem_bytes, const SliceRegion& scope,
                            const std::vector<DeviceId>& devices) {
  const auto src_at = placements(src, shape);
  const auto dst_at = placements(dst, shape);
  // Boxes of the involved devices, sources first, each side by ascending id.
  const std::set<DeviceId> involved(devices.begin(), devices.end());
  std::vector<const SliceRegion*> boxes;
  std::vector<DeviceId> who;
  size_t n_src = 0;
  for (const auto* side : {&src_at, &dst_at}) {
    for (const auto& [d, r] : *side)
      if (involved.count(d)) {
        if (r.partial_count > 1)
          fail(Errc::PartialUnderBsr, "device " + std::to_string(d) + " holds a Partial piece; BSR moves whole values");
        boxes.push_back(&r);
        who.push_back(d);
      }
    if (side == &src_at) n_src = boxes.size();
  }
  BsrTable table;
  detail::CoverGrid(scope, boxes).walk([&](const SliceRegion& cell, const detail::CoverSet& cover) {
    BsrRow row;
    row.tensor_id = tensor_id;
    row.region = cell;
    row.bytes = cell.cells() * elem_bytes;
    cover.each([&](size_t b) { (b < n_src ? row.owners : row.requesters).push_back(who[b]); });
    table.rows.push_back(std::move(row));
  });
  return table;
}

BsrTable build_table(const HetAnnotation& src, const HetAnnotation& dst, const Shape& shape, int tensor_id,
                     int elem_bytes) {
  for (const auto& [a, side] : {std::pair{&src, "source"}, std::pair{&dst, "destination"}})
    if (a->has_partial())
      fail(Errc::PartialUnderBsr, std::string("the ") + side + " " + a->str() +
                                      " holds Partial values, which a batched send-receive cannot move");
  std::vector<DeviceId> devs = src.all_devices();
  const std::vector<DeviceId> more = dst.all_devices();
  devs.insert(devs.end(), more.begin(), more.end());
  return build_table_scoped(src, dst, shape, tensor_id, elem_bytes, SliceRegion::whole(shape), devs);
}

// ---------------------------------------------------------------- plans
int64_t BsrPlan::total_bytes() const {
  return std::accumulate(transfers.begin(), transfers.end(), int64_t{0},
                         [](int64_t s, const Transfer& t) { return s + t.bytes; });
}

std::map<DeviceId, int64_t> BsrPlan::send_load() const {
  std::map<DeviceId, int64_t> load;
  for (const Transfer& t : transfers) load[t.sender] += t.bytes;
  return load;
}

namespace {

// Sender choice for one receiver among a row's owners (ascending ids).
// Without a bandwidth map: the lowest id.  With one: the best link, then the
// least bytes sent so far in this plan, then the lowest id.
class SenderChooser {
 public:
  explicit SenderChooser(const Bandwidth* bw) : bw_(bw) {}

  DeviceId choose(const std::vector<DeviceId>& owners, DeviceId receiver) const {
    if (!bw_) return owners.front();
    DeviceId best = owners.front();
    double best_bw = bw_->get(best, receiver);
    for (DeviceId o : owners) {
      const double b = bw_->get(o, receiver);
      if (b > best_bw || (b == best_bw && sent(o) < sent(best))) {
        best = o;
        best_bw = b;
      }
    }
    return best;
  }
  void charge(DeviceId sender, int64_t bytes) { sent_[sender] += bytes; }

 private:
  int64_t sent(DeviceId d) const {
    const auto it = sent_.find(d);
    return it == sent_.end() ? 0 : it->second;
  }
  const Bandwidth* bw_;
  std::unordered_map<DeviceId, int64_t> sent_;
};

// Fusion groups: transfer indices grouped by (sender, receiver), groups in
// ascending pair order, indices ascending within a group.
std::vector<FusionGroup> fusion_groups(const std::vector<Transfer>& xfer) {
  std::vector<int> order(xfer.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return std::pair{xfer[a].sender, xfer[a].receiver} < std::pair{xfer[b].sender, xfer[b].receiver};
  });
  std::vector<FusionGroup> groups;
  for (int i : order) {
    const Transfer& t = xfer[i];
    if (groups.empty() || groups.back().sender != t.sender || groups.back().receiver != t.receiver)
      groups.push_back({t.sender, t.receiver, {}});
    groups.back().transfer_indices.push_back(i);
  }
  return groups;
}

// A row as the planner sees it: the tensor it belongs to may differ from the
// table row's own tensor_id when one table serves several identical tensors.
struct RowRef {
  int tensor;
  const BsrRow* row;
};

BsrPlan plan_rows(const std::vector<RowRef>& rows, const Bandwidth* bw) {
  BsrPlan plan;
  SenderChooser chooser(bw);
  std::vector<DeviceId> owners, receivers;
  for (const auto& [tensor, row] : rows) {
    if (row->requesters.empty()) continue;
    if (row->owners.empty())
      fail(Errc::NoOwner, "nobody holds " + row->region.str() + " of tensor " + std::to_string(tensor));
    owners.assign(row->owners.begin(), row->owners.end());
    receivers.assign(row->requesters.begin(), row->requesters.end());
    std::sort(owners.begin(), owners.end());
    std::sort(receivers.begin(), receivers.end());
    for (DeviceId r : receivers) {
      if (std::binary_search(owners.begin(), owners.end(), r)) {
        plan.local_copies.push_back({r, tensor, row->region});
        continue;
      }
      const DeviceId snd = chooser.choose(owners, r);
      plan.transfers.push_back({tensor, row->region, snd, r, row->bytes});
      chooser.charge(snd, row->bytes);
    }
  }
  plan.fusion_groups = fusion_groups(plan.transfers);
  return plan;
}

std::vector<RowRef> rows_of(const BsrTable& t) {
  std::vector<RowRef> v;
  v.reserve(t.rows.size());
  for (const BsrRow& r : t.rows) v.push_back({r.tensor_id, &r});
  return v;
}

// fuse over (tensor, table) pairs: rows ordered by (tensor, region bounds).
BsrPlan fuse_rows(std::vector<RowRef> rows, const Bandwidth& bw) {
  std::stable_sort(rows.begin(), rows.end(), [](const RowRef& a, const RowRef& b) {
    return a.tensor != b.tensor ? a.tensor < b.tensor : a.row->region.bounds < b.row->region.bounds;
  });
  return plan_rows(rows, &bw);
}

}  // namespace

BsrPlan make_plan(const BsrTable& table, const Bandwidth& bandwidth) { return plan_rows(rows_of(table), &bandwidth); }

BsrPlan make_plan_naive(const BsrTable& table) { return plan_rows(rows_of(table), nullptr); }

BsrPlan fuse(const std::vector<BsrTable>& tables, const Bandwidth& bandwidth) {
  // every tensor id belongs to one table
  std::map<int, size_t> owner_table;
  std::vector<RowRef> rows;
  for (size_t k = 0; k < tables.size(); ++k)
    for (const BsrRow& r : tables[k].rows) {
      const auto [it, fresh] = owner_table.emplace(r.tensor_id, k);
      if (!fresh && it->second != k)
        fail(Errc::ParseError, "tensor " + std::to_string(r.tensor_id) + " appears in two fused tables");
      rows.push_back({r.tensor_id, &r});
    }
  return fuse_rows(std::move(rows), bandwidth);
}

namespace detail {

BsrPlan fuse_relabelled(const std::vector<std::pair<int, const BsrTable*>>& tables, const Bandwidth& bandwidth) {
  std::set<int> ids;
  std::vector<RowRef> rows;
  for (const auto& [tensor, table] : tables) {
    if (table->rows.empty()) continue;
    if (!ids.insert(tensor).second)
      fail(Errc::ParseError, "tensor " + std::to_string(tensor) + " appears in two fused tables");
    for (const BsrRow& r : table->rows) rows.push_back({tensor, &r});
  }
  return fuse_rows(std::move(rows), bandwidth);
}

}  // namespace detail

std::map<DeviceId, VolumeEntry> volume_report(const BsrPlan& plan, const std::map<DeviceId, int>& node_of) {
  std::map<DeviceId, VolumeEntry> report;
  for (const auto& [d, n] : node_of) report.emplace(d, VolumeEntry{});
  auto node = [&](DeviceId d, const char* role) {
    const auto it = node_of.find(d);
    if (it == node_of.end()) fail(Errc::UnknownDevice, std::string(role) + " " + std::to_string(d) + " has no node");
    return it->second;
  };
  for (const Transfer& t : plan.transfers) {
    const int from = node(t.sender, "sender");  // sender checked first
    const bool same_node = from == node(t.receiver, "receiver");
    VolumeEntry& v = report[t.sender];
    (same_node ? v.intra_bytes : v.inter_bytes) += t.bytes;
  }
  return report;
}

}  // namespace hshard
