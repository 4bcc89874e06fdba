// hshard-b200 planner: graph-switch planning.
#include "hshard/switch.hpp"

#include <algorithm>
#include <chrono>
#include <string>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>

#include "hshard/graph.hpp"
#include "planner_internal.hpp"

namespace hshard {

std::vector<SwitchEntry> diff_strategies(const CompGraph& graph, int a, int b,
                                         const std::map<std::string, int64_t>& bindings) {
  std::vector<ParamLayouts> params;
  for (const OpNode& n : graph.nodes()) {
    if (n.kind != OpKind::Parameter) continue;  // only weights migrate
    const TensorRef& t = graph.tensor(n.outputs.at(0));
    const auto &sa = t.slots.at(a), &sb = t.slots.at(b);
    if (!sa || !sb)
      fail(Errc::UndeducedStrategy, "parameter " + std::to_string(t.id) + " has no annotation for strategy " +
                                        std::to_string(sa ? b : a) + " (deduce_graph first)");
    params.push_back({t.id, bind_shape(t.shape, bindings), *sa, *sb});
  }
  return diff_strategies(params);
}

std::vector<SwitchEntry> diff_strategies(const std::vector<ParamLayouts>& params) {
  std::vector<SwitchEntry> out;
  for (const ParamLayouts& p : params)
    if (!annotations_equal(p.a, p.b)) out.push_back({p.tensor_id, p.a, p.b, p.shape});
  return out;
}

SwitchPlan plan_switch(const std::vector<SwitchEntry>& diff, DType dtype,
                       const Bandwidth& bandwidth) {
  SwitchPlan sp;
  sp.diff = diff;
  sp.dtype = dtype;
  // build_table per parameter.  A model's parameters repeat a handful of
  // (src, dst, shape) triples (cfg4: 291 tensors, 12 triples), and a table
  // depends on the tensor only through BsrRow::tensor_id, so each distinct
  // triple is built once and its rows relabelled (same table, same order).
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<BsrTable> distinct;
  std::vector<std::pair<int, size_t>> uses;  // (tensor id, index into distinct)
  uses.reserve(diff.size());
  std::unordered_map<std::string, size_t> seen;  // triple -> its table
  for (const SwitchEntry& e : diff) {
    std::string key = e.src.str();
    key += '>';
    key += e.dst.str();
    key += '@';
    key += join_ints(e.shape);
    auto it = seen.find(key);
    if (it == seen.end()) {
      it = seen.emplace(std::move(key), distinct.size()).first;
      distinct.push_back(build_table(e.src, e.dst, e.shape, e.tensor_id, dtype_width(dtype)));
    }
    uses.emplace_back(e.tensor_id, it->second);
  }
  std::vector<std::pair<int, const BsrTable*>> tables;
  tables.reserve(uses.size());
  for (const auto& [tid, k] : uses) tables.emplace_back(tid, &distinct[k]);
  const auto t1 = std::chrono::steady_clock::now();
  sp.plan = detail::fuse_relabelled(tables, bandwidth);
  if (std::getenv("HS_COMPILE_TRACE"))
    std::fprintf(stderr, "[plan] build_table %.2f ms, fuse %.2f ms (%zu tables, %zu distinct)\n",
                 std::chrono::duration<double, std::milli>(t1 - t0).count(),
                 std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(), tables.size(),
                 distinct.size());
  return sp;
}

}  // namespace hshard
