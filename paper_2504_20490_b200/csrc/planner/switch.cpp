// hshard-b200 planner: graph-switch planning.
#include "hshard/switch.hpp"

#include "hshard/graph.hpp"

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
  std::vector<BsrTable> tables;
  tables.reserve(diff.size());
  for (const SwitchEntry& e : diff)
    tables.push_back(build_table(e.src, e.dst, e.shape, e.tensor_id, dtype_width(dtype)));
  sp.plan = fuse(tables, bandwidth);
  return sp;
}

}  // namespace hshard
