// hshard-b200 planner: graph-switch planning.
#include "hshard/switch.hpp"

namespace hshard {

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
