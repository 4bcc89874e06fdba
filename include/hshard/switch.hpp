// hshard-b200: graph-switch parameter redistribution.
//
// The reference specifies diff_strategies / plan_switch / apply_switch only in
// prose; there is no reference code.  Planning here is the
// SPEC's recipe on the reference primitives: build_table per changed
// parameter (bsr.hpp:50) then one global fuse() (bsr.hpp:96).  Execution is
// in hshard/exec.hpp.
#pragma once

#include <map>
#include <string>

#include "hshard/bsr.hpp"

namespace hshard {

// One parameter whose annotation changes (SPEC.md:413-418 output element).
struct SwitchEntry {
  int tensor_id = 0;
  HetAnnotation src;
  HetAnnotation dst;
  Shape shape;
};

// A parameter's layout under two strategies (a CompGraph's slots supply them
// through the overload below).
struct ParamLayouts {
  int tensor_id = 0;
  Shape shape;
  HetAnnotation a;
  HetAnnotation b;
};

// Changed parameters only; annotations_equal pairs are omitted.
std::vector<SwitchEntry> diff_strategies(const std::vector<ParamLayouts>& params);

class CompGraph;
// SPEC.md:413-418 as specified: the Parameters of a deduced graph whose
// annotation differs between strategies a and b, shapes bound with
// `bindings` (graph.hpp).  UndeducedStrategy if a slot is empty.
std::vector<SwitchEntry> diff_strategies(const CompGraph& graph, int a, int b,
                                         const std::map<std::string, int64_t>& bindings = {});

struct SwitchPlan {
  std::vector<SwitchEntry> diff;  // tensor order of the plan
  DType dtype = DType::F32;
  BsrPlan plan;                   // fused: one fusion group per (sender, receiver)
};

// build_table per entry (elem bytes = dtype width), then fuse.
// Throws PartialUnderBsr for Partial parameters.
SwitchPlan plan_switch(const std::vector<SwitchEntry>& diff, DType dtype,
                       const Bandwidth& bandwidth = Bandwidth::uniform());

}  // namespace hshard
