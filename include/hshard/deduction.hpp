// hshard-b200: sharding deduction over a CompGraph (reference deduction.hpp:19-31).
#pragma once

#include "hshard/graph.hpp"

namespace hshard {

// Convert every annotation to the largest hsize among them and require one
// device-group union; DgUnionMismatch means an explicit CommOp is needed.
std::vector<HetAnnotation> unify_inputs(const std::vector<HetAnnotation>& annos);

// Output annotations of one non-leaf op from its (unified) input annotations.
std::vector<HetAnnotation> deduce_op(const CompGraph& graph, const OpNode& node,
                                     const std::vector<HetAnnotation>& input_annos);

// Fill every tensor slot of `strategy` from the leaf / CommOp annotations;
// errors carry the failing node id.  Only CommOps change device groups.
void deduce_graph(CompGraph& graph, int strategy);

}  // namespace hshard
