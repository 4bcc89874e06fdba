// hshard-b200 C ABI: planner entry points (include/hshard_c.h).
#include <chrono>
#include <unordered_map>
#include <cstdio>
#include <cstdlib>
#include <cstdlib>
#include <cstring>
#include <map>
#include <sstream>
#include <variant>

#include "capi_common.hpp"
#include "hshard/deduction.hpp"
#include "hshard/graph.hpp"
#include "hshard/specialize.hpp"
#include "hshard/resolve.hpp"
#include "hshard/switch.hpp"

using namespace hshard;

namespace hshard::capi {

thread_local std::string g_last_error;

int fail_code(Errc e, const std::string& msg) {
  g_last_error = msg;
  return 1 + static_cast<int>(e);
}

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

Shape to_shape(const int64_t* shape, int ndim) {
  if (ndim < 0 || (ndim > 0 && !shape)) fail(Errc::ShapeMismatch, "bad shape");
  return Shape(shape, shape + ndim);
}

DType to_dtype(int code) {
  if (code < 0 || code > static_cast<int>(DType::BF16)) fail(Errc::ParseError, "bad dtype code");
  return static_cast<DType>(code);
}

}  // namespace hshard::capi

using namespace hshard::capi;

extern "C" {

const char* hs_last_error(void) { return g_last_error.c_str(); }
const char* hs_errc_name(int errc) { return errc_name(static_cast<Errc>(errc)); }
void hs_free(void* p) { std::free(p); }
int hs_version(void) { return 1; }

int hs_classify(const char* src, const char* dst, const int64_t* shape, int ndim, int dtype,
                const char* bw, hs_plan** out) {
  return guarded([&] {
    auto plan = std::make_unique<hs_plan>();
    plan->comm = classify(parse_annotation(src), parse_annotation(dst), to_shape(shape, ndim),
                          to_dtype(dtype), parse_bandwidth(bw ? bw : "u"));
    *out = plan.release();
  });
}

int hs_plan_switch(int n, const int* tensor_ids, const char* const* src, const char* const* dst,
                   const int64_t* shapes_flat, const int* ndims, int dtype, const char* bw,
                   hs_plan** out) {
  return guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<SwitchEntry> diff;
    const int64_t* cursor = shapes_flat;
    // a model repeats a handful of annotation texts: parse each once
    std::unordered_map<std::string, HetAnnotation> parsed;
    auto anno = [&](const char* text) -> const HetAnnotation& {
      auto it = parsed.find(text);
      if (it == parsed.end()) it = parsed.emplace(text, parse_annotation(text)).first;
      return it->second;
    };
    for (int i = 0; i < n; ++i) {
      SwitchEntry e;
      e.tensor_id = tensor_ids[i];
      e.src = anno(src[i]);
      e.dst = anno(dst[i]);
      e.shape = to_shape(cursor, ndims[i]);
      cursor += ndims[i];
      diff.push_back(std::move(e));
    }
    if (std::getenv("HS_COMPILE_TRACE"))
      std::fprintf(stderr, "[plan] parse %zu entries %.2f ms\n", diff.size(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    auto plan = std::make_unique<hs_plan>();
    plan->sw = plan_switch(diff, to_dtype(dtype), parse_bandwidth(bw ? bw : "u"));
    *out = plan.release();
  });
}

int hs_plan_dump(const hs_plan* plan, char** json) {
  return guarded([&] {
    *json = dup_string(plan->comm ? dump_plan(*plan->comm) : dump_bsr(plan->sw->plan));
  });
}

void hs_plan_destroy(hs_plan* plan) { delete plan; }

int hs_volume_report(const hs_plan* plan, int n, const int* devices, const int* nodes, char** json) {
  return guarded([&] {
    std::map<DeviceId, int> node_of;
    for (int i = 0; i < n; ++i) node_of[devices[i]] = nodes[i];
    BsrPlan merged;  // a switch's fused plan, or every Bsr step of a CommPlan
    if (plan->sw) {
      merged = plan->sw->plan;
    } else {
      for (const auto* ph : {&plan->comm->bottom_phase, &plan->comm->top_phase})
        for (const CommStep& st : *ph)
          if (st.bsr) merged.transfers.insert(merged.transfers.end(), st.bsr->transfers.begin(), st.bsr->transfers.end());
    }
    std::string o = "{";
    bool first = true;
    for (const auto& [d, v] : volume_report(merged, node_of)) {
      o += std::string(first ? "" : ",") + "\"" + std::to_string(d) + "\":[" + std::to_string(v.intra_bytes) + "," +
           std::to_string(v.inter_bytes) + "]";
      first = false;
    }
    *json = capi::dup_string(o + "}");
  });
}

int hs_build_table(const char* src, const char* dst, const int64_t* shape, int ndim,
                   int tensor_id, int elem_bytes, char** json) {
  return guarded([&] {
    *json = dup_string(dump_table(build_table(parse_annotation(src), parse_annotation(dst),
                                              to_shape(shape, ndim), tensor_id, elem_bytes)));
  });
}

int hs_make_plan(const char* src, const char* dst, const int64_t* shape, int ndim,
                 int elem_bytes, const char* bw, int naive, char** json) {
  return guarded([&] {
    const BsrTable t =
        build_table(parse_annotation(src), parse_annotation(dst), to_shape(shape, ndim), 0, elem_bytes);
    *json = dup_string(dump_bsr(naive ? make_plan_naive(t) : make_plan(t, parse_bandwidth(bw ? bw : "u"))));
  });
}

int hs_placement(const char* anno, const int64_t* shape, int ndim, int device, int64_t* lo,
                 int64_t* hi, int* ord) {
  return guarded([&] {
    const SliceRegion r = placement(parse_annotation(anno), to_shape(shape, ndim), device);
    for (int d = 0; d < ndim; ++d) {
      lo[d] = r.bounds[d][0];
      hi[d] = r.bounds[d][1];
    }
    ord[0] = r.partial_index;
    ord[1] = r.partial_count;
    ord[2] = r.replica_index;
    ord[3] = r.replica_count;
  });
}

int hs_convert_hsize(const char* anno, int target, char** out) {
  return guarded([&] { *out = dup_string(convert_hsize(parse_annotation(anno), target).str()); });
}

int hs_annotations_equal(const char* a, const char* b, int* eq) {
  return guarded([&] { *eq = annotations_equal(parse_annotation(a), parse_annotation(b)) ? 1 : 0; });
}

int hs_validate(const char* anno, const int64_t* shape, int ndim, char** json) {
  return guarded([&] {
    std::string s = "[";
    const auto issues = validate(parse_annotation(anno), to_shape(shape, ndim));
    for (size_t i = 0; i < issues.size(); ++i)
      s += std::string(i ? "," : "") + "\"" + errc_name(issues[i].code) + "\"";
    *json = dup_string(s + "]");
  });
}

int hs_align_shard_specs(const char* a, const char* b, char** json) {
  return guarded([&] {
    const auto f = align_shard_specs(parse_shard_spec(a), parse_shard_spec(b));
    if (!f) {
      *json = dup_string("null");
      return;
    }
    std::string s = "[";
    for (size_t i = 0; i < f->size(); ++i)
      s += std::string(i ? "," : "") + "[" + std::to_string((*f)[i].key_a) + "," +
           std::to_string((*f)[i].key_b) + "," + std::to_string((*f)[i].count) + "]";
    *json = dup_string(s + "]");
  });
}

}  // extern "C"

// ---------------------------------------------------------------- strategy source
namespace {

std::string jquote(const std::string& v) {
  std::string o = "\"";
  for (char c : v) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

std::map<std::string, int64_t> parse_bindings(const char* text) {
  std::map<std::string, int64_t> b;
  if (!text) return b;
  std::stringstream ss(text);
  for (std::string item; std::getline(ss, item, ',');) {
    if (item.find_first_not_of(' ') == std::string::npos) continue;
    const auto eq = item.find('=');
    if (eq == std::string::npos) fail(Errc::ParseError, "binding '" + item + "' lacks '='");
    std::string k = item.substr(0, eq);
    k.erase(0, k.find_first_not_of(' '));
    k.erase(k.find_last_not_of(' ') + 1);
    b[k] = std::stoll(item.substr(eq + 1));
  }
  return b;
}

}  // namespace

extern "C" {

int hs_graph_deduce(const char* graph, char** json) {
  return capi::guarded([&] {
    CompGraph g = parse_graph(graph);
    std::string o = "{\"tensors\":[";
    for (const TensorRef& t : g.tensors())
      o += std::string(t.id ? "," : "") + "{\"id\":" + std::to_string(t.id) + ",\"name\":" + jquote(t.name) +
           ",\"kind\":" + jquote(op_kind_name(g.node(t.producer).kind)) + ",\"shape\":" +
           jquote(sym_shape_str(t.shape)) + ",\"dtype\":" + jquote(dtype_name(t.dtype)) +
           ",\"producer\":" + std::to_string(t.producer) + "}";
    o += "],\"topo\":[";
    const auto order = g.topo_order();
    for (size_t i = 0; i < order.size(); ++i) o += (i ? "," : "") + std::to_string(order[i]);
    o += "],\"symbols\":[";
    const auto syms = g.symbols();
    for (size_t i = 0; i < syms.size(); ++i) o += (i ? "," : "") + jquote(syms[i]);
    o += "],\"strategies\":[";
    for (int s = 0; s < g.strategy_count(); ++s) {
      o += s ? "," : "";
      try {
        deduce_graph(g, s);
        o += "{\"ok\":1,\"slots\":[";
        for (const TensorRef& t : g.tensors())
          o += std::string(t.id ? "," : "") + (t.slots.at(s) ? jquote(t.slots.at(s)->str()) : "null");
        o += "]}";
      } catch (const Error& e) {
        o += "{\"ok\":0,\"error\":" + jquote(errc_name(e.code())) + ",\"message\":" + jquote(e.what()) + "}";
      }
    }
    *json = capi::dup_string(o + "]}");
  });
}

int hs_graph_diff(const char* graph, int a, int b, const char* bindings, char** json) {
  return capi::guarded([&] {
    CompGraph g = parse_graph(graph);
    deduce_graph(g, a);
    if (b != a) deduce_graph(g, b);
    const auto diff = diff_strategies(g, a, b, parse_bindings(bindings));
    std::string o = "[";
    for (size_t i = 0; i < diff.size(); ++i) {
      const SwitchEntry& e = diff[i];
      o += std::string(i ? "," : "") + "{\"tensor\":" + std::to_string(e.tensor_id) + ",\"name\":" +
           jquote(g.tensor(e.tensor_id).name) + ",\"src\":" + jquote(e.src.str()) + ",\"dst\":" +
           jquote(e.dst.str()) + ",\"shape\":[" + join_ints(e.shape) + "]}";
    }
    *json = capi::dup_string(o + "]");
  });
}

int hs_graph_specialize(const char* graph, int strategy, const char* bindings, char** json) {
  return capi::guarded([&] {
    CompGraph g = parse_graph(graph);
    deduce_graph(g, strategy);
    const auto bind = parse_bindings(bindings);
    std::string o = "{\"phases\":{";
    bool first = true;
    for (const auto& [id, ph] : node_phases(g, strategy)) {
      o += std::string(first ? "" : ",") + "\"" + std::to_string(id) + "\":" + jquote(exec_phase_name(ph));
      first = false;
    }
    o += "},\"exec_graphs\":[";
    const auto egs = instantiate_all(g, strategy, bind);
    for (size_t i = 0; i < egs.size(); ++i) {
      o += std::string(i ? "," : "") + "{\"device\":" + std::to_string(egs[i].device) + ",\"nodes\":[";
      for (size_t k = 0; k < egs[i].nodes.size(); ++k) {
        const ExecNode& n = egs[i].nodes[k];
        o += std::string(k ? "," : "") + "{\"node\":" + std::to_string(n.node_id) + ",\"comm\":" +
             (n.is_comm ? "1" : "0") + ",\"phase\":" + jquote(exec_phase_name(n.phase)) +
             ",\"plan\":" + (n.plan ? dump_plan(*n.plan) : std::string("null")) + "}";
      }
      o += "]}";
    }
    o += "]";
    try {
      const auto pipes = construct_pipelines(g, strategy, bind);
      o += ",\"pipelines\":[";
      for (size_t p = 0; p < pipes.size(); ++p) {
        o += p ? ",[" : "[";
        for (size_t st = 0; st < pipes[p].stages.size(); ++st) {
          std::vector<int64_t> devs(pipes[p].stages[st].begin(), pipes[p].stages[st].end());
          o += std::string(st ? "," : "") + "[" + join_ints(devs) + "]";
        }
        o += "]";
      }
      o += "]";
    } catch (const Error& e) {
      o += ",\"pipelines_error\":" + jquote(errc_name(e.code()));
    }
    *json = capi::dup_string(o + "}");
  });
}

}  // extern "C"
