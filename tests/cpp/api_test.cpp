// C++ API test: exercises libhshard_b200.so exactly as a reference (hshard)
// user would -- same headers, names and calls -- and checks SPEC examples.
//   api_test cpu   planner + host Tensor / scatter / reassemble (no GPU)
//   api_test gpu   execute_plan / apply_switch on the B200
#include <cstdio>
#include <cstdlib>
#include <string>

#include "hshard/deduction.hpp"
#include "hshard/graph.hpp"
#include "hshard/resolve.hpp"
#include "hshard/sim.hpp"
#include "hshard/switch.hpp"

using namespace hshard;

static int failures = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "%s:%d CHECK(%s)\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

static Tensor iota(Shape s, DType dt, double scale = 1.0) {
  Tensor t(s, dt);
  for (size_t i = 0; i < t.data.size(); ++i) t.data[i] = static_cast<double>((i * 7) % 13) * scale - 5;
  return t;
}

static bool comm_kind_ok(const CompGraph& g, int node) {
  return g.node(node).kind == OpKind::CommOp && !g.comm_once(node);  // fed by a placeholder path
}

static void cpu_tests() {
  const DeviceGroup g4({0, 1, 2, 3});
  // Fig 6 bottom-tier table
  auto kind = [](const CommPlan& p) { return p.bottom_phase.at(0).kind; };
  CHECK(kind(classify(HetAnnotation::single(g4, {{kPartial, 4}}), HetAnnotation::single(g4, {{kDuplicate, 4}}), {8, 8})) == StepKind::AllReduce);
  CHECK(kind(classify(HetAnnotation::single(g4, {{kPartial, 4}}), HetAnnotation::single(g4, {{0, 4}}), {8, 8})) == StepKind::ReduceScatter);
  CHECK(kind(classify(HetAnnotation::single(g4, {{0, 4}}), HetAnnotation::single(g4, {{kDuplicate, 4}}), {8, 8})) == StepKind::AllGather);
  // placement example
  auto a = HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2})}, {{{1, 2}}, {}}, 0, {Rational(1, 2), Rational(1, 2)});
  const SliceRegion r = placement(a, {4, 4}, 1);
  CHECK(r.str() == "[0,2)x[2,4)");
  // text round trip of the reference str() form
  CHECK(parse_annotation(a.str()).str() == a.str());
  // PartialUnderBsr
  bool threw = false;
  try {
    classify(HetAnnotation::single(g4, {{kPartial, 4}}), HetAnnotation::single(DeviceGroup({0, 1}), {{0, 2}}), {8, 8});
  } catch (const Error& e) {
    threw = e.code() == Errc::PartialUnderBsr;
  }
  CHECK(threw);
  // Tensor box ops
  Tensor t = iota({6, 5}, DType::F32);
  SliceRegion box;
  box.bounds = {{{1, 4}}, {{2, 5}}};
  Tensor s = t.slice(box);
  CHECK(s.shape == Shape({3, 3}) && s.data[0] == t.data[1 * 5 + 2]);
  Tensor z = Tensor::zeros({6, 5}, DType::F32);
  z.write_slice(box, s);
  z.add_slice(box, s);
  CHECK(z.data[2 * 5 + 3] == 2 * t.data[2 * 5 + 3]);
  // scatter -> reassemble is the identity (Split / Duplicate / Partial / hdim)
  const std::vector<HetAnnotation> annos = {
      HetAnnotation::single(g4, {{0, 2}, {kDuplicate, 2}}),
      HetAnnotation::single(g4, {{kPartial, 2}, {1, 2}}),
      HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{1, 2}}, {{kDuplicate, 2}}}, 0,
                          {Rational(2, 3), Rational(1, 3)}),
      HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{1, 2}}, {{kPartial, 2}}}, kPartial),
  };
  const Tensor x = iota({6, 4}, DType::F64);
  for (const auto& an : annos) CHECK(reassemble(an, scatter(an, x), x.shape).bit_equal(x));
  // fused switch conservation
  std::vector<SwitchEntry> diff = {
      {1, HetAnnotation::single(DeviceGroup({0, 1}), {{0, 2}}), HetAnnotation::single(g4, {{0, 4}}), {16, 8}},
      {2, HetAnnotation::single(DeviceGroup({0, 1}), {{kDuplicate, 2}}), HetAnnotation::single(DeviceGroup({2, 3}), {{1, 2}}), {8, 8}},
  };
  const SwitchPlan sp = plan_switch(diff, DType::BF16);
  int64_t unfused = 0;
  for (const auto& e : diff) unfused += make_plan(build_table(e.src, e.dst, e.shape, e.tensor_id, 2), Bandwidth::uniform()).total_bytes();
  CHECK(sp.plan.total_bytes() == unfused);

  // strategy source, as a reference user builds it (graph.hpp / deduction.hpp):
  // Megatron MLP under TP2 and TP4, deduced, then diffed into switch entries
  CompGraph g;
  const int s1 = g.add_strategy();
  const int gx = g.placeholder("x", {SymDim::sym("B"), SymDim::lit(64)}, DType::F32);
  const int w1 = g.parameter("w1", {SymDim::lit(64), SymDim::lit(256)}, DType::F32);
  const int h = g.elementwise(EwFunc::Gelu, g.dot(gx, w1));
  const int w2 = g.parameter("w2", {SymDim::lit(256), SymDim::lit(64)}, DType::F32);
  const int y = g.comm(g.dot(h, w2));
  const DeviceGroup t2({0, 1});
  for (int s : {0, s1}) {
    const DeviceGroup& tg = s == 0 ? t2 : g4;
    const int n = tg.size();
    g.set_annotation(gx, s, HetAnnotation::single(tg, {{kDuplicate, n}}));
    g.set_annotation(w1, s, HetAnnotation::single(tg, {{1, n}}));
    g.set_annotation(w2, s, HetAnnotation::single(tg, {{0, n}}));
    g.set_annotation(y, s, HetAnnotation::single(tg, {{kDuplicate, n}}));
    deduce_graph(g, s);
  }
  CHECK(g.tensor(g.node(y).inputs[0]).slots[0]->ds_union[0].count_of(kPartial) == 2);  // row-parallel
  const auto moves = diff_strategies(g, 0, s1, {{"B", 8}});
  CHECK(moves.size() == 2 && moves[0].shape == Shape({64, 256}));
  CHECK(comm_kind_ok(g, y));
}

static void gpu_tests() {
  const DeviceGroup g4({0, 1, 2, 3});
  // config-2-shaped hierarchical Partial -> Split(1), bf16 on the grid (exact)
  auto src = HetAnnotation::make({g4, DeviceGroup({4, 5, 6, 7})}, {{{kPartial, 4}}, {{kDuplicate, 2}, {kPartial, 2}}}, kPartial);
  auto dst = HetAnnotation::make({g4, DeviceGroup({4, 5, 6, 7})}, {{{1, 4}}, {{kDuplicate, 2}, {1, 2}}}, 1);
  const Shape shape{64, 128};
  const CommPlan plan = classify(src, dst, shape, DType::BF16);
  const Tensor x = iota(shape, DType::BF16);
  TrafficLog log;
  auto out = execute_plan(plan, scatter(src, x), &log);
  CHECK(reassemble(dst, out, shape).bit_equal(x));
  CHECK(log.total() > 0);
  // every step kind, f32 (exact small integers)
  const std::vector<std::pair<HetAnnotation, HetAnnotation>> pairs = {
      {HetAnnotation::single(g4, {{kPartial, 4}}), HetAnnotation::single(g4, {{kDuplicate, 4}})},
      {HetAnnotation::single(g4, {{0, 4}}), HetAnnotation::single(g4, {{kDuplicate, 4}})},
      {HetAnnotation::single(g4, {{0, 4}}), HetAnnotation::single(DeviceGroup({4, 5, 6, 7}), {{0, 4}})},
      {HetAnnotation::single(g4, {{0, 2}, {kDuplicate, 2}}), HetAnnotation::single(g4, {{1, 4}})},
      {HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{0, 2}}, {{0, 2}}}, kPartial),
       HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{0, 2}}, {{0, 2}}}, kDuplicate)},
      {HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{kDuplicate, 2}}, {{kDuplicate, 2}}}, 0,
                           {Rational(3, 4), Rational(1, 4)}),
       HetAnnotation::make({DeviceGroup({0, 1}), DeviceGroup({2, 3})}, {{{kDuplicate, 2}}, {{kDuplicate, 2}}}, kDuplicate)},
  };
  for (const auto& [s, d] : pairs) {
    const Tensor v = iota({16, 8}, DType::F32);
    const CommPlan p = classify(s, d, {16, 8}, DType::F32);
    CHECK(reassemble(d, execute_plan(p, scatter(s, v)), v.shape).bit_equal(v));
  }
  // apply_switch round trip
  std::vector<SwitchEntry> diff = {
      {1, HetAnnotation::single(DeviceGroup({0, 1}), {{0, 2}}), HetAnnotation::single(g4, {{1, 4}}), {16, 8}},
      {2, HetAnnotation::single(DeviceGroup({0, 1}), {{kDuplicate, 2}}), HetAnnotation::single(DeviceGroup({2, 3}), {{0, 2}}), {8, 8}},
  };
  std::vector<SwitchEntry> back;
  for (const auto& e : diff) back.push_back({e.tensor_id, e.dst, e.src, e.shape});
  std::map<ShardKey, Tensor> state;
  for (const auto& e : diff)
    for (auto& [d, t] : scatter(e.src, iota(e.shape, DType::BF16, e.tensor_id))) state[{e.tensor_id, d}] = t;
  auto moved = apply_switch(plan_switch(diff, DType::BF16), state);
  auto restored = apply_switch(plan_switch(back, DType::BF16), moved);
  CHECK(restored.size() == state.size());
  for (const auto& [k, t] : state) CHECK(restored.at(k).bit_equal(t));
  bool missing = false;
  try {
    apply_switch(plan_switch(diff, DType::BF16), moved);  // applying twice
  } catch (const Error& e) {
    missing = e.code() == Errc::MissingShard;
  }
  CHECK(missing);
  // the SPEC's state-to-state form over the reference's SimState / DeviceState
  SimState sim;
  for (const auto& e : diff)
    for (auto& [d, t] : scatter(e.src, iota(e.shape, DType::BF16, e.tensor_id)))
      sim.devices[d].store[e.tensor_id] = {placement(e.src, e.shape, d), t};
  const SimState moved_sim = apply_switch(sim, plan_switch(diff, DType::BF16));
  CHECK(moved_sim.traffic.total() > 0);
  for (const auto& e : diff) {
    std::map<DeviceId, Tensor> shards;
    for (const auto& [d, ds] : moved_sim.devices)
      if (ds.store.count(e.tensor_id)) shards[d] = ds.store.at(e.tensor_id).second;
    CHECK(reassemble(e.dst, shards, e.shape).bit_equal(iota(e.shape, DType::BF16, e.tensor_id)));
  }
  const SimState back_sim = apply_switch(moved_sim, plan_switch(back, DType::BF16));
  for (const auto& [d, ds] : sim.devices)
    for (const auto& [tid, rt] : ds.store) CHECK(back_sim.devices.at(d).store.at(tid).second.bit_equal(rt.second));
  bool twice = false;
  try {
    apply_switch(moved_sim, plan_switch(diff, DType::BF16));
  } catch (const Error& e) {
    twice = e.code() == Errc::MissingShard;
  }
  CHECK(twice);
  // repeated execute_plan of one plan reuses its cached context and program
  for (int r = 0; r < 3; ++r) CHECK(reassemble(dst, execute_plan(plan, scatter(src, x)), shape).bit_equal(x));
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    cpu_tests();
    if (mode == "gpu") gpu_tests();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %d failures\n", mode.c_str(), failures);
  return failures ? 1 : 0;
}
