// ORACLE / TEST INFRASTRUCTURE ONLY -- never linked into the product.
//
// Line-protocol driver over the *reference* hshard planner compiled from
// /root/reference/proj/src (see oracle/Makefile).  It parses annotations in
// the reference's own HetAnnotation::str() format
// (annotation.cpp:146-170), calls the reference's classify / build_table /
// make_plan / fuse / placement / convert_hsize, and prints a canonical JSON
// dump that the product planner (paper_2504_20490_b200/csrc/planner) must
// reproduce byte-for-byte.  The same format is emitted by
// paper_2504_20490_b200/csrc/planner/dump.cpp.
//
// It also hosts the "reference-faithful" CPU executor (command X): the plan
// from the reference planner executed with the reference's own per-cell
// Tensor primitives (tensor.cpp:84-114) following SPEC.md:467-495 and
// SURVEY.md Appendix C.  That executor is the CPU baseline of bench.py
// (--impl reference) and a second pin for the numpy oracle.
//
// Commands (one per stdin line, fields separated by '|'):
//   C|dtype|shape|bw|src|dst                  classify          -> plan JSON
//   T|elem_bytes|shape|tid|src|dst            build_table       -> table JSON
//   M|bw|naive|elem_bytes|shape|src|dst       make_plan(_naive) -> bsr JSON
//   F|bw|n  + n lines  tid|elem_bytes|shape|src|dst   fuse      -> bsr JSON
//   R|bw|n|d:node,...  + n lines (as F)         fuse + volume_report
//   P|shape|anno                              placement of every device
//   H|anno|target                             convert_hsize
//   Q|anno|anno                               annotations_equal
//   A|ds|ds                                   align_shard_specs
//   V|shape|anno                              validate (issue codes)
//   X|dtype|shape|bw|src|dst|seed|mode|reps|emit[|threads[|warmup]]
//                                             reference-primitive executor
//   N|dtype|shape|bw|src|dst|seed|mode|reps|threads|warmup|outdir
//                                             native-dtype memcpy executor
//   W|dtype|bw|n|seed|reps|threads|warmup + n lines tid|shape|src|dst
//                                             the same for a fused switch
//                                             (oracle/native_exec.inc)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <iostream>
#include <optional>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hshard/bsr.hpp"
#include "hshard/deduction.hpp"
#include "hshard/graph.hpp"
#include "hshard/resolve.hpp"
#include "hshard/specialize.hpp"
#include "hshard/tensor.hpp"

using namespace hshard;

namespace {

std::vector<std::string> split(const std::string& s, char sep) {
  std::vector<std::string> out;
  std::string cur;
  for (char c : s) {
    if (c == sep) {
      out.push_back(cur);
      cur.clear();
    } else {
      cur.push_back(c);
    }
  }
  out.push_back(cur);
  return out;
}

std::string trim(const std::string& s) {
  size_t a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  size_t b = s.find_last_not_of(" \t\r\n");
  return s.substr(a, b - a + 1);
}

Shape parse_shape(const std::string& s) {
  Shape out;
  for (auto& t : split(trim(s), ','))
    if (!trim(t).empty()) out.push_back(std::stoll(t));
  return out;
}

ShardSpec parse_ds(const std::string& text) {
  // "{k:c,k:c}"
  std::string s = trim(text);
  ShardSpec ds;
  if (s.size() < 2 || s.front() != '{' || s.back() != '}')
    throw std::runtime_error("bad ds " + s);
  s = s.substr(1, s.size() - 2);
  if (trim(s).empty()) return ds;
  for (auto& e : split(s, ',')) {
    auto kv = split(e, ':');
    ds.entries.push_back({std::stoi(kv.at(0)), std::stoi(kv.at(1))});
  }
  return ds;
}

// Parses "hsize=H hdim=D [(a,b){k:c}; (e){}] ratios=1/2,1/2".
HetAnnotation parse_anno(const std::string& text) {
  std::string s = trim(text);
  size_t hd = s.find("hdim=");
  int hdim = std::stoi(s.substr(hd + 5));
  size_t lb = s.find('['), rb = s.rfind(']');
  std::string body = s.substr(lb + 1, rb - lb - 1);
  std::vector<DeviceGroup> groups;
  std::vector<ShardSpec> specs;
  for (auto& part : split(body, ';')) {
    std::string p = trim(part);
    size_t lp = p.find('('), rp = p.find(')');
    std::vector<DeviceId> devs;
    std::string ids = p.substr(lp + 1, rp - lp - 1);
    if (!trim(ids).empty())
      for (auto& t : split(ids, ',')) devs.push_back(std::stoi(t));
    groups.emplace_back(devs);
    specs.push_back(parse_ds(p.substr(rp + 1)));
  }
  std::vector<Rational> ratios;
  size_t rp = s.find("ratios=", rb);
  if (rp != std::string::npos)
    for (auto& t : split(trim(s.substr(rp + 7)), ','))
      ratios.push_back(Rational::parse(trim(t)));
  return HetAnnotation::make(groups, specs, hdim, ratios);
}

Bandwidth parse_bw(const std::string& text) {
  // "u" | "d=<default>;a-b=w;..."
  std::string s = trim(text);
  Bandwidth bw = Bandwidth::uniform();
  if (s.empty() || s == "u") return bw;
  for (auto& item : split(s, ';')) {
    std::string it = trim(item);
    if (it.empty()) continue;
    auto eq = it.find('=');
    std::string k = it.substr(0, eq);
    double v = std::stod(it.substr(eq + 1));
    if (k == "d") {
      bw.default_bw = v;
    } else {
      auto ab = split(k, '-');
      bw.set(std::stoi(ab.at(0)), std::stoi(ab.at(1)), v);
    }
  }
  return bw;
}

DType parse_dtype(const std::string& s) { return dtype_from_name(trim(s)); }

// ---- canonical JSON -------------------------------------------------------
std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o.push_back('\\');
    o.push_back(c);
  }
  return o + "\"";
}

template <class T>
std::string jints(const std::vector<T>& v) {
  std::string o = "[";
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) o += ",";
    o += std::to_string(v[i]);
  }
  return o + "]";
}

std::string jreg(const SliceRegion& r) {
  std::string o = "[";
  for (size_t i = 0; i < r.bounds.size(); ++i) {
    if (i) o += ",";
    o += "[" + std::to_string(r.bounds[i][0]) + "," + std::to_string(r.bounds[i][1]) + "]";
  }
  o += "]";
  if (r.partial_count != 1 || r.replica_count != 1 || r.partial_index != 0 ||
      r.replica_index != 0)
    o = "{\"b\":" + o + ",\"p\":[" + std::to_string(r.partial_index) + "," +
        std::to_string(r.partial_count) + "],\"q\":[" +
        std::to_string(r.replica_index) + "," + std::to_string(r.replica_count) + "]}";
  return o;
}

std::string jbsr(const BsrPlan& p) {
  std::string o = "{\"local\":[";
  for (size_t i = 0; i < p.local_copies.size(); ++i) {
    const auto& c = p.local_copies[i];
    if (i) o += ",";
    o += "[" + std::to_string(c.device) + "," + std::to_string(c.tensor_id) + "," +
         jreg(c.region) + "]";
  }
  o += "],\"xfer\":[";
  for (size_t i = 0; i < p.transfers.size(); ++i) {
    const auto& t = p.transfers[i];
    if (i) o += ",";
    o += "[" + std::to_string(t.tensor_id) + "," + jreg(t.region) + "," +
         std::to_string(t.sender) + "," + std::to_string(t.receiver) + "," +
         std::to_string(t.bytes) + "]";
  }
  o += "],\"fg\":[";
  for (size_t i = 0; i < p.fusion_groups.size(); ++i) {
    const auto& g = p.fusion_groups[i];
    if (i) o += ",";
    o += "[" + std::to_string(g.sender) + "," + std::to_string(g.receiver) + "," +
         jints(g.transfer_indices) + "]";
  }
  return o + "]}";
}

std::string jstep(const CommStep& s) {
  std::string o = "{\"kind\":" + jstr(step_kind_name(s.kind)) +
                  ",\"sub\":" + std::to_string(s.subgroup) + ",\"groups\":[";
  for (size_t i = 0; i < s.groups.size(); ++i) {
    if (i) o += ",";
    o += jints(s.groups[i]);
  }
  o += "],\"pairs\":[";
  for (size_t i = 0; i < s.pairs.size(); ++i) {
    if (i) o += ",";
    o += "[" + std::to_string(s.pairs[i].first) + "," + std::to_string(s.pairs[i].second) + "]";
  }
  o += "],\"slices\":[";
  for (size_t i = 0; i < s.slices.size(); ++i) {
    if (i) o += ",";
    o += "{\"reg\":" + jreg(s.slices[i].region) + ",\"c\":" + jints(s.slices[i].contributors) +
         ",\"r\":" + jints(s.slices[i].receivers) + "}";
  }
  o += "],\"bsr\":";
  o += s.bsr ? jbsr(*s.bsr) : std::string("null");
  return o + "}";
}

std::string jplan(const CommPlan& p, const std::string& dtype_label) {
  std::string o = "{\"src\":" + jstr(p.src.str()) + ",\"dst\":" + jstr(p.dst.str()) +
                  ",\"mid\":" + (p.mid ? jstr(p.mid->str()) : std::string("null")) +
                  ",\"shape\":" + jints(p.shape) + ",\"dtype\":" + jstr(dtype_label) +
                  ",\"bottom\":[";
  for (size_t i = 0; i < p.bottom_phase.size(); ++i) {
    if (i) o += ",";
    o += jstep(p.bottom_phase[i]);
  }
  o += "],\"top\":[";
  for (size_t i = 0; i < p.top_phase.size(); ++i) {
    if (i) o += ",";
    o += jstep(p.top_phase[i]);
  }
  return o + "]}";
}

std::string jtable(const BsrTable& t) {
  std::string o = "{\"rows\":[";
  for (size_t i = 0; i < t.rows.size(); ++i) {
    const auto& r = t.rows[i];
    if (i) o += ",";
    o += "[" + std::to_string(r.tensor_id) + "," + jreg(r.region) + "," + jints(r.owners) +
         "," + jints(r.requesters) + "," + std::to_string(r.bytes) + "]";
  }
  return o + "]}";
}

// ---- counter-hash data generator (mirrors oracle/datagen.py and the CUDA
// fill kernel) ----------------------------
uint32_t mix32(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x;
}

uint32_t hash3(uint32_t seed, uint32_t key, uint64_t lin) {
  uint32_t h = mix32(seed * 0x9E3779B1U + key * 0x85EBCA77U + 0x165667B1U);
  h = mix32(h ^ static_cast<uint32_t>(lin));
  h = mix32(h ^ static_cast<uint32_t>(lin >> 32) ^ 0x27D4EB2FU);
  return h;
}

uint32_t piece_key(int tensor_id, int level, int g, int p) {
  return static_cast<uint32_t>(tensor_id) * 1000003U + static_cast<uint32_t>(level) * 7919U +
         static_cast<uint32_t>(g) * 131U + static_cast<uint32_t>(p);
}

double grid_value(uint32_t h) { return static_cast<double>((h >> 8) % 8) - 4.0; }

// Value stored by a device with top piece index tg (-1: none, the whole
// logical value), subgroup g, bottom partial ordinal (p of P), at linear
// index `lin` of the logical tensor.  Grid mode only (exact integers).
double piece_value(uint32_t seed, int tid, int hsize, int tg, int g, int p, int P,
                   uint64_t lin) {
  double x = grid_value(hash3(seed, piece_key(tid, 0, 0, 0), lin));
  double t = x;
  if (tg >= 0) {
    if (tg < hsize - 1) {
      t = grid_value(hash3(seed, piece_key(tid, 1, tg, 0), lin));
    } else {
      double s = 0;
      for (int k = 0; k < hsize - 1; ++k)
        s += grid_value(hash3(seed, piece_key(tid, 1, k, 0), lin));
      t = x - s;
    }
  }
  if (P == 1) return t;
  if (p < P - 1) return grid_value(hash3(seed, piece_key(tid, 2, g, p), lin));
  double s = 0;
  for (int k = 0; k < P - 1; ++k) s += grid_value(hash3(seed, piece_key(tid, 2, g, k), lin));
  return t - s;
}

uint64_t linear_index(const Shape& shape, const std::vector<int64_t>& idx) {
  uint64_t off = 0;
  for (size_t i = 0; i < shape.size(); ++i) off = off * shape[i] + idx[i];
  return off;
}

Tensor make_shard(const HetAnnotation& a, const Shape& shape, DeviceId d, uint32_t seed,
                  int tid, DType dt) {
  SliceRegion r = placement(a, shape, d);
  int g = a.subgroup_of(d);
  int tg = a.effective_hdim() == kPartial ? g : -1;
  Tensor t(r.extents(), dt);
  int64_t pos = 0;
  for_each_cell(r, [&](const std::vector<int64_t>& idx) {
    t.data[pos++] = piece_value(seed, tid, a.hsize, tg, g, r.partial_index, r.partial_count,
                                linear_index(shape, idx));
  });
  return t;
}

// Translate a logical box into the local box of a shard whose placement is
// `owner`.
SliceRegion local_box(const SliceRegion& owner, const SliceRegion& logical) {
  SliceRegion out;
  for (size_t i = 0; i < logical.bounds.size(); ++i)
    out.bounds.push_back(
        {logical.bounds[i][0] - owner.bounds[i][0], logical.bounds[i][1] - owner.bounds[i][0]});
  return out;
}

using ShardMap = std::map<DeviceId, std::pair<SliceRegion, Tensor>>;

ShardMap init_target(const HetAnnotation& a, const Shape& shape, DType dt) {
  ShardMap out;
  for (DeviceId d : a.all_devices()) {
    SliceRegion r = placement(a, shape, d);
    out.emplace(d, std::make_pair(r, Tensor(r.extents(), dt)));
  }
  return out;
}

// Phase semantics per SURVEY Appendix C (restating SPEC.md:467-495) using the
// reference's Tensor::slice / write_slice / add_slice.  Reductions use
// ascending device id order; values are doubles (tensor.hpp:24).
// Work units are (target device d, row band k of K): band k is rows
// [lo + n*k/K, lo + n*(k+1)/K) of dim 0 of d's target box, and every logical
// region written to d is clipped to it, so units write disjoint cells and the
// primitives run unchanged on all host threads (unit u = d*K + k runs on
// thread u % nthreads).  Whole-shard assignments (Identity / SendRecv) are
// band 0's.
struct Unit {
  int tid = 0, nthreads = 1, K = 1;
};

std::optional<SliceRegion> clip(const SliceRegion& logical, const SliceRegion& target, int k, int K) {
  if (K == 1) return logical;
  SliceRegion band;
  band.bounds = target.bounds;
  const int64_t lo = target.bounds[0][0], n = target.bounds[0][1] - lo;
  band.bounds[0] = {lo + n * k / K, lo + n * (k + 1) / K};
  if (band.bounds[0][0] >= band.bounds[0][1]) return std::nullopt;
  return intersect(logical, band);
}

void run_step(const CommStep& step, const HetAnnotation& phase_src, const ShardMap& in,
              ShardMap& out, const Unit& U) {
  auto mine = [&](DeviceId d, int k) { return (static_cast<int64_t>(d) * U.K + k) % U.nthreads == U.tid; };
  auto piece = [&](DeviceId m, const SliceRegion& logical) {
    const auto& [reg, ten] = in.at(m);
    return ten.slice(local_box(reg, logical));
  };
  auto put = [&](DeviceId d, const SliceRegion& logical, const Tensor& v, bool add) {
    auto& [reg, ten] = out.at(d);
    if (add)
      ten.add_slice(local_box(reg, logical), v);
    else
      ten.write_slice(local_box(reg, logical), v);
  };
  switch (step.kind) {
    case StepKind::Identity:
      for (DeviceId d : phase_src.dg_union.at(step.subgroup).devices)
        if (mine(d, 0)) out.at(d).second = in.at(d).second;
      break;
    case StepKind::SendRecv:
      for (auto [s, r] : step.pairs)
        if (mine(r, 0)) out.at(r).second = in.at(s).second;
      break;
    case StepKind::AllReduce:
    case StepKind::ReduceScatter:
      for (const auto& grp : step.groups) {
        std::vector<DeviceId> order(grp.begin(), grp.end());
        std::sort(order.begin(), order.end());
        for (DeviceId d : grp) {
          SliceRegion target = out.at(d).first;
          SliceRegion whole;
          whole.bounds = target.bounds;
          for (DeviceId m : order) {
            if (!in.at(m).first.covers(whole)) throw Error(Errc::ShapeMismatch, "unexecutable");
          }
          for (int k = 0; k < U.K; ++k) {
            if (!mine(d, k)) continue;
            auto box = clip(whole, target, k, U.K);
            if (!box) continue;
            bool first = true;
            for (DeviceId m : order) {
              put(d, *box, piece(m, *box), !first);
              first = false;
            }
          }
        }
      }
      break;
    case StepKind::AllGather:
      for (const auto& grp : step.groups) {
        for (DeviceId d : grp) {
          SliceRegion target = out.at(d).first;
          int64_t covered = 0;
          for (DeviceId m : grp) {
            auto isect = intersect(in.at(m).first, target);
            if (isect) covered += isect->cells();
          }
          if (covered != target.cells()) throw Error(Errc::ShapeMismatch, "unexecutable");
          for (int k = 0; k < U.K; ++k) {
            if (!mine(d, k)) continue;
            for (DeviceId m : grp) {
              auto isect = intersect(in.at(m).first, target);
              if (!isect) continue;
              auto box = clip(*isect, target, k, U.K);
              if (box) put(d, *box, piece(m, *box), false);
            }
          }
        }
      }
      break;
    case StepKind::SplitAllReduce:
    case StepKind::SplitReduceScatter:
    case StepKind::SplitAllGather:
      for (const auto& sc : step.slices) {
        for (DeviceId r : sc.receivers) {
          const SliceRegion& rr = out.at(r).first;
          std::vector<DeviceId> cs(sc.contributors.begin(), sc.contributors.end());
          std::sort(cs.begin(), cs.end());
          for (int k = 0; k < U.K; ++k) {
            if (!mine(r, k)) continue;
            auto box = clip(sc.region, rr, k, U.K);
            if (!box) continue;
            bool any = false;
            for (DeviceId c : cs) {
              const SliceRegion& cr = in.at(c).first;
              if (cr.partial_index % rr.partial_count != rr.partial_index) continue;
              put(r, *box, piece(c, *box), any);
              any = true;
            }
            if (!any) {
              Tensor z(box->extents(), out.at(r).second.dtype);
              put(r, *box, z, false);
            }
          }
        }
      }
      break;
    case StepKind::Bsr:
      for (int k = 0; k < U.K; ++k) {
        for (const auto& c : step.bsr->local_copies) {
          if (!mine(c.device, k)) continue;
          auto box = clip(c.region, out.at(c.device).first, k, U.K);
          if (box) put(c.device, *box, piece(c.device, *box), false);
        }
        for (const auto& fg : step.bsr->fusion_groups)
          for (int i : fg.transfer_indices) {
            const auto& t = step.bsr->transfers[i];
            if (!mine(t.receiver, k)) continue;
            auto box = clip(t.region, out.at(t.receiver).first, k, U.K);
            if (box) put(t.receiver, *box, piece(t.sender, *box), false);
          }
      }
      break;
  }
}

void run_phase(const std::vector<CommStep>& steps, const HetAnnotation& phase_src,
               const ShardMap& in, ShardMap& out, int nthreads) {
  // K bands per target so that targets x bands covers every thread
  const int K = std::max<int>(1, (nthreads + static_cast<int>(out.size()) - 1) / std::max<int>(1, out.size()));
  if (nthreads <= 1) {
    for (const auto& s : steps) run_step(s, phase_src, in, out, Unit{});
    return;
  }
  std::vector<std::thread> pool;
  std::vector<std::exception_ptr> errs(nthreads);
  for (int t = 0; t < nthreads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (const auto& s : steps) run_step(s, phase_src, in, out, Unit{t, nthreads, K});
      } catch (...) {
        errs[t] = std::current_exception();
      }
    });
  for (auto& th : pool) th.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}

// The functional executor (sim.hpp:77-79): fresh target states per run; the
// source map is read in place (no per-run copy of the inputs).
ShardMap run_plan(const CommPlan& plan, const ShardMap& src, DType dt, int nthreads) {
  if (plan.bottom_phase.empty() && plan.top_phase.empty()) return src;
  const ShardMap* cur = &src;
  ShardMap mid;
  if (!plan.bottom_phase.empty()) {
    mid = init_target(plan.bottom_target(), plan.shape, dt);
    run_phase(plan.bottom_phase, plan.src, *cur, mid, nthreads);
    if (plan.top_phase.empty()) return mid;
    cur = &mid;
  }
  ShardMap next = init_target(plan.dst, plan.shape, dt);
  run_phase(plan.top_phase, plan.mid ? *plan.mid : plan.src, *cur, next, nthreads);
  return next;
}

std::string cmd_execute(const std::vector<std::string>& f) {
  DType dt = parse_dtype(f.at(1));
  Shape shape = parse_shape(f.at(2));
  Bandwidth bw = parse_bw(f.at(3));
  HetAnnotation src = parse_anno(f.at(4)), dst = parse_anno(f.at(5));
  uint32_t seed = static_cast<uint32_t>(std::stoul(f.at(6)));
  int reps = std::stoi(f.at(8));
  int emit = std::stoi(f.at(9));
  int nthreads = f.size() > 10 ? std::stoi(f.at(10)) : 1;
  int warmup = f.size() > 11 ? std::stoi(f.at(11)) : 0;
  CommPlan plan = classify(src, dst, shape, dt, bw);
  ShardMap in;
  for (DeviceId d : src.all_devices())  // regions first, payloads generated in parallel below
    in.emplace(d, std::make_pair(placement(src, shape, d), Tensor(Shape{}, dt)));
  {
    std::vector<std::thread> gen;
    for (DeviceId d : src.all_devices())
      gen.emplace_back([&, d] { in.at(d).second = make_shard(src, shape, d, seed, 0, dt); });
    for (auto& th : gen) th.join();
  }
  ShardMap out;
  for (int r = 0; r < warmup; ++r) out = run_plan(plan, in, dt, nthreads);
  double best = 1e30, total = 0;
  for (int r = 0; r < std::max(1, reps); ++r) {
    auto t0 = std::chrono::steady_clock::now();
    out = run_plan(plan, in, dt, nthreads);
    auto t1 = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(t1 - t0).count();
    best = std::min(best, sec);
    total += sec;
  }
  int64_t dst_bytes = 0;
  std::string o = "{\"seconds\":" + std::to_string(best) +
                  ",\"mean\":" + std::to_string(total / std::max(1, reps)) +
                  ",\"reps\":" + std::to_string(std::max(1, reps)) +
                  ",\"threads\":" + std::to_string(nthreads) + ",\"shards\":{";
  bool first = true;
  for (auto& [d, rt] : out) {
    dst_bytes += rt.first.cells() * dtype_width(dt);
    double sum = 0, wsum = 0;
    for (size_t i = 0; i < rt.second.data.size(); ++i) {
      sum += rt.second.data[i];
      wsum += rt.second.data[i] * static_cast<double>((i % 1013) + 1);
    }
    if (!first) o += ",";
    first = false;
    std::ostringstream os;
    os.precision(17);
    os << "\"" << d << "\":{\"sum\":" << sum << ",\"wsum\":" << wsum;
    if (emit) {
      os << ",\"v\":[";
      for (size_t i = 0; i < rt.second.data.size(); ++i) os << (i ? "," : "") << rt.second.data[i];
      os << "]";
    }
    os << "}";
    o += os.str();
  }
  o += "},\"dst_bytes\":" + std::to_string(dst_bytes) + "}";
  return o;
}

#include "native_exec.inc"

// G|stmt&stmt&...: build the reference CompGraph from the line form of
// include/hshard/graph.hpp (parse_graph), deduce every strategy with the
// reference deduce_graph (deduction.cpp:318-353), print the slots.
CompGraph parse_program(const std::string& program) {
  CompGraph g;
  bool first = true;
  for (const std::string& raw : split(program, '&')) {
    const std::string st = trim(raw);
    if (st.empty()) continue;
    std::istringstream is(st);
    std::vector<std::string> w;
    for (std::string x; is >> x;) w.push_back(x);
    auto shape_from = [&](size_t k) {
      SymShape sh;
      for (size_t i = k; i < w.size(); ++i) sh.push_back(SymDim::parse(w[i]));
      return sh;
    };
    const std::string& op = w[0];
    if (op == "strategies") {
      if (!first) throw std::runtime_error("strategies must come first");
      for (int k = 1; k < std::stoi(w.at(1)); ++k) g.add_strategy();
    } else if (op == "placeholder") {
      g.placeholder(w.at(1), shape_from(3), parse_dtype(w.at(2)));
    } else if (op == "parameter") {
      g.parameter(w.at(1), shape_from(3), parse_dtype(w.at(2)));
    } else if (op == "elementwise") {
      g.elementwise(ew_func_from_name(w.at(1)), std::stoi(w.at(2)));
    } else if (op == "dot") {
      g.dot(std::stoi(w.at(1)), std::stoi(w.at(2)));
    } else if (op == "sum") {
      g.sum(std::stoi(w.at(1)), std::stoi(w.at(2)));
    } else if (op == "reshape") {
      g.reshape(std::stoi(w.at(1)), shape_from(2));
    } else if (op == "comm") {
      g.comm(std::stoi(w.at(1)), w.at(2) == "auto" ? std::nullopt : std::optional<bool>(w.at(2) == "1"));
    } else if (op == "annotate") {
      // annotation text = everything after the third word
      size_t pos = 0;
      for (int k = 0; k < 3; ++k) {
        pos = st.find_first_not_of(" ", pos);
        pos = st.find(' ', pos);
      }
      g.set_annotation(std::stoi(w.at(1)), std::stoi(w.at(2)), parse_anno(st.substr(pos)));
    } else {
      throw std::runtime_error("unknown statement " + op);
    }
    first = false;
  }
  return g;
}

std::string cmd_graph(const std::string& program) {
  CompGraph g = parse_program(program);
  std::string o = "{\"topo\":" + jints(g.topo_order()) + ",\"strategies\":[";
  for (int s = 0; s < g.strategy_count(); ++s) {
    if (s) o += ",";
    try {
      deduce_graph(g, s);
      o += "{\"ok\":1,\"slots\":[";
      for (const auto& t : g.tensors())
        o += std::string(t.id ? "," : "") + (t.slots.at(s) ? jstr(t.slots.at(s)->str()) : "null");
      o += "]}";
    } catch (const Error& e) {
      o += "{\"ok\":0,\"error\":" + jstr(errc_name(e.code())) + "}";
    }
  }
  return o + "]}";
}

// S|strategy|bindings|program: the reference's node_phases, instantiate_all
// and construct_pipelines (specialize.cpp:31-270) on a deduced strategy.
std::string cmd_specialize(const std::vector<std::string>& f, const std::string& line) {
  const int strategy = std::stoi(f.at(1));
  std::map<std::string, int64_t> bind;
  for (const auto& kv : split(f.at(2), ','))
    if (!trim(kv).empty()) bind[trim(split(kv, '=').at(0))] = std::stoll(split(kv, '=').at(1));
  const size_t at = line.find('|', line.find('|', line.find('|') + 1) + 1);
  CompGraph g = parse_program(line.substr(at + 1));
  deduce_graph(g, strategy);
  std::string o = "{\"phases\":{";
  bool first = true;
  for (const auto& [id, ph] : node_phases(g, strategy)) {
    o += std::string(first ? "" : ",") + "\"" + std::to_string(id) + "\":" + jstr(exec_phase_name(ph));
    first = false;
  }
  o += "},\"exec_graphs\":[";
  const auto egs = instantiate_all(g, strategy, bind);
  for (size_t i = 0; i < egs.size(); ++i) {
    o += std::string(i ? "," : "") + "{\"device\":" + std::to_string(egs[i].device) + ",\"nodes\":[";
    for (size_t k = 0; k < egs[i].nodes.size(); ++k) {
      const auto& n = egs[i].nodes[k];
      o += std::string(k ? "," : "") + "{\"node\":" + std::to_string(n.node_id) + ",\"comm\":" +
           (n.is_comm ? "1" : "0") + ",\"phase\":" + jstr(exec_phase_name(n.phase)) + ",\"plan\":" +
           (n.plan ? jplan(*n.plan, dtype_name(n.plan->dtype)) : std::string("null")) + "}";
    }
    o += "]}";
  }
  o += "]";
  try {
    const auto pipes = construct_pipelines(g, strategy, bind);
    o += ",\"pipelines\":[";
    for (size_t p = 0; p < pipes.size(); ++p) {
      o += p ? ",[" : "[";
      for (size_t st = 0; st < pipes[p].stages.size(); ++st) o += std::string(st ? "," : "") + jints(pipes[p].stages[st]);
      o += "]";
    }
    o += "]";
  } catch (const Error& e) {
    o += ",\"pipelines_error\":" + jstr(errc_name(e.code()));
  }
  return o + "}";
}

std::string handle(const std::string& line, std::istream& in) {
  auto f = split(line, '|');
  const std::string& c = f.at(0);
  if (c == "C") {
    DType dt = parse_dtype(f.at(1));
    auto plan = classify(parse_anno(f.at(4)), parse_anno(f.at(5)), parse_shape(f.at(2)), dt,
                         parse_bw(f.at(3)));
    return jplan(plan, dtype_name(dt));
  }
  if (c == "T") {
    auto t = build_table(parse_anno(f.at(4)), parse_anno(f.at(5)), parse_shape(f.at(2)),
                         std::stoi(f.at(3)), std::stoi(f.at(1)));
    return jtable(t);
  }
  if (c == "M") {
    Bandwidth bw = parse_bw(f.at(1));
    bool naive = f.at(2) == "1";
    auto t = build_table(parse_anno(f.at(5)), parse_anno(f.at(6)), parse_shape(f.at(4)), 0,
                         std::stoi(f.at(3)));
    return jbsr(naive ? make_plan_naive(t) : make_plan(t, bw));
  }
  if (c == "F") {
    Bandwidth bw = parse_bw(f.at(1));
    int n = std::stoi(f.at(2));
    std::vector<BsrTable> tables;
    std::vector<std::string> lines(n);
    for (int i = 0; i < n; ++i) std::getline(in, lines[i]);
    for (int i = 0; i < n; ++i) {
      auto g = split(lines[i], '|');
      tables.push_back(build_table(parse_anno(g.at(3)), parse_anno(g.at(4)), parse_shape(g.at(2)),
                                   std::stoi(g.at(0)), std::stoi(g.at(1))));
    }
    return jbsr(fuse(tables, bw));
  }
  if (c == "R") {  // R|bw|n|d:node,d:node,...  + n lines tid|elem_bytes|shape|src|dst
    Bandwidth bw = parse_bw(f.at(1));
    int n = std::stoi(f.at(2));
    std::map<DeviceId, int> node_of;
    for (auto& kv : split(trim(f.at(3)), ','))
      if (!trim(kv).empty()) node_of[std::stoi(split(kv, ':').at(0))] = std::stoi(split(kv, ':').at(1));
    std::vector<BsrTable> tables;
    std::vector<std::string> lines(n);
    for (int i = 0; i < n; ++i) std::getline(in, lines[i]);
    for (int i = 0; i < n; ++i) {
      auto g = split(lines[i], '|');
      tables.push_back(build_table(parse_anno(g.at(3)), parse_anno(g.at(4)), parse_shape(g.at(2)),
                                   std::stoi(g.at(0)), std::stoi(g.at(1))));
    }
    std::string o = "{";
    bool first = true;
    for (const auto& [d, v] : volume_report(fuse(tables, bw), node_of)) {
      o += std::string(first ? "" : ",") + "\"" + std::to_string(d) + "\":[" + std::to_string(v.intra_bytes) +
           "," + std::to_string(v.inter_bytes) + "]";
      first = false;
    }
    return o + "}";
  }
  if (c == "P") {
    Shape shape = parse_shape(f.at(1));
    HetAnnotation a = parse_anno(f.at(2));
    std::vector<DeviceId> devs = a.all_devices();
    std::sort(devs.begin(), devs.end());
    std::string o = "{";
    for (size_t i = 0; i < devs.size(); ++i) {
      if (i) o += ",";
      o += "\"" + std::to_string(devs[i]) + "\":" + jstr(placement(a, shape, devs[i]).str());
    }
    return o + "}";
  }
  if (c == "H") return jstr(convert_hsize(parse_anno(f.at(1)), std::stoi(f.at(2))).str());
  if (c == "Q") return annotations_equal(parse_anno(f.at(1)), parse_anno(f.at(2))) ? "true" : "false";
  if (c == "A") {
    auto r = align_shard_specs(parse_ds(f.at(1)), parse_ds(f.at(2)));
    if (!r) return "null";
    std::string o = "[";
    for (size_t i = 0; i < r->size(); ++i) {
      if (i) o += ",";
      o += "[" + std::to_string((*r)[i].key_a) + "," + std::to_string((*r)[i].key_b) + "," +
           std::to_string((*r)[i].count) + "]";
    }
    return o + "]";
  }
  if (c == "V") {
    auto issues = validate(parse_anno(f.at(2)), parse_shape(f.at(1)));
    std::string o = "[";
    for (size_t i = 0; i < issues.size(); ++i) {
      if (i) o += ",";
      o += jstr(errc_name(issues[i].code));
    }
    return o + "]";
  }
  if (c == "X") return cmd_execute(f);
  if (c == "N") return cmd_native(f);
  if (c == "W") return cmd_native_switch(f, in);
  if (c == "G") return cmd_graph(line.substr(2));
  if (c == "S") return cmd_specialize(f, line);
  return "{\"error\":\"UnknownCommand\"}";
}

}  // namespace

int main() {
  std::ios::sync_with_stdio(false);
  std::string line;
  while (std::getline(std::cin, line)) {
    if (trim(line).empty()) continue;
    std::string out;
    try {
      out = handle(line, std::cin);
    } catch (const Error& e) {
      out = "{\"error\":" + jstr(errc_name(e.code())) + "}";
    } catch (const std::exception& e) {
      out = "{\"error\":\"Exception\",\"what\":" + jstr(e.what()) + "}";
    }
    std::cout << out << "\n";
    std::cout.flush();
  }
  return 0;
}
