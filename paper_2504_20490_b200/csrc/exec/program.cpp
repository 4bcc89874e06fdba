// hshard-b200 executor: plan -> box tasks -> (fusion, output merging) -> device tables.
//
// Lowering restates the executor semantics the reference specifies but never
// implements (checked against
// oracle/executor.py):
//   Identity / SendRecv / Bsr / AllGather pieces -> copy tasks
//   AllReduce / ReduceScatter -> per member: sum over the group, ascending id
//   Split collectives -> per (slice, receiver): sum of contributors whose
//     bottom partial ordinal p_c satisfies p_c mod P_r == p_r, ascending id;
//     zero-fill when none does.
// Every task is checked at compile time: a step whose members cannot produce
// the target box (the reference's align_shard_specs defect)
// throws Errc::UnexecutableStep instead of producing garbage.
//
// Two rewrites then cut HBM traffic without changing a single result bit:
//   * phase fusion: a phase-2 task that reads the intermediate (mid) shards
//     is split along the boxes of the phase-1 tasks that produced them and
//     reads their inputs directly, as a grouped sum that rounds each
//     phase-1 group exactly where the materialised mid would have;
//   * output merging: tasks with identical inputs (replicas, SplitAG fan-out)
//     become one task with several outputs, so inputs are read once.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <numeric>
#include <set>
#include <sstream>
#include <tuple>
#include <unordered_map>

#include "hshard_c.h"
#include "nccl_dyn.hpp"
#include "planner_internal.hpp"
#include "program.hpp"

namespace hshard::exec {

namespace {

constexpr int64_t kItemBytes = 64 * 1024;     // register path, output bytes per item
constexpr int64_t kTmaItemBytes = 32 * 1024;  // TMA path upper bound (also <= stage / nterms)
constexpr int kBlocksPerSm = 2;

// Host-side item geometry of one TMA task (TmaTask minus the record fields).
struct TmaGeom {
  int32_t task, mode, per, cpr;
  int64_t count;
};
constexpr int kSlots = 9;
// HS_PROG_BULK_STORE: a copy's outputs stored by TMA bulk stores (the rest from
// registers, so the TMA unit still has room for the loads feeding the stages)
constexpr int kBulkStoreOutputs = 2;

// A task's inputs -- phase, tensor, (rank), box, terms, groups -- as raw words:
// tasks with equal keys compute the same values (output merging, sharing).
std::string input_key(const BoxTask& t, bool with_rank) {
  std::string k;
  k.reserve(64 + 16 * t.box.bounds.size() + 8 * (t.terms.size() + t.groups.size()));
  auto put = [&k](int64_t v) { k.append(reinterpret_cast<const char*>(&v), sizeof v); };
  put(t.phase);
  put(t.tensor);
  put(with_rank ? t.rank : -1);
  put(static_cast<int64_t>(t.box.bounds.size()));
  for (const auto& b : t.box.bounds) {
    put(b[0]);
    put(b[1]);
  }
  put(static_cast<int64_t>(t.terms.size()));
  for (const Operand& o : t.terms) put((static_cast<int64_t>(o.state) << 32) | static_cast<uint32_t>(o.dev));
  for (int g : t.groups) put(g);
  return k;
}

SliceRegion bounds_only(const SliceRegion& r) {
  SliceRegion b;
  b.bounds = r.bounds;
  return b;
}

std::vector<int64_t> row_major_strides(const Shape& ext) {
  std::vector<int64_t> s(ext.size(), 1);
  for (int i = static_cast<int>(ext.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * ext[i + 1];
  return s;
}

int64_t cells_of(const SliceRegion& r) { return r.cells(); }

}  // namespace

ShardLoc& Program::loc(int state, int tensor, DeviceId d) {
  const bool dense = tensor >= 0 && tensor < n_tensors_ && d >= 0 && d < n_virt_;
  const size_t slot = dense ? static_cast<size_t>(tensor) * n_virt_ + d : 0;
  if (dense && static_cast<size_t>(state) < dense_.size() && !dense_[state].empty())
    if (ShardLoc* p = dense_[state][slot]) return *p;
  auto it = states_[state].find({tensor, d});
  if (it == states_[state].end())
    fail(Errc::MissingShard, "no shard for tensor slot " + std::to_string(tensor) + " on device " +
                                 std::to_string(d));
  if (dense) {
    if (dense_.size() <= static_cast<size_t>(state)) dense_.resize(state + 1);
    if (dense_[state].empty()) dense_[state].assign(static_cast<size_t>(n_tensors_) * n_virt_, nullptr);
    dense_[state][slot] = &it->second;
  }
  return it->second;
}

Program::Program(Context& ctx, const CommPlan* comm, const SwitchPlan* sw,
                 const std::vector<int>& v_to_rank, const size_t* src_off, const size_t* dst_off,
                 int flags, const void* const* src_ptr, const void* const* dst_ptr)
    : ctx_(ctx), flags_(flags), n_virt_(static_cast<int>(v_to_rank.size())), v_to_rank_(v_to_rank) {
  if (!comm == !sw) fail(Errc::UnsupportedOp, "program needs exactly one plan");
  if (!ctx_.peers_open()) fail(Errc::CommError, "open peers before compiling");
  for (int r : v_to_rank_)
    if (r < 0 || r >= ctx_.world()) fail(Errc::UnknownDevice, "virtual device mapped to bad rank");
  const DType dt = comm ? comm->dtype : sw->dtype;
  dtype_ = static_cast<int>(dt);
  es_ = dtype_width(dt);

  std::vector<std::pair<const HetAnnotation*, const HetAnnotation*>> annos;
  if (comm) {
    shapes_.push_back(comm->shape);
    annos.emplace_back(&comm->src, &comm->dst);
  } else {
    for (const SwitchEntry& e : sw->diff) {
      shapes_.push_back(e.shape);
      annos.emplace_back(&e.src, &e.dst);
    }
  }
  n_tensors_ = static_cast<int>(shapes_.size());
  const bool has_mid = comm && comm->mid.has_value();
  states_.resize(has_mid ? 3 : 2);
  mid_state_ = has_mid ? 1 : -1;
  final_state_ = states_.size() - 1;

  const bool ptr_mode = src_ptr || dst_ptr;
  if (ptr_mode && (flags_ & HS_PROG_CE_RELAY))
    fail(Errc::UnsupportedOp, "copy-engine relays need arena shards");
  // placements per distinct (annotation, shape): a model's parameters repeat a
  // few layouts, and placements() validates the annotation each time
  std::unordered_map<std::string, std::map<DeviceId, SliceRegion>> placed;
  auto placements_of = [&](const HetAnnotation& a, const Shape& shape) -> const std::map<DeviceId, SliceRegion>& {
    std::string key = a.str();
    key += '@';
    key += join_ints(shape);
    auto it = placed.find(key);
    if (it == placed.end()) it = placed.emplace(std::move(key), placements(a, shape)).first;
    return it->second;
  };
  auto add_state = [&](int state, int t, const HetAnnotation& a, const size_t* offs,
                       const void* const* ptrs = nullptr) {
    for (const auto& [d, reg] : placements_of(a, shapes_[t])) {
      if (d < 0 || d >= n_virt_)
        fail(Errc::UnknownDevice, "device " + std::to_string(d) + " has no rank mapping");
      ShardLoc L;
      L.region = reg;
      L.rank = v_to_rank_[d];
      L.offset = offs ? offs[static_cast<size_t>(t) * n_virt_ + d] : SIZE_MAX;
      if (ptrs) {
        L.ptr = static_cast<char*>(const_cast<void*>(ptrs[static_cast<size_t>(t) * n_virt_ + d]));
        L.offset = SIZE_MAX;
      }
      // Every rank's arena has the same size: a caller-supplied offset must
      // leave room for the whole shard (hs_fill_shard / hs_ctx_read check the same).
      if (L.offset != SIZE_MAX) {
        const size_t bytes = static_cast<size_t>(reg.cells()) * static_cast<size_t>(es_);
        if (L.offset > ctx_.arena_bytes() || bytes > ctx_.arena_bytes() - L.offset)
          fail(Errc::ShapeMismatch, "shard of device " + std::to_string(d) + " at offset " +
                                        std::to_string(L.offset) + " (" + std::to_string(bytes) +
                                        " bytes) exceeds the arena");
      }
      L.subgroup = a.subgroup_of(d);
      L.eff_hdim = a.effective_hdim();
      auto& m = states_[state];  // keys arrive in ascending (tensor, device) order
      m.insert_or_assign(m.end(), std::pair<int, DeviceId>{t, d}, L);
    }
  };
  for (int t = 0; t < n_tensors_; ++t) {
    add_state(0, t, *annos[t].first, ptr_mode ? nullptr : src_off, src_ptr);
    add_state(static_cast<int>(states_.size()) - 1, t, *annos[t].second, ptr_mode ? nullptr : dst_off, dst_ptr);
  }
  if (has_mid) add_state(1, 0, *comm->mid, nullptr);
  clock_.mark("placements");

  for (const auto& [key, L] : states_[0])
    if (L.rank == ctx_.rank() && present(L)) {
      host_src_.emplace_back(key.second, key.first, ctx_.is_analysis() ? nullptr : addr_of(L),
                             L.region.cells() * es_);
      stats_.src_bytes += L.region.cells() * es_;
    }
  for (const auto& [key, L] : states_.back())
    if (L.rank == ctx_.rank() && present(L)) {
      host_dst_.emplace_back(key.second, key.first, ctx_.is_analysis() ? nullptr : addr_of(L),
                             L.region.cells() * es_);
      stats_.dst_bytes += L.region.cells() * es_;
    }
  lower(comm, sw);
}

Program::~Program() {
  if (dev_block_) {
    cudaDeviceSynchronize();  // no launch may still read the tables
    pool_->free(dev_block_);  // (the context itself may already be gone)
  }
  for (cudaEvent_t e : host_ev_)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : ce_events_) cudaEventDestroy(e);
  if (ce_stream_) cudaStreamDestroy(ce_stream_);
  if (ce_dev_) cudaFree(ce_dev_);
  for (cudaEvent_t e : events_) cudaEventDestroy(e);
}

void Program::set_profiling(bool on) {
  profiling_ = on;
  events_used_ = 0;
}

int Program::phase_ms(double* out, int n) {
  for (int p = 0; p < n; ++p) out[p] = 0;
  const size_t per_run = 2 * static_cast<size_t>(n_phases_);
  if (per_run == 0) return 0;
  const int runs = static_cast<int>(events_used_ / per_run);
  for (int r = 0; r < runs; ++r)
    for (int p = 0; p < n_phases_ && p < n; ++p) {
      float ms = 0;
      cudaEvent_t a = events_[r * per_run + 2 * p], b = events_[r * per_run + 2 * p + 1];
      cuda_check(cudaEventSynchronize(b), "event sync");
      cuda_check(cudaEventElapsedTime(&ms, a, b), "event elapsed");
      out[p] += ms;
    }
  return runs;
}

// ---------------------------------------------------------------- lowering
void Program::lower(const CommPlan* comm, const SwitchPlan* sw) {
  std::vector<BoxTask> tasks;
  auto covered = [this](int state, int t, DeviceId d, const SliceRegion& box, const char* why) {
    const ShardLoc& L = loc(state, t, d);
    if (!L.region.covers(box))
      fail(Errc::UnexecutableStep, std::string(why) + ": device " + std::to_string(d) + " holds " +
                                       L.region.str() + ", needs " + box.str());
  };
  auto emit = [&](int phase, StepKind kind, int t, int tgt, DeviceId dd, const SliceRegion& box,
                  int src, const std::vector<DeviceId>& from, const char* why) {
    BoxTask task;
    task.phase = phase;
    task.kind = kind;
    task.tensor = t;
    task.box = bounds_only(box);
    covered(tgt, t, dd, task.box, why);
    task.dsts.push_back({tgt, dd});
    task.rank = loc(tgt, t, dd).rank;
    for (DeviceId m : from) {
      covered(src, t, m, task.box, why);
      task.terms.push_back({src, m});
    }
    // Zero-width top-tier slices give empty boxes: no work.
    if (cells_of(task.box) == 0) return;
    tasks.push_back(std::move(task));
  };
  auto region_of = [this](int state, DeviceId d) { return loc(state, 0, d).region; };

  auto lower_step = [&](const CommStep& step, const HetAnnotation& phase_src, int src, int tgt,
                        int phase) {
    switch (step.kind) {
      case StepKind::Identity:
        for (DeviceId d : phase_src.dg_union.at(step.subgroup).devices)
          emit(phase, step.kind, 0, tgt, d, region_of(src, d), src, {d}, "Identity");
        break;
      case StepKind::SendRecv:
        for (const auto& [s, r] : step.pairs) {
          const SliceRegion a = bounds_only(region_of(src, s)), b = bounds_only(region_of(tgt, r));
          if (a.bounds != b.bounds) fail(Errc::UnexecutableStep, "SendRecv shard boxes differ");
          emit(phase, step.kind, 0, tgt, r, b, src, {s}, "SendRecv");
        }
        break;
      case StepKind::AllReduce:
      case StepKind::ReduceScatter:
        for (const auto& grp : step.groups) {
          std::vector<DeviceId> order(grp.begin(), grp.end());
          std::sort(order.begin(), order.end());
          for (DeviceId d : grp)
            emit(phase, step.kind, 0, tgt, d, region_of(tgt, d), src, order, step_kind_name(step.kind));
        }
        break;
      case StepKind::AllGather:
        for (const auto& grp : step.groups)
          for (DeviceId d : grp) {
            const SliceRegion want = bounds_only(region_of(tgt, d));
            std::vector<SliceRegion> pieces;
            int64_t got = 0;
            for (DeviceId m : grp) {
              auto isect = intersect(region_of(src, m), want);
              if (!isect) continue;
              for (const SliceRegion& p : pieces)
                if (intersect(p, *isect))
                  fail(Errc::UnexecutableStep, "AllGather members overlap on " + isect->str());
              pieces.push_back(*isect);
              got += isect->cells();
              emit(phase, step.kind, 0, tgt, d, *isect, src, {m}, "AllGather");
            }
            if (got != want.cells())
              fail(Errc::UnexecutableStep, "AllGather group cannot assemble " + want.str() +
                                               " on device " + std::to_string(d));
          }
        break;
      case StepKind::SplitAllReduce:
      case StepKind::SplitReduceScatter:
      case StepKind::SplitAllGather:
        for (const SliceCollective& sc : step.slices) {
          std::vector<DeviceId> cs(sc.contributors.begin(), sc.contributors.end());
          std::sort(cs.begin(), cs.end());
          for (DeviceId r : sc.receivers) {
            const SliceRegion& rr = region_of(tgt, r);
            std::vector<DeviceId> from;
            for (DeviceId c : cs)
              if (region_of(src, c).partial_index % rr.partial_count == rr.partial_index)
                from.push_back(c);
            emit(phase, step.kind, 0, tgt, r, sc.region, src, from, step_kind_name(step.kind));
          }
        }
        break;
      case StepKind::Bsr: {
        const BsrPlan& b = *step.bsr;
        for (const LocalCopy& c : b.local_copies)
          emit(phase, step.kind, 0, tgt, c.device, c.region, src, {c.device}, "Bsr local");
        for (const FusionGroup& g : b.fusion_groups)
          for (int i : g.transfer_indices) {
            const Transfer& t = b.transfers[i];
            emit(phase, step.kind, 0, tgt, t.receiver, t.region, src, {t.sender}, "Bsr");
          }
        break;
      }
    }
  };

  if (comm) {
    int cur = 0;
    const HetAnnotation* cur_anno = &comm->src;
    const int last = static_cast<int>(states_.size()) - 1;
    int phase = 0;
    if (!comm->bottom_phase.empty()) {
      const int tgt = comm->mid ? 1 : last;
      for (const CommStep& s : comm->bottom_phase) lower_step(s, *cur_anno, cur, tgt, phase);
      cur = tgt;
      cur_anno = comm->mid ? &*comm->mid : &comm->dst;
      ++phase;
    }
    if (!comm->top_phase.empty()) {
      for (const CommStep& s : comm->top_phase) lower_step(s, *cur_anno, cur, last, phase);
      ++phase;
    }
    n_phases_ = phase;
  } else {
    std::map<int, int> slot;
    for (int t = 0; t < n_tensors_; ++t) slot[sw->diff[t].tensor_id] = t;
    auto slot_of = [&](int tid) {
      auto it = slot.find(tid);
      if (it == slot.end()) fail(Errc::MissingShard, "plan names unknown tensor " + std::to_string(tid));
      return it->second;
    };
    for (const LocalCopy& c : sw->plan.local_copies)
      emit(0, StepKind::Bsr, slot_of(c.tensor_id), 1, c.device, c.region, 0, {c.device}, "switch local");
    for (const FusionGroup& g : sw->plan.fusion_groups)
      for (int i : g.transfer_indices) {
        const Transfer& t = sw->plan.transfers[i];
        emit(0, StepKind::Bsr, slot_of(t.tensor_id), 1, t.receiver, t.region, 0, {t.sender}, "switch");
      }
    n_phases_ = 1;
  }
  stats_.plan_phases = n_phases_;
  clock_.mark("lowering");

  // ---- rewrites (results are bit-identical by construction; see header)
  nccl_mode_ = ctx_.world() > 1 && (flags_ & HS_PROG_NCCL);
  if (nccl_mode_) {
    // baseline transport: plain pulls, no peer stores (the rewrites below
    // that store into peers are off); remote inputs are staged in stage_for_nccl()
    if (!ctx_.nccl_comm() && !ctx_.is_analysis()) fail(Errc::CommError, "HS_PROG_NCCL needs hs_ctx_nccl_init first");
    flags_ |= HS_PROG_NO_RELAY | HS_PROG_NO_SHARE | HS_PROG_PULL_COPIES;
    flags_ &= ~(HS_PROG_PUSH_ALL | HS_PROG_FUSE_PHASES);
  }
  ce_mode_ = ctx_.world() > 1 && (flags_ & HS_PROG_CE_RELAY) && !nccl_mode_;
  if (ce_mode_) {
    // producers run where their mid box lives; nothing else stores remotely
    flags_ |= HS_PROG_NO_SHARE | HS_PROG_PULL_COPIES;
    flags_ &= ~(HS_PROG_PUSH_ALL | HS_PROG_FUSE_PHASES | HS_PROG_PULL_MID | HS_PROG_NO_RELAY | HS_PROG_SPLIT_RELAY);
    if (const char* e = std::getenv("HS_CE_CHUNKS")) ce_chunks_ = std::max(1, std::atoi(e));
  }
  if (ctx_.world() > 1 && !(flags_ & HS_PROG_NO_REPLICA)) choose_replicas(tasks);
  clock_.mark("rewrites:replicas");
  const bool two_phase = mid_state_ >= 0 && n_phases_ == 2 && !(flags_ & HS_PROG_NO_FUSE);
  auto rank_of = [this](const Operand& o, int t) { return loc(o.state, t, o.dev).rank; };
  // Cross-rank rewrites (world > 1), each behind a flag because which wins
  // depends on the plan's balance (executor.autotune() times the variants):
  //   share -- identical tasks on several ranks become per-rank chunks;
  //   push  -- single-output copies run on the rank holding the input.
  //   push-all -- every copy runs on the input's rank, even one that stores
  //               to several outputs (moves work off busy receivers).
  auto finish = [&](std::vector<BoxTask> ts) {
    if (ctx_.world() > 1 && !(flags_ & HS_PROG_NO_SHARE)) ts = spread_shared(std::move(ts));
    clock_.mark("rewrites:share");
    if (ctx_.world() > 1 && (flags_ & HS_PROG_PUSH_ALL))
      for (BoxTask& t : ts)
        if (t.terms.size() == 1) {
          const int src = rank_of(t.terms[0], t.tensor);
          if (src != t.rank) {
            t.rank = src;
            stats_.pushed_copies += 1;
          }
        }
    if (!(flags_ & HS_PROG_NO_MERGE)) ts = merge_outputs(std::move(ts));
    if (ctx_.world() > 1 && !(flags_ & HS_PROG_PULL_COPIES))
      for (BoxTask& t : ts)
        if (t.terms.size() == 1 && t.dsts.size() == 1) {
          const int src = rank_of(t.terms[0], t.tensor);
          if (src != t.rank) {
            t.rank = src;
            stats_.pushed_copies += 1;
          }
        }
    return ts;
  };
  if (two_phase && (ctx_.world() == 1 || (flags_ & HS_PROG_FUSE_PHASES))) {
    // world 1: fuse everything fusable (HS_PROG_FUSE_PHASES forces it at
    // world > 1, pulling raw inputs over NVLink)
    tasks = finish(fuse_phases(std::move(tasks), RelayMode::None));
  } else if (two_phase && !(flags_ & HS_PROG_NO_RELAY)) {
    // world > 1: relays for remote mid reads.  A task that waits for a relay
    // fuses its local groups too (least HBM traffic) unless
    // HS_PROG_RELAY_KEEP_LOCAL asks to compute them before the barrier,
    // concurrently with the remote producers.
    const RelayMode mode = (flags_ & HS_PROG_SPLIT_RELAY)        ? RelayMode::Split
                           : (flags_ & HS_PROG_PULL_MID)           ? RelayMode::Pull
                           : (flags_ & HS_PROG_RELAY_KEEP_LOCAL) ? RelayMode::KeepLocal
                                                                 : RelayMode::FuseLocal;
    tasks = finish(fuse_phases(std::move(tasks), mode));
    stats_.model_ms[0] = estimate_seconds(tasks, n_phases_) * 1e3;
    if (ce_mode_) tasks = ce_relay(std::move(tasks));
  } else {
    tasks = finish(std::move(tasks));
  }

  if (ctx_.world() > 1 && (flags_ & HS_PROG_FANOUT_ONCE) && !nccl_mode_ && !ce_mode_)
    tasks = fanout_once(std::move(tasks));
  if (nccl_mode_) stage_for_nccl(tasks);
  if (ce_mode_ && ce_copies_.empty()) ce_mode_ = false;  // no relay to move
  clock_.mark("rewrites");

  // world > 1: both plan phases in one launch with per-chunk ready flags
  // (kept only if every producer / consumer piece runs on the TMA path).
  std::vector<BoxTask> unstreamed;
  if (ctx_.world() > 1 && n_phases_ == 2 && !nccl_mode_ && !(flags_ & (HS_PROG_NO_STREAM | HS_PROG_NO_TMA))) {
    std::vector<BoxTask> st = stream_phases(tasks);
    if (!st.empty()) {
      unstreamed = std::move(tasks);
      tasks = std::move(st);
      streamed_ = true;
    }
  }

  // Symmetric placement of the intermediate (mid) and relay shards still in
  // use: every rank packs its own densely from one common base.
  if (mid_state_ >= 0) {
    std::set<std::pair<int, DeviceId>> used_keys;  // (state, dev)
    for (const BoxTask& t : tasks)
      for (const auto* ops : {&t.dsts, &t.terms})
        for (const Operand& o : *ops)
          if (o.state >= mid_state_ && o.state != static_cast<int>(final_state_) &&
              o.state < staging_state_)
            used_keys.insert({o.state, o.dev});
    if (!used_keys.empty()) {
      std::vector<size_t> used(ctx_.world(), 0);
      for (const auto& [st, dev] : used_keys) {
        ShardLoc& L = states_[st].at({0, dev});
        size_t& u = used[L.rank];
        u = (u + 255) & ~size_t{255};
        L.offset = u;
        u += static_cast<size_t>(L.region.cells()) * es_;
      }
      const size_t base = ctx_.alloc(*std::max_element(used.begin(), used.end()) + 256);
      for (const auto& [st, dev] : used_keys) states_[st].at({0, dev}).offset += base;
    }
  }

  if (streamed_) {
    bool ok = true;
    for (const BoxTask& t : tasks)
      if ((t.wait >= 0 || !t.targets.empty()) && !tma_capable(t)) ok = false;
    if (!ok) {
      tasks = std::move(unstreamed);
      streamed_ = false;
    } else {
      n_phases_ = 1;
      // symmetric flag array (same offset on every rank), zeroed before the
      // first run's opening barrier
      std::vector<int> nflags(ctx_.world(), 0);
      for (const BoxTask& t : tasks)
        if (t.wait >= 0) nflags[t.rank] = std::max(nflags[t.rank], t.wait + 1);
      const size_t bytes = static_cast<size_t>(*std::max_element(nflags.begin(), nflags.end())) * 4;
      flag_off_ = ctx_.alloc(bytes + 256);
      if (!ctx_.is_analysis()) {
        cuda_check(cudaMemsetAsync(ctx_.arena() + flag_off_, 0, bytes + 256, ctx_.stream()), "memset(flags)");
        cuda_check(cudaStreamSynchronize(ctx_.stream()), "memset(flags) sync");
      }
    }
  }
  stats_.streamed = streamed_;
  if (ce_mode_) {
    // copy geometry (mid box on the sender == relay box on the receiver, same
    // region layout) and the symmetric chunk flag words
    ce_geometry();
    const size_t bytes = static_cast<size_t>(ctx_.world()) * ce_chunks_ * 4;
    ce_flag_off_ = ctx_.alloc(bytes + 256);
    if (!ctx_.is_analysis()) {
      cuda_check(cudaMemsetAsync(ctx_.arena() + ce_flag_off_, 0, bytes + 256, ctx_.stream()), "memset(ce flags)");
      cuda_check(cudaStreamSynchronize(ctx_.stream()), "memset(ce flags) sync");
    }
  }
  stats_.ce_relay = ce_mode_;

  // Stores into peers' destination shards in the last launch need a closing
  // barrier (relay / intermediate stores are consumed inside the run).
  for (const BoxTask& t : tasks)
    if (t.phase == n_phases_ - 1 || ce_mode_)
      for (const Operand& o : t.dsts)
        remote_final_writes_ = remote_final_writes_ ||
                               (o.state == static_cast<int>(final_state_) && rank_of(o, t.tensor) != t.rank);

  // The host-buffer path copies in only the source shards some task (on any
  // rank) reads: replicas the program never sources from (replica choice,
  // fusion) stay on the host -- cfg2e reads 6 of its 8 partials.
  {
    std::set<std::pair<int, DeviceId>> read;
    for (const BoxTask& t : tasks)
      for (const Operand& o : t.terms)
        if (o.state == 0) read.insert({t.tensor, o.dev});
    std::vector<std::tuple<DeviceId, int, char*, size_t>> kept;
    for (const auto& h : host_src_)
      if (read.count({std::get<1>(h), std::get<0>(h)})) kept.push_back(h);
    stats_.h2d_bytes = 0;
    for (const auto& h : kept) stats_.h2d_bytes += static_cast<int64_t>(std::get<3>(h));
    host_src_ = std::move(kept);
  }

  // ---- algorithmic byte accounting over ALL ranks' tasks, then keep ours
  const int me = ctx_.rank();
  std::vector<BoxTask> mine;
  stats_.phase_bytes.assign(n_phases_, {0, 0, 0});
  // My kernels: local reads / local writes / NVLink (remote reads + remote
  // stores) per phase.  Per GPU: nvlink_in = bytes arriving (my remote reads
  // + peers' stores into me), nvlink_out = bytes leaving.
  for (BoxTask& t : tasks) {
    const int64_t bytes = cells_of(t.box) * es_;
    const bool mine_task = t.rank == me;
    auto& pb = stats_.phase_bytes[t.phase];
    for (const Operand& o : t.terms) {
      const int r = rank_of(o, t.tensor);
      if (mine_task && r == me) {
        stats_.hbm_read += bytes;
        pb[0] += bytes;
      } else if (mine_task) {
        stats_.nvlink_in += bytes;
        pb[2] += bytes;
      } else if (r == me) {
        stats_.nvlink_out += bytes;
      }
    }
    for (const Operand& o : t.dsts) {
      const int r = rank_of(o, t.tensor);
      if (mine_task && r == me) {
        stats_.hbm_write += bytes;
        pb[1] += bytes;
      } else if (mine_task) {
        stats_.nvlink_out += bytes;
        pb[2] += bytes;
      } else if (r == me) {
        stats_.nvlink_in += bytes;
      }
    }
    if (mine_task) mine.push_back(std::move(t));
  }
  for (const CeCopy& c : ce_copies_) {
    const int64_t b = static_cast<int64_t>(c.width * c.height * c.planes);
    if (c.sender == me) stats_.nvlink_out += b;
    if (c.receiver == me) stats_.nvlink_in += b;
  }
  if (ctx_.is_analysis()) analysed_ = mine;
  clock_.mark("accounting");
  for (const BoxTask& t : mine) {
    for (const Operand& o : t.dsts)
      if (!present(loc(o.state, t.tensor, o.dev)))
        fail(Errc::MissingShard, "destination shard of device " + std::to_string(o.dev) + " has no buffer");
    for (const Operand& o : t.terms)
      if (!present(loc(o.state, t.tensor, o.dev)))
        fail(Errc::MissingShard, "source shard of device " + std::to_string(o.dev) + " has no buffer");
  }
  build_tables(mine);
  clock_.mark("tables");
  if (ce_mode_ && !ctx_.is_analysis()) ce_build();
}

// ---------------------------------------------------------------- replicas
// A term may be read from any device holding the SAME VALUES on its box: the
// same bottom partial piece, the same top-tier piece (subgroup, when the top
// tier is Partial), and -- when that piece is a partial (P > 1) -- the same
// subgroup, since subgroups of an hdim -1 annotation may decompose the value
// differently.  Duplicate replicas of a valid state are bit-identical
// (reassemble's precondition), so results do not change
// (SURVEY App. B7).  Policy: a replica on the executing rank if any, else the
// one whose rank has served the fewest bytes so far.
void Program::choose_replicas(std::vector<BoxTask>& tasks) {
  std::vector<int64_t> egress(ctx_.world(), 0);
  for (BoxTask& t : tasks) {
    const int64_t bytes = t.box.cells() * es_;
    for (Operand& o : t.terms) {
      const ShardLoc& cur = loc(o.state, t.tensor, o.dev);
      if (cur.rank == t.rank) continue;
      DeviceId best = o.dev;
      int best_rank = cur.rank;
      // the state's shards of this tensor only (keys are ordered (tensor, device))
      const auto& st = states_[o.state];
      for (auto it = st.lower_bound({t.tensor, std::numeric_limits<DeviceId>::min()});
           it != st.end() && it->first.first == t.tensor; ++it) {
        const auto& [key, L] = *it;
        if (key.second == o.dev) continue;
        const bool same = L.region.covers(t.box) &&
                          L.region.partial_index == cur.region.partial_index &&
                          L.region.partial_count == cur.region.partial_count &&
                          (cur.eff_hdim != kPartial || L.subgroup == cur.subgroup) &&
                          (cur.region.partial_count == 1 || L.subgroup == cur.subgroup);
        if (!same) continue;
        const bool better = (L.rank == t.rank && best_rank != t.rank) ||
                            (best_rank != t.rank && L.rank != t.rank && egress[L.rank] < egress[best_rank]);
        if (better) {
          best = key.second;
          best_rank = L.rank;
        }
      }
      if (best != o.dev) {
        o.dev = best;
        stats_.replica_swaps += 1;
      }
      if (best_rank != t.rank) egress[best_rank] += bytes;
    }
  }
}

// ---------------------------------------------------------------- fusion / relays
// Per phase-2 term reading an intermediate (mid) shard c:
//   FUSE  -- read the phase-1 producers' inputs directly (grouped, rounded
//            where mid would have been); needs every input on this rank at
//            world > 1 so fusion never adds NVLink traffic;
//   RELAY -- (world > 1, c on another rank) the phase-1 producers also store
//            their result straight into a relay copy of c in this rank's HBM
//            (a remote store from the reducing kernel: transfer and reduction
//            overlap), and the phase-2 term reads it locally;
//   KEEP  -- read the materialised mid shard.
std::vector<BoxTask> Program::fuse_phases(std::vector<BoxTask> tasks, RelayMode mode) {
  const bool relay = mode != RelayMode::None;
  enum Policy { FUSE, KEEP, RELAY };
  auto rank_of = [this](const Operand& o, int t) { return loc(o.state, t, o.dev).rank; };
  std::map<DeviceId, std::vector<int>> producers;
  for (int i = 0; i < static_cast<int>(tasks.size()); ++i)
    if (tasks[i].phase == 0 && tasks[i].dsts.size() == 1 && tasks[i].dsts[0].state == mid_state_)
      producers[tasks[i].dsts[0].dev].push_back(i);

  int relay_state = -1;
  auto relay_operand = [&](DeviceId c, int q) {
    if (relay_state < 0) {
      relay_state = static_cast<int>(states_.size());
      states_.emplace_back();
    }
    const DeviceId id = c * ctx_.world() + q;
    auto& m = states_[relay_state];
    if (!m.count({0, id})) {
      ShardLoc L = loc(mid_state_, 0, c);
      L.rank = q;
      L.offset = SIZE_MAX;
      m[{0, id}] = L;
    }
    return Operand{relay_state, id};
  };

  // Split: the boxes of each kept producer that some consumer actually reads
  // locally (the other rows go out as relays only).
  const bool split = mode == RelayMode::Split;
  int64_t split_64ths = 32;  // share of the rows relayed (exploration knob)
  if (const char* e = std::getenv("HS_SPLIT_RELAY_64THS")) split_64ths = std::clamp(std::atol(e), 1L, 63L);
  std::vector<std::vector<SliceRegion>> keep_at(tasks.size());
  std::vector<BoxTask> out;
  std::vector<char> keep_local(tasks.size(), 0);
  // producer -> consumer rank -> boxes that rank actually reads
  std::vector<std::map<int, std::vector<SliceRegion>>> relay_to(tasks.size());
  bool any_unfused = false;

  for (int i = 0; i < static_cast<int>(tasks.size()); ++i) {
    const BoxTask& T = tasks[i];
    if (T.phase != 1) continue;
    if (T.terms.empty()) {  // zero-fill reads nothing
      out.push_back(T);
      continue;
    }
    const int q = T.rank;
    const size_t nt = T.terms.size();
    std::vector<Policy> pol(nt, KEEP);
    std::vector<std::vector<int>> prod(nt);
    for (size_t j = 0; j < nt; ++j) {
      const Operand& o = T.terms[j];
      if (o.state != mid_state_ || !T.groups.empty()) continue;
      bool fusable = true;
      for (int p : producers[o.dev])
        if (intersect(tasks[p].box, T.box)) {
          prod[j].push_back(p);
          fusable = fusable && !tasks[p].terms.empty() && tasks[p].groups.empty();
          if (relay)
            for (const Operand& in : tasks[p].terms) fusable = fusable && rank_of(in, T.tensor) == q;
        }
      if (relay && rank_of(o, T.tensor) != q)
        pol[j] = mode == RelayMode::Pull ? KEEP : RELAY;
      else if (fusable && !prod[j].empty())
        pol[j] = FUSE;
    }
    // world > 1: a task that waits for a relay anyway keeps its local groups
    // in phase 1's producers (they run concurrently with the remote ones)
    // instead of redoing them after the barrier.
    bool needs_relay = false;
    for (Policy p : pol) needs_relay = needs_relay || p == RELAY;
    // Split: rows [lo, band) of the task read relays, rows [band, hi) pull.
    const int64_t row_lo = T.box.bounds.empty() ? 0 : T.box.bounds[0][0];
    const int64_t row_hi = T.box.bounds.empty() ? 0 : T.box.bounds[0][1];
    const int64_t band = split && needs_relay && row_hi - row_lo >= 2
                             ? std::clamp(row_lo + (row_hi - row_lo) * split_64ths / 64, row_lo + 1, row_hi - 1)
                             : row_hi;
    auto band_box = [&](bool first) {
      SliceRegion b = T.box;
      b.bounds[0] = first ? std::array<int64_t, 2>{row_lo, band} : std::array<int64_t, 2>{band, row_hi};
      return b;
    };
    if (mode == RelayMode::KeepLocal && needs_relay)
      for (Policy& p : pol)
        if (p == FUSE) p = KEEP;
    auto build = [&](std::vector<BoxTask>& cells) {
      detail::Cuts cuts(T.box.bounds.size());
      for (size_t d = 0; d < cuts.size(); ++d) {
        const int64_t lo = T.box.bounds[d][0], hi = T.box.bounds[d][1];
        std::set<int64_t> s{lo, hi};
        for (size_t j = 0; j < nt; ++j)
          if (pol[j] == FUSE)
            for (int p : prod[j])
              for (int64_t v : tasks[p].box.bounds[d])
                if (lo < v && v < hi) s.insert(v);
        if (d == 0 && band < row_hi) s.insert(band);
        cuts[d].assign(s.begin(), s.end());
      }
      bool ok = true;
      detail::for_each_grid_cell(cuts, [&](const SliceRegion& cell) {
        if (!ok) return;
        BoxTask N = T;
        N.box = cell;
        N.terms.clear();
        N.groups.clear();
        bool nested = false;
        for (size_t j = 0; j < nt; ++j) {
          if (pol[j] == FUSE) {
            const BoxTask* src = nullptr;
            for (int p : prod[j])
              if (tasks[p].box.covers(cell)) src = &tasks[p];
            if (!src) {
              ok = false;
              return;
            }
            N.terms.insert(N.terms.end(), src->terms.begin(), src->terms.end());
            N.groups.push_back(static_cast<int>(src->terms.size()));
            nested = nested || src->terms.size() > 1;
          } else {
            const bool relayed = pol[j] == RELAY && (cell.bounds.empty() || cell.bounds[0][0] < band);
            N.terms.push_back(relayed ? relay_operand(T.terms[j].dev, q) : T.terms[j]);
            N.groups.push_back(1);
          }
        }
        if (!nested) N.groups.clear();
        if (N.terms.size() > static_cast<size_t>(kMaxTerms) || N.groups.size() > 16) ok = false;
        cells.push_back(std::move(N));
      });
      return ok;
    };
    std::vector<BoxTask> cells;
    if (!build(cells)) {  // too many terms: stop fusing this task
      for (Policy& p : pol)
        if (p == FUSE) p = KEEP;
      cells.clear();
      build(cells);
    }
    for (size_t j = 0; j < nt; ++j) {
      if (pol[j] == FUSE) continue;
      any_unfused = true;
      if (T.terms[j].state != mid_state_) continue;
      for (int p : producers[T.terms[j].dev]) {
        if (pol[j] != RELAY) {
          keep_local[p] = 1;
          if (auto need = intersect(tasks[p].box, T.box)) keep_at[p].push_back(*need);
        } else if (band < row_hi) {  // split: first band relayed, second kept for the pull
          if (auto need = intersect(tasks[p].box, band_box(true))) relay_to[p][q].push_back(*need);
          if (auto need = intersect(tasks[p].box, band_box(false))) {
            keep_local[p] = 1;
            keep_at[p].push_back(*need);
          }
        } else if (auto need = intersect(tasks[p].box, T.box)) {
          relay_to[p][q].push_back(*need);
        }
      }
    }
    bool fused_any = false, all_fused = true;
    for (Policy p : pol) {
      fused_any = fused_any || p == FUSE;
      all_fused = all_fused && p == FUSE;
    }
    if (fused_any) stats_.fused_tasks += static_cast<int64_t>(cells.size());
    // A fully fused task reads only phase-1 inputs: at world > 1 it runs in
    // phase 1 (before the barrier) alongside the producers.
    if (relay && all_fused)
      for (BoxTask& c : cells) c.phase = 0;
    for (BoxTask& c : cells) out.push_back(std::move(c));
  }
  std::vector<BoxTask> result;
  for (int i = 0; i < static_cast<int>(tasks.size()); ++i) {
    if (tasks[i].phase != 0) continue;
    const BoxTask& P = tasks[i];
    const bool is_producer = P.dsts.size() == 1 && P.dsts[0].state == mid_state_;
    if (!is_producer || relay_to[i].empty()) {
      if (!is_producer || keep_local[i]) result.push_back(P);
      continue;
    }
    // Split the producer along the boxes remote consumers read, so each
    // piece is stored exactly where it is consumed (and locally if needed).
    const DeviceId c = P.dsts[0].dev;
    detail::Cuts cuts(P.box.bounds.size());
    for (size_t d = 0; d < cuts.size(); ++d) {
      const int64_t lo = P.box.bounds[d][0], hi = P.box.bounds[d][1];
      std::set<int64_t> s{lo, hi};
      for (const auto& [q, boxes] : relay_to[i])
        for (const SliceRegion& b : boxes)
          for (int64_t v : b.bounds[d])
            if (lo < v && v < hi) s.insert(v);
      if (split)
        for (const SliceRegion& b : keep_at[i])
          for (int64_t v : b.bounds[d])
            if (lo < v && v < hi) s.insert(v);
      cuts[d].assign(s.begin(), s.end());
    }
    detail::for_each_grid_cell(cuts, [&](const SliceRegion& cell) {
      BoxTask piece = P;
      piece.box = cell;
      piece.dsts.clear();
      bool local = keep_local[i];
      if (split && local) {  // only the rows some consumer reads from the local mid
        local = false;
        for (const SliceRegion& b : keep_at[i]) local = local || b.covers(cell);
      }
      if (local) piece.dsts.push_back(P.dsts[0]);
      for (const auto& [q, boxes] : relay_to[i]) {
        bool read = false;
        for (const SliceRegion& b : boxes) read = read || b.covers(cell);
        if (read) {
          piece.dsts.push_back(relay_operand(c, q));
          stats_.relay_outputs += 1;
        }
      }
      if (!piece.dsts.empty()) result.push_back(std::move(piece));
    });
  }
  for (BoxTask& t : out) result.push_back(std::move(t));
  bool any_late = false;
  for (const BoxTask& t : result) any_late = any_late || t.phase == 1;
  if (!any_unfused || !any_late) {  // one phase left: one launch, no barrier between
    for (BoxTask& t : result) t.phase = 0;
    n_phases_ = 1;
  }
  return result;
}

// ---------------------------------------------------------------- NCCL baseline
// HS_PROG_NCCL: every remote input of every task is first copied (a local
// "pack" task on the owner) into a per-(phase, sender, receiver) message,
// the messages of a phase go out as one ncclGroupStart / ncclSend x peers /
// ncclRecv x peers / ncclGroupEnd, and the task reads its input from the
// receive buffer.  Plan phase p becomes launched phases 2p (pack) and 2p+1
// (compute).  This is the NCCL-carried executor the peer-memory kernels are
// measured against.
void Program::stage_for_nccl(std::vector<BoxTask>& tasks) {
  const int W = ctx_.world();
  const int P = n_phases_;
  staging_state_ = static_cast<int>(states_.size());
  const int send_state = staging_state_, recv_state = staging_state_ + 1;
  states_.emplace_back();
  states_.emplace_back();
  struct Chunk {
    int phase, src, dst, tensor;
    size_t off;
    DeviceId id;
  };
  std::vector<Chunk> chunks;
  std::vector<std::map<std::pair<int, int>, size_t>> msg(P);  // (src, dst) -> bytes
  std::vector<BoxTask> packs;
  DeviceId next = 0;
  for (BoxTask& t : tasks) {
    for (Operand& o : t.terms) {
      const ShardLoc& L = loc(o.state, t.tensor, o.dev);
      if (L.rank == t.rank) continue;
      size_t& u = msg[t.phase][{L.rank, t.rank}];
      u = (u + 255) & ~size_t{255};
      const size_t off = u;
      u += static_cast<size_t>(t.box.cells()) * es_;
      const DeviceId id = next++;
      ShardLoc S;
      S.region = t.box;
      S.rank = L.rank;
      states_[send_state][{t.tensor, id}] = S;
      S.rank = t.rank;
      states_[recv_state][{t.tensor, id}] = S;
      BoxTask pack;
      pack.phase = t.phase;
      pack.kind = t.kind;
      pack.tensor = t.tensor;
      pack.box = t.box;
      pack.rank = L.rank;
      pack.dsts = {Operand{send_state, id}};
      pack.terms = {o};
      packs.push_back(std::move(pack));
      chunks.push_back({t.phase, L.rank, t.rank, t.tensor, off, id});
      o = Operand{recv_state, id};
    }
  }
  // Message layout: every rank's send area ordered by (phase, receiver), its
  // receive area by (phase, sender); both sides agree on chunk offsets.
  std::vector<std::map<std::pair<int, int>, size_t>> send_at(W), recv_at(W);
  std::vector<size_t> send_total(W, 0), recv_total(W, 0);
  for (int p = 0; p < P; ++p)
    for (const auto& [pair, bytes] : msg[p]) {
      send_at[pair.first][{p, pair.second}] = send_total[pair.first];
      send_total[pair.first] += (bytes + 255) & ~size_t{255};
      recv_at[pair.second][{p, pair.first}] = recv_total[pair.second];
      recv_total[pair.second] += (bytes + 255) & ~size_t{255};
    }
  const size_t send_base = ctx_.alloc(*std::max_element(send_total.begin(), send_total.end()) + 256);
  const size_t recv_base = ctx_.alloc(*std::max_element(recv_total.begin(), recv_total.end()) + 256);
  for (const Chunk& c : chunks) {
    states_[send_state][{c.tensor, c.id}].offset = send_base + send_at[c.src][{c.phase, c.dst}] + c.off;
    states_[recv_state][{c.tensor, c.id}].offset = recv_base + recv_at[c.dst][{c.phase, c.src}] + c.off;
  }
  const int me = ctx_.rank();
  exchanges_.assign(P, {});
  for (int p = 0; p < P; ++p)
    for (const auto& [pair, bytes] : msg[p]) {
      if (pair.first == me) {
        exchanges_[p].push_back({pair.second, true, send_base + send_at[me][{p, pair.second}], bytes});
        stats_.nvlink_out += static_cast<int64_t>(bytes);
      }
      if (pair.second == me) {
        exchanges_[p].push_back({pair.first, false, recv_base + recv_at[me][{p, pair.first}], bytes});
        stats_.nvlink_in += static_cast<int64_t>(bytes);
      }
    }
  for (BoxTask& t : tasks) t.phase = 2 * t.phase + 1;
  for (BoxTask& t : packs) t.phase = 2 * t.phase;
  tasks.insert(tasks.end(), std::make_move_iterator(packs.begin()), std::make_move_iterator(packs.end()));
  n_phases_ = 2 * P;
}

// ---------------------------------------------------------------- cost model
// Seconds for a task list: per phase, the slowest rank's max of HBM bytes /
// 6.3 TB/s, NVLink-in / 0.7 TB/s and NVLink-out / 0.7 TB/s (peer reads are
// served by the owner's HBM and leave through its links), plus one barrier
// per phase.  Only used to choose between equivalent rewrites.
double Program::estimate_seconds(const std::vector<BoxTask>& tasks, int phases) {
  struct Load {
    double hbm = 0, in = 0, out = 0;
  };
  const int W = ctx_.world();
  std::vector<std::vector<Load>> load(phases, std::vector<Load>(W));
  for (const BoxTask& t : tasks) {
    const double bytes = static_cast<double>(t.box.cells()) * es_;
    auto& L = load.at(t.phase);
    const int r = t.rank;
    for (const Operand& o : t.terms) {
      const int ro = loc(o.state, t.tensor, o.dev).rank;
      L[ro].hbm += bytes;
      if (ro != r) {
        L[r].in += bytes;
        L[ro].out += bytes;
      }
    }
    for (const Operand& o : t.dsts) {
      const int ro = loc(o.state, t.tensor, o.dev).rank;
      L[ro].hbm += bytes;
      if (ro != r) {
        L[r].out += bytes;
        L[ro].in += bytes;
      }
    }
  }
  double total = 0;
  for (const auto& per : load) {
    double worst = 0;
    for (const Load& l : per) worst = std::max({worst, l.hbm / 6.3e12, l.in / 7.0e11, l.out / 7.0e11});
    total += worst + 8e-6;
  }
  return total;
}

// ---------------------------------------------------------------- cross-rank sharing
// world > 1: tasks that compute the same values (same phase, tensor, box,
// inputs, groups) on several ranks -- AllReduce members, SplitAllReduce /
// SplitAllGather receivers, replicas of one shard -- are cut into one chunk
// per rank along the box's outermost splittable dim; each rank computes its
// chunk once and stores it to every output (local or over NVLink).  A
// reduce-scatter + all-gather, with the inputs of each chunk read once.
std::vector<BoxTask> Program::spread_shared(std::vector<BoxTask> tasks) {
  std::unordered_map<std::string, std::vector<int>> same;
  std::vector<std::string> order;
  same.reserve(tasks.size() * 2);
  for (int i = 0; i < static_cast<int>(tasks.size()); ++i) {
    std::string k = input_key(tasks[i], false);
    auto [it, fresh] = same.try_emplace(k);
    if (fresh) order.push_back(std::move(k));
    it->second.push_back(i);
  }
  std::vector<BoxTask> out;
  out.reserve(tasks.size());
  for (const std::string& key : order) {
    const std::vector<int>& idx = same.find(key)->second;
    std::set<int> ranks;
    std::vector<Operand> dsts;
    for (int i : idx) {
      ranks.insert(tasks[i].rank);
      for (const Operand& o : tasks[i].dsts)
        if (std::find(dsts.begin(), dsts.end(), o) == dsts.end()) dsts.push_back(o);
    }
    const BoxTask& T = tasks[idx.front()];
    int split = -1;
    for (size_t d = 0; d < T.box.bounds.size() && split < 0; ++d)
      if (T.box.bounds[d][1] - T.box.bounds[d][0] >= static_cast<int64_t>(ranks.size())) split = static_cast<int>(d);
    const bool worth = ranks.size() >= 2 && split >= 0;
    if (!worth || dsts.size() > static_cast<size_t>(kMaxOuts) || T.terms.empty()) {
      for (int i : idx) out.push_back(std::move(tasks[i]));
      continue;
    }
    const int64_t lo = T.box.bounds[split][0], ext = T.box.bounds[split][1] - lo;
    const int R = static_cast<int>(ranks.size());
    int c = 0;
    for (int r : ranks) {
      BoxTask chunk = T;
      chunk.rank = r;
      chunk.dsts = dsts;
      chunk.box.bounds[split] = {lo + ext * c / R, lo + ext * (c + 1) / R};
      ++c;
      stats_.shared_chunks += 1;
      out.push_back(std::move(chunk));
    }
  }
  return out;
}

// ---------------------------------------------------------------- output merging
std::vector<BoxTask> Program::merge_outputs(std::vector<BoxTask> tasks) {
  std::unordered_map<std::string, int> index;
  index.reserve(tasks.size() * 2);
  std::vector<BoxTask> out;
  out.reserve(tasks.size());
  for (BoxTask& t : tasks) {
    const std::string k = input_key(t, true);
    auto it = index.find(k);
    if (it != index.end() && out[it->second].dsts.size() < static_cast<size_t>(kMaxOuts)) {
      BoxTask& m = out[it->second];
      m.dsts.insert(m.dsts.end(), t.dsts.begin(), t.dsts.end());
      continue;
    }
    index[k] = static_cast<int>(out.size());
    out.push_back(std::move(t));
  }
  return out;
}

// ---------------------------------------------------------------- fan-out once
// HS_PROG_FANOUT_ONCE: a last-phase task that stores its result into several
// destination shards on the same remote rank keeps one of those stores; the
// remote rank copies that shard's box into the others in a new last phase
// (streamed like any phase-1 consumer when it applies).  NVLink carries each
// result once per GPU instead of once per virtual device.
std::vector<BoxTask> Program::fanout_once(std::vector<BoxTask> tasks) {
  const int last = n_phases_ - 1;
  std::vector<BoxTask> copies;
  for (BoxTask& t : tasks) {
    if (t.phase != last) continue;
    std::map<int, std::vector<Operand>> remote;
    for (const Operand& o : t.dsts) {
      const int r = loc(o.state, t.tensor, o.dev).rank;
      if (r != t.rank && o.state == static_cast<int>(final_state_)) remote[r].push_back(o);
    }
    std::set<Operand> dropped;
    for (const auto& [r, os] : remote) {
      if (os.size() < 2) continue;
      BoxTask c;
      c.phase = last + 1;
      c.kind = t.kind;
      c.tensor = t.tensor;
      c.rank = r;
      c.box = t.box;
      c.terms = {os[0]};
      c.dsts.assign(os.begin() + 1, os.end());
      dropped.insert(os.begin() + 1, os.end());
      copies.push_back(std::move(c));
    }
    if (!dropped.empty())
      t.dsts.erase(std::remove_if(t.dsts.begin(), t.dsts.end(), [&](const Operand& o) { return dropped.count(o) > 0; }),
                   t.dsts.end());
  }
  if (copies.empty()) return tasks;
  n_phases_ = last + 2;
  for (BoxTask& c : copies) tasks.push_back(std::move(c));
  return tasks;
}

// ---------------------------------------------------------------- copy-engine relays
// HS_PROG_CE_RELAY: an SM moves only ~5-6 GB/s over NVLink (loads or stores),
// so NVLink-bound and HBM-bound work compete for SMs; the copy engines move
// 650+ GB/s with no SM and no HBM-rate loss (measured, tools/ce_probe.py).
// Relay producers therefore write their result into their own mid box, in K
// row chunks (one launch each); after chunk k the rank's copy stream copies
// it into every consumer's relay buffer (2-D DMA from the same offsets) and
// signals the consumer; the consumers of chunk k wait for that signal.  The
// phases become: [0, K) producer chunks, K the other phase-1 work (runs while
// the DMA moves), K+1+k consumers of chunk k, 2K+1 the other phase-2 work.
std::vector<BoxTask> Program::ce_relay(std::vector<BoxTask> tasks) {
  const int W = ctx_.world(), K = ce_chunks_;
  auto is_relay = [&](int st) { return st > static_cast<int>(final_state_) && st < staging_state_; };
  bool any = false;
  for (const BoxTask& t : tasks)
    for (const Operand& o : t.dsts) any = any || is_relay(o.state);
  if (!any) return tasks;
  const int64_t rows = shapes_.at(0).at(0);
  std::vector<int64_t> cut(K + 1);
  for (int k = 0; k <= K; ++k) cut[k] = rows * k / K;
  std::vector<BoxTask> out;
  for (BoxTask& t : tasks) {
    bool prod = false, cons = false;
    for (const Operand& o : t.dsts) prod = prod || is_relay(o.state);
    for (const Operand& o : t.terms) cons = cons || is_relay(o.state);
    if (!prod && !cons) {
      t.phase = t.phase == 0 ? K : 2 * K + 1;
      out.push_back(std::move(t));
      continue;
    }
    const int64_t lo = t.box.bounds[0][0], hi = t.box.bounds[0][1];
    for (int64_t a = lo; a < hi;) {
      const int k = static_cast<int>(std::upper_bound(cut.begin(), cut.end(), a) - cut.begin()) - 1;
      const int64_t b = std::min(hi, cut[k + 1]);
      BoxTask piece = t;
      piece.box.bounds[0] = {a, b};
      if (prod) {
        std::vector<Operand> dsts;
        for (const Operand& o : t.dsts) {
          if (!is_relay(o.state)) {
            dsts.push_back(o);
            continue;
          }
          const DeviceId c = o.dev / W;
          const int q = static_cast<int>(o.dev % W);
          const Operand mid{mid_state_, c};
          if (loc(mid_state_, 0, c).rank != piece.rank)
            fail(Errc::UnsupportedOp, "copy-engine relay: producer not on its mid box's rank");
          if (std::find(dsts.begin(), dsts.end(), mid) == dsts.end()) dsts.push_back(mid);
          CeCopy cp{};
          cp.chunk = k;
          cp.sender = piece.rank;
          cp.receiver = q;
          // geometry: filled once offsets exist (ce_geometry below); keep the
          // operands in the offsets for now
          cp.src_off = static_cast<size_t>(c);
          cp.dst_off = static_cast<size_t>(o.dev);
          cp.planes = static_cast<size_t>(o.state);
          ce_boxes_.push_back(piece.box);
          ce_mid_dev_.push_back(c);
          ce_relay_dev_.push_back(o.dev);
          ce_copies_.push_back(cp);
        }
        piece.dsts = std::move(dsts);
        piece.phase = k;
      } else {
        piece.phase = K + 1 + k;
      }
      out.push_back(std::move(piece));
      a = b;
    }
  }
  n_phases_ = 2 * K + 2;
  return out;
}

void Program::ce_geometry() {
  for (size_t i = 0; i < ce_copies_.size(); ++i) {
    CeCopy& c = ce_copies_[i];
    const DeviceId mid_dev = static_cast<DeviceId>(c.src_off), relay_dev = static_cast<DeviceId>(c.dst_off);
    const int relay_state = static_cast<int>(c.planes);
    const ShardLoc& S = loc(mid_state_, 0, mid_dev);
    const ShardLoc& D = loc(relay_state, 0, relay_dev);
    const SliceRegion& box = ce_boxes_[i];
    const std::vector<int64_t> st = row_major_strides(S.region.extents());
    int64_t off = 0;
    for (size_t d = 0; d < box.bounds.size(); ++d) off += (box.bounds[d][0] - S.region.bounds[d][0]) * st[d];
    // merge dims contiguous in the region, drop unit outer dims
    std::vector<int64_t> ext, str;
    const Shape e = box.extents();
    for (size_t d = 0; d < e.size(); ++d) {
      if (e[d] == 1 && d + 1 < e.size()) continue;
      if (!ext.empty() && str.back() == e[d] * st[d]) {
        ext.back() *= e[d];
        str.back() = st[d];
        continue;
      }
      ext.push_back(e[d]);
      str.push_back(st[d]);
    }
    if (ext.size() > 3) fail(Errc::UnsupportedOp, "copy-engine relay of a box with more than 3 strided dims");
    while (ext.size() < 3) {
      ext.insert(ext.begin(), 1);
      str.insert(str.begin(), 0);
    }
    c.planes = static_cast<size_t>(ext[0]);
    c.plane_stride = static_cast<size_t>(str[0] * es_);
    c.height = static_cast<size_t>(ext[1]);
    c.pitch = static_cast<size_t>((ext[1] > 1 ? str[1] : ext[2]) * es_);
    c.width = static_cast<size_t>(ext[2] * es_);
    c.src_off = S.offset + static_cast<size_t>(off * es_);
    c.dst_off = D.offset + static_cast<size_t>(off * es_);
  }
}

void Program::ce_build() {
  const int me = ctx_.rank(), K = ce_chunks_;
  std::vector<std::set<int>> to(K), from(K);
  for (const CeCopy& c : ce_copies_) {
    if (c.sender == me) to[c.chunk].insert(c.receiver);
    if (c.receiver == me) from[c.chunk].insert(c.sender);
  }
  auto word = [&](int rank, int sender, int k) {
    return reinterpret_cast<unsigned int*>(ctx_.arena_of(rank) + ce_flag_off_) + sender * K + k;
  };
  std::vector<unsigned int*> host;
  std::vector<size_t> t0(K), w0(K);
  ce_ntargets_.assign(K, 0);
  ce_nwaits_.assign(K, 0);
  for (int k = 0; k < K; ++k) {
    t0[k] = host.size();
    for (int q : to[k]) host.push_back(word(q, me, k));
    ce_ntargets_[k] = static_cast<int>(to[k].size());
    w0[k] = host.size();
    for (int p : from[k]) host.push_back(word(me, p, k));
    ce_nwaits_[k] = static_cast<int>(from[k].size());
  }
  cuda_check(cudaMalloc(&ce_dev_, std::max<size_t>(1, host.size()) * sizeof(unsigned int*)), "cudaMalloc(ce)");
  cuda_check(cudaMemcpy(ce_dev_, host.data(), host.size() * sizeof(unsigned int*), cudaMemcpyHostToDevice),
             "cudaMemcpy(ce)");
  auto* base = static_cast<unsigned int**>(ce_dev_);
  ce_targets_.resize(K);
  ce_waits_.resize(K);
  for (int k = 0; k < K; ++k) {
    ce_targets_[k] = base + t0[k];
    ce_waits_[k] = const_cast<const unsigned int**>(base + w0[k]);
  }
  cuda_check(cudaStreamCreateWithFlags(&ce_stream_, cudaStreamNonBlocking), "cudaStreamCreate(ce)");
  ce_events_.resize(K);
  for (cudaEvent_t& e : ce_events_) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event(ce)");
  int signals = 0, waits = 0;
  for (int k = 0; k < K; ++k) {
    signals += ce_ntargets_[k] > 0;
    waits += ce_nwaits_[k] > 0;
  }
  stats_.kernels_per_run += signals + waits - n_phases_ + 1;  // one barrier per run, not one per phase
}

void Program::ce_run_phase_post(int k, cudaStream_t s) {
  const int me = ctx_.rank();
  if (!ce_ntargets_[k]) return;
  cuda_check(cudaEventRecord(ce_events_[k], s), "event record(ce)");
  cuda_check(cudaStreamWaitEvent(ce_stream_, ce_events_[k], 0), "stream wait(ce)");
  for (const CeCopy& c : ce_copies_) {
    if (c.sender != me || c.chunk != k) continue;
    for (size_t p = 0; p < c.planes; ++p)
      cuda_check(cudaMemcpy2DAsync(ctx_.arena_of(c.receiver) + c.dst_off + p * c.plane_stride, c.pitch,
                                   ctx_.arena() + c.src_off + p * c.plane_stride, c.pitch, c.width, c.height,
                                   cudaMemcpyDeviceToDevice, ce_stream_),
                 "copy-engine relay");
  }
  cuda_check(launch_signal(ce_targets_[k], ce_ntargets_[k], runs_, ce_stream_), "signal launch");
}

// ---------------------------------------------------------------- streaming
// world > 1, two plan phases: ONE launch instead of phase / barrier / phase.
// Producer tasks (phase 0, an output a phase-1 task reads) and their consumers
// are cut along dim 0 at common multiples of ~kChunkBytes of the operand's
// rows.  Every consumer piece gets a ready flag on its rank; each producer
// piece it reads adds 1 to that flag once per run when its last item has
// landed (kernels.cuh SigDesc), and the consumer's loads wait for
// epoch * need.  Results are unchanged: the same tasks, cut, run in the same
// order of terms.  Returns {} when no phase-1 task reads a phase-0 output.
std::vector<BoxTask> Program::stream_phases(const std::vector<BoxTask>& in) {
  using Key = std::tuple<int, int, DeviceId>;  // (state, tensor, device)
  auto key = [](const BoxTask& t, const Operand& o) { return Key{o.state, t.tensor, o.dev}; };
  int64_t chunk_bytes = 2 << 20;
  if (const char* e = std::getenv("HS_STREAM_CHUNK_KB")) chunk_bytes = std::max(1L, std::atol(e)) << 10;

  std::map<Key, std::vector<int>> writers;
  for (int i = 0; i < static_cast<int>(in.size()); ++i)
    if (in[i].phase == 0)
      for (const Operand& o : in[i].dsts) writers[key(in[i], o)].push_back(i);
  std::map<Key, int64_t> rows;  // chunk rows of each operand read across the phases
  std::vector<int64_t> cut_rows(in.size(), 0);
  auto note = [&](int i, const Key& k) {
    auto [it, fresh] = rows.try_emplace(k, 0);
    if (fresh) {
      const ShardLoc& L = loc(std::get<0>(k), std::get<1>(k), std::get<2>(k));
      int64_t row_bytes = es_;
      for (size_t d = 1; d < L.region.bounds.size(); ++d) row_bytes *= L.region.bounds[d][1] - L.region.bounds[d][0];
      it->second = std::max<int64_t>(1, chunk_bytes / row_bytes);
    }
    cut_rows[i] = cut_rows[i] ? std::min(cut_rows[i], it->second) : it->second;
  };
  bool any = false;
  for (int i = 0; i < static_cast<int>(in.size()); ++i) {
    if (in[i].phase != 1) continue;
    for (const Operand& o : in[i].terms) {
      auto it = writers.find(key(in[i], o));
      if (it == writers.end()) continue;
      for (int p : it->second)
        if (intersect(in[p].box, in[i].box)) {
          note(i, it->first);
          note(p, it->first);
          any = true;
        }
    }
  }
  if (!any) return {};

  std::vector<BoxTask> out;
  for (int i = 0; i < static_cast<int>(in.size()); ++i) {
    const BoxTask& T = in[i];
    const int64_t R = cut_rows[i];
    const int64_t lo = T.box.bounds[0][0], hi = T.box.bounds[0][1];
    if (!R || hi - lo <= R) {
      out.push_back(T);
      continue;
    }
    for (int64_t a = lo; a < hi;) {
      const int64_t b = std::min(hi, (a / R + 1) * R);
      BoxTask piece = T;
      piece.box.bounds[0] = {a, b};
      out.push_back(std::move(piece));
      a = b;
    }
  }
  std::map<Key, std::vector<int>> w2;
  for (int j = 0; j < static_cast<int>(out.size()); ++j)
    if (out[j].phase == 0)
      for (const Operand& o : out[j].dsts) w2[key(out[j], o)].push_back(j);
  std::vector<int> flags(ctx_.world(), 0);
  for (int j = 0; j < static_cast<int>(out.size()); ++j) {
    if (out[j].phase != 1) continue;
    std::set<int> deps;
    for (const Operand& o : out[j].terms) {
      auto it = w2.find(key(out[j], o));
      if (it == w2.end()) continue;
      for (int p : it->second)
        if (intersect(out[p].box, out[j].box)) deps.insert(p);
    }
    if (deps.empty()) continue;
    out[j].wait = flags[out[j].rank]++;
    out[j].need = static_cast<int>(deps.size());
    for (int p : deps) out[p].targets.emplace_back(out[j].rank, out[j].wait);
  }
  for (BoxTask& t : out) t.phase = 0;
  return out;
}

// A task's box with unit outer dims dropped and dims contiguous for every
// operand merged (outputs first, then terms): what the device tables hold.
struct Program::Flat {
  std::vector<int64_t> ext;                // outermost first
  std::vector<std::vector<int64_t>> st;    // per operand: element strides
  std::vector<const ShardLoc*> locs;
  std::vector<int64_t> elem_off;           // per operand: box origin in its shard
  int vec_bytes = 0;                       // widest vector legal for every operand
};

Program::Flat Program::flatten(const BoxTask& bt) {
  Flat f;
  std::vector<std::vector<int64_t>> full;
  auto add = [&](const Operand& o) {
    const ShardLoc& L = loc(o.state, bt.tensor, o.dev);
    full.push_back(row_major_strides(L.region.extents()));
    int64_t off = 0;
    for (size_t i = 0; i < bt.box.bounds.size(); ++i) off += (bt.box.bounds[i][0] - L.region.bounds[i][0]) * full.back()[i];
    f.locs.push_back(&L);
    f.elem_off.push_back(off);
  };
  for (const Operand& o : bt.dsts) add(o);
  for (const Operand& o : bt.terms) add(o);
  const Shape box = bt.box.extents();
  const size_t nd = box.size();
  f.st.resize(full.size());
  for (size_t i = 0; i < nd; ++i) {
    if (box[i] == 1 && i + 1 < nd) continue;  // the innermost (stride-1) dim always stays
    f.ext.push_back(box[i]);
    for (size_t k = 0; k < full.size(); ++k) f.st[k].push_back(full[k][i]);
  }
  for (int i = static_cast<int>(f.ext.size()) - 2; i >= 0; --i) {
    bool merge = true;
    for (size_t k = 0; k < full.size(); ++k) merge = merge && f.st[k][i] == f.ext[i + 1] * f.st[k][i + 1];
    if (!merge) continue;
    f.ext[i] *= f.ext[i + 1];
    f.ext.erase(f.ext.begin() + i + 1);
    for (auto& s : f.st) {
      s[i] = s[i + 1];
      s.erase(s.begin() + i + 1);
    }
  }
  if (f.ext.empty()) {
    f.ext.push_back(1);
    for (auto& s : f.st) s.push_back(1);
  }
  // Alignment from arena offsets (every rank's arena base is 256-byte
  // aligned) or from the caller's buffer addresses.
  const int rd = static_cast<int>(f.ext.size());
  auto ok = [&](int v) {
    if ((f.ext.back() * es_) % v) return false;
    for (size_t k = 0; k < f.locs.size(); ++k) {
      const uint64_t a = f.locs[k]->ptr ? reinterpret_cast<uintptr_t>(f.locs[k]->ptr) : f.locs[k]->offset;
      if ((a + f.elem_off[k] * es_) % v) return false;
      for (int j = 0; j + 1 < rd; ++j)
        if ((f.st[k][j] * es_) % v) return false;
    }
    return true;
  };
  int vb = 16;
  while (vb > es_ && !ok(vb)) vb /= 2;
  f.vec_bytes = std::max(vb, es_);
  return f;
}

bool Program::tma_capable(const BoxTask& bt) { return tma_capable(bt, flatten(bt)); }

bool Program::tma_capable(const BoxTask& bt, const Flat& f) {
  bool all_local = true;
  for (const ShardLoc* L : f.locs) all_local = all_local && L->rank == bt.rank;
  return f.vec_bytes == 16 && (all_local || !(flags_ & HS_PROG_NO_TMA_PEER)) && !(flags_ & HS_PROG_NO_TMA) &&
         f.ext.size() <= 4;
}

// ---------------------------------------------------------------- tables
void Program::build_tables(const std::vector<BoxTask>& tasks) {
  struct Host {
    std::vector<TaskDesc> tasks;
    std::vector<TermDesc> terms;
    std::vector<const BoxTask*> src;  // the BoxTask of each TaskDesc
    // [0] unused (TMA items are decoded from `tma`); [1..4] register copy/zero by
    // width 16, 8, 4, 2; [5..8] register reduce
    std::vector<WorkItem> items[kSlots];
    std::vector<TmaGeom> tma;  // TMA tasks in launch (queue) order
    int64_t tma_items() const {
      int64_t n = 0;
      for (const TmaGeom& g : tma) n += g.count;
      return n;
    }
  };
  auto slot_of = [](int vb, bool tma, bool reduce) {
    return tma ? 0 : (vb == 16 ? 1 : vb == 8 ? 2 : vb == 4 ? 3 : 4) + (reduce ? 4 : 0);
  };
  std::vector<Host> ph(n_phases_);
  stats_.phases = n_phases_;
  clock_.mark("tables:init");

  for (const BoxTask& bt : tasks) {
    Host& H = ph.at(bt.phase);
    if (static_cast<int>(bt.terms.size()) > kMaxTerms) fail(Errc::UnsupportedOp, "more than 16 terms in one task");
    if (static_cast<int>(bt.dsts.size()) > kMaxOuts) fail(Errc::UnsupportedOp, "more than 8 outputs in one task");
    const Flat f = flatten(bt);
    const size_t nout = bt.dsts.size();
    const int rd = static_cast<int>(f.ext.size());
    if (rd > 4) fail(Errc::UnsupportedOp, "box needs more than 4 strided dims");
    for (int64_t e : f.ext)
      if (e > INT32_MAX) fail(Errc::UnsupportedOp, "box dim >= 2^31");
    TaskDesc td{};
    for (int j = 0; j < 4; ++j) td.n[j] = j < rd ? static_cast<int32_t>(f.ext[rd - 1 - j]) : 1;
    const int vb = f.vec_bytes;
    td.vec_bytes = vb;
    td.out0 = static_cast<int32_t>(H.terms.size());
    td.nout = static_cast<int32_t>(nout);
    td.term0 = td.out0 + td.nout;
    td.nterms = static_cast<int32_t>(bt.terms.size());
    td.ngroups = static_cast<int32_t>(bt.groups.size());
    for (size_t g = 0; g < bt.groups.size(); ++g) td.gsize[g] = static_cast<uint8_t>(bt.groups[g]);
    for (size_t k = 0; k < f.locs.size(); ++k) {
      TermDesc tm{};
      tm.base = addr_of(*f.locs[k]) + f.elem_off[k] * es_;
      for (int j = 1; j < 4; ++j) tm.stride[j - 1] = j < rd ? f.st[k][rd - 1 - j] : 0;
      H.terms.push_back(tm);
    }
    const bool tma = tma_capable(bt, f);
    if ((bt.wait >= 0 || !bt.targets.empty()) && !tma)
      fail(Errc::UnsupportedOp, "streamed task is not TMA-capable");  // lower() checks first
    const int32_t task_id = static_cast<int32_t>(H.tasks.size());
    H.tasks.push_back(td);
    H.src.push_back(&bt);
    stats_.tasks += 1;
    stats_.terms += td.nterms;
    stats_.outputs += td.nout;
    (td.nterms == 0 ? stats_.zero_tasks : td.nterms == 1 ? stats_.copy_tasks : stats_.reduce_tasks) += 1;

    // Work items: never crossing a (dim2, dim3) plane; TMA items also fit a
    // pipeline stage (nterms x item bytes <= kStageBytes).
    const int64_t row_vecs = static_cast<int64_t>(td.n[0]) * es_ / vb;
    int64_t item_bytes = kItemBytes;
    if (tma) {
      const int64_t cap = (flags_ & HS_PROG_SMALL_ITEMS) ? kTmaItemBytes / 2 : kTmaItemBytes;
      item_bytes = std::min<int64_t>(cap, kStageBytes / std::max(1, td.nterms));
    }
    const int64_t target = std::max<int64_t>(1, item_bytes / vb);
    const int64_t planes = static_cast<int64_t>(td.n[2]) * td.n[3];
    if (tma) {
      // TMA items are decoded on the device from the task (kernels.cu
      // tma_record): only the geometry is recorded here.
      TmaGeom g{task_id, 0, 0, 0, 0};
      if (row_vecs >= target) {
        g.mode = 0;
        g.per = static_cast<int32_t>(target);
        g.cpr = static_cast<int32_t>((row_vecs + target - 1) / target);
        g.count = planes * td.n[1] * g.cpr;
      } else {
        g.mode = 1;
        g.per = static_cast<int32_t>(std::max<int64_t>(1, target / row_vecs));
        g.cpr = (td.n[1] + g.per - 1) / g.per;
        g.count = planes * g.cpr;
      }
      if (g.count > INT32_MAX) fail(Errc::UnsupportedOp, "more than 2^31 items in one task");
      H.tma.push_back(g);
      continue;
    }
    std::vector<WorkItem>& items = H.items[slot_of(vb, tma, td.nterms >= 2)];
    for (int64_t pl = 0; pl < planes; ++pl) {
      if (row_vecs >= target) {
        for (int32_t r = 0; r < td.n[1]; ++r)
          for (int64_t c = 0; c < row_vecs; c += target)
            items.push_back({task_id, r, 1, static_cast<int32_t>(pl), static_cast<int32_t>(c),
                             static_cast<int32_t>(std::min(target, row_vecs - c))});
      } else {
        const int32_t rows = static_cast<int32_t>(std::max<int64_t>(1, target / row_vecs));
        for (int32_t r = 0; r < td.n[1]; r += rows)
          items.push_back({task_id, r, std::min(rows, td.n[1] - r), static_cast<int32_t>(pl), 0,
                           static_cast<int32_t>(row_vecs)});
      }
    }
  }

  clock_.mark("items");
  // Streamed launches: signalling tasks' SigDescs and flag addresses; TMA
  // items reordered into the two queues (signalling work first, then other
  // non-waiting work; then waiting work), each by the piece's position along
  // dim 0 so consumers follow their producers' progress.
  std::vector<SigDesc> sigs;
  std::vector<unsigned int*> targets;
  std::vector<std::vector<int32_t>> task_sig(n_phases_);
  std::vector<int32_t> n_first(n_phases_, 0);
  std::vector<double> first_frac(n_phases_, 1.0);
  for (int p = 0; p < n_phases_; ++p) {
    Host& H = ph[p];
    task_sig[p].assign(H.tasks.size(), -1);
    if (H.tma_items() > INT32_MAX) fail(Errc::UnsupportedOp, "more than 2^31 TMA items in one launch");
    if (!streamed_) {
      n_first[p] = static_cast<int32_t>(H.tma_items());
      continue;
    }
    for (const TmaGeom& g : H.tma) {
      const BoxTask& bt = *H.src[g.task];
      if (bt.targets.empty() || g.count == 0) continue;
      task_sig[p][g.task] = static_cast<int32_t>(sigs.size());
      sigs.push_back({static_cast<uint32_t>(sigs.size()), static_cast<uint32_t>(g.count),
                      static_cast<uint32_t>(targets.size()), static_cast<uint32_t>(bt.targets.size())});
      for (const auto& [r, flag] : bt.targets)
        targets.push_back(reinterpret_cast<unsigned int*>(ctx_.arena_of(r) + flag_off_) + flag);
    }
    auto rank_key = [&](const TmaGeom& g) {
      const BoxTask& bt = *H.src[g.task];
      const int queue = bt.wait >= 0 ? 2 : bt.targets.empty() ? 1 : 0;
      const double pos = static_cast<double>(bt.box.bounds[0][0]) / std::max<int64_t>(1, shapes_[bt.tensor][0]);
      return std::make_pair(queue, pos);
    };
    // tasks (each a contiguous run of items) into the two queues
    std::stable_sort(H.tma.begin(), H.tma.end(),
                     [&](const TmaGeom& a, const TmaGeom& b) { return rank_key(a) < rank_key(b); });
    // CTAs of the first queue in proportion to its modelled time (HBM bytes
    // at 6.5 TB/s vs NVLink bytes at 0.77 TB/s, whichever binds).
    double hbm[2] = {0, 0}, nv[2] = {0, 0};
    for (size_t k = 0; k < H.tasks.size(); ++k) {
      const BoxTask& bt = *H.src[k];
      const int q = bt.wait >= 0 ? 1 : 0;
      const double bytes = static_cast<double>(bt.box.cells()) * es_;
      for (const auto* ops : {&bt.dsts, &bt.terms})
        for (const Operand& o : *ops) (loc(o.state, bt.tensor, o.dev).rank == bt.rank ? hbm : nv)[q] += bytes;
    }
    for (const TmaGeom& g : H.tma) n_first[p] += H.src[g.task]->wait < 0 ? static_cast<int32_t>(g.count) : 0;
    const double t0 = std::max(hbm[0] / 6.5e12, nv[0] / 7.7e11), t1 = std::max(hbm[1] / 6.5e12, nv[1] / 7.7e11);
    first_frac[p] = t0 + t1 > 0 ? t0 / (t0 + t1) : 1.0;
    if (const int share = (flags_ >> 16) & 0xff) first_frac[p] = share / 64.0;
  }

  clock_.mark("queues");
  // HS_PROG_INTERLEAVE (unstreamed multi-GPU launches): tasks with NVLink
  // operands first, then local-only tasks; the record expansion merges the two
  // item ranges evenly in launch order.
  std::vector<int> interleave(n_phases_, 0);
  if (ctx_.world() > 1 && !streamed_ && (flags_ & HS_PROG_INTERLEAVE))
    for (int p = 0; p < n_phases_; ++p) {
      Host& H = ph[p];
      auto remote = [&](const TmaGeom& g) {
        const BoxTask& bt = *H.src[g.task];
        for (const auto* ops : {&bt.dsts, &bt.terms})
          for (const Operand& o : *ops)
            if (loc(o.state, bt.tensor, o.dev).rank != bt.rank) return true;
        return false;
      };
      std::stable_partition(H.tma.begin(), H.tma.end(), remote);
      int64_t na = 0;
      for (const TmaGeom& g : H.tma) na += remote(g) ? g.count : 0;
      interleave[p] = static_cast<int>(na);
    }

  // TMA task descriptors in item order (+ a sentinel whose item0 is the item
  // count); the producer warp decodes every item's record from them.
  std::vector<std::vector<TmaTask>> ttasks(n_phases_);
  std::vector<int> rec_words(n_phases_, kTmaHeadWords);
  for (int p = 0; p < n_phases_; ++p) {
    const Host& H = ph[p];
    int64_t item0 = 0;
    for (const TmaGeom& g : H.tma) {
      const TaskDesc& td = H.tasks[g.task];
      const BoxTask& bt = *H.src[g.task];
      rec_words[p] = std::max(rec_words[p], kTmaHeadWords + td.nterms + td.nout);
      TmaTask tt{};
      tt.item0 = static_cast<int32_t>(item0);
      tt.nterms = td.nterms;
      tt.nout = td.nout;
      tt.ngroups = td.ngroups;
      tt.wait = bt.wait;
      tt.sig = task_sig[p][g.task];
      tt.need = bt.need;
      tt.mode = g.mode;
      tt.n1 = td.n[1];
      tt.n2 = td.n[2];
      tt.row_vecs = static_cast<int32_t>(static_cast<int64_t>(td.n[0]) * es_ / 16);
      tt.per = g.per;
      tt.cpr = g.cpr;
      tt.term0 = td.term0;
      tt.out0 = td.out0;
      std::memcpy(tt.gsize, td.gsize, sizeof(tt.gsize));
      ttasks[p].push_back(tt);
      item0 += g.count;
    }
    TmaTask sentinel{};
    sentinel.item0 = static_cast<int32_t>(item0);
    ttasks[p].push_back(sentinel);
  }

  clock_.mark("records");
  // One device block for every phase's tables.
  size_t total = 0;
  auto reserve = [&total](size_t bytes) {
    const size_t off = (total + 255) & ~size_t{255};
    total = off + bytes;
    return off;
  };
  struct Offs {
    size_t tasks, terms, items[kSlots], ttasks, recs, sched;
  };
  std::vector<Offs> offs(n_phases_);
  for (int p = 0; p < n_phases_; ++p) {
    offs[p].tasks = reserve(ph[p].tasks.size() * sizeof(TaskDesc));
    offs[p].terms = reserve(ph[p].terms.size() * sizeof(TermDesc));
    for (int v = 0; v < kSlots; ++v) offs[p].items[v] = reserve(ph[p].items[v].size() * sizeof(WorkItem));
    offs[p].ttasks = reserve(ttasks[p].size() * sizeof(TmaTask));
    offs[p].sched = reserve(4 * sizeof(int));  // zero-initialised scheduler words
  }
  const size_t sigs_off = reserve(sigs.size() * sizeof(SigDesc));
  const size_t targets_off = reserve(targets.size() * sizeof(unsigned int*));
  const size_t done_off = reserve(sigs.size() * sizeof(unsigned long long));  // zero: no items done yet
  // The TMA records are written on the device (expanded from the task
  // descriptors below): reserved after everything that is uploaded.
  const size_t upload = total;
  for (int p = 0; p < n_phases_; ++p)
    offs[p].recs = reserve(static_cast<size_t>(ph[p].tma_items()) * rec_words[p] * sizeof(uint4));
  std::vector<char> host(std::max<size_t>(upload, 1));
  for (int p = 0; p < n_phases_; ++p) {
    std::memcpy(host.data() + offs[p].tasks, ph[p].tasks.data(), ph[p].tasks.size() * sizeof(TaskDesc));
    std::memcpy(host.data() + offs[p].terms, ph[p].terms.data(), ph[p].terms.size() * sizeof(TermDesc));
    for (int v = 0; v < kSlots; ++v)
      std::memcpy(host.data() + offs[p].items[v], ph[p].items[v].data(),
                  ph[p].items[v].size() * sizeof(WorkItem));
    std::memcpy(host.data() + offs[p].ttasks, ttasks[p].data(), ttasks[p].size() * sizeof(TmaTask));
  }
  std::memcpy(host.data() + sigs_off, sigs.data(), sigs.size() * sizeof(SigDesc));
  std::memcpy(host.data() + targets_off, targets.data(), targets.size() * sizeof(unsigned int*));
  clock_.mark("pack");
  char* base = nullptr;
  if (!ctx_.is_analysis()) {
    pool_ = ctx_.tables();
    dev_block_ = pool_->alloc(total);
    cuda_check(cudaMemcpy(dev_block_, host.data(), host.size(), cudaMemcpyHostToDevice),
               "cudaMemcpy(tables)");
    base = static_cast<char*>(dev_block_);
  }
  clock_.mark("upload");
  dphases_.assign(n_phases_, {});
  const int max_grid = ctx_.sm_count() * kBlocksPerSm;
  int launches = 0;
  for (int p = 0; p < n_phases_; ++p) {
    DevicePhase& d = dphases_[p];
    int64_t n = 0;
    for (int v = 0; v < kSlots; ++v) {
      const int32_t cnt = static_cast<int32_t>(v == 0 ? ph[p].tma_items() : ph[p].items[v].size());
      n += cnt;
      if (!cnt) continue;
      Launch l;
      l.tables = PhaseTables{};
      l.tables.tasks = reinterpret_cast<TaskDesc*>(base + offs[p].tasks);
      l.tables.terms = reinterpret_cast<TermDesc*>(base + offs[p].terms);
      l.tables.items = reinterpret_cast<WorkItem*>(base + offs[p].items[v]);
      l.tables.ttasks = reinterpret_cast<const TmaTask*>(base + offs[p].ttasks);
      l.tables.recs = reinterpret_cast<const uint4*>(base + offs[p].recs);
      l.tables.n_ttasks = static_cast<int32_t>(ttasks[p].size()) - 1;
      l.tables.sched = reinterpret_cast<int*>(base + offs[p].sched);
      l.tables.n_items = cnt;
      l.tables.rec_words = rec_words[p];
      l.tma = v == 0;
      l.reduce = v >= 5;
      l.vec_bytes = v == 0 ? 16 : 16 >> ((v - 1) % 4);
      l.grid = l.tma ? std::max(1, std::min<int>(cnt, tma_grid(ctx_.sm_count())))
                     : std::max(1, std::min<int>(cnt, max_grid));
      l.tables.n_first = cnt;
      l.tables.first_ctas = l.grid;
      l.tables.error = ctx_.error_flag();
      l.tables.bulk_store = (flags_ & HS_PROG_BULK_STORE) ? kBulkStoreOutputs : 0;
      // Programmatic dependent launch on one GPU only: at N > 1 the launches
      // open with cross-rank barriers and gain little; an autotune sweep at N=2
      // once failed with a launch error that did not reproduce, so the
      // multi-rank path keeps plain stream order.
      l.tables.pdl = !(flags_ & HS_PROG_NO_PDL) && ctx_.world() == 1;
      if (l.tma && std::getenv("HS_TRACE") && !ctx_.is_analysis()) {
        stats_.trace_off = ctx_.alloc(static_cast<size_t>(l.grid) * 64);
        stats_.trace_ctas = l.grid;
        l.tables.trace = reinterpret_cast<unsigned long long*>(ctx_.arena() + stats_.trace_off);
      }
      if (l.tma && !ctx_.is_analysis())
        cuda_check(launch_expand_records(l.tables, dtype_, const_cast<uint4*>(l.tables.recs), l.tables.rec_words,
                                         ctx_.sm_count(), interleave[p], ctx_.stream()),
                   "expand records");
      if (l.tma) {
        stats_.tma_items += cnt;
        if (streamed_) {
          // two dynamic queues; no CTA takes a signalling item after a waiting one
          l.tables.n_static = 0;
          l.tables.n_first = n_first[p];
          int fc = static_cast<int>(l.grid * first_frac[p] + 0.5);
          if (n_first[p] == 0) fc = 0;
          else if (n_first[p] == cnt) fc = l.grid;
          else fc = std::min(l.grid - 1, std::max(1, fc));
          l.tables.first_ctas = fc;
          l.tables.sigs = reinterpret_cast<const SigDesc*>(base + sigs_off);
          l.tables.targets = reinterpret_cast<unsigned int* const*>(base + targets_off);
          l.tables.done = reinterpret_cast<unsigned long long*>(base + done_off);
          l.tables.wait_flags = reinterpret_cast<const unsigned int*>(ctx_.arena() + flag_off_);
        } else {
          // Single GPU: items are uniform local work, a static round-robin is
          // best (no atomic on the producer's critical path).  Multi-GPU: local
          // and NVLink items differ in cost, so the last ~1/16 are dynamic.
          // HS_PROG_STATIC_LOCAL: a multi-GPU launch of local-only items of one
          // task shape is dealt statically too.  Which wins is plan-dependent
          // (pull-mid cfg2e's producer phase: 80 -> 71 us; cfg5 S3->S4: 8%
          // slower), so it is a variant the autotuner times.
          bool uniform_local = (flags_ & HS_PROG_STATIC_LOCAL) != 0;
          const BoxTask* first = ph[p].src.empty() ? nullptr : ph[p].src.front();
          for (const BoxTask* bt : ph[p].src) {
            uniform_local = uniform_local && bt->terms.size() == first->terms.size() &&
                            bt->dsts.size() == first->dsts.size();
            for (const auto* ops : {&bt->dsts, &bt->terms})
              for (const Operand& o : *ops)
                uniform_local = uniform_local && loc(o.state, bt->tensor, o.dev).rank == bt->rank;
          }
          l.tables.n_static = ctx_.world() == 1 || uniform_local
                                  ? cnt
                                  : static_cast<int32_t>((static_cast<int64_t>(cnt) * 15 / 16) / l.grid * l.grid);
        }
      }
      d.launches.push_back(l);
      ++launches;
    }
    // The phase's opening barrier runs in the prologue of its first launch
    // when that is a TMA kernel (not the register path): one launch and its
    // gap fewer per barrier.
    // HS_SEPARATE_BARRIERS=1: ranks share a GPU (oversubscribed validation runs) --
    // a persistent kernel spinning in a folded barrier can hold the time-sliced GPU
    // while the co-resident peer that must arrive waits for a slice
    static const bool separate = std::getenv("HS_SEPARATE_BARRIERS") != nullptr;
    d.fold_barrier = ctx_.world() > 1 && !nccl_mode_ && !ce_mode_ && !(flags_ & HS_PROG_SEPARATE_BARRIERS) &&
                     !separate && !d.launches.empty() && d.launches[0].tma;
    stats_.items += n;
    stats_.phase_items.push_back(n);
  }
  // the records are complete before any stream can run the program
  if (!ctx_.is_analysis()) cuda_check(cudaStreamSynchronize(ctx_.stream()), "expand records sync");
  int barriers = ctx_.world() > 1 && !nccl_mode_ ? n_phases_ + (remote_final_writes_ ? 1 : 0) : 0;
  for (const DevicePhase& d : dphases_) barriers -= d.fold_barrier ? 1 : 0;
  stats_.kernels_per_run = launches + barriers;
}

// ---------------------------------------------------------------- run
void Program::run(cudaStream_t s) {
  if (ctx_.is_analysis()) fail(Errc::UnsupportedOp, "analysis programs do not run");
  if (!s) s = ctx_.stream();
  auto event = [&]() {
    if (events_used_ == events_.size()) {
      cudaEvent_t e;
      cuda_check(cudaEventCreate(&e), "cudaEventCreate");
      events_.push_back(e);
    }
    cuda_check(cudaEventRecord(events_[events_used_], s), "cudaEventRecord");
    ++events_used_;
  };
  // Before each phase every rank has finished everything earlier on its
  // stream: sources are ready, the previous phase's outputs are visible, and
  // the previous run's readers are done.  A program whose kernels store into
  // peers' destination shards ends with one more barrier, so a rank's own
  // destinations are complete when its stream is (callers still sync all
  // ranks before modifying sources).
  ++runs_;
  if (ce_mode_) {
    const int K = ce_chunks_;
    ctx_.barrier(s);
    for (int p = 0; p < n_phases_; ++p) {
      const int kc = p - K - 1;
      if (kc >= 0 && kc < K && ce_nwaits_[kc])
        cuda_check(launch_wait_flags(ce_waits_[kc], ce_nwaits_[kc], runs_, 20ull * 1000 * 1000 * 1000,
                                     ctx_.error_flag(), s),
                   "wait launch");
      if (profiling_) event();
      for (const Launch& l : dphases_[p].launches) {
        PhaseTables t = l.tables;
        t.epoch = runs_;
        cuda_check(launch_phase(t, dtype_, l.vec_bytes, l.tma, l.reduce, l.grid, s), "box_phase launch");
      }
      if (profiling_) event();
      if (p < K) ce_run_phase_post(p, s);
    }
    if (remote_final_writes_) ctx_.barrier(s);
    return;
  }
  for (int p = 0; p < n_phases_; ++p) {
    const bool fold = dphases_[p].fold_barrier;
    const unsigned int bar_epoch = fold ? ctx_.next_epoch() : 0;
    if (!nccl_mode_ && !fold) ctx_.barrier(s);
    if (profiling_) event();
    for (size_t i = 0; i < dphases_[p].launches.size(); ++i) {
      const Launch& l = dphases_[p].launches[i];
      PhaseTables t = l.tables;
      t.epoch = runs_;
      if (fold && i == 0) {
        t.bar_flags = ctx_.peer_flag_table();
        t.bar_world = ctx_.world();
        t.bar_rank = ctx_.rank();
        t.bar_epoch = bar_epoch;
      }
      cuda_check(launch_phase(t, dtype_, l.vec_bytes, l.tma, l.reduce, l.grid, s), "box_phase launch");
    }
    if (nccl_mode_ && p % 2 == 0 && !exchanges_[p / 2].empty()) {
      // the pack phase is followed by the phase's message exchange
      ncclComm_t comm = static_cast<ncclComm_t>(ctx_.nccl_comm());
      const nccl::Api& n = nccl::api();
      nccl::check(n.GroupStart(), "ncclGroupStart");
      for (const Exchange& x : exchanges_[p / 2]) {
        char* ptr = ctx_.arena() + x.offset;
        if (x.send)
          nccl::check(n.Send(ptr, x.bytes, ncclChar, x.peer, comm, s), "ncclSend");
        else
          nccl::check(n.Recv(ptr, x.bytes, ncclChar, x.peer, comm, s), "ncclRecv");
      }
      nccl::check(n.GroupEnd(), "ncclGroupEnd");
    }
    if (profiling_) event();
  }
  if (remote_final_writes_ && !nccl_mode_) ctx_.barrier(s);
}

void Program::run_host_async(const void* const* src_host, void* const* dst_host, cudaStream_t h2d,
                             cudaStream_t compute, cudaStream_t d2h) {
  // [0] inputs landed, [1] run done, [2] outputs read.  A repeated call waits
  // for its previous run to finish reading the sources before overwriting them,
  // and for its previous D2H before the run overwrites the destinations (an
  // event never recorded is already complete).
  for (cudaEvent_t& e : host_ev_)
    if (!e) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
  cuda_check(cudaStreamWaitEvent(h2d, host_ev_[1], 0), "stream wait");
  for (const auto& [d, t, off, bytes] : host_src_) {
    const void* h = src_host[static_cast<size_t>(t) * n_virt_ + d];
    if (h) cuda_check(cudaMemcpyAsync(off, h, bytes, cudaMemcpyHostToDevice, h2d), "H2D");
  }
  cuda_check(cudaEventRecord(host_ev_[0], h2d), "event record");
  cuda_check(cudaStreamWaitEvent(compute, host_ev_[0], 0), "stream wait");
  cuda_check(cudaStreamWaitEvent(compute, host_ev_[2], 0), "stream wait");
  run(compute);
  // host_ev_[1] (which the next call's H2D into these sources waits for) is
  // recorded after every rank has finished this run: peers read this rank's
  // sources over NVLink.  run() already ends with this barrier when its last
  // launch stores into peers' destinations.
  if (ctx_.world() > 1 && !nccl_mode_ && !remote_final_writes_) ctx_.barrier(compute);
  cuda_check(cudaEventRecord(host_ev_[1], compute), "event record");
  cuda_check(cudaStreamWaitEvent(d2h, host_ev_[1], 0), "stream wait");
  for (const auto& [d, t, off, bytes] : host_dst_) {
    void* h = dst_host[static_cast<size_t>(t) * n_virt_ + d];
    if (h) cuda_check(cudaMemcpyAsync(h, off, bytes, cudaMemcpyDeviceToHost, d2h), "D2H");
  }
  cuda_check(cudaEventRecord(host_ev_[2], d2h), "event record");
}

void Program::run_host(const void* const* src_host, void* const* dst_host) {
  cudaStream_t s = ctx_.stream();
  for (const auto& [d, t, off, bytes] : host_src_) {
    const void* h = src_host[static_cast<size_t>(t) * n_virt_ + d];
    if (h) cuda_check(cudaMemcpyAsync(off, h, bytes, cudaMemcpyHostToDevice, s), "H2D");
  }
  run(s);
  // Peers read this rank's sources over NVLink during their run: the next
  // call's H2D (stream order: after this barrier) must not overwrite them
  // before every rank has finished this run.
  if (ctx_.world() > 1 && !nccl_mode_ && !remote_final_writes_) ctx_.barrier(s);
  for (const auto& [d, t, off, bytes] : host_dst_) {
    void* h = dst_host[static_cast<size_t>(t) * n_virt_ + d];
    if (h) cuda_check(cudaMemcpyAsync(h, off, bytes, cudaMemcpyDeviceToHost, s), "D2H");
  }
  cuda_check(cudaStreamSynchronize(s), "run_host sync");
  ctx_.check_barrier_error();
}

std::string Program::tasks_json() const {
  auto kind = [this](int state) -> const char* {
    if (state == 0) return "src";
    if (state == static_cast<int>(final_state_)) return "dst";
    if (state == mid_state_) return "mid";
    if (state >= staging_state_) return state == staging_state_ ? "send" : "recv";
    return "relay";
  };
  std::ostringstream o;
  o << "[";
  bool first = true;
  for (const BoxTask& t : analysed_) {
    o << (first ? "" : ",") << "{\"phase\":" << t.phase << ",\"tensor\":" << t.tensor << ",\"rank\":" << t.rank
      << ",\"box\":[";
    first = false;
    for (size_t d = 0; d < t.box.bounds.size(); ++d)
      o << (d ? "," : "") << "[" << t.box.bounds[d][0] << "," << t.box.bounds[d][1] << "]";
    auto ops = [&](const std::vector<Operand>& v) {
      o << "[";
      for (size_t i = 0; i < v.size(); ++i) {
        const ShardLoc& L = states_[v[i].state].at({t.tensor, v[i].dev});
        o << (i ? "," : "") << "[\"" << kind(v[i].state) << "\"," << v[i].dev << "," << L.rank << "]";
      }
      o << "]";
    };
    o << "],\"dsts\":";
    ops(t.dsts);
    o << ",\"terms\":";
    ops(t.terms);
    o << ",\"groups\":[";
    for (size_t g = 0; g < t.groups.size(); ++g) o << (g ? "," : "") << t.groups[g];
    o << "],\"wait\":" << t.wait << ",\"need\":" << t.need << ",\"targets\":[";
    for (size_t g = 0; g < t.targets.size(); ++g)
      o << (g ? "," : "") << "[" << t.targets[g].first << "," << t.targets[g].second << "]";
    o << "]}";
  }
  // copy-engine relays as pseudo-tasks between the producer chunk (phase k)
  // and its consumers (phase K+1+k): read the sender's mid box, write the
  // receiver's relay box
  for (size_t i = 0; i < ce_copies_.size(); ++i) {
    const CeCopy& c = ce_copies_[i];
    if (c.sender != ctx_.rank()) continue;
    const SliceRegion& b = ce_boxes_[i];
    o << (first ? "" : ",") << "{\"phase\":" << c.chunk << ".5,\"tensor\":0,\"rank\":" << c.sender
      << ",\"copy\":1,\"box\":[";
    first = false;
    for (size_t d = 0; d < b.bounds.size(); ++d) o << (d ? "," : "") << "[" << b.bounds[d][0] << "," << b.bounds[d][1] << "]";
    o << "],\"dsts\":[[\"relay\"," << ce_relay_dev_[i] << "," << c.receiver << "]],\"terms\":[[\"mid\","
      << ce_mid_dev_[i] << "," << c.sender << "]],\"groups\":[],\"wait\":-1,\"need\":0,\"targets\":[]}";
  }
  o << "]";
  return o.str();
}

std::string Program::stats_json() const {
  std::ostringstream o;
  o << "{\"phases\":" << stats_.phases << ",\"plan_phases\":" << stats_.plan_phases
    << ",\"tasks\":" << stats_.tasks << ",\"items\":" << stats_.items << ",\"terms\":" << stats_.terms
    << ",\"outputs\":" << stats_.outputs << ",\"copy_tasks\":" << stats_.copy_tasks
    << ",\"reduce_tasks\":" << stats_.reduce_tasks << ",\"zero_tasks\":" << stats_.zero_tasks
    << ",\"tma_items\":" << stats_.tma_items << ",\"fused_tasks\":" << stats_.fused_tasks
    << ",\"relay_outputs\":" << stats_.relay_outputs << ",\"replica_swaps\":" << stats_.replica_swaps
    << ",\"shared_chunks\":" << stats_.shared_chunks << ",\"pushed_copies\":" << stats_.pushed_copies
    << ",\"model_ms\":[" << stats_.model_ms[0] << "," << stats_.model_ms[1] << "]"
    << ",\"hbm_read\":" << stats_.hbm_read << ",\"hbm_write\":" << stats_.hbm_write
    << ",\"nvlink_in\":" << stats_.nvlink_in << ",\"nvlink_out\":" << stats_.nvlink_out
    << ",\"dst_bytes\":" << stats_.dst_bytes << ",\"src_bytes\":" << stats_.src_bytes
    << ",\"h2d_bytes\":" << stats_.h2d_bytes
    << ",\"kernels_per_run\":" << stats_.kernels_per_run << ",\"streamed\":" << (stats_.streamed ? 1 : 0)
    << ",\"ce_relay\":" << (stats_.ce_relay ? 1 : 0) << ",\"ce_copies\":" << ce_copies_.size()
    << ",\"trace_off\":" << stats_.trace_off << ",\"trace_ctas\":" << stats_.trace_ctas
    << ",\"phase_items\":[";
  for (size_t i = 0; i < stats_.phase_items.size(); ++i) o << (i ? "," : "") << stats_.phase_items[i];
  o << "],\"phase_bytes\":[";
  for (size_t i = 0; i < stats_.phase_bytes.size(); ++i)
    o << (i ? "," : "") << "[" << stats_.phase_bytes[i][0] << "," << stats_.phase_bytes[i][1] << ","
      << stats_.phase_bytes[i][2] << "]";
  o << "],\"phase_kernels\":[";  // kernel of each launch, per launched phase
  for (size_t p = 0; p < dphases_.size(); ++p) {
    o << (p ? "," : "") << "[";
    for (size_t i = 0; i < dphases_[p].launches.size(); ++i) {
      const Launch& l = dphases_[p].launches[i];
      const char* name = !l.tma                                      ? "box_phase_kernel"
                         : l.tables.sigs                             ? "box_phase_tma_kernel"
                         : l.tables.n_static >= l.tables.n_items     ? "box_phase_tma_static_kernel"
                                                                     : "box_phase_tma_tail_kernel";
      o << (i ? "," : "") << "\"" << name << "\"";
    }
    o << "]";
  }
  o << "],\"dtype\":" << dtype_ << ",\"rank\":" << ctx_.rank() << "}";
  return o.str();
}

}  // namespace hshard::exec
