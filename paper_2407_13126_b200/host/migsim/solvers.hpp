// SPDX-License-Identifier: Apache-2.0
//
// B200 drop-in for the reference planner header proj/include/migsim/solvers.hpp.
//
// Same namespace, types and signatures as the reference (solvers.hpp:20-579):
//   SolveOptions, precheck_scenario, throw_if_infeasible,
//   engine::{allowed_sizes, FrontKey, FrontKeyHash, DpState, dp_better,
//            status_dominates},
//   solve_bruteforce, solve_dp.
// Put this directory ahead of the reference's include directory (or replace
// the file) and every existing caller -- tests, baselines.hpp, ilp.hpp, the
// per-window driver -- runs its searches on the GPU unchanged. The other
// reference headers (catalog/workload/plan_types/space/evaluate/predictor)
// are used as they are: they hold the data types and the cheap host tables.
//
// What moves to the device (through the C ABI, include/migsim_b200.h):
//   precheck_scenario  -> mgs_precheck     (option space built on the GPU)
//   solve_bruteforce   -> mgs_bruteforce   (every sequence scored on the GPU)
//   solve_dp           -> mgs_solve_window (the whole DP device-resident)
// There is no CPU search here and no fallback: a missing library is a link
// error, a missing GPU is migsim::Error("device.cuda").
//
// Threading: each host thread gets its own device context (mgs_ctx) on
// device $MIGSIM_B200_DEVICE (default 0). SolveOptions::workers is accepted
// and, as in the reference, never changes results.
#pragma once

#include <array>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "migsim/evaluate.hpp"
#include "migsim/predictor.hpp"
#include "migsim/space.hpp"
#include "migsim_b200.h"

namespace migsim {

struct SolveOptions {
  int workers = 1;                // accepted; results are identical for any value
  size_t state_budget = 4000000;  // max DP frontier states per step
  double bruteforce_cap = 5e7;    // gate on |options|^S
};

namespace b200 {

// One device context per host thread (mgs_ctx is not thread-safe).
inline mgs_ctx* context() {
  struct Holder {
    mgs_ctx* h = nullptr;
    ~Holder() {
      if (h) mgs_close(h);
    }
  };
  thread_local Holder holder;
  if (!holder.h) {
    const char* env = std::getenv("MIGSIM_B200_DEVICE");
    const int dev = env ? std::atoi(env) : 0;
    const int st = mgs_open(dev, &holder.h);
    if (st != MGS_OK) fail(mgs_status_code(st), "cannot open the B200 planner on device " + std::to_string(dev));
  }
  return holder.h;
}

// PlanContext (+ forecast) marshalled into the C ABI's flat problem. Owns
// the arrays the mgs_problem points into.
struct Problem {
  engine::Tables t;
  std::vector<int32_t> slot_offset, slot_size, slot_start;
  std::vector<int64_t> forecast;
  mgs_problem p{};

  Problem(const PlanContext& ctx, const ArrivalForecast* fc, size_t state_budget, int workers)
      : t(engine::Tables::build(ctx)) {  // input.scenario / input.catalog as the reference
    const Catalog& cat = ctx.scenario->catalog;
    slot_offset.push_back(0);
    for (const auto& cfg : cat.configurations) {  // file order; slots sorted by slice_start
      for (const auto& s : cfg.slots) {
        slot_size.push_back(s.size);
        slot_start.push_back(s.slice_start);
      }
      slot_offset.push_back(static_cast<int32_t>(slot_size.size()));
    }
    p.lattice.n_configs = static_cast<int32_t>(cat.configurations.size());
    p.lattice.gpc_count = cat.gpc_count;
    p.lattice.slot_offset = slot_offset.data();
    p.lattice.slot_size = slot_size.data();
    p.lattice.slot_start = slot_start.data();
    mgs_tables& tb = p.tables;
    tb.models = t.models;
    tb.steps = t.steps;
    for (int m = 0; m < t.models; ++m) {
      for (int k = 0; k < MGS_SIZES; ++k) {
        tb.cap_by_size[m][k] = t.cap_by_size[m][k];
        tb.rt_by_size[m][k] = t.rt_by_size[m][k];
      }
      tb.floor_gpcs[m] = t.floor_gpcs[m];
      tb.psi[m] = t.psi[m];
      tb.acc_pre[m] = t.acc_pre[m];
      tb.acc_post[m] = t.acc_post[m];
    }
    bool has_initial = false;
    const auto init = engine::initial_masks(t, ctx, &has_initial);
    p.has_initial = has_initial ? 1 : 0;
    for (int m = 0; m < engine::kMaxModels; ++m) p.init_mask[m] = init[m];
    p.state_budget = state_budget;
    p.workers = workers;
    if (fc) {
      const int S = t.steps;
      forecast.assign(static_cast<size_t>(t.models) * S, 0);
      for (int m = 0; m < t.models && m < static_cast<int>(fc->counts.size()); ++m) {
        const auto& row = fc->counts[m];
        for (int s = 0; s < S && s < static_cast<int>(row.size()); ++s) forecast[static_cast<size_t>(m) * S + s] = row[s];
      }
      p.forecast = forecast.data();
      p.forecast_len = S;
    }
  }
};

// The reference's precheck messages (solvers.hpp:31-66) with model names.
inline Violation violation_of(const engine::Tables& t, const mgs_violation& v) {
  const std::string name = v.model >= 0 ? t.sc->models[v.model].profile.name : std::string();
  switch (v.code) {
    case MGS_ERR_DEPLOYMENT_FLOOR:
      if (v.model < 0)
        return {"deployment-floor",
                "deployment-floor unsatisfiable: no configuration deploys every inference task simultaneously", -1, ""};
      return {"deployment-floor", "deployment-floor unsatisfiable: no catalog instance reaches " +
                                      std::to_string(t.floor_gpcs[v.model]) + " GPCs for model " + name,
              -1, name + ":i"};
    case MGS_ERR_RETRAINING_WINDOW:
      return {"retraining-window",
              "model " + name + ": every retraining time exceeds the window (" + std::to_string(t.steps) + " steps)",
              -1, name + ":r"};
    default:
      return {"no-coexistence-configuration",
              "no-coexistence-configuration: no configuration runs " + name + ":r alongside every inference task", -1,
              name + ":r"};
  }
}

[[noreturn]] inline void rethrow(int status, const mgs_error& e) {
  fail(mgs_status_code(status), e.message);
}

// Space::to_allocation (space.hpp:213-227) from a configuration index and the
// per-slot labels the device returns.
inline Allocation to_allocation(const Scenario& sc, int config, const int8_t* labels, int second) {
  const auto& cfg = sc.catalog.configurations.at(config);
  Allocation a;
  a.second = second;
  a.configuration_id = cfg.id;
  for (size_t i = 0; i < cfg.slots.size(); ++i) {
    const int lab = labels[i];
    if (lab == 0) continue;
    const int m = (lab - 1) / 2;
    const std::string& name = sc.models[m].profile.name;
    const TaskId task = (lab - 1) % 2 == 0 ? inference_task(name) : retraining_task(name);
    a.assignments[task].insert(cfg.slots[i].id);
  }
  return a;
}

inline AllocationSequence to_sequence(const PlanContext& ctx, const std::vector<int32_t>& config,
                                      const std::vector<int8_t>& labels) {
  AllocationSequence seq;
  seq.window_index = ctx.window;
  for (size_t s = 0; s < config.size(); ++s)
    seq.allocations.push_back(
        to_allocation(*ctx.scenario, config[s], labels.data() + s * MGS_MAX_SLOTS, static_cast<int>(s)));
  return seq;
}

inline void check_horizon(const engine::Tables& t, const ArrivalForecast& forecast) {
  for (int m = 0; m < t.models; ++m)  // solvers.hpp:250-252
    if (static_cast<int>(forecast.counts.at(m).size()) != t.steps)
      fail("input.forecast", "forecast horizon != window size");
}

}  // namespace b200

// Necessary feasibility conditions (solvers.hpp:27-69), evaluated over the
// option space the GPU enumerates.
inline std::vector<Violation> precheck_scenario(const PlanContext& ctx) {
  b200::Problem pb(ctx, nullptr, 0, 1);
  mgs_violation v[3 * MGS_MAX_MODELS + 1];
  int32_t n = 0;
  mgs_error err{};
  const int st = mgs_precheck(b200::context(), &pb.p.lattice, &pb.p.tables, v, 3 * MGS_MAX_MODELS + 1, &n, &err);
  if (st != MGS_OK) b200::rethrow(st, err);
  std::vector<Violation> out;
  for (int i = 0; i < n; ++i) out.push_back(b200::violation_of(pb.t, v[i]));
  return out;
}

inline void throw_if_infeasible(const std::vector<Violation>& v) {
  if (!v.empty()) fail("infeasible." + v.front().code, v.front().message);
}

namespace engine {

// Retraining sizes a tenant may hold at step s given its status (solvers.hpp:79-97).
inline bool allowed_sizes(const Tables& t, const StatusCodec& codec, int m, int status, int s,
                          std::array<int8_t, 9>* sizes, int* count) {
  *count = 0;
  if (codec.is_running(status)) {
    sizes->at((*count)++) = static_cast<int8_t>(codec.run_size(status));
  } else if (status == codec.done()) {
    sizes->at((*count)++) = 0;
  } else {
    if (t.min_rt[m] >= 0 && s + 1 + t.min_rt[m] <= t.steps) sizes->at((*count)++) = 0;
    for (int k = 1; k <= 7; ++k) {
      const long long rt = t.rt_by_size[m][k];
      if (rt >= 1 && s + rt <= t.steps) sizes->at((*count)++) = static_cast<int8_t>(k);
    }
  }
  return *count > 0;
}

// DP state key / record types (solvers.hpp:99-121); the device keeps the same
// information as structure-of-arrays frontiers.
struct FrontKey {
  uint64_t status = 0;
  std::array<uint32_t, kMaxModels> mask{};
  bool operator==(const FrontKey&) const = default;
};
struct FrontKeyHash {
  size_t operator()(const FrontKey& k) const {
    uint64_t h = 1469598103934665603ull ^ k.status;  // FNV-1a over the fields
    for (uint32_t m : k.mask) h = (h ^ m) * 1099511628211ull;
    h *= 1099511628211ull;
    return static_cast<size_t>(h ^ (h >> 29));
  }
};
struct DpState {
  FrontKey key;
  double value = 0.0;
  int parent = -1;
  int option = -1;
  uint64_t lex = 0;  // (parent lex rank << 32) | option index
  uint32_t rank = 0;
};

// Higher value wins, then smaller lex (solvers.hpp:123-126).
inline bool dp_better(double va, uint64_t la, double vb, uint64_t lb) { return va != vb ? va > vb : la < lb; }

// done >= running >= longer-remaining running at equal size (solvers.hpp:128-134).
inline bool status_dominates(const StatusCodec& codec, int a, int b) {
  if (a == b || a == codec.done()) return true;
  return codec.is_running(a) && codec.is_running(b) && codec.run_size(a) == codec.run_size(b) &&
         codec.run_rem(a) <= codec.run_rem(b);
}

}  // namespace engine

// Exhaustive search (solvers.hpp:143-228): every sequence scored on the GPU;
// the lexicographically smallest optimal sequence, exactly like the DFS.
inline AllocationSequence solve_bruteforce(const PlanContext& ctx, const ArrivalForecast& forecast,
                                           const SolveOptions& opt = {}) {
  b200::Problem pb(ctx, &forecast, opt.state_budget, opt.workers);
  throw_if_infeasible(precheck_scenario(ctx));
  b200::check_horizon(pb.t, forecast);
  const int S = pb.t.steps;
  std::vector<int32_t> config(S);
  std::vector<int8_t> labels(static_cast<size_t>(S) * MGS_MAX_SLOTS);
  double objective = 0.0;
  mgs_error err{};
  const int st = mgs_bruteforce(b200::context(), &pb.p, opt.bruteforce_cap, nullptr, config.data(), labels.data(),
                                &objective, &err);
  if (st != MGS_OK) b200::rethrow(st, err);
  return b200::to_sequence(ctx, config, labels);
}

// The per-window reconfiguration decision (solvers.hpp:242-579): the whole
// cross-slot max-plus DP runs on the device, same procedure and tie-breaks.
inline AllocationSequence solve_dp(const PlanContext& ctx, const ArrivalForecast& forecast,
                                   const SolveOptions& opt = {}) {
  b200::Problem pb(ctx, &forecast, opt.state_budget, opt.workers);
  throw_if_infeasible(precheck_scenario(ctx));
  b200::check_horizon(pb.t, forecast);
  const int S = pb.t.steps;
  std::vector<int32_t> config(S);
  std::vector<int8_t> labels(static_cast<size_t>(S) * MGS_MAX_SLOTS);
  double objective = 0.0;
  mgs_error err{};
  const int st = mgs_solve_window(b200::context(), &pb.p, nullptr, config.data(), labels.data(), &objective, nullptr,
                                  &err);
  if (st != MGS_OK) b200::rethrow(st, err);
  return b200::to_sequence(ctx, config, labels);
}

}  // namespace migsim
