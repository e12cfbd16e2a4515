// SPDX-License-Identifier: Apache-2.0
//
// Device plumbing shared by the B200 drop-in headers (migsim/solvers.hpp,
// migsim/evaluate.hpp) and the widened host API (migsim_b200/extras.hpp):
// the per-thread device context, the PlanContext -> mgs_problem marshal, the
// error mapping back to migsim::Error, and the option -> Allocation decode.
#pragma once

#include <cstdlib>
#include <string>
#include <vector>

#include "migsim/predictor.hpp"
#include "migsim/space.hpp"
#include "migsim_b200.h"

namespace migsim {

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

}  // namespace migsim
