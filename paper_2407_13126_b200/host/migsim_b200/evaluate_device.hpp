// SPDX-License-Identifier: Apache-2.0
//
// check_feasible and evaluate_plan on the device, with the reference's types,
// error codes and messages (evaluate.hpp:55-210), for ANY allocation sequence
// resolve_step can read (not only the planner's enumerated options):
//   b200::check_feasible(ctx, seq)                    -> mgs_check_feasible_batch
//   b200::evaluate_plan(ctx, seq, arrivals, ov, verify) -> mgs_evaluate_views_batch
// The drop-in evaluate.hpp (host/dropin/migsim/) forwards the reference names
// here; tests/dropin/extras_test.cpp compares both with the unmodified
// reference functions. The host keeps what needs names: window length,
// second-index, validate_allocation (catalog.hpp, unchanged) and the message
// text, formatted from the device's records.
#pragma once

#include <limits>
#include <string>
#include <vector>

#include "migsim/space.hpp"
#include "migsim_b200/device.hpp"

namespace migsim {

namespace b200 {

// One allocation sequence as the device's plan steps: configuration index in
// catalog order and per-slot task bits (bit 2m inference, 2m+1 retraining).
// Throws like resolve_step for unknown configurations / models.
struct PlanSteps {
  std::vector<int32_t> config;
  std::vector<uint8_t> tasks;

  void add(const engine::Tables& t, const Catalog& cat, const Allocation& a) {
    const MigConfiguration* cfg = t.config(a.configuration_id);
    if (!cfg) fail("plan.unknown-configuration", "allocation names unknown configuration '" + a.configuration_id + "'");
    config.push_back(static_cast<int32_t>(cfg - cat.configurations.data()));
    const size_t base = tasks.size();
    tasks.resize(base + MGS_MAX_SLOTS, 0);
    for (size_t k = 0; k < cfg->slots.size() && k < MGS_MAX_SLOTS; ++k)
      for (const auto& [task, slots] : a.assignments) {
        if (slots.find(cfg->slots[k].id) == slots.end()) continue;
        const int m = t.model_of(task);
        if (m < 0) fail("plan.unknown-model", "allocation names unknown model '" + task.model + "'");
        tasks[base + k] |= static_cast<uint8_t>(1u << (2 * m + (task.kind == TaskKind::Inference ? 0 : 1)));
      }
  }
};

// The reference's text for one device violation record (evaluate.hpp:82-144).
inline Violation violation_text(const engine::Tables& t, const mgs_plan_violation& v) {
  const std::string name = t.sc->models[v.model].profile.name;
  switch (v.code) {
    case MGS_VIOL_DEPLOYMENT_FLOOR:
      return {"deployment-floor",
              "step " + std::to_string(v.step) + ": inference task " + name + ":i holds no single instance of size >= " +
                  std::to_string(v.detail[1]) + " (weaker GPC-sum check: " +
                  (v.detail[0] ? "satisfied" : "also violated") + ")",
              v.step, name + ":i"};
    case MGS_VIOL_RETRAINING_NOT_LAUNCHED:
      return {"retraining-not-launched", "retraining task " + name + ":r is never launched within the window", -1,
              name + ":r"};
    case MGS_VIOL_RETRAINING_INTERRUPTED:
      return {"retraining-interrupted",
              "retraining task " + name + ":r must keep a constant GPC count from start to finish (" +
                  (v.detail[0] ? "GPC count changed mid-run" : "run has gaps") + ")",
              v.step, name + ":r"};
    case MGS_VIOL_RETRAINING_SIZE:
      return {"retraining-size", "retraining task " + name + ":r runs on " + std::to_string(v.detail[0]) +
                                     " GPCs but no retraining time is defined for that size",
              v.step, name + ":r"};
    case MGS_VIOL_RETRAINING_INCOMPLETE:
      return {"retraining-incomplete", "retraining task " + name + ":r runs " + std::to_string(v.detail[0]) +
                                           " steps but needs " + std::to_string(v.detail[1]) + " on " +
                                           std::to_string(v.detail[2]) + " GPCs to complete within the window",
              v.step, name + ":r"};
    default:
      return {"retraining-overrun", "retraining task " + name + ":r holds its instance for " +
                                        std::to_string(v.detail[0]) + " steps but completes after " +
                                        std::to_string(v.detail[1]),
              v.step, name + ":r"};
  }
}

}  // namespace b200

namespace b200 {

// check_feasible (evaluate.hpp:55-146): empty iff the sequence satisfies every
// constraint family.
inline std::vector<Violation> check_feasible(const PlanContext& ctx, const AllocationSequence& seq) {
  using namespace engine;
  Problem pb(ctx, nullptr, 0, 1);
  const Tables& t = pb.t;
  std::vector<Violation> out;
  const int S = t.steps;
  if (static_cast<int>(seq.allocations.size()) != S) {
    out.push_back({"window-length", "plan has " + std::to_string(seq.allocations.size()) + " steps, window needs " +
                                        std::to_string(S),
                   -1, ""});
    return out;
  }
  PlanSteps steps;
  for (int s = 0; s < S; ++s) {
    const Allocation& a = seq.allocations[s];
    if (a.second != s)
      out.push_back({"second-index", "allocation at position " + std::to_string(s) + " is labeled second " +
                                         std::to_string(a.second),
                     s, ""});
    for (const auto& v : validate_allocation(ctx.scenario->catalog, a)) out.push_back({v.code, v.message, s, ""});
    if (!t.config(a.configuration_id)) return out;  // cannot resolve further
    steps.add(t, ctx.scenario->catalog, a);
  }
  const int cap = S * t.models + t.models;
  std::vector<mgs_plan_violation> rec(cap);
  int32_t n = 0;
  mgs_error err{};
  const int st = mgs_check_feasible_batch(context(), &pb.p, steps.config.data(), steps.tasks.data(), 1, rec.data(),
                                          cap, &n, &err);
  if (st != MGS_OK) rethrow(st, err);
  for (int i = 0; i < n && i < cap; ++i) out.push_back(violation_text(t, rec[i]));
  return out;
}

// evaluate_plan (evaluate.hpp:153-210): expected valid-request count of the
// sequence against the arrivals; breakdown step-major, model-minor.
inline PlanScore evaluate_plan(const PlanContext& ctx, const AllocationSequence& seq,
                               const std::vector<std::vector<long long>>& arrivals,
                               const OverheadOverrides* overhead = nullptr, bool verify_feasibility = true) {
  using namespace engine;
  if (verify_feasibility) {
    const auto violations = b200::check_feasible(ctx, seq);
    if (!violations.empty())
      fail("plan.infeasible",
           "evaluate_plan: infeasible plan: " + violations.front().code + ": " + violations.front().message);
  }
  Problem pb(ctx, nullptr, 0, 1);
  const Tables& t = pb.t;
  const int S = t.steps, M = t.models;
  if (static_cast<int>(seq.allocations.size()) != S) fail("plan.infeasible", "plan length != window size");
  std::vector<int64_t> arr(static_cast<size_t>(M) * S);
  for (int m = 0; m < M; ++m) {
    const auto& row = arrivals.at(m);
    if (static_cast<int>(row.size()) < S) fail("input.arrivals", "arrivals shorter than the window");
    for (int s = 0; s < S; ++s) arr[static_cast<size_t>(m) * S + s] = row[s];
  }
  PlanSteps steps;
  for (const auto& a : seq.allocations) steps.add(t, ctx.scenario->catalog, a);
  std::vector<double> psi;
  if (overhead && !overhead->empty()) {
    psi.assign(static_cast<size_t>(S) * M, std::numeric_limits<double>::quiet_NaN());
    for (const auto& [key, v] : *overhead)
      if (key.first >= 0 && key.first < M && key.second >= 0 && key.second < S)
        psi[static_cast<size_t>(key.second) * M + key.first] = v;
  }
  double total = 0.0;
  std::vector<mgs_score_entry> ent(static_cast<size_t>(S) * M);
  mgs_error err{};
  const int st = mgs_evaluate_views_batch(context(), &pb.p, steps.config.data(), steps.tasks.data(), 1,
                                          psi.empty() ? nullptr : psi.data(), arr.data(), 1, 0, &total, ent.data(),
                                          nullptr, nullptr, &err);
  if (st != MGS_OK) rethrow(st, err);
  PlanScore score;
  score.total = total;
  score.breakdown.reserve(ent.size());
  for (int s = 0; s < S; ++s)
    for (int m = 0; m < M; ++m) {
      const mgs_score_entry& e = ent[static_cast<size_t>(s) * M + m];
      score.breakdown.push_back({s, m, e.throughput, e.completion != 0, e.overhead_loss, e.goodput});
    }
  return score;
}

}  // namespace b200
}  // namespace migsim
