// SPDX-License-Identifier: Apache-2.0
//
// C++ host API for the GPU paths next to the planner, with
// the reference's types and semantics. Include after the migsim headers; link
// libmigsim_b200.so.
//
//   b200::plan_window_boundary(ctx, forecast)  == plan_window_boundary   baselines.hpp:139-289
//   b200::apply_preinit(ctx, seq)              == apply_preinit(ctx, seq, plan_preinit(cat, seq))
//                                                                         preinit.hpp:41-114
//   b200::run_requests(sc, plans, seed)        == run_requests           simulator.hpp:209-275
//   b200::run_fluid(sc, plans)                 == run_fluid              simulator.hpp:171-203
//                                                 (any allocation resolve_step reads)
//   b200::check_feasible / b200::evaluate_plan == check_feasible / evaluate_plan
//                                                 (evaluate_device.hpp) evaluate.hpp:55-210
//   b200::evaluate_totals(ctx, seqs, traces, overrides)
//                                              == evaluate_plan(...).total for plans x traces
//                                                 (verify_feasibility = false)  evaluate.hpp:153-210
// Results are bit-identical to the reference functions (tests/dropin/extras_test.cpp).
//
// Plan representation: run_fluid, check_feasible and evaluate_plan read ANY
// allocation sequence resolve_step can read (PlanSteps: configuration + per-slot
// task bits). run_requests, apply_preinit and evaluate_totals map every step to
// one of the planner's enumerated options (Space::build) and throw
// plan.infeasible for a step that is not one (several inference slots of one
// tenant, broken floors, shared instances): the planners' and baselines' plans
// always are options.
#pragma once

#include <map>
#include <vector>

#include "migsim/preinit.hpp"
#include "migsim/simulator.hpp"
#include "migsim/solvers.hpp"  // precheck_scenario (the drop-in's or the reference's)
#include "migsim_b200/device.hpp"
#include "migsim_b200/evaluate_device.hpp"

namespace migsim::b200 {

// option index of each step of a sequence (the enumeration's lex order)
inline std::vector<int32_t> option_indices(const PlanContext& ctx, const Problem& pb, const AllocationSequence& seq) {
  const int S = pb.t.steps;
  int64_t n = 0;
  mgs_error err{};
  int st = mgs_enumerate(context(), &pb.p.lattice, &pb.p.tables, &n, 0, nullptr, nullptr, nullptr, nullptr, nullptr, &err);
  if (st != MGS_OK) rethrow(st, err);
  std::vector<int32_t> cfg(n);
  std::vector<int8_t> lab(static_cast<size_t>(n) * MGS_MAX_SLOTS);
  st = mgs_enumerate(context(), &pb.p.lattice, &pb.p.tables, &n, n, cfg.data(), lab.data(), nullptr, nullptr, nullptr,
                     &err);
  if (st != MGS_OK) rethrow(st, err);
  std::map<std::vector<int>, int32_t> index;  // Space::encode of one step -> option
  const auto& configs = ctx.scenario->catalog.configurations;
  for (int64_t o = 0; o < n; ++o) {
    std::vector<int> key{cfg[o]};
    for (size_t k = 0; k < configs[cfg[o]].slots.size(); ++k) key.push_back(lab[o * MGS_MAX_SLOTS + k]);
    index.emplace(std::move(key), static_cast<int32_t>(o));
  }
  engine::Space sp;  // encode() needs only the tables
  sp.tables = pb.t;
  const std::vector<int> enc = sp.encode(seq);
  std::vector<int32_t> out;
  for (size_t i = 0; i < enc.size();) {
    const int c = enc[i];
    const size_t w = 1 + configs[c].slots.size();
    auto it = index.find(std::vector<int>(enc.begin() + i, enc.begin() + i + w));
    if (it == index.end()) fail("plan.infeasible", "plan step is not an enumerated option");
    out.push_back(it->second);
    i += w;
  }
  if (static_cast<int>(out.size()) != S) fail("input.plan", "plan length != window size");
  return out;
}

inline AllocationSequence plan_window_boundary(const PlanContext& ctx, const ArrivalForecast& forecast) {
  Problem pb(ctx, &forecast, 4000000, 1);
  throw_if_infeasible(precheck_scenario(ctx));
  check_horizon(pb.t, forecast);
  const int S = pb.t.steps;
  std::vector<int32_t> config(S);
  std::vector<int8_t> labels(static_cast<size_t>(S) * MGS_MAX_SLOTS);
  mgs_error err{};
  const int st = mgs_window_boundary(context(), &pb.p, nullptr, config.data(), labels.data(), nullptr, &err);
  if (st != MGS_OK) rethrow(st, err);
  return to_sequence(ctx, config, labels);
}

inline EffectivePlan apply_preinit(const PlanContext& ctx, const AllocationSequence& seq) {
  Problem pb(ctx, nullptr, 4000000, 1);
  const std::vector<int32_t> plan = option_indices(ctx, pb, seq);
  const int S = pb.t.steps, M = pb.t.models;
  std::vector<uint8_t> ov(static_cast<size_t>(S) * M);
  mgs_error err{};
  const int st = mgs_preinit(context(), &pb.p, plan.data(), 1, ov.data(), nullptr, &err);
  if (st != MGS_OK) rethrow(st, err);
  EffectivePlan out;
  out.seq = seq;
  for (int s = 0; s < S; ++s)
    for (int m = 0; m < M; ++m)
      if (ov[static_cast<size_t>(s) * M + m]) out.overrides[{m, s}] = 0.0;
  return out;
}

// Overrides as the device's zero-psi flags (the only value apply_preinit produces).
inline void override_flags(const OverheadOverrides& ov, int S, int M, uint8_t* flags) {
  for (const auto& [key, v] : ov) {
    if (v != 0.0) fail("input.overrides", "only zero psi_eff overrides (pre-initialisation) are supported on the device");
    if (key.first < 0 || key.first >= M || key.second < 0 || key.second >= S) continue;
    flags[static_cast<size_t>(key.second) * M + key.first] = 1;
  }
}

inline Metrics run_requests(const Scenario& sc, const std::vector<EffectivePlan>& plans, uint64_t seed) {
  const int W = static_cast<int>(plans.size());
  if (W != sc.window_count) fail("input.plan", "plan count != window count");
  PlanContext ctx0{&sc, 0, std::nullopt};
  Problem pb(ctx0, nullptr, 4000000, 1);
  const int S = pb.t.steps, M = pb.t.models;
  std::vector<int32_t> plan;
  std::vector<uint8_t> ov(static_cast<size_t>(W) * S * M, 0);
  bool any_ov = false;
  for (int w = 0; w < W; ++w) {
    PlanContext ctx{&sc, w, std::nullopt};
    const auto idx = option_indices(ctx, pb, plans[w].seq);
    plan.insert(plan.end(), idx.begin(), idx.end());
    override_flags(plans[w].overrides, S, M, ov.data() + static_cast<size_t>(w) * S * M);
    any_ov = any_ov || !plans[w].overrides.empty();
  }
  std::vector<int64_t> arrivals(static_cast<size_t>(M) * W * S);
  for (int m = 0; m < M; ++m)
    for (int g = 0; g < W * S; ++g) arrivals[static_cast<size_t>(m) * W * S + g] = sc.trace.counts[m][g];
  std::vector<double> acc_pre(static_cast<size_t>(W) * M), acc_post(static_cast<size_t>(W) * M), slo(M);
  for (int w = 0; w < W; ++w)
    for (int m = 0; m < M; ++m) {
      acc_pre[w * M + m] = sc.models[m].retraining.accuracy_pre[w];
      acc_post[w * M + m] = sc.models[m].retraining.accuracy_post[w];
    }
  for (int m = 0; m < M; ++m) slo[m] = slo_target(sc.models[m].profile);
  std::vector<mgs_job_metrics> out(static_cast<size_t>(W) * M);
  mgs_error err{};
  const int st = mgs_replay_requests(context(), &pb.p, W, acc_pre.data(), acc_post.data(), slo.data(), sc.step_seconds,
                                     plan.data(), 1, any_ov ? ov.data() : nullptr, arrivals.data(), 1, &seed, 1,
                                     out.data(), &err);
  if (st != MGS_OK) rethrow(st, err);
  std::vector<WindowMetrics> windows;  // per-window metrics, then the reference's own assembly
  for (int w = 0; w < W; ++w) {
    WindowMetrics wm;
    wm.window = w;
    for (int m = 0; m < M; ++m) {
      const mgs_job_metrics& r = out[static_cast<size_t>(w) * M + m];
      JobMetrics j;
      j.model = sc.models[m].profile.name;
      j.received = r.received;
      j.served = r.served;
      j.timely = r.timely;
      j.correct = r.correct;
      j.valid = r.valid;
      j.dropped = r.dropped;
      j.queued_at_end = r.queued_at_end;
      j.reconfigurations = r.reconfigurations;
      j.overhead_seconds = r.overhead_seconds;
      detail_sim::finalize_fractions(j);
      wm.jobs.push_back(j);
    }
    windows.push_back(std::move(wm));
  }
  return detail_sim::assemble(sc, windows);
}

// evaluate_plan(...).total (verify_feasibility = false) for every plan x trace,
// one launch; totals[i * traces.size() + t].
inline std::vector<double> evaluate_totals(const PlanContext& ctx, const std::vector<AllocationSequence>& seqs,
                                           const std::vector<std::vector<std::vector<long long>>>& traces,
                                           const std::vector<const OverheadOverrides*>& overrides = {}) {
  Problem pb(ctx, nullptr, 4000000, 1);
  const int S = pb.t.steps, M = pb.t.models;
  std::vector<int32_t> plans;
  std::vector<uint8_t> ov(seqs.size() * S * M, 0);
  for (size_t i = 0; i < seqs.size(); ++i) {
    const auto idx = option_indices(ctx, pb, seqs[i]);
    plans.insert(plans.end(), idx.begin(), idx.end());
    if (i < overrides.size() && overrides[i]) override_flags(*overrides[i], S, M, ov.data() + i * S * M);
  }
  std::vector<int64_t> arr;
  for (const auto& tr : traces)
    for (int m = 0; m < M; ++m) {
      if (static_cast<int>(tr.at(m).size()) != S) fail("input.arrivals", "arrival series length != window size");
      arr.insert(arr.end(), tr[m].begin(), tr[m].end());
    }
  std::vector<double> totals(seqs.size() * traces.size());
  mgs_error err{};
  const int st = mgs_evaluate_batch(context(), &pb.p, plans.data(), static_cast<int32_t>(seqs.size()),
                                    overrides.empty() ? nullptr : ov.data(), arr.data(),
                                    static_cast<int32_t>(traces.size()), totals.data(), nullptr, &err);
  if (st != MGS_OK) rethrow(st, err);
  return totals;
}

// run_fluid (simulator.hpp:171-203, build_series :72-131) on the device: the
// plans are read as general allocations (PlanSteps), overrides as doubles.
inline Metrics run_fluid(const Scenario& sc, const std::vector<EffectivePlan>& plans) {
  const int W = static_cast<int>(plans.size());
  if (W != sc.window_count) fail("input.plan", "plan count != window count");
  PlanContext ctx0{&sc, 0, std::nullopt};
  Problem pb(ctx0, nullptr, 4000000, 1);
  const int S = pb.t.steps, M = pb.t.models;
  PlanSteps steps;
  std::vector<double> psi;
  for (int w = 0; w < W; ++w) {
    const auto& seq = plans[w].seq;
    if (static_cast<int>(seq.allocations.size()) != S) fail("input.plan", "plan length != window size");
    for (const auto& a : seq.allocations) steps.add(pb.t, sc.catalog, a);
    if (!plans[w].overrides.empty() && psi.empty())
      psi.assign(static_cast<size_t>(W) * S * M, std::numeric_limits<double>::quiet_NaN());
    for (const auto& [key, v] : plans[w].overrides)
      if (key.first >= 0 && key.first < M && key.second >= 0 && key.second < S)
        psi[(static_cast<size_t>(w) * S + key.second) * M + key.first] = v;
  }
  std::vector<int64_t> arrivals(static_cast<size_t>(M) * W * S);
  for (int m = 0; m < M; ++m)
    for (int g = 0; g < W * S; ++g) arrivals[static_cast<size_t>(m) * W * S + g] = sc.trace.counts[m][g];
  std::vector<double> acc_pre(static_cast<size_t>(W) * M), acc_post(static_cast<size_t>(W) * M);
  for (int w = 0; w < W; ++w)
    for (int m = 0; m < M; ++m) {
      acc_pre[w * M + m] = sc.models[m].retraining.accuracy_pre[w];
      acc_post[w * M + m] = sc.models[m].retraining.accuracy_post[w];
    }
  std::vector<mgs_job_metrics> out(static_cast<size_t>(W) * M);
  mgs_error err{};
  const int st = mgs_run_fluid(context(), &pb.p, W, acc_pre.data(), acc_post.data(), sc.step_seconds,
                               steps.config.data(), steps.tasks.data(), 1, psi.empty() ? nullptr : psi.data(),
                               arrivals.data(), 1, out.data(), &err);
  if (st != MGS_OK) rethrow(st, err);
  std::vector<WindowMetrics> windows;
  for (int w = 0; w < W; ++w) {
    WindowMetrics wm;
    wm.window = w;
    for (int m = 0; m < M; ++m) {
      const mgs_job_metrics& r = out[static_cast<size_t>(w) * M + m];
      JobMetrics j;
      j.model = sc.models[m].profile.name;
      j.received = r.received;
      j.served = r.served;
      j.timely = r.timely;
      j.correct = r.correct;
      j.valid = r.valid;
      j.reconfigurations = r.reconfigurations;
      j.overhead_seconds = r.overhead_seconds;
      detail_sim::finalize_fractions(j);
      wm.jobs.push_back(j);
    }
    windows.push_back(std::move(wm));
  }
  return detail_sim::assemble(sc, windows);
}

}  // namespace migsim::b200
