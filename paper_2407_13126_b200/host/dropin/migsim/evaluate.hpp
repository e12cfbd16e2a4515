// SPDX-License-Identifier: Apache-2.0
//
// B200 drop-in for the reference header proj/include/migsim/evaluate.hpp.
//
// Same namespace, types and signatures (evaluate.hpp:14-226):
//   engine::StepView, engine::resolve_step   host (the other reference headers
//                                             -- preinit, simulator, baselines
//                                             -- read allocations through it)
//   check_feasible                            device: mgs_check_feasible_batch
//   evaluate_plan                             device: mgs_evaluate_views_batch
//   final_ranges                              host (window-to-window carry)
// The host side keeps only what needs names and strings: the window-length
// and second-index checks, validate_allocation (catalog.hpp, unchanged), and
// the reference's violation messages, formatted from the device's records.
// Any allocation resolve_step can read is accepted -- several inference
// slots per tenant, shared instances, plans that break a constraint family --
// not only the planner's enumerated options.
#pragma once

#include <climits>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "migsim/space.hpp"
#include "migsim_b200/evaluate_device.hpp"

namespace migsim {

namespace engine {

// Per-step resolved view of one allocation (evaluate.hpp:16-23).
struct StepView {
  std::array<uint32_t, kMaxModels> infer_mask{};
  std::array<double, kMaxModels> infer_cap{};
  std::array<int, kMaxModels> retrain_size{};        // 0 = none
  std::array<int, kMaxModels> retrain_slot_count{};  // for validation
  uint32_t occupied_slices = 0;
};

// resolve_step (evaluate.hpp:25-47): the configuration's slots in slice-start
// order, each slot's tasks in TaskId order, so capability sums fold in the
// order every scorer uses.
inline StepView resolve_step(const Tables& t, const Allocation& a) {
  const MigConfiguration* cfg = t.config(a.configuration_id);
  if (!cfg) fail("plan.unknown-configuration", "allocation names unknown configuration '" + a.configuration_id + "'");
  StepView v{};
  for (const InstanceSlot& slot : cfg->slots) {
    for (const auto& entry : a.assignments) {
      if (entry.second.find(slot.id) == entry.second.end()) continue;
      const TaskId& task = entry.first;
      const int m = t.model_of(task);
      if (m < 0) fail("plan.unknown-model", "allocation names unknown model '" + task.model + "'");
      v.occupied_slices |= ((1u << slot.size) - 1u) << slot.slice_start;
      if (task.kind == TaskKind::Inference) {
        v.infer_mask[m] |= 1u << t.universe.find({slot.slice_start, slot.size});
        v.infer_cap[m] += t.cap_by_size[m][slot.size];
      } else {
        v.retrain_size[m] = slot.size;
        ++v.retrain_slot_count[m];
      }
    }
  }
  return v;
}

}  // namespace engine

// check_feasible (evaluate.hpp:55-146) on the device.
inline std::vector<Violation> check_feasible(const PlanContext& ctx, const AllocationSequence& seq) {
  return b200::check_feasible(ctx, seq);
}

// evaluate_plan (evaluate.hpp:153-210) on the device.
inline PlanScore evaluate_plan(const PlanContext& ctx, const AllocationSequence& seq,
                               const std::vector<std::vector<long long>>& arrivals,
                               const OverheadOverrides* overhead = nullptr, bool verify_feasibility = true) {
  return b200::evaluate_plan(ctx, seq, arrivals, overhead, verify_feasibility);
}

// Final slot sets of a sequence, for the next window's context (evaluate.hpp:213-226).
inline std::map<TaskId, std::set<SlotRange>> final_ranges(const Scenario& sc, const AllocationSequence& seq) {
  std::map<TaskId, std::set<SlotRange>> out;
  if (seq.allocations.empty()) return out;
  const Allocation& last = seq.allocations.back();
  const MigConfiguration* cfg = sc.catalog.find(last.configuration_id);
  if (!cfg) fail("plan.unknown-configuration", "unknown configuration '" + last.configuration_id + "'");
  for (const auto& [task, ids] : last.assignments)
    for (const auto& id : ids)
      if (const InstanceSlot* slot = cfg->find_slot(id)) out[task].insert({slot->slice_start, slot->size});
  return out;
}

}  // namespace migsim
