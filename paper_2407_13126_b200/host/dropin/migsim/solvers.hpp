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

#include "migsim/evaluate.hpp"  // the drop-in (device check_feasible / evaluate_plan)
#include "migsim/predictor.hpp"
#include "migsim/space.hpp"
#include "migsim_b200/device.hpp"

namespace migsim {

struct SolveOptions {
  int workers = 1;                // accepted; results are identical for any value
  size_t state_budget = 4000000;  // max DP frontier states per step
  double bruteforce_cap = 5e7;    // gate on |options|^S
};



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
