// The C++ host API for the widened GPU paths (paper_2407_13126_b200/host/
// migsim_b200/extras.hpp) against the UNMODIFIED reference functions, on the
// reference's own randomized scenarios and plans (tests/test_util.hpp):
// plan_window_boundary, plan_preinit + apply_preinit, evaluate_plan with
// overrides, and run_requests -- all compared bit for bit.
// TEST INFRASTRUCTURE: built by tests/dropin/Makefile, run by tests/test_dropin.py.
#include <catch_amalgamated.hpp>

#include <cstring>
#include <random>

#include "migsim/baselines.hpp"
#include "migsim/simulator.hpp"
#include "migsim_b200/extras.hpp"
#include "test_util.hpp"

using namespace migsim;

namespace {

ArrivalForecast window0(const Scenario& sc) {
  ArrivalForecast fc;
  for (size_t m = 0; m < sc.models.size(); ++m) fc.counts.push_back(sc.window_arrivals(static_cast<int>(m), 0));
  return fc;
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

// random_feasible_plan gives up (std::runtime_error) on some scenarios
bool try_plan(const Scenario& sc, std::mt19937& rng, bool sparse, AllocationSequence* out) {
  try {
    *out = testutil::random_feasible_plan(sc, rng, sparse);
    return true;
  } catch (const std::runtime_error&) {
    return false;
  }
}

std::string code_of(const std::function<void()>& f) {
  try {
    f();
  } catch (const Error& e) {
    return e.code();
  }
  return "ok";
}

}  // namespace

TEST_CASE("GPU plan_window_boundary equals the reference on randomized scenarios") {
  std::mt19937 rng(20241017);
  int compared = 0;
  for (int iter = 0; iter < 60; ++iter) {
    INFO("iteration " << iter);
    Scenario sc = testutil::random_oracle_scenario(rng);
    PlanContext ctx{&sc, 0, std::nullopt};
    ArrivalForecast fc = window0(sc);
    AllocationSequence ref, gpu;
    const std::string rc = code_of([&] { ref = plan_window_boundary(ctx, fc); });
    const std::string gc = code_of([&] { gpu = b200::plan_window_boundary(ctx, fc); });
    CHECK(rc == gc);
    if (rc != "ok" || gc != "ok") continue;
    engine::Space sp = engine::Space::build(ctx);
    CHECK(sp.encode(ref) == sp.encode(gpu));
    ++compared;
  }
  CHECK(compared >= 20);
}

TEST_CASE("GPU pre-initialisation, evaluate_plan and run_requests equal the reference") {
  std::mt19937 rng(777001);
  int overrides = 0;
  for (int iter = 0; iter < 40; ++iter) {
    INFO("iteration " << iter);
    Scenario sc = testutil::random_oracle_scenario(rng);
    PlanContext ctx{&sc, 0, std::nullopt};
    AllocationSequence seq = testutil::random_feasible_plan(sc, rng, true);
    EffectivePlan ref = apply_preinit(ctx, seq, plan_preinit(sc.catalog, seq));
    EffectivePlan gpu = b200::apply_preinit(ctx, seq);
    CHECK(ref.overrides == gpu.overrides);
    overrides += static_cast<int>(ref.overrides.size());
    const auto counts = window0(sc).counts;
    const double ref_total = evaluate_plan(ctx, seq, counts, &ref.overrides, false).total;
    const auto totals = b200::evaluate_totals(ctx, {seq}, {counts}, {&ref.overrides});
    CHECK(same_bits(ref_total, totals.at(0)));
    for (uint64_t seed : {1ull, 99ull}) {
      const Metrics a = run_requests(sc, {ref}, seed);
      const Metrics b = b200::run_requests(sc, {gpu}, seed);
      REQUIRE(a.jobs.size() == b.jobs.size());
      for (size_t m = 0; m < a.jobs.size(); ++m) {
        CHECK(same_bits(a.jobs[m].received, b.jobs[m].received));
        CHECK(same_bits(a.jobs[m].served, b.jobs[m].served));
        CHECK(same_bits(a.jobs[m].timely, b.jobs[m].timely));
        CHECK(same_bits(a.jobs[m].correct, b.jobs[m].correct));
        CHECK(same_bits(a.jobs[m].valid, b.jobs[m].valid));
        CHECK(same_bits(a.jobs[m].dropped, b.jobs[m].dropped));
        CHECK(same_bits(a.jobs[m].goodput, b.jobs[m].goodput));
        CHECK(same_bits(a.jobs[m].overhead_seconds, b.jobs[m].overhead_seconds));
        CHECK(a.jobs[m].reconfigurations == b.jobs[m].reconfigurations);
      }
      CHECK(same_bits(a.system_goodput, b.system_goodput));
    }
  }
  CHECK(overrides > 0);
}

namespace {

// A random structural mutation of a plan step (the constraint families of
// check_feasible, shared instances, extra inference slots, dropped tasks).
AllocationSequence mutate(const Scenario& sc, AllocationSequence seq, std::mt19937& rng) {
  const int S = static_cast<int>(seq.allocations.size());
  const int kind = static_cast<int>(rng() % 7);
  Allocation& a = seq.allocations[rng() % S];
  const MigConfiguration* cfg = sc.catalog.find(a.configuration_id);
  const std::string m = sc.models[rng() % sc.models.size()].profile.name;
  const std::string slot = cfg->slots[rng() % cfg->slots.size()].id;
  switch (kind) {
    case 0: a.assignments.erase(retraining_task(m)); break;             // gap / not launched / incomplete
    case 1: a.assignments.erase(inference_task(m)); break;              // deployment floor
    case 2: a.assignments[inference_task(m)].insert(slot); break;       // extra slot, maybe shared
    case 3: a.assignments[retraining_task(m)] = {slot}; break;          // size change / overrun
    case 4: a.assignments[retraining_task(m)].insert(slot); break;      // multi-instance retraining
    case 5: a.second += 1; break;                                       // second-index
    default: {                                                          // another configuration
      const auto& c2 = sc.catalog.configurations[rng() % sc.catalog.configurations.size()];
      a.configuration_id = c2.id;
      a.assignments.clear();
      a.assignments[inference_task(m)] = {c2.slots[0].id};
    }
  }
  return seq;
}

}  // namespace

TEST_CASE("GPU check_feasible and evaluate_plan equal the reference on random and mutated plans") {
  std::mt19937 rng(4242);
  int infeasible = 0, compared = 0;
  for (int iter = 0; iter < 40; ++iter) {
    INFO("iteration " << iter);
    Scenario sc = testutil::random_oracle_scenario(rng);
    PlanContext ctx{&sc, 0, std::nullopt};
    const auto counts = window0(sc).counts;
    AllocationSequence base;
    if (!try_plan(sc, rng, iter % 2 == 0, &base)) continue;
    for (int k = 0; k < 6; ++k) {
      AllocationSequence seq = k == 0 ? base : mutate(sc, base, rng);
      if (k >= 4) seq = mutate(sc, seq, rng);
      std::vector<Violation> ref, gpu;
      const std::string rc = code_of([&] { ref = check_feasible(ctx, seq); });
      const std::string gc = code_of([&] { gpu = b200::check_feasible(ctx, seq); });
      CHECK(rc == gc);
      REQUIRE(ref.size() == gpu.size());
      for (size_t i = 0; i < ref.size(); ++i) {
        CHECK(ref[i].code == gpu[i].code);
        CHECK(ref[i].message == gpu[i].message);
        CHECK(ref[i].second == gpu[i].second);
        CHECK(ref[i].task == gpu[i].task);
      }
      infeasible += ref.empty() ? 0 : 1;
      for (bool verify : {true, false}) {
        PlanScore a, b;
        std::string am, bm;
        const std::string ra = code_of([&] {
          try {
            a = evaluate_plan(ctx, seq, counts, nullptr, verify);
          } catch (const Error& e) {
            am = e.what();
            throw;
          }
        });
        const std::string rb = code_of([&] {
          try {
            b = b200::evaluate_plan(ctx, seq, counts, nullptr, verify);
          } catch (const Error& e) {
            bm = e.what();
            throw;
          }
        });
        CHECK(ra == rb);
        CHECK(am == bm);
        if (ra != "ok" || rb != "ok") continue;
        CHECK(same_bits(a.total, b.total));
        REQUIRE(a.breakdown.size() == b.breakdown.size());
        for (size_t i = 0; i < a.breakdown.size(); ++i) {
          CHECK(same_bits(a.breakdown[i].throughput, b.breakdown[i].throughput));
          CHECK(same_bits(a.breakdown[i].overhead_loss, b.breakdown[i].overhead_loss));
          CHECK(same_bits(a.breakdown[i].goodput, b.breakdown[i].goodput));
          CHECK(a.breakdown[i].completion == b.breakdown[i].completion);
        }
        ++compared;
      }
    }
  }
  CHECK(infeasible >= 30);
  CHECK(compared >= 150);
}

TEST_CASE("GPU run_fluid equals the reference, with and without overrides") {
  std::mt19937 rng(515151);
  for (int iter = 0; iter < 40; ++iter) {
    INFO("iteration " << iter);
    Scenario sc = testutil::random_oracle_scenario(rng);
    PlanContext ctx{&sc, 0, std::nullopt};
    AllocationSequence seq;
    if (!try_plan(sc, rng, true, &seq)) continue;
    EffectivePlan plain{seq, {}};
    EffectivePlan pre = apply_preinit(ctx, seq, plan_preinit(sc.catalog, seq));
    EffectivePlan odd{seq, {{{0, 1}, 0.25}, {{0, 2}, 1.75}}};  // arbitrary psi_eff, incl. spill > 1
    for (const EffectivePlan& ep : {plain, pre, odd}) {
      const Metrics a = run_fluid(sc, {ep});
      const Metrics b = b200::run_fluid(sc, {ep});
      REQUIRE(a.jobs.size() == b.jobs.size());
      for (size_t m = 0; m < a.jobs.size(); ++m) {
        CHECK(same_bits(a.jobs[m].received, b.jobs[m].received));
        CHECK(same_bits(a.jobs[m].served, b.jobs[m].served));
        CHECK(same_bits(a.jobs[m].timely, b.jobs[m].timely));
        CHECK(same_bits(a.jobs[m].correct, b.jobs[m].correct));
        CHECK(same_bits(a.jobs[m].valid, b.jobs[m].valid));
        CHECK(same_bits(a.jobs[m].goodput, b.jobs[m].goodput));
        CHECK(same_bits(a.jobs[m].accuracy, b.jobs[m].accuracy));
        CHECK(same_bits(a.jobs[m].overhead_seconds, b.jobs[m].overhead_seconds));
        CHECK(a.jobs[m].reconfigurations == b.jobs[m].reconfigurations);
      }
      CHECK(same_bits(a.system_goodput, b.system_goodput));
      CHECK(same_bits(a.total_overhead_seconds, b.total_overhead_seconds));
    }
  }
}
