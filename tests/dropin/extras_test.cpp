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
