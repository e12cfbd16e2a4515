// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// Driver around the UNMODIFIED reference planner (header-only C++20 under
// /root/reference/proj/include, compiled in place by oracle/Makefile into
// oracle/_ref/). It is the ground truth the CPU restatement and the GPU path
// are pinned against, and the CPU baseline arm of bench.py.
//
//   migref solve <scenario.scn> [window] [--workers N] [--budget B] [--chain] [--bf]
//       load_scenario (workload.hpp:337) -> solve_dp (solvers.hpp:242) [and
//       solve_bruteforce (:143)] -> evaluate_plan (evaluate.hpp:153); prints
//       one JSON object: plan encoding (space.hpp:231), objective bits, per-(s,m)
//       SLO-attained throughput bits, wall time, or the Error code.
//       --wb adds plan_window_boundary (baselines.hpp:139-289) under "wb".
//       --chain re-plans with initial = final_ranges(first plan)
//       (solver_test.cpp:130-147 semantics).
//   migref replay <scenario.scn> <seed>...
//       run_requests (simulator.hpp:209-275) of the window-0 solve_dp plan
//       (no pre-initialisation overrides) for each seed; prints per-model
//       JobMetrics counters as hex bits.
//   migref preinit <scenario.scn> <seed>
//       plan_preinit + apply_preinit (preinit.hpp:41-114) of the window-0
//       solve_dp plan: overrides, evaluate_plan total with them,
//       overhead_summary, and run_requests of the EffectivePlan.
//   migref drive <scenario.scn> <predictor> [max_windows] [lookback] [psi]
//       the per-window planning loop from the reference's
//       pieces: predict_arrivals (oracle for window 0) -> solve_dp with the
//       carried final_ranges -> evaluate_plan on forecast and actual counts.
//   migref replay-windows <scenario.scn> <seed>
//       run_requests over every window of the scenario for the plans of the
//       per-window loop (oracle forecasts, carried final_ranges); prints the
//       per-window JobMetrics counters and each window's plan encoding.
//   migref gen-random <seed> <count> <outdir> [--no-drop]
//       the reference's own randomized oracle corpus generator
//       (tests/test_util.hpp:104-181), written to files with
//       write_scenario_files (workload.hpp:422) so other implementations
//       read identical inputs.
//   migref gen-multi <seed> <count> <outdir> <M> <S_lo> <S_hi> <est_cap>
//       the same generator shape (test_util.hpp:104-181: mt19937, rng() % n,
//       finalize_scenario, precheck, |O|^S estimate, solvability through
//       solve_dp) widened to M = 3..4 tenants on A100 configurations with
//       enough slots to anchor every tenant. Only meaningful when built
//       against the patched headers (migref_patched, see oracle/Makefile):
//       the unmodified solve_dp rejects every M >= 3 window
//       (solvers.hpp:359,401,414 narrow the packed status to int).
//
// The shared-library build exports migref_solve_file() for bench.py.
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#ifndef MIGSIM_DATA_DIR
#define MIGSIM_DATA_DIR "/nonexistent"
#endif
#include "migsim/baselines.hpp"
#include "migsim/simulator.hpp"
#include "migsim/solvers.hpp"
#include "test_util.hpp"  // reference tests/test_util.hpp (via -I)

using namespace migsim;

namespace {

std::string hexbits(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  char buf[32];
  std::snprintf(buf, sizeof buf, "%016" PRIx64, b);
  return buf;
}

std::string json_str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') { o += '\\'; o += c; }
    else if (c == '\n') o += "\\n";
    else o += c;
  }
  return o + "\"";
}

ArrivalForecast window_forecast(const Scenario& sc, int w) {
  ArrivalForecast fc;
  for (size_t m = 0; m < sc.models.size(); ++m) fc.counts.push_back(sc.window_arrivals(static_cast<int>(m), w));
  return fc;
}

std::string plan_json(const PlanContext& ctx, const AllocationSequence& seq, const ArrivalForecast& fc) {
  engine::Space sp = engine::Space::build(ctx);
  auto enc = sp.encode(seq);
  PlanScore sc = evaluate_plan(ctx, seq, fc.counts);
  std::string o = "{\"encode\":[";
  for (size_t i = 0; i < enc.size(); ++i) o += (i ? "," : "") + std::to_string(enc[i]);
  o += "],\"obj\":\"" + hexbits(sc.total) + "\",\"objective\":" + fmt_real(sc.total) + ",\"thr\":[";
  for (size_t i = 0; i < sc.breakdown.size(); ++i) o += std::string(i ? "," : "") + "\"" + hexbits(sc.breakdown[i].throughput) + "\"";
  o += "]}";
  return o;
}

std::string initial_json(const std::map<TaskId, std::set<SlotRange>>& init) {
  std::string o = "[";
  bool first = true;
  for (const auto& [task, ranges] : init)
    for (const auto& [start, size] : ranges) {
      o += std::string(first ? "" : ",") + "[" + json_str(task.model) + "," +
           (task.kind == TaskKind::Inference ? "\"i\"" : "\"r\"") + "," + std::to_string(start) + "," +
           std::to_string(size) + "]";
      first = false;
    }
  return o + "]";
}

template <class F>
std::string guarded(F&& f) {
  try {
    return f();
  } catch (const Error& e) {
    return "{\"error\":" + json_str(e.code()) + ",\"message\":" + json_str(e.what()) + "}";
  }
}

int cmd_solve(int argc, char** argv) {
  if (argc < 3) return 2;
  std::string path = argv[2];
  int window = 0;
  SolveOptions opt;
  bool chain = false, bf = false, wb = false;
  for (int i = 3; i < argc; ++i) {
    std::string a = argv[i];
    if (a == "--workers") opt.workers = std::atoi(argv[++i]);
    else if (a == "--budget") opt.state_budget = std::strtoull(argv[++i], nullptr, 10);
    else if (a == "--chain") chain = true;
    else if (a == "--bf") bf = true;
    else if (a == "--wb") wb = true;
    else window = std::atoi(a.c_str());
  }
  std::string out = guarded([&] {
    Scenario sc = load_scenario(path);
    PlanContext ctx{&sc, window, std::nullopt};
    ArrivalForecast fc = window_forecast(sc, window);
    auto t0 = std::chrono::steady_clock::now();
    AllocationSequence dp = solve_dp(ctx, fc, opt);
    double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::string o = "{\"dp\":" + plan_json(ctx, dp, fc) + ",\"seconds\":" + fmt_real(secs) +
                    ",\"options\":" + std::to_string(engine::Space::build(ctx).options.size());
    if (bf) o += ",\"bf\":" + guarded([&] { return plan_json(ctx, solve_bruteforce(ctx, fc, opt), fc); });
    if (wb) o += ",\"wb\":" + guarded([&] { return plan_json(ctx, plan_window_boundary(ctx, fc), fc); });
    if (chain) {
      PlanContext chained = ctx;
      chained.initial = final_ranges(sc, dp);
      o += ",\"chain\":{\"initial\":" + initial_json(*chained.initial) +
           ",\"dp\":" + guarded([&] { return plan_json(chained, solve_dp(chained, fc, opt), fc); });
      if (bf) o += ",\"bf\":" + guarded([&] { return plan_json(chained, solve_bruteforce(chained, fc, opt), fc); });
      if (wb) o += ",\"wb\":" + guarded([&] { return plan_json(chained, plan_window_boundary(chained, fc), fc); });
      o += "}";
    }
    return o + "}";
  });
  std::printf("%s\n", out.c_str());
  return 0;
}

int cmd_replay(int argc, char** argv) {
  if (argc < 4) return 2;
  std::string out = guarded([&] {
    Scenario sc = load_scenario(argv[2]);
    PlanContext ctx{&sc, 0, std::nullopt};
    ArrivalForecast fc = window_forecast(sc, 0);
    AllocationSequence dp = solve_dp(ctx, fc);
    std::vector<EffectivePlan> plans{EffectivePlan{dp, {}}};
    std::string o = "{\"runs\":[";
    for (int i = 3; i < argc; ++i) {
      const uint64_t seed = std::strtoull(argv[i], nullptr, 10);
      Metrics mt = run_requests(sc, plans, seed);
      o += std::string(i > 3 ? "," : "") + "{\"seed\":" + std::to_string(seed) + ",\"jobs\":[";
      for (size_t m = 0; m < mt.jobs.size(); ++m) {
        const JobMetrics& j = mt.jobs[m];
        o += std::string(m ? "," : "") + "[\"" + hexbits(j.received) + "\",\"" + hexbits(j.served) + "\",\"" +
             hexbits(j.timely) + "\",\"" + hexbits(j.correct) + "\",\"" + hexbits(j.valid) + "\",\"" +
             hexbits(j.dropped) + "\",\"" + hexbits(j.queued_at_end) + "\"," + std::to_string(j.reconfigurations) +
             ",\"" + hexbits(j.overhead_seconds) + "\"]";
      }
      o += "]}";
    }
    return o + "]}";
  });
  std::printf("%s\n", out.c_str());
  return 0;
}

std::string jobs_json(const Metrics& mt) {
  std::string o = "[";
  for (size_t m = 0; m < mt.jobs.size(); ++m) {
    const JobMetrics& j = mt.jobs[m];
    o += std::string(m ? "," : "") + "[\"" + hexbits(j.received) + "\",\"" + hexbits(j.served) + "\",\"" +
         hexbits(j.timely) + "\",\"" + hexbits(j.correct) + "\",\"" + hexbits(j.valid) + "\",\"" +
         hexbits(j.dropped) + "\",\"" + hexbits(j.queued_at_end) + "\"," + std::to_string(j.reconfigurations) +
         ",\"" + hexbits(j.overhead_seconds) + "\"]";
  }
  return o + "]";
}

std::string preinit_json(const Scenario& sc, const PlanContext& ctx, const ArrivalForecast& fc,
                         const AllocationSequence& seq, uint64_t seed) {
  auto actions = plan_preinit(sc.catalog, seq);
  EffectivePlan eff = apply_preinit(ctx, seq, actions);
  engine::Space sp = engine::Space::build(ctx);
  auto enc = sp.encode(seq);
  std::string o = "{\"encode\":[";
  for (size_t i = 0; i < enc.size(); ++i) o += (i ? "," : "") + std::to_string(enc[i]);
  o += "],\"overrides\":[";
  bool first = true;
  for (const auto& [key, v] : eff.overrides) {
    o += std::string(first ? "" : ",") + "[" + std::to_string(key.first) + "," + std::to_string(key.second) + "]";
    first = false;
  }
  PlanScore ps = evaluate_plan(ctx, seq, fc.counts, &eff.overrides);
  OverheadSummary os = overhead_summary(ctx, seq, &eff.overrides);
  o += "],\"actions\":" + std::to_string(actions.size()) + ",\"obj\":\"" + hexbits(ps.total) +
       "\",\"reconfigurations\":" + std::to_string(os.reconfigurations) + ",\"overhead\":\"" +
       hexbits(os.total_overhead) + "\",\"seed\":" + std::to_string(seed) +
       ",\"jobs\":" + jobs_json(run_requests(sc, {eff}, seed)) + "}";
  return o;
}

int cmd_preinit(int argc, char** argv) {
  if (argc < 4) return 2;
  const int n_random = argc > 4 ? std::atoi(argv[4]) : 0;
  std::string out = guarded([&] {
    Scenario sc = load_scenario(argv[2]);
    const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
    PlanContext ctx{&sc, 0, std::nullopt};
    ArrivalForecast fc = window_forecast(sc, 0);
    std::string o = "{\"dp\":" + preinit_json(sc, ctx, fc, solve_dp(ctx, fc), seed) + ",\"random\":[";
    std::mt19937 rng(static_cast<unsigned>(seed));
    for (int k = 0; k < n_random; ++k)  // sparse random feasible plans leave pre-initialisation room to act
      o += std::string(k ? "," : "") + preinit_json(sc, ctx, fc, testutil::random_feasible_plan(sc, rng, true), seed);
    return o + "]}";
  });
  std::printf("%s\n", out.c_str());
  return 0;
}

int cmd_drive(int argc, char** argv) {
  if (argc < 4) return 2;
  std::string out = guarded([&] {
    Scenario sc = load_scenario(argv[2]);
    PredictorSpec spec = parse_predictor_spec(argv[3]);
    const int S = sc.window_size, M = static_cast<int>(sc.models.size());
    std::optional<std::map<TaskId, std::set<SlotRange>>> initial;
    std::string o = "{\"windows\":[";
    const int W = argc > 4 ? std::min(sc.window_count, std::atoi(argv[4])) : sc.window_count;
    // sliding lookahead: the predictor sees only the last `lookback` windows
    const int lookback = argc > 5 ? std::atoi(argv[5]) : (1 << 30);
    if (argc > 6)  // reconfiguration-cost sweep point: every tenant's psi
      for (auto& e : sc.models) e.profile.reconfig_overhead = std::atof(argv[6]);
    for (int w = 0; w < W; ++w) {
      ArrivalForecast actual = window_forecast(sc, w);
      ArrivalForecast fc;
      if (spec.kind == PredictorKind::Oracle || w == 0) {
        fc = predict_arrivals(PredictorSpec{}, {}, S, S, &actual.counts);
      } else {
        std::vector<std::vector<long long>> history(M);
        const int from = std::max(0, w - lookback);
        for (int m = 0; m < M; ++m)
          history[m].assign(sc.trace.counts[m].begin() + static_cast<long>(from) * S,
                            sc.trace.counts[m].begin() + static_cast<long>(w) * S);
        fc = predict_arrivals(spec, history, S, S, &actual.counts);
      }
      PlanContext ctx{&sc, w, initial};
      AllocationSequence dp = solve_dp(ctx, fc);
      engine::Space sp = engine::Space::build(ctx);
      auto enc = sp.encode(dp);
      o += std::string(w ? "," : "") + "{\"encode\":[";
      for (size_t i = 0; i < enc.size(); ++i) o += (i ? "," : "") + std::to_string(enc[i]);
      o += "],\"forecast\":[";
      for (int m = 0; m < M; ++m) {
        o += std::string(m ? "," : "") + "[";
        for (int s = 0; s < S; ++s) o += (s ? "," : "") + std::to_string(fc.counts[m][s]);
        o += "]";
      }
      o += "],\"obj\":\"" + hexbits(evaluate_plan(ctx, dp, fc.counts).total) + "\",\"realized\":\"" +
           hexbits(evaluate_plan(ctx, dp, actual.counts).total) + "\"}";
      initial = final_ranges(sc, dp);
    }
    return o + "]}";
  });
  std::printf("%s\n", out.c_str());
  return 0;
}

int cmd_replay_windows(int argc, char** argv) {
  if (argc < 4) return 2;
  std::string out = guarded([&] {
    Scenario sc = load_scenario(argv[2]);
    const uint64_t seed = std::strtoull(argv[3], nullptr, 10);
    std::optional<std::map<TaskId, std::set<SlotRange>>> initial;
    std::vector<EffectivePlan> plans;
    std::string o = "{\"encode\":[";
    for (int w = 0; w < sc.window_count; ++w) {
      PlanContext ctx{&sc, w, initial};
      ArrivalForecast fc = window_forecast(sc, w);
      AllocationSequence dp = solve_dp(ctx, fc);
      auto enc = engine::Space::build(ctx).encode(dp);
      o += std::string(w ? "," : "") + "[";
      for (size_t i = 0; i < enc.size(); ++i) o += (i ? "," : "") + std::to_string(enc[i]);
      o += "]";
      plans.push_back(EffectivePlan{dp, {}});
      initial = final_ranges(sc, dp);
    }
    Metrics mt = run_requests(sc, plans, seed);
    o += "],\"windows\":[";
    for (size_t w = 0; w < mt.windows.size(); ++w) {
      Metrics one;
      one.jobs = mt.windows[w].jobs;
      o += std::string(w ? "," : "") + jobs_json(one);
    }
    return o + "],\"totals\":" + jobs_json(mt) + "}";
  });
  std::printf("%s\n", out.c_str());
  return 0;
}

int cmd_gen_random(int argc, char** argv) {
  if (argc < 5) return 2;
  unsigned seed = static_cast<unsigned>(std::strtoul(argv[2], nullptr, 10));
  int count = std::atoi(argv[3]);
  std::string dir = argv[4];
  bool allow_drop = !(argc > 5 && std::string(argv[5]) == "--no-drop");
  std::mt19937 rng(seed);
  for (int i = 0; i < count; ++i) {
    Scenario sc = testutil::random_oracle_scenario(rng, allow_drop);
    std::string stem = "rnd_" + std::to_string(seed) + "_" + std::to_string(i);
    write_scenario_files(sc, dir, stem);
    std::printf("%s/%s.scn\n", dir.c_str(), stem.c_str());
  }
  return 0;
}

// Multi-tenant sibling of testutil::random_oracle_scenario (test_util.hpp:
// 104-181). RT tables are sparse (random subsets of sizes) so the option space
// stays small enough for the brute-force cross-check.
Scenario random_multi_scenario(std::mt19937& rng, int M, int S_lo, int S_hi, double est_cap) {
  static const std::vector<std::string> pool = {
      "config 4_2_1 4@0 2@4 1@6\n",         "config 4_1_1_1 4@0 1@4 1@5 1@6\n",
      "config 3_2_2 2@0 2@2 3@4\n",         "config 3_2_1_1 2@0 1@2 1@3 3@4\n",
      "config 3_1_1_1_1 1@0 1@1 1@2 1@3 3@4\n", "config 2_2_2_1 2@0 2@2 2@4 1@6\n",
      "config 2_2_1_1_1 2@0 2@2 1@4 1@5 1@6\n",
  };
  auto pick_real = [&](double lo, double hi) {
    return lo + (hi - lo) * (static_cast<double>(rng() % 10000) / 10000.0);
  };
  for (int attempt = 0; attempt < 2000; ++attempt) {
    int S = S_lo + static_cast<int>(rng() % static_cast<unsigned>(S_hi - S_lo + 1));
    // M >= 4 needs five slots (four anchored tenants + one retraining): draw
    // from the pool's tail (3_1_1_1_1, 2_2_2_1, 2_2_1_1_1)
    const int lo = M >= 4 ? 4 : 0;
    int nconfigs = 1 + static_cast<int>(rng() % (M >= 4 ? 2 : 3));
    std::set<int> chosen;
    while (static_cast<int>(chosen.size()) < nconfigs)
      chosen.insert(lo + static_cast<int>(rng() % static_cast<unsigned>(pool.size() - lo)));
    std::string text;
    for (int i : chosen) text += pool[i];
    Catalog cat = load_catalog_text(text);
    std::vector<ModelEntry> models;
    for (int m = 0; m < M; ++m) {
      ModelEntry e;
      e.profile.name = "t" + std::to_string(m);
      e.profile.gflops = pick_real(1.0, 20.0);
      e.profile.min_deploy_gpcs = M >= 4 ? 1 : 1 + static_cast<int>(rng() % 2);
      e.profile.latency_full = 0.01;
      e.profile.reconfig_overhead = std::vector<double>{0.0, 0.3, 0.7, 1.0}[rng() % 4];
      double cap = 4.0 + rng() % 8;
      for (int k = 1; k <= 7; ++k) {
        e.profile.capability[k] = cap;
        cap += rng() % 10;
      }
      // sparse nonincreasing RT table: few retraining sizes keep |O| small
      long long rt1 = 1 + static_cast<long long>(rng() % static_cast<unsigned>(S));
      long long drop = rng() % 2;
      for (int k = 1; k <= 7; ++k)
        if (rng() % 3 == 0) e.retraining.rt_table[k] = std::max<long long>(1, rt1 - drop * (k - 1));
      if (e.retraining.rt_table.empty() || (M >= 4 && !e.retraining.rt_table.count(1)))
        e.retraining.rt_table[1] = std::max<long long>(rt1, e.retraining.rt_table.empty() ? 1 : e.retraining.rt_table.begin()->second);
      double pre = pick_real(0.2, 0.9);
      double post = rng() % 4 == 0 ? pick_real(0.1, pre) : pick_real(pre, 1.0);
      e.retraining.accuracy_pre = {pre};
      e.retraining.accuracy_post = {post};
      models.push_back(std::move(e));
    }
    InferenceTrace trace;
    for (int m = 0; m < M; ++m) {
      std::vector<long long> counts;
      bool zero = rng() % 12 == 0;
      for (int s = 0; s < S; ++s) counts.push_back(zero ? 0 : rng() % 30);
      trace.counts.push_back(std::move(counts));
    }
    Scenario sc;
    try {
      sc = finalize_scenario(std::move(cat), std::move(models), std::move(trace), S, 1, 1.0);
    } catch (const Error& e) {
      if (std::getenv("MIGREF_GEN_DEBUG")) std::fprintf(stderr, "finalize: %s\n", e.what());
      continue;
    }
    PlanContext ctx{&sc, 0, std::nullopt};
    if (!precheck_scenario(ctx).empty()) {
      if (std::getenv("MIGREF_GEN_DEBUG")) std::fprintf(stderr, "precheck\n");
      continue;
    }
    auto space = engine::Space::build(ctx);
    if (std::pow(static_cast<double>(space.options.size()), S) > est_cap) {
      if (std::getenv("MIGREF_GEN_DEBUG")) std::fprintf(stderr, "estimate %zu^%d\n", space.options.size(), S);
      continue;
    }
    try {
      ArrivalForecast fc = window_forecast(sc, 0);
      (void)solve_dp(ctx, fc);
    } catch (const Error& e) {
      if (std::getenv("MIGREF_GEN_DEBUG")) std::fprintf(stderr, "solve: %s\n", e.code().c_str());
      continue;
    }
    return sc;
  }
  throw std::runtime_error("random_multi_scenario: no scenario found");
}

int cmd_gen_multi(int argc, char** argv) {
  if (argc < 9) return 2;
  unsigned seed = static_cast<unsigned>(std::strtoul(argv[2], nullptr, 10));
  int count = std::atoi(argv[3]);
  std::string dir = argv[4];
  int M = std::atoi(argv[5]), S_lo = std::atoi(argv[6]), S_hi = std::atoi(argv[7]);
  double est_cap = std::atof(argv[8]);
  std::mt19937 rng(seed);
  for (int i = 0; i < count; ++i) {
    Scenario sc = random_multi_scenario(rng, M, S_lo, S_hi, est_cap);
    std::string stem = "m" + std::to_string(M) + "_" + std::to_string(seed) + "_" + std::to_string(i);
    write_scenario_files(sc, dir, stem);
    std::printf("%s/%s.scn\n", dir.c_str(), stem.c_str());
  }
  return 0;
}

}  // namespace

extern "C" {
// CPU baseline entry for bench.py: one solve_dp of window `window` of the
// scenario file. Returns 0 on success, 1 on a migsim::Error (code copied).
int migref_solve_file(const char* scn, int window, int workers, double* seconds, double* objective,
                      int* encode, int encode_cap, int* encode_len, char* err_code, int err_cap) {
  try {
    Scenario sc = load_scenario(scn);
    PlanContext ctx{&sc, window, std::nullopt};
    ArrivalForecast fc = window_forecast(sc, window);
    SolveOptions opt;
    opt.workers = workers;
    auto t0 = std::chrono::steady_clock::now();
    AllocationSequence dp = solve_dp(ctx, fc, opt);
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *objective = evaluate_plan(ctx, dp, fc.counts).total;
    auto enc = engine::Space::build(ctx).encode(dp);
    *encode_len = static_cast<int>(enc.size());
    for (int i = 0; i < encode_cap && i < static_cast<int>(enc.size()); ++i) encode[i] = enc[i];
    return 0;
  } catch (const Error& e) {
    if (err_cap > 0) std::snprintf(err_code, err_cap, "%s", e.code().c_str());
    return 1;
  }
}
}

#ifndef MIGREF_NO_MAIN
int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: migref solve|gen-random ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  if (cmd == "solve") return cmd_solve(argc, argv);
  if (cmd == "gen-random") return cmd_gen_random(argc, argv);
  if (cmd == "gen-multi") return cmd_gen_multi(argc, argv);
  if (cmd == "replay") return cmd_replay(argc, argv);
  if (cmd == "preinit") return cmd_preinit(argc, argv);
  if (cmd == "drive") return cmd_drive(argc, argv);
  if (cmd == "replay-windows") return cmd_replay_windows(argc, argv);
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
#endif
