// plan_horizon: the per-window planning loop over a long horizon, in C++ on
// the reference's own planner API (the per-window loop SPEC.md:484 describes
// and the reference's CLI placeholder, proj/tools/main.cpp:4-7, leaves out),
// with a sliding lookahead, a reconfiguration-cost (psi) sweep, and the work
// sharded over the GPUs of one box (one process per GPU, NCCL through the
// library's C ABI).
//
//   plan_horizon <scenario.scn>... [--predictor oracle|persistence|ewma:<a>]
//                [--lookback L] [--psi v1,v2,...] [--windows W]
//                [--world N --rank R --id-file PATH] [--device D]
//
// Units are (scenario, psi) pairs; psi replaces every tenant's
// reconfig_overhead. For window w of every unit:
//   forecast = predict_arrivals(predictor, the last L windows of history,
//              S, S, actual window-w counts)        predictor.hpp:53-91
//              (the lookahead slides with the window; window 0 and the
//              oracle predictor use the actual counts)
//   plans    = mgs_solve_batch_sharded over all units: rank r solves its
//              block as batched lanes, the plans are all-gathered   (GPU)
//   initial  = final_ranges(plan)                   evaluate.hpp:213-226
//   objective / realized = evaluate_plan on forecast / actual counts (GPU,
//              the drop-in evaluate.hpp)
// Rank 0 prints one JSON object: per unit and window the plan encoding
// (Space::encode), objective and realized Goodput bits; per psi the realized
// total over the units; the best psi (per-shard best combined with
// mgs_shard_best: all-reduce(max) over NVLink).
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>

#include "migsim/solvers.hpp"
#include "migsim/workload.hpp"
#include "migsim_b200/device.hpp"

using namespace migsim;

namespace {

std::string hexbits(double v) {
  uint64_t b;
  std::memcpy(&b, &v, 8);
  char s[24];
  std::snprintf(s, sizeof s, "%016llx", static_cast<unsigned long long>(b));
  return s;
}

std::vector<double> parse_list(const std::string& text) {
  std::vector<double> out;
  std::stringstream ss(text);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(parse_real(tok, "psi"));
  return out;
}

// rank 0 publishes the NCCL id in a file; the others wait for it
void exchange_id(int rank, const std::string& path, uint8_t* id) {
  if (rank == 0) {
    if (mgs_nccl_unique_id(id) != MGS_OK) fail("device.nccl", "cannot create an NCCL unique id");
    const std::string tmp = path + ".tmp";
    std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<const char*>(id), MGS_NCCL_ID_BYTES);
    std::rename(tmp.c_str(), path.c_str());
    return;
  }
  for (int i = 0; i < 6000; ++i) {
    std::ifstream in(path, std::ios::binary);
    if (in && in.read(reinterpret_cast<char*>(id), MGS_NCCL_ID_BYTES)) return;
    std::this_thread::sleep_for(std::chrono::milliseconds(10));
  }
  fail("device.nccl", "timed out waiting for the NCCL id file " + path);
}

struct Unit {
  Scenario sc;
  double psi = -1.0;  // < 0: the scenario's own reconfig_overhead
  std::optional<std::map<TaskId, std::set<SlotRange>>> initial;
  std::vector<int32_t> opt_config;  // option -> configuration / labels (Space::build on the device)
  std::vector<int8_t> opt_labels;
  std::string json;
  double realized_total = 0.0;
  std::string error;
};

}  // namespace

int main(int argc, char** argv) {
  std::vector<std::string> paths;
  std::string predictor = "oracle", id_file = "/tmp/plan_horizon.ncclid";
  int lookback = 1 << 30, windows = -1, world = 1, rank = 0, device = -1;
  std::vector<double> psis;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) fail("input.argument", "missing value after " + a);
      return argv[++i];
    };
    if (a == "--predictor") predictor = next();
    else if (a == "--lookback") lookback = std::atoi(next().c_str());
    else if (a == "--psi") psis = parse_list(next());
    else if (a == "--windows") windows = std::atoi(next().c_str());
    else if (a == "--world") world = std::atoi(next().c_str());
    else if (a == "--rank") rank = std::atoi(next().c_str());
    else if (a == "--id-file") id_file = next();
    else if (a == "--device") device = std::atoi(next().c_str());
    else paths.push_back(a);
  }
  try {
    if (paths.empty()) fail("input.argument", "usage: plan_horizon <scenario.scn>... [options]");
    if (lookback < 1) fail("input.argument", "--lookback must be >= 1");
    const PredictorSpec spec = parse_predictor_spec(predictor);
    if (device < 0) device = rank;
    setenv("MIGSIM_B200_DEVICE", std::to_string(device).c_str(), 1);
    mgs_ctx* ctx = b200::context();
    if (world > 1) {
      uint8_t id[MGS_NCCL_ID_BYTES];
      exchange_id(rank, id_file, id);
      mgs_error err{};
      const int st = mgs_shard_init(ctx, world, rank, id, &err);
      if (st != MGS_OK) b200::rethrow(st, err);
    }
    // units = scenarios x psi points, in that order on every rank
    std::vector<Unit> units;
    for (const auto& p : paths) {
      const Scenario sc = load_scenario(p);
      if (psis.empty()) psis.push_back(-1.0);
      for (double psi : psis) {
        Unit u;
        u.sc = sc;
        u.psi = psi;
        if (psi >= 0.0)
          for (auto& e : u.sc.models) e.profile.reconfig_overhead = psi;
        units.push_back(std::move(u));
      }
    }
    const int W = windows > 0 ? std::min(windows, units[0].sc.window_count) : units[0].sc.window_count;
    for (const auto& u : units)
      if (u.sc.window_count < W || u.sc.window_size != units[0].sc.window_size)
        fail("input.argument", "scenarios must share the window size and have >= W windows");
    const int S = units[0].sc.window_size;
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::string> unit_windows(units.size());
    for (int w = 0; w < W; ++w) {
      std::vector<b200::Problem> probs;
      std::vector<ArrivalForecast> fcs, actuals;
      probs.reserve(units.size());
      for (auto& u : units) {
        const int M = static_cast<int>(u.sc.models.size());
        ArrivalForecast actual;
        for (int m = 0; m < M; ++m) actual.counts.push_back(u.sc.window_arrivals(m, w));
        ArrivalForecast fc;
        if (spec.kind == PredictorKind::Oracle || w == 0) {
          fc = predict_arrivals(PredictorSpec{}, {}, S, S, &actual.counts);
        } else {  // the sliding lookahead: forecast from the last `lookback` windows
          const int from = std::max(0, w - lookback);
          std::vector<std::vector<long long>> history(M);
          for (int m = 0; m < M; ++m)
            history[m].assign(u.sc.trace.counts[m].begin() + static_cast<long>(from) * S,
                              u.sc.trace.counts[m].begin() + static_cast<long>(w) * S);
          fc = predict_arrivals(spec, history, S, S, &actual.counts);
        }
        PlanContext pc{&u.sc, w, u.initial};
        probs.emplace_back(pc, &fc, 4000000, 1);
        fcs.push_back(std::move(fc));
        actuals.push_back(std::move(actual));
      }
      // Problem keeps pointers into its own vectors: re-point after the moves
      std::vector<mgs_problem> flat;
      for (size_t i = 0; i < probs.size(); ++i) {
        auto& pb = probs[i];
        pb.p.lattice.slot_offset = pb.slot_offset.data();
        pb.p.lattice.slot_size = pb.slot_size.data();
        pb.p.lattice.slot_start = pb.slot_start.data();
        pb.p.forecast = pb.forecast.data();
        flat.push_back(pb.p);
      }
      const int n = static_cast<int>(units.size());
      std::vector<int32_t> opt(static_cast<size_t>(n) * S), status(n);
      std::vector<double> obj(n);
      mgs_error err{};
      const int st = mgs_solve_batch_sharded(ctx, flat.data(), n, S, opt.data(), obj.data(), status.data(), &err);
      if (st != MGS_OK) b200::rethrow(st, err);
      for (int i = 0; i < n; ++i) {
        Unit& u = units[i];
        if (!u.error.empty()) continue;
        if (status[i] != MGS_OK) {
          u.error = mgs_status_code(status[i]);
          continue;
        }
        if (u.opt_config.empty()) {  // the option space of this unit's lattice + tables
          int64_t no = 0;
          mgs_error e2{};
          int rc = mgs_enumerate(ctx, &flat[i].lattice, &flat[i].tables, &no, 0, nullptr, nullptr, nullptr, nullptr,
                                 nullptr, &e2);
          if (rc != MGS_OK) b200::rethrow(rc, e2);
          u.opt_config.resize(no);
          u.opt_labels.resize(static_cast<size_t>(no) * MGS_MAX_SLOTS);
          rc = mgs_enumerate(ctx, &flat[i].lattice, &flat[i].tables, &no, no, u.opt_config.data(), u.opt_labels.data(),
                             nullptr, nullptr, nullptr, &e2);
          if (rc != MGS_OK) b200::rethrow(rc, e2);
        }
        std::vector<int32_t> cfg(S);
        std::vector<int8_t> lab(static_cast<size_t>(S) * MGS_MAX_SLOTS);
        for (int s = 0; s < S; ++s) {
          const int o = opt[static_cast<size_t>(i) * S + s];
          cfg[s] = u.opt_config[o];
          std::memcpy(&lab[static_cast<size_t>(s) * MGS_MAX_SLOTS], &u.opt_labels[static_cast<size_t>(o) * MGS_MAX_SLOTS],
                      MGS_MAX_SLOTS);
        }
        PlanContext pc{&u.sc, w, u.initial};
        const AllocationSequence seq = b200::to_sequence(pc, cfg, lab);
        const double objective = evaluate_plan(pc, seq, fcs[i].counts, nullptr, false).total;
        const double realized = evaluate_plan(pc, seq, actuals[i].counts, nullptr, false).total;
        u.realized_total += realized;
        engine::Space sp;
        sp.tables = probs[i].t;
        const auto enc = sp.encode(seq);
        std::string o = std::string(w ? "," : "") + "{\"encode\":[";
        for (size_t k = 0; k < enc.size(); ++k) o += (k ? "," : "") + std::to_string(enc[k]);
        o += "],\"obj\":\"" + hexbits(objective) + "\",\"realized\":\"" + hexbits(realized) + "\"}";
        unit_windows[i] += o;
        u.initial = final_ranges(u.sc, seq);
      }
    }
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    // per-psi realized totals (identical on every rank: every rank holds every plan);
    // the best psi: each rank proposes the best of the psi points it owns (j % world),
    // combined with an all-reduce(max) over the ranks
    const int P = static_cast<int>(psis.size());
    std::vector<double> per_psi(P, 0.0);
    std::vector<int> failed(P, 0);
    for (size_t i = 0; i < units.size(); ++i) {
      per_psi[i % P] += units[i].realized_total;
      failed[i % P] += units[i].error.empty() ? 0 : 1;
    }
    double mine = 0.0;
    int mine_j = -1;
    for (int j = rank; j < P; j += world)
      if (!failed[j] && (mine_j < 0 || per_psi[j] > mine)) {
        mine = per_psi[j];
        mine_j = j;
      }
    double best = mine;
    int32_t owner = 0;
    if (world > 1) {
      mgs_error err{};
      const int st = mgs_shard_best(ctx, mine, &best, &owner, &err);
      if (st != MGS_OK) b200::rethrow(st, err);
    }
    int best_j = -1;
    for (int j = 0; j < P; ++j)
      if (!failed[j] && per_psi[j] == best && best_j < 0) best_j = j;
    if (rank == 0) {
      std::string o = "{\"world\":" + std::to_string(world) + ",\"windows\":" + std::to_string(W) +
                      ",\"seconds\":" + std::to_string(secs) + ",\"predictor\":\"" + spec.str() +
                      "\",\"lookback\":" + std::to_string(std::min(lookback, W)) + ",\"units\":[";
      for (size_t i = 0; i < units.size(); ++i) {
        o += std::string(i ? "," : "") + "{\"scenario\":\"" + paths[i / P] + "\",\"psi\":" +
             (units[i].psi >= 0 ? fmt_real(units[i].psi) : std::string("null"));
        if (!units[i].error.empty()) o += ",\"error\":\"" + units[i].error + "\"";
        o += ",\"realized_total\":\"" + hexbits(units[i].realized_total) + "\",\"windows\":[" + unit_windows[i] + "]}";
      }
      o += "],\"per_psi\":[";
      for (int j = 0; j < P; ++j)
        o += std::string(j ? "," : "") + "{\"psi\":" + (psis[j] >= 0 ? fmt_real(psis[j]) : std::string("null")) +
             ",\"realized_total\":" + fmt_real(per_psi[j]) + ",\"failed_units\":" + std::to_string(failed[j]) + "}";
      o += "],\"best_psi\":" + (best_j >= 0 && psis[best_j] >= 0 ? fmt_real(psis[best_j]) : std::string("null")) +
           ",\"best_realized_total\":" + fmt_real(best) + ",\"best_owner_rank\":" + std::to_string(owner) + "}";
      std::printf("%s\n", o.c_str());
    }
    return 0;
  } catch (const Error& e) {
    std::fprintf(stderr, "plan_horizon: %s: %s\n", e.code().c_str(), e.what());
    return 1;
  }
}
