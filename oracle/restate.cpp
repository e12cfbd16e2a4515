// TEST INFRASTRUCTURE ONLY — the CPU restatement of the reference planner's
// hot path, used by tests/ and bench.py's cpu_baseline leg as a CHECKER. The
// product (paper_2407_13126_b200) never links or calls this file.
//
// Parity pinning: this restatement is checked against the unmodified reference
// (oracle/_ref/migref, built from /root/reference by oracle/Makefile) on the
// golden corpus in tests/golden/ (tests/test_oracle.py). Each function cites
// the reference lines it restates (paths relative to proj/include/migsim/).
//
// Deliberate difference: packed statuses are kept in uint64_t end to end. The
// reference narrows them to int at solvers.hpp:359,401,414,461, which drops
// tenants >= 2; for M <= 2 both are identical because codes
// fit 16 bits and the upper half is zero.
//
// Built with -ffp-contract=off so x86 never contracts to FMA (the reference's
// Release build has no -march, hence no FMA either).
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "migsim_b200.h"

namespace {

constexpr int KM = MGS_MAX_MODELS;

struct Tables {  // engine::Tables (space.hpp:32-86)
  int S = 0, M = 0;
  std::vector<std::pair<int, int>> universe;  // uid -> (start, size), first-appearance order (:56-64)
  std::map<std::pair<int, int>, int> uid_of;
  double cap[KM][8]{};
  long long rt[KM][8]{};
  int floor_[KM]{};
  double loss[KM]{};  // reconfig_loss_fraction(psi) = psi < 1 ? psi : 1 (plan_types.hpp:68)
  double pre[KM]{}, post[KM]{};
  long long min_rt[KM]{};  // -1 if none (:79-83)
};

struct Option {  // engine::Option (space.hpp:100-114)
  int config = 0;
  std::array<int8_t, MGS_MAX_SLOTS> labels{};
  std::array<uint32_t, KM> mask{};
  std::array<double, KM> cap{};
  std::array<int8_t, KM> rsize{};
  int sig = 0;
};

struct Fail {
  int code;
  std::string msg;
  int step = 0;
  uint64_t frontier = 0;
  int model = -1;
};

void set_err(mgs_error* e, const Fail& f) {
  if (!e) return;
  e->code = f.code;
  e->step = f.step;
  e->frontier = f.frontier;
  e->model = f.model;
  std::snprintf(e->message, sizeof e->message, "%s", f.msg.c_str());
}

Tables build_tables(const mgs_lattice& lat, const mgs_tables& in) {
  Tables t;
  if (in.models > KM) throw Fail{MGS_ERR_INPUT_SCENARIO, "at most 4 models are supported"};  // :49-50
  t.S = in.steps;
  t.M = in.models;
  for (int c = 0; c < lat.n_configs; ++c)
    for (int i = lat.slot_offset[c]; i < lat.slot_offset[c + 1]; ++i) {
      std::pair<int, int> r{lat.slot_start[i], lat.slot_size[i]};
      if (!t.uid_of.count(r)) {
        t.uid_of[r] = static_cast<int>(t.universe.size());
        t.universe.push_back(r);
      }
    }
  if (t.universe.size() > 30) throw Fail{MGS_ERR_INPUT_CATALOG, "catalog has more than 30 distinct instances"};  // :65
  for (int m = 0; m < t.M; ++m) {
    for (int k = 0; k < 8; ++k) {
      t.cap[m][k] = in.cap_by_size[m][k];
      t.rt[m][k] = in.rt_by_size[m][k];
    }
    t.floor_[m] = in.floor_gpcs[m];
    t.loss[m] = in.psi[m] < 1.0 ? in.psi[m] : 1.0;
    t.pre[m] = in.acc_pre[m];
    t.post[m] = in.acc_post[m];
    t.min_rt[m] = -1;
    for (int k = 1; k <= 7; ++k) {
      long long r = t.rt[m][k];
      if (r >= 1 && r <= t.S && (t.min_rt[m] < 0 || r < t.min_rt[m])) t.min_rt[m] = r;
    }
  }
  return t;
}

// Space::build (space.hpp:126-210): per configuration in catalog order, a
// depth-first product over per-slot labels in ascending order with per-slot
// admissibility; emitted options are lexicographic.
std::vector<Option> enumerate(const mgs_lattice& lat, const Tables& t) {
  std::vector<Option> out;
  for (int c = 0; c < lat.n_configs; ++c) {
    const int base = lat.slot_offset[c], n = lat.slot_offset[c + 1] - base;
    std::vector<int> uid(n);
    for (int i = 0; i < n; ++i) uid[i] = t.uid_of.at({lat.slot_start[base + i], lat.slot_size[base + i]});
    std::array<int8_t, MGS_MAX_SLOTS> labels{};
    const int maxl = 2 * t.M;
    auto admissible = [&](int depth, int lab) {  // :178-192
      if (lab == 0) return true;
      int m = (lab - 1) / 2, size = lat.slot_size[base + depth];
      if ((lab - 1) % 2 == 0) return t.cap[m][size] > 0.0;
      long long r = t.rt[m][size];
      if (!(r >= 1 && r <= t.S)) return false;
      for (int i = 0; i < depth; ++i)
        if (labels[i] == lab) return false;
      return true;
    };
    auto emit = [&]() {  // :141-165
      Option o;
      o.config = c;
      o.labels = labels;
      bool anchored[KM] = {};
      for (int i = 0; i < n; ++i) {
        int lab = labels[i];
        if (!lab) continue;
        int m = (lab - 1) / 2, size = lat.slot_size[base + i];
        if ((lab - 1) % 2 == 0) {
          o.mask[m] |= 1u << uid[i];
          o.cap[m] += t.cap[m][size];  // summed in slot (slice_start) order
          if (size >= t.floor_[m]) anchored[m] = true;
        } else {
          o.rsize[m] = static_cast<int8_t>(size);
        }
      }
      for (int m = 0; m < t.M; ++m)
        if (!anchored[m]) return;
      int sig = 0;
      for (int m = t.M - 1; m >= 0; --m) sig = sig * 8 + o.rsize[m];  // Option::signature :109-113
      o.sig = sig;
      out.push_back(o);
    };
    // recursive form of the iterative product (:167-204)
    auto rec = [&](auto&& self, int depth) -> void {
      for (int lab = 0; lab <= maxl; ++lab) {
        if (!admissible(depth, lab)) continue;
        labels[depth] = static_cast<int8_t>(lab);
        if (depth + 1 == n) emit();
        else self(self, depth + 1);
      }
      labels[depth] = 0;
    };
    if (n > 0) rec(rec, 0);
  }
  return out;
}

// StatusCodec (space.hpp:259-298), with 64-bit packing throughout.
struct Codec {
  int S, M;
  static constexpr int done = 1;
  int running(int k, long long rem) const { return 2 + (k - 1) * S + static_cast<int>(rem - 1); }
  static bool is_running(int c) { return c >= 2; }
  int run_size(int c) const { return (c - 2) / S + 1; }
  long long run_rem(int c) const { return (c - 2) % S + 1; }
  uint64_t pack(const std::array<int, KM>& st) const {
    uint64_t key = 0;
    for (int m = M - 1; m >= 0; --m) key = (key << 16) | static_cast<uint64_t>(st[m]);
    return key;
  }
  std::array<int, KM> unpack(uint64_t key) const {
    std::array<int, KM> st{};
    for (int m = 0; m < M; ++m) {
      st[m] = static_cast<int>(key & 0xffff);
      key >>= 16;
    }
    return st;
  }
  int advance(const Tables& t, int m, int status, int size, int s) const {  // :286-297
    if (is_running(status)) {
      if (size != run_size(status)) return -1;
      return run_rem(status) == 1 ? done : running(size, run_rem(status) - 1);
    }
    if (status == done) return size == 0 ? done : -1;
    if (size == 0) return 0;
    long long r = t.rt[m][size];
    if (r < 1 || s + r > t.S) return -1;
    return r == 1 ? done : running(size, r - 1);
  }
};

inline double eff_cap(double raw, double loss) { return raw - loss * raw; }           // plan_types.hpp:69
inline double thr_of(double recv, double cap) { return recv < cap ? recv : cap; }      // plan_types.hpp:70-72
inline bool better(double va, uint64_t la, double vb, uint64_t lb) {                  // dp_better solvers.hpp:123-126
  if (va != vb) return va > vb;
  return la < lb;
}

// precheck_scenario (solvers.hpp:27-69); message text as the reference
// builds it, with model names replaced by "model <m>" (the C++ drop-in
// re-renders them with names).
void precheck(const mgs_lattice& lat, const Tables& t, const std::vector<Option>& opts) {
  std::vector<Fail> out;
  for (int m = 0; m < t.M; ++m) {
    bool anchor = false;
    for (int i = 0; i < lat.slot_offset[lat.n_configs]; ++i)
      if (lat.slot_size[i] >= t.floor_[m]) anchor = true;
    if (!anchor) {
      out.push_back({MGS_ERR_DEPLOYMENT_FLOOR, "deployment-floor unsatisfiable: no catalog instance reaches " +
                                                   std::to_string(t.floor_[m]) + " GPCs for model <" + std::to_string(m) + ">", 0, 0, m});
      continue;
    }
    if (t.min_rt[m] < 0)
      out.push_back({MGS_ERR_RETRAINING_WINDOW, "model <" + std::to_string(m) + ">: every retraining time exceeds the window (" +
                                                    std::to_string(t.S) + " steps)", 0, 0, m});
  }
  if (!out.empty()) throw out.front();
  std::map<int, int> by_sig;
  for (const auto& o : opts) by_sig[o.sig]++;
  if (!by_sig.count(0))
    throw Fail{MGS_ERR_DEPLOYMENT_FLOOR,
               "deployment-floor unsatisfiable: no configuration deploys every inference task simultaneously"};
  for (int m = 0; m < t.M; ++m) {
    bool co = false;
    for (const auto& [sig, n] : by_sig)
      if ((sig >> (3 * m)) & 7) co = true;
    if (!co)
      throw Fail{MGS_ERR_NO_COEXISTENCE, "no-coexistence-configuration: no configuration runs <" + std::to_string(m) +
                                             ">:r alongside every inference task", 0, 0, m};
  }
}

struct Prepared {
  Tables t;
  std::vector<Option> opts;
  std::map<int, std::vector<int>> by_sig;  // Space::by_signature (:207-208)
};

Prepared prepare(const mgs_problem& p, bool check) {
  Prepared P;
  P.t = build_tables(p.lattice, p.tables);
  P.opts = enumerate(p.lattice, P.t);
  if (check) precheck(p.lattice, P.t, P.opts);
  for (size_t i = 0; i < P.opts.size(); ++i) P.by_sig[P.opts[i].sig].push_back(static_cast<int>(i));
  return P;
}

// ub_suffix (solvers.hpp:258-280) and the greedy incumbent (:282-322).
void goodput_reductions(const mgs_problem& p, const Prepared& P, std::vector<double>* ub, double* incumbent,
                        std::vector<int>* greedy) {
  const Tables& t = P.t;
  const int S = t.S, M = t.M;
  Codec codec{S, M};
  double acc_max[KM]{};
  for (int m = 0; m < M; ++m) acc_max[m] = std::max(t.pre[m], t.post[m]);
  ub->assign(S + 1, 0.0);
  for (int s = S - 1; s >= 0; --s) {
    double best = 0.0;
    for (const auto& o : P.opts) {
      double v = 0.0;
      for (int m = 0; m < M; ++m) v += acc_max[m] * thr_of(static_cast<double>(p.forecast[m * p.forecast_len + s]), o.cap[m]);
      best = std::max(best, v);
    }
    (*ub)[s] = (*ub)[s + 1] + best;
  }
  *incumbent = -std::numeric_limits<double>::infinity();
  greedy->assign(S, -1);
  std::array<int, KM> st{};
  std::array<uint32_t, KM> mask{};
  for (int m = 0; m < M; ++m) mask[m] = p.has_initial ? p.init_mask[m] : 0u;
  double value = 0.0;
  bool alive = true;
  for (int s = 0; s < S && alive; ++s) {
    bool charge = s > 0 || p.has_initial;
    double best_v = 0.0;
    int best_o = -1;
    std::array<int, KM> best_st{};
    for (size_t oi = 0; oi < P.opts.size(); ++oi) {
      const Option& o = P.opts[oi];
      std::array<int, KM> ns{};
      bool ok = true;
      for (int m = 0; m < M && ok; ++m) {
        ns[m] = codec.advance(t, m, st[m], o.rsize[m], s);
        ok = ns[m] >= 0 && !(ns[m] == 0 && (t.min_rt[m] < 0 || s + 1 + t.min_rt[m] > S));
      }
      if (!ok) continue;
      double v = value;
      for (int m = 0; m < M; ++m) {
        double acc = st[m] == Codec::done ? t.post[m] : t.pre[m];
        bool changed = charge && mask[m] != o.mask[m];
        double eff = eff_cap(o.cap[m], changed ? t.loss[m] : 0.0);
        v += thr_of(static_cast<double>(p.forecast[m * p.forecast_len + s]), eff) * acc;
      }
      if (best_o < 0 || v > best_v) {
        best_v = v;
        best_o = static_cast<int>(oi);
        best_st = ns;
      }
    }
    if (best_o < 0) {
      alive = false;
      break;
    }
    (*greedy)[s] = best_o;
    value = best_v;
    st = best_st;
    mask = P.opts[best_o].mask;
  }
  if (alive) {
    bool all_done = true;
    for (int m = 0; m < M; ++m) all_done = all_done && st[m] == Codec::done;
    if (all_done) *incumbent = value;
  }
}

struct State {  // DpState (solvers.hpp:99-120)
  uint64_t status = 0;
  std::array<uint32_t, KM> mask{};
  double value = 0.0;
  int parent = -1, option = -1;
  uint64_t lex = 0;
  uint32_t rank = 0;
};

struct KeyHash {
  size_t operator()(const std::pair<uint64_t, std::array<uint32_t, KM>>& k) const {
    uint64_t h = 1469598103934665603ull ^ k.first;
    for (uint32_t m : k.second) h = (h ^ m) * 1099511628211ull;
    return static_cast<size_t>(h ^ (h >> 29));
  }
};
struct MaskHash {
  size_t operator()(const std::array<uint32_t, KM>& k) const {
    uint64_t h = 14695981039346656037ull;
    for (uint32_t m : k) h = (h ^ m) * 1099511628211ull;
    return static_cast<size_t>(h ^ (h >> 31));
  }
};

bool status_dominates(const Codec& c, int a, int b) {  // solvers.hpp:128-134
  if (a == b) return true;
  if (a == Codec::done) return true;
  if (Codec::is_running(a) && Codec::is_running(b) && c.run_size(a) == c.run_size(b)) return c.run_rem(a) <= c.run_rem(b);
  return false;
}

// solve_dp (solvers.hpp:242-579), single-threaded (the reference's result is
// worker-independent, solver_test.cpp:149-162).
std::vector<int> solve(const mgs_problem& p, mgs_stats* stats) {
  if (p.tables.models < 1) throw Fail{MGS_ERR_ARGUMENT, "models must be >= 1"};
  Prepared P = prepare(p, true);
  const Tables& t = P.t;
  const int S = t.S, M = t.M;
  if (p.forecast_len != S) throw Fail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};  // :250-252
  Codec codec{S, M};
  std::array<uint32_t, KM> init_mask{};
  for (int m = 0; m < M; ++m) init_mask[m] = p.has_initial ? p.init_mask[m] : 0u;
  auto recv = [&](int m, int s) { return static_cast<double>(p.forecast[m * p.forecast_len + s]); };

  double acc_max[KM]{}, cap_max[KM]{};
  bool dominance_ok = true;
  for (int m = 0; m < M; ++m) {
    acc_max[m] = std::max(t.pre[m], t.post[m]);
    dominance_ok = dominance_ok && t.post[m] >= t.pre[m];
    for (const auto& o : P.opts) cap_max[m] = std::max(cap_max[m], o.cap[m]);
  }
  double band = 1e-9;
  for (int m = 0; m < M; ++m) band += t.loss[m] * cap_max[m] * acc_max[m];  // :266-267
  std::vector<double> ub;
  std::vector<int> greedy;
  double incumbent;
  goodput_reductions(p, P, &ub, &incumbent, &greedy);

  // dedup statistic: distinct inference-mask tuples per signature
  std::map<int, int> cand_per_sig;
  {
    std::map<int, std::vector<std::array<uint32_t, KM>>> tmp;
    for (const auto& o : P.opts) tmp[o.sig].push_back(o.mask);
    for (auto& [sig, v] : tmp) {
      std::sort(v.begin(), v.end());
      cand_per_sig[sig] = static_cast<int>(std::unique(v.begin(), v.end()) - v.begin());
    }
  }
  uint64_t n_cand = 0;
  for (auto& [sig, n] : cand_per_sig) n_cand += n;

  std::vector<std::vector<State>> F(S + 1);
  {
    State root;
    root.mask = init_mask;
    F[0] = {root};
  }
  struct Best {
    double value = -std::numeric_limits<double>::infinity();
    uint64_t lex = ~0ull;
    int idx = -1;
  };
  using SubKey = std::array<uint32_t, KM>;
  uint64_t tr_ref = 0, tr = 0, ftot = 0, fpeak = 0;

  const bool trace = std::getenv("MGS_ORACLE_TRACE") != nullptr;
  for (int s = 0; s < S; ++s) {
    const auto& cur = F[s];
    size_t n_units_step = 0;
    uint64_t tr_before = tr;
    if (cur.empty()) throw Fail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};  // :348
    const bool charge = s > 0 || p.has_initial;
    std::unordered_map<uint64_t, std::vector<int>> groups;  // :351-353
    for (size_t i = 0; i < cur.size(); ++i) groups[cur[i].status].push_back(static_cast<int>(i));

    std::unordered_map<std::pair<uint64_t, std::array<uint32_t, KM>>, State, KeyHash> merged;
    for (auto& [status, idxs] : groups) {
      std::array<int, KM> st = codec.unpack(status);
      // subset representatives (:367-378)
      std::vector<std::unordered_map<SubKey, Best, MaskHash>> by_subset(1u << M);
      for (int i : idxs) {
        for (unsigned sub = 0; sub < (1u << M); ++sub) {
          SubKey key{};
          for (int m = 0; m < M; ++m) key[m] = (sub & (1u << m)) ? cur[i].mask[m] : 0xdeadbeefu;
          Best& b = by_subset[sub][key];
          if (better(cur[i].value, cur[i].lex, b.value, b.lex)) b = {cur[i].value, cur[i].lex, i};
        }
      }
      // signatures compatible with this status (:379-411, allowed_sizes :79-97)
      std::array<std::vector<int>, KM> sizes;
      bool alive = true;
      for (int m = 0; m < M; ++m) {
        int c = st[m];
        if (Codec::is_running(c)) sizes[m] = {codec.run_size(c)};
        else if (c == Codec::done) sizes[m] = {0};
        else {
          if (t.min_rt[m] >= 0 && s + 1 + t.min_rt[m] <= S) sizes[m].push_back(0);
          for (int k = 1; k <= 7; ++k)
            if (t.rt[m][k] >= 1 && s + t.rt[m][k] <= S) sizes[m].push_back(k);
        }
        if (sizes[m].empty()) alive = false;
      }
      if (!alive) continue;
      std::array<int, KM> pick{};
      std::vector<std::pair<uint64_t, const std::vector<int>*>> units;
      auto rec = [&](auto&& self, int m) -> void {
        if (m == M) {
          int sig = 0;
          std::array<int, KM> ns{};
          for (int mm = M - 1; mm >= 0; --mm) sig = sig * 8 + sizes[mm][pick[mm]];
          for (int mm = 0; mm < M; ++mm) {
            ns[mm] = codec.advance(t, mm, st[mm], sizes[mm][pick[mm]], s);
            if (ns[mm] < 0 || (ns[mm] == 0 && (t.min_rt[mm] < 0 || s + 1 + t.min_rt[mm] > S))) return;
          }
          auto it = P.by_sig.find(sig);
          if (it == P.by_sig.end()) return;
          units.emplace_back(codec.pack(ns), &it->second);
          return;
        }
        for (size_t c = 0; c < sizes[m].size(); ++c) {
          pick[m] = static_cast<int>(c);
          self(self, m + 1);
        }
      };
      rec(rec, 0);
      // transitions (:420-471)
      n_units_step += units.size();
      for (auto& [packed, olist] : units) {
        tr_ref += olist->size();
        tr += cand_per_sig[P.opts[olist->front()].sig];
        for (int oi : *olist) {
          const Option& o = P.opts[oi];
          double bonus[KM]{};
          for (int m = 0; m < M; ++m) {
            double acc = st[m] == Codec::done ? t.post[m] : t.pre[m];
            double c_changed = thr_of(recv(m, s), eff_cap(o.cap[m], charge ? t.loss[m] : 0.0)) * acc;
            bonus[m] = charge ? thr_of(recv(m, s), o.cap[m]) * acc - c_changed : 0.0;
          }
          Best chosen;
          for (unsigned sub = 0; sub < (1u << M); ++sub) {  // :435-447
            SubKey key{};
            double extra = 0.0;
            for (int m = 0; m < M; ++m) {
              if (sub & (1u << m)) {
                key[m] = o.mask[m];
                extra += bonus[m];
              } else {
                key[m] = 0xdeadbeefu;
              }
            }
            auto it = by_subset[sub].find(key);
            if (it == by_subset[sub].end()) continue;
            double cand = it->second.value + extra;
            if (better(cand, it->second.lex, chosen.value, chosen.lex)) chosen = {cand, it->second.lex, it->second.idx};
          }
          if (chosen.idx < 0) continue;
          const State& pred = cur[chosen.idx];
          double v = pred.value;  // exact fold (:451-458)
          for (int m = 0; m < M; ++m) {
            bool changed = charge && pred.mask[m] != o.mask[m];
            double acc = st[m] == Codec::done ? t.post[m] : t.pre[m];
            v += thr_of(recv(m, s), eff_cap(o.cap[m], changed ? t.loss[m] : 0.0)) * acc;
          }
          if (v + ub[s + 1] < incumbent) continue;  // :459
          State ns;
          ns.status = packed;
          ns.mask = o.mask;
          ns.value = v;
          ns.parent = chosen.idx;
          ns.option = oi;
          ns.lex = (static_cast<uint64_t>(pred.rank) << 32) | static_cast<uint64_t>(oi);
          auto [it2, ins] = merged.emplace(std::make_pair(ns.status, ns.mask), ns);
          if (!ins && better(ns.value, ns.lex, it2->second.value, it2->second.lex)) it2->second = ns;
        }
      }
    }
    std::vector<State> next;
    next.reserve(merged.size());
    for (auto& [k, st] : merged) next.push_back(st);
    size_t n_merged = next.size();
    {  // band (:499-511)
      std::unordered_map<uint64_t, double> best;
      for (const auto& st : next) {
        auto [it, ins] = best.emplace(st.status, st.value);
        if (!ins) it->second = std::max(it->second, st.value);
      }
      std::vector<State> kept;
      for (auto& st : next)
        if (st.value >= best[st.status] - band) kept.push_back(st);
      next.swap(kept);
    }
    if (dominance_ok) {  // (:514-537)
      std::unordered_map<SubKey, std::vector<int>, MaskHash> by_mask;
      for (size_t i = 0; i < next.size(); ++i) by_mask[next[i].mask].push_back(static_cast<int>(i));
      std::vector<char> dead(next.size(), 0);
      for (auto& [mk, idxs] : by_mask) {
        if (idxs.size() > 64) continue;
        for (int a : idxs) {
          if (dead[a]) continue;
          auto sa = codec.unpack(next[a].status);
          for (int b : idxs) {
            if (a == b || dead[b] || dead[a]) continue;
            auto sb = codec.unpack(next[b].status);
            bool dom = true;
            for (int m = 0; m < M && dom; ++m) dom = status_dominates(codec, sa[m], sb[m]);
            if (dom && better(next[a].value, next[a].lex, next[b].value, next[b].lex)) dead[b] = 1;
          }
        }
      }
      std::vector<State> kept;
      for (size_t i = 0; i < next.size(); ++i)
        if (!dead[i]) kept.push_back(next[i]);
      next.swap(kept);
    }
    if (next.size() > p.state_budget)  // :539-542
      throw Fail{MGS_ERR_STATE_BUDGET,
                 "dynamic-program frontier reached " + std::to_string(next.size()) + " states at step " +
                     std::to_string(s + 1) + " (budget " + std::to_string(p.state_budget) + ")",
                 s + 1, next.size()};
    std::vector<int> order(next.size());  // ranks (:544-548)
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return next[a].lex < next[b].lex; });
    for (size_t r = 0; r < order.size(); ++r) next[order[r]].rank = static_cast<uint32_t>(r);
    if (trace) {
      // detailed distribution stats for kernel design
      size_t gh[4] = {0, 0, 0, 0};
      for (auto& [st_, idxs] : groups) gh[idxs.size() <= 32 ? 0 : idxs.size() <= 128 ? 1 : idxs.size() <= 1024 ? 2 : 3]++;
      std::unordered_map<int, int> kids;
      for (auto& st_ : next) kids[st_.parent]++;
      size_t kh[4] = {0, 0, 0, 0}; int kmax = 0;
      for (auto& [p_, c_] : kids) { kh[c_ <= 1 ? 0 : c_ <= 32 ? 1 : c_ <= 256 ? 2 : 3]++; kmax = std::max(kmax, c_); }
      std::unordered_map<SubKey, int, MaskHash> pc;
      for (auto& st_ : next) pc[st_.mask]++;
      size_t db = 0, dm = 0;
      for (auto& [k_, c_] : pc) if (c_ >= 2 && c_ <= 64) { db++; dm += c_; }
      std::fprintf(stderr, "  groups<=32:%zu <=128:%zu <=1024:%zu >1024:%zu | kids 1:%zu <=32:%zu <=256:%zu >256:%zu max %d | dom buckets %zu members %zu of %zu pids\n",
                   gh[0], gh[1], gh[2], gh[3], kh[0], kh[1], kh[2], kh[3], kmax, db, dm, pc.size());
    }
    if (trace) {
      size_t gmax = 0;
      for (auto& [st_, idxs] : groups) gmax = std::max(gmax, idxs.size());
      std::unordered_map<uint64_t, int> ns_count;
      for (auto& st_ : next) ns_count[st_.status]++;
      std::fprintf(stderr, "step %d frontier %zu groups %zu gmax %zu units %zu tr %llu merged %zu kept %zu nsgroups %zu\n", s,
                   cur.size(), groups.size(), gmax, n_units_step, (unsigned long long)(tr - tr_before), n_merged, next.size(), ns_count.size());
    }
    ftot += next.size();
    fpeak = std::max<uint64_t>(fpeak, next.size());
    F[s + 1] = std::move(next);
  }
  std::array<int, KM> done{};
  for (int m = 0; m < M; ++m) done[m] = Codec::done;
  const uint64_t all_done = codec.pack(done);
  const State* best = nullptr;
  for (const auto& st : F[S])
    if (st.status == all_done && (!best || better(st.value, st.lex, best->value, best->lex))) best = &st;
  if (!best) throw Fail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};
  std::vector<int> chosen(S);
  const State* sp = best;
  for (int s = S - 1; s >= 0; --s) {
    chosen[s] = sp->option;
    sp = s > 0 ? &F[s][sp->parent] : nullptr;
  }
  if (stats) {
    stats->options = P.opts.size();
    stats->candidates = n_cand;
    stats->transitions_ref = tr_ref;
    stats->transitions = tr;
    stats->frontier_total = ftot;
    stats->frontier_peak = fpeak;
  }
  return chosen;
}

// evaluate_plan(verify=false) over option indices (evaluate.hpp:153-210).
double evaluate(const mgs_problem& p, const Prepared& P, const int32_t* plan, const int64_t* arrivals, int alen,
                double* thr_out) {
  const Tables& t = P.t;
  const int S = t.S, M = t.M;
  int finish_after[KM];
  for (int m = 0; m < M; ++m) {
    finish_after[m] = std::numeric_limits<int>::max();
    for (int s = S - 1; s >= 0; --s)
      if (P.opts[plan[s]].rsize[m] > 0) {
        finish_after[m] = s + 1;
        break;
      }
  }
  double total = 0.0;
  for (int s = 0; s < S; ++s) {
    const Option& o = P.opts[plan[s]];
    for (int m = 0; m < M; ++m) {
      bool changed = s == 0 ? (p.has_initial && o.mask[m] != p.init_mask[m]) : (o.mask[m] != P.opts[plan[s - 1]].mask[m]);
      double eff = eff_cap(o.cap[m], changed ? t.loss[m] : 0.0);
      double thr = thr_of(static_cast<double>(arrivals[m * alen + s]), eff);
      double acc = s >= finish_after[m] ? t.post[m] : t.pre[m];
      total += thr * acc;
      if (thr_out) thr_out[s * M + m] = thr;
    }
  }
  return total;
}

}  // namespace

extern "C" {

int oracle_enumerate(const mgs_lattice* lat, const mgs_tables* tab, int64_t* n, int64_t cap, int32_t* config,
                     int8_t* labels, uint32_t* mask, double* icap, int8_t* rsize, mgs_error* err) {
  try {
    Tables t = build_tables(*lat, *tab);
    auto opts = enumerate(*lat, t);
    *n = static_cast<int64_t>(opts.size());
    for (int64_t i = 0; i < cap && i < *n; ++i) {
      const Option& o = opts[i];
      if (config) config[i] = o.config;
      for (int k = 0; k < MGS_MAX_SLOTS; ++k)
        if (labels) labels[i * MGS_MAX_SLOTS + k] = o.labels[k];
      for (int m = 0; m < KM; ++m) {
        if (mask) mask[i * KM + m] = o.mask[m];
        if (icap) icap[i * KM + m] = o.cap[m];
        if (rsize) rsize[i * KM + m] = o.rsize[m];
      }
    }
    return 0;
  } catch (const Fail& f) {
    set_err(err, f);
    return f.code;
  }
}

int oracle_goodput_table(const mgs_problem* p, double* ub, double* incumbent, int32_t* greedy, mgs_error* err) {
  try {
    Prepared P = prepare(*p, false);
    std::vector<double> u;
    std::vector<int> g;
    goodput_reductions(*p, P, &u, incumbent, &g);
    for (size_t i = 0; i < u.size(); ++i) ub[i] = u[i];
    if (greedy)
      for (size_t i = 0; i < g.size(); ++i) greedy[i] = g[i];
    return 0;
  } catch (const Fail& f) {
    set_err(err, f);
    return f.code;
  }
}

int oracle_solve_window(const mgs_problem* p, int32_t* out_option, double* objective, mgs_stats* stats,
                        mgs_error* err) {
  try {
    auto chosen = solve(*p, stats);
    for (size_t s = 0; s < chosen.size(); ++s) out_option[s] = chosen[s];
    if (objective) {
      Prepared P = prepare(*p, false);
      *objective = evaluate(*p, P, out_option, p->forecast, p->forecast_len, nullptr);
    }
    return 0;
  } catch (const Fail& f) {
    set_err(err, f);
    return f.code;
  }
}

int oracle_evaluate(const mgs_problem* p, const int32_t* plan, const int64_t* arrivals, int32_t arrivals_len,
                    double* total, double* thr, mgs_error* err) {
  try {
    Prepared P = prepare(*p, false);
    if (arrivals_len < P.t.S) throw Fail{MGS_ERR_INPUT_ARRIVALS, "arrivals shorter than the window"};
    for (int s = 0; s < P.t.S; ++s)
      if (plan[s] < 0 || plan[s] >= static_cast<int32_t>(P.opts.size())) throw Fail{MGS_ERR_ARGUMENT, "option index out of range"};
    *total = evaluate(*p, P, plan, arrivals, arrivals_len, thr);
    return 0;
  } catch (const Fail& f) {
    set_err(err, f);
    return f.code;
  }
}
}
