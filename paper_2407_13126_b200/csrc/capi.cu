// C ABI (include/migsim_b200.h): thin POD layer over the device planner.
// Every entry point catches planner / CUDA failures and maps them to the
// reference's error codes; nothing here falls back to a CPU computation.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <new>

#include <functional>

#include "ctx.cuh"


namespace mgs {
bool solve_dp_v2_supported(const Prepared& pr, const DevSpace& sp);
void solve_dp_v2(Ctx& c, const mgs_problem& p, const Prepared& pr, const DevSpace& sp, const double* d_recv,
                 const double* d_ub, const double* d_incumbent, SolveOut& out);
void evaluate_batch(Ctx& c, const Prepared& pr, const DevSpace& sp, const int32_t* d_plans, int n_plans,
                    const int64_t* d_arr, int n_traces, double* d_total, double* d_thr, const uint8_t* d_overrides);
}

namespace {

using mgs::Ctx;
using mgs::PlanFail;

void fill_err(mgs_error* e, int code, const std::string& msg, int step = 0, uint64_t frontier = 0, int model = -1) {
  if (!e) return;
  e->code = code;
  e->step = step;
  e->frontier = frontier;
  e->model = model;
  std::snprintf(e->message, sizeof e->message, "%s", msg.c_str());
}

template <class F>
int guarded(mgs_error* err, F&& f) {
  if (err) fill_err(err, MGS_OK, "");
  try {
    f();
    return MGS_OK;
  } catch (const PlanFail& pf) {
    fill_err(err, pf.code, pf.msg, pf.step, pf.frontier, pf.model);
    return pf.code;
  } catch (const mgs::CudaFail& cf) {
    fill_err(err, MGS_ERR_CUDA,
             std::string("CUDA error ") + cudaGetErrorString(cf.err) + " at " + cf.what + ":" + std::to_string(cf.line));
    return MGS_ERR_CUDA;
  } catch (const std::bad_alloc&) {
    fill_err(err, MGS_ERR_CUDA, "host allocation failed");
    return MGS_ERR_CUDA;
  }
}

mgs::Prepared prepare_problem(const mgs_problem& p) {
  mgs::Prepared pr = mgs::prepare_tables(p.lattice, p.tables);
  pr.has_initial = p.has_initial ? 1 : 0;
  for (int m = 0; m < MGS_MAX_MODELS; ++m) pr.init_mask[m] = p.has_initial ? p.init_mask[m] : 0u;
  return pr;
}

__global__ void k_to_double(const int64_t* in, double* out, int n) {  // static_cast<double>(count)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = static_cast<double>(in[i]);
}

// forecast [M][forecast_len] -> device doubles [M][S]
double* upload_forecast(Ctx& c, const mgs_problem& p, int M, int S) {
  if (!p.forecast) throw PlanFail{MGS_ERR_ARGUMENT, "forecast is null"};
  int64_t* d_i = c.buf<int64_t>("forecast_i64", static_cast<size_t>(M) * S);
  double* d_f = c.buf<double>("forecast_f64", static_cast<size_t>(M) * S);
  if (p.forecast_len == S) {
    MGS_CUDA_OK(cudaMemcpyAsync(d_i, p.forecast, static_cast<size_t>(M) * S * 8, cudaMemcpyHostToDevice, c.stream));
  } else {
    MGS_CUDA_OK(cudaMemcpy2DAsync(d_i, S * 8, p.forecast, p.forecast_len * 8, static_cast<size_t>(S) * 8, M,
                                  cudaMemcpyHostToDevice, c.stream));
  }
  k_to_double<<<mgs::ceil_div(M * S, 256), 256, 0, c.stream>>>(d_i, d_f, M * S);
  ++c.kernel_launches;
  return d_f;
}

// evaluate_plan(...).total of one plan on the device (forecast_i64 resident)
double plan_total(Ctx& c, const mgs::Prepared& pr, const mgs::DevSpace& sp, const std::vector<int32_t>& plan) {
  const int M = pr.t.M, S = pr.t.S;
  int32_t* d_plan = c.buf<int32_t>("plan_eval", S);
  double* d_total = c.buf<double>("plan_total", 1);
  MGS_CUDA_OK(cudaMemcpyAsync(d_plan, plan.data(), S * 4, cudaMemcpyHostToDevice, c.stream));
  int64_t* d_arr = c.buf<int64_t>("forecast_i64", static_cast<size_t>(M) * S);
  mgs::evaluate_batch(c, pr, sp, d_plan, 1, d_arr, 1, d_total, nullptr, nullptr);
  double* h = c.pinned.get<double>(1);
  MGS_CUDA_OK(cudaMemcpyAsync(h, d_total, 8, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  return *h;
}

void copy_plan_labels(Ctx& c, const mgs::DevSpace& sp, const std::vector<int32_t>& plan, int32_t* out_config,
                      int8_t* out_labels) {
  if (!out_config && !out_labels) return;
  std::vector<int32_t> cfg(sp.n_opt);
  std::vector<int8_t> lab(static_cast<size_t>(sp.n_opt) * MGS_MAX_SLOTS);
  MGS_CUDA_OK(cudaMemcpyAsync(cfg.data(), sp.opt_config, sp.n_opt * 4, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(lab.data(), sp.opt_labels, lab.size(), cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  for (size_t s = 0; s < plan.size(); ++s) {
    const int o = plan[s];
    if (out_config) out_config[s] = cfg[o];
    if (out_labels)
      for (int k = 0; k < MGS_MAX_SLOTS; ++k) out_labels[s * MGS_MAX_SLOTS + k] = lab[static_cast<size_t>(o) * MGS_MAX_SLOTS + k];
  }
}

// the chosen plan's options, configurations, labels and objective packed for
// one device->host copy: [S] int32 options | [S] int32 configs | [S][8] labels | total
__global__ void k_gather_plan(const int32_t* opt_config, const int8_t* opt_labels, const int32_t* plan,
                              const double* total, int S, uint8_t* out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < S) {
    const int o = plan[s];
    reinterpret_cast<int32_t*>(out)[s] = o;
    reinterpret_cast<int32_t*>(out)[S + s] = opt_config[o];
    for (int k = 0; k < MGS_MAX_SLOTS; ++k)
      out[static_cast<size_t>(S) * 8 + static_cast<size_t>(s) * MGS_MAX_SLOTS + k] =
          static_cast<uint8_t>(opt_labels[static_cast<size_t>(o) * MGS_MAX_SLOTS + k]);
  }
  if (s == 0) {
    const double v = *total;
    uint8_t* dst = out + static_cast<size_t>(S) * (8 + MGS_MAX_SLOTS);
    for (int b = 0; b < 8; ++b) dst[b] = reinterpret_cast<const uint8_t*>(&v)[b];
  }
}

void solve_one(Ctx& c, const mgs_problem& p, int32_t* out_option, int32_t* out_config, int8_t* out_labels,
               double* out_objective, mgs_stats* stats) {
  MGS_CUDA_OK(cudaEventRecord(c.ev0, c.stream));
  c.timer.reset();
  c.open_phase = -1;
  c.kernel_launches = 0;
  c.phase(0);
  mgs::Prepared pr = prepare_problem(p);
  mgs::DevSpace sp;
  mgs::build_space(c, p.lattice, pr, sp);
  mgs::precheck_space(c, p.lattice, pr, sp);  // throw_if_infeasible(precheck_scenario) first (solvers.hpp:245)
  const int M = pr.t.M, S = pr.t.S;
  if (p.forecast_len != S) throw PlanFail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};  // :250-252
  c.phase(1);
  double* d_recv = upload_forecast(c, p, M, S);
  double* d_ub = c.buf<double>("ub_suffix", S + 1);
  double* d_inc = c.buf<double>("incumbent", 1);
  int32_t* d_greedy = c.buf<int32_t>("greedy", S);
  mgs::goodput_reductions(c, pr, sp, d_recv, d_ub, d_inc, d_greedy);
  mgs::SolveOut out;
  if (mgs::solve_dp_v2_supported(pr, sp)) {
    c.phase(3);  // one persistent launch covers units..ranks
    mgs::solve_dp_v2(c, p, pr, sp, d_recv, d_ub, d_inc, out);
  } else {
    mgs::solve_dp(c, p, pr, sp, d_recv, d_ub, d_inc, out);
  }
  // objective = evaluate_plan(...).total of the chosen plan and the plan's
  // configurations / labels, gathered on the device; one read-back of
  // S*(4+4+8)+8 bytes for the whole solve
  c.phase(7);
  int32_t* d_plan = c.buf<int32_t>("plan_eval", S);
  if (out.d_options) {
    MGS_CUDA_OK(cudaMemcpyAsync(d_plan, out.d_options, S * 4, cudaMemcpyDeviceToDevice, c.stream));
  } else {
    MGS_CUDA_OK(cudaMemcpyAsync(d_plan, out.options.data(), S * 4, cudaMemcpyHostToDevice, c.stream));
  }
  double* d_total = c.buf<double>("plan_total", 1);
  int64_t* d_arr = c.buf<int64_t>("forecast_i64", static_cast<size_t>(M) * S);
  mgs::evaluate_batch(c, pr, sp, d_plan, 1, d_arr, 1, d_total, nullptr, nullptr);
  const size_t rb = static_cast<size_t>(S) * (4 + 4 + MGS_MAX_SLOTS) + 8;
  uint8_t* d_rb = c.buf<uint8_t>("plan_readback", rb);
  k_gather_plan<<<mgs::ceil_div(S, 128), 128, 0, c.stream>>>(sp.opt_config, sp.opt_labels, d_plan, d_total, S, d_rb);
  ++c.kernel_launches;
  uint8_t* h_rb = c.pinned.get<uint8_t>(rb);
  MGS_CUDA_OK(cudaMemcpyAsync(h_rb, d_rb, rb, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  out.options.assign(reinterpret_cast<const int32_t*>(h_rb), reinterpret_cast<const int32_t*>(h_rb) + S);
  const int32_t* h_cfg = reinterpret_cast<const int32_t*>(h_rb) + S;
  const int8_t* h_lab = reinterpret_cast<const int8_t*>(h_rb + static_cast<size_t>(S) * 8);
  double total = 0.0;
  std::memcpy(&total, h_rb + static_cast<size_t>(S) * (8 + MGS_MAX_SLOTS), 8);
  if (out_config) std::memcpy(out_config, h_cfg, static_cast<size_t>(S) * 4);
  if (out_labels) std::memcpy(out_labels, h_lab, static_cast<size_t>(S) * MGS_MAX_SLOTS);
  c.phase(-1);
  MGS_CUDA_OK(cudaEventRecord(c.ev1, c.stream));
  MGS_CUDA_OK(cudaEventSynchronize(c.ev1));
  float ms = 0.f;
  MGS_CUDA_OK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
  out.stats.device_ms = ms;
  c.phase_totals(out.stats.phase_ms);
  out.stats.kernel_launches = c.kernel_launches;
  if (out_option)
    for (int s = 0; s < S; ++s) out_option[s] = out.options[s];
  if (out_objective) *out_objective = total;
  if (stats) *stats = out.stats;
}

}  // namespace

// the same exception-to-status mapping for the other translation units (shard.cu)
int mgs_guarded_call(mgs_error* err, const std::function<void()>& f) { return guarded(err, f); }

extern "C" {

const char* mgs_version(void) { return "paper_2407_13126_b200 0.1 (sm_100a)"; }

const char* mgs_status_code(int status) {
  switch (status) {
    case MGS_OK: return "ok";
    case MGS_ERR_INPUT_SCENARIO: return "input.scenario";
    case MGS_ERR_INPUT_CATALOG: return "input.catalog";
    case MGS_ERR_INPUT_FORECAST: return "input.forecast";
    case MGS_ERR_INPUT_ARRIVALS: return "input.arrivals";
    case MGS_ERR_DEPLOYMENT_FLOOR: return "infeasible.deployment-floor";
    case MGS_ERR_RETRAINING_WINDOW: return "infeasible.retraining-window";
    case MGS_ERR_NO_COEXISTENCE: return "infeasible.no-coexistence-configuration";
    case MGS_ERR_INFEASIBLE_JOINT: return "infeasible.joint";
    case MGS_ERR_STATE_BUDGET: return "planner.state-budget";
    case MGS_ERR_PLAN_INFEASIBLE: return "plan.infeasible";
    case MGS_ERR_CUDA: return "device.cuda";
    case MGS_ERR_ARGUMENT: return "input.argument";
    case MGS_ERR_BRUTEFORCE_CAP: return "planner.bruteforce-cap";
    case MGS_ERR_WINDOW_BOUNDARY: return "infeasible.window-boundary";
    default: return "unknown";
  }
}

int mgs_open(int device, mgs_ctx** out) {
  if (!out) return MGS_ERR_ARGUMENT;
  *out = nullptr;
  return guarded(nullptr, [&] {
    int n = 0;
    MGS_CUDA_OK(cudaGetDeviceCount(&n));
    if (device < 0 || device >= n) throw PlanFail{MGS_ERR_ARGUMENT, "no such CUDA device"};
    MGS_CUDA_OK(cudaSetDevice(device));
    auto* h = new mgs_ctx();
    h->c.device = device;
    MGS_CUDA_OK(cudaDeviceGetAttribute(&h->c.sm_count, cudaDevAttrMultiProcessorCount, device));
    MGS_CUDA_OK(cudaStreamCreateWithFlags(&h->c.own_stream, cudaStreamNonBlocking));
    h->c.stream = h->c.own_stream;
    MGS_CUDA_OK(cudaEventCreate(&h->c.ev0));
    MGS_CUDA_OK(cudaEventCreate(&h->c.ev1));
    *out = h;
  });
}

int mgs_set_stream(mgs_ctx* ctx, void* stream) {
  if (!ctx) return MGS_ERR_ARGUMENT;
  ctx->c.stream = stream ? static_cast<cudaStream_t>(stream) : ctx->c.own_stream;
  return MGS_OK;
}

void mgs_close(mgs_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->c.device);
  delete ctx;
}

int mgs_enumerate(mgs_ctx* ctx, const mgs_lattice* lattice, const mgs_tables* tables, int64_t* n_options, int64_t cap,
                  int32_t* config, int8_t* labels, uint32_t* infer_mask, double* infer_cap, int8_t* retrain_size,
                  mgs_error* err) {
  if (!ctx || !lattice || !tables || !n_options) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = mgs::prepare_tables(*lattice, *tables);
    mgs::DevSpace sp;
    mgs::build_space(c, *lattice, pr, sp);
    *n_options = sp.n_opt;
    const int64_t n = std::min<int64_t>(cap, sp.n_opt);
    if (n > 0) {
      if (config) MGS_CUDA_OK(cudaMemcpyAsync(config, sp.opt_config, n * 4, cudaMemcpyDeviceToHost, c.stream));
      if (labels) MGS_CUDA_OK(cudaMemcpyAsync(labels, sp.opt_labels, n * MGS_MAX_SLOTS, cudaMemcpyDeviceToHost, c.stream));
      if (infer_mask) MGS_CUDA_OK(cudaMemcpyAsync(infer_mask, sp.opt_mask, n * 16, cudaMemcpyDeviceToHost, c.stream));
      if (infer_cap) MGS_CUDA_OK(cudaMemcpyAsync(infer_cap, sp.opt_cap, n * 32, cudaMemcpyDeviceToHost, c.stream));
      if (retrain_size) MGS_CUDA_OK(cudaMemcpyAsync(retrain_size, sp.opt_rsize, n * 4, cudaMemcpyDeviceToHost, c.stream));
    }
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int mgs_goodput_table(mgs_ctx* ctx, const mgs_problem* p, double* ub_suffix, double* incumbent, int32_t* greedy_option,
                      mgs_error* err) {
  if (!ctx || !p) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    const int M = pr.t.M, S = pr.t.S;
    if (p->forecast_len < S) throw PlanFail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};
    if (sp.n_opt == 0) throw PlanFail{MGS_ERR_DEPLOYMENT_FLOOR, "no options"};
    double* d_recv = upload_forecast(c, *p, M, S);
    double* d_ub = c.buf<double>("ub_suffix", S + 1);
    double* d_inc = c.buf<double>("incumbent", 1);
    int32_t* d_greedy = c.buf<int32_t>("greedy", S);
    mgs::goodput_reductions(c, pr, sp, d_recv, d_ub, d_inc, d_greedy);
    if (ub_suffix) MGS_CUDA_OK(cudaMemcpyAsync(ub_suffix, d_ub, (S + 1) * 8, cudaMemcpyDeviceToHost, c.stream));
    if (incumbent) MGS_CUDA_OK(cudaMemcpyAsync(incumbent, d_inc, 8, cudaMemcpyDeviceToHost, c.stream));
    if (greedy_option) MGS_CUDA_OK(cudaMemcpyAsync(greedy_option, d_greedy, S * 4, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int mgs_precheck(mgs_ctx* ctx, const mgs_lattice* lattice, const mgs_tables* tables, mgs_violation* out, int32_t cap,
                 int32_t* n_out, mgs_error* err) {
  if (!ctx || !lattice || !tables || !n_out || cap < 0 || (cap > 0 && !out)) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = mgs::prepare_tables(*lattice, *tables);
    mgs::DevSpace sp;
    mgs::build_space(c, *lattice, pr, sp);
    const auto v = mgs::collect_violations(c, *lattice, pr, sp);
    *n_out = static_cast<int32_t>(v.size());
    for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) out[i] = mgs_violation{v[i].first, v[i].second};
  });
}

int mgs_bruteforce(mgs_ctx* ctx, const mgs_problem* p, double bruteforce_cap, int32_t* out_option, int32_t* out_config,
                   int8_t* out_labels, double* out_objective, mgs_error* err) {
  if (!ctx || !p) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    c.kernel_launches = 0;
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    mgs::precheck_space(c, p->lattice, pr, sp);  // throw_if_infeasible(precheck_scenario) (solvers.hpp:146)
    const int M = pr.t.M, S = pr.t.S;
    if (p->forecast_len != S) throw PlanFail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};
    const double estimate = std::pow(static_cast<double>(sp.n_opt), S);  // solvers.hpp:153-158
    if (estimate > bruteforce_cap) {
      char a[64], b[64];
      std::snprintf(a, sizeof a, "%.9g", estimate);
      std::snprintf(b, sizeof b, "%.9g", bruteforce_cap);
      throw PlanFail{MGS_ERR_BRUTEFORCE_CAP, std::string("brute-force space estimate ") + a + " (=" +
                                                 std::to_string(sp.n_opt) + "^" + std::to_string(S) +
                                                 ") exceeds the cap " + b};
    }
    double* d_recv = upload_forecast(c, *p, M, S);
    std::vector<int32_t> plan;
    if (!mgs::bruteforce(c, pr, sp, d_recv, plan))
      throw PlanFail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};
    const double total = plan_total(c, pr, sp, plan);
    copy_plan_labels(c, sp, plan, out_config, out_labels);
    if (out_option)
      for (int s = 0; s < S; ++s) out_option[s] = plan[s];
    if (out_objective) *out_objective = total;
  });
}

int mgs_window_boundary(mgs_ctx* ctx, const mgs_problem* p, int32_t* out_option, int32_t* out_config,
                        int8_t* out_labels, double* out_objective, mgs_error* err) {
  if (!ctx || !p) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    c.kernel_launches = 0;
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    mgs::precheck_space(c, p->lattice, pr, sp);  // throw_if_infeasible(precheck_scenario) (baselines.hpp:141)
    const int M = pr.t.M, S = pr.t.S;
    if (p->forecast_len != S) throw PlanFail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};
    double* d_recv = upload_forecast(c, *p, M, S);
    std::vector<int32_t> plan;
    if (!mgs::window_boundary(c, pr, sp, p->lattice, d_recv, plan))
      throw PlanFail{MGS_ERR_WINDOW_BOUNDARY, "no window-boundary plan can complete every retraining"};
    const double total = plan_total(c, pr, sp, plan);
    copy_plan_labels(c, sp, plan, out_config, out_labels);
    if (out_option)
      for (int s = 0; s < S; ++s) out_option[s] = plan[s];
    if (out_objective) *out_objective = total;
  });
}

int mgs_replay_requests(mgs_ctx* ctx, const mgs_problem* p, int32_t windows, const double* acc_pre, const double* acc_post,
                        const double* slo, double step_seconds, const int32_t* plans, int32_t n_plans,
                        const uint8_t* overrides, const int64_t* arrivals, int32_t n_traces, const uint64_t* seeds,
                        int32_t n_seeds, mgs_job_metrics* out, mgs_error* err) {
  if (!ctx || !p || !slo || windows < 1 || n_plans < 0 || n_traces < 0 || n_seeds < 0 || !(step_seconds > 0))
    return MGS_ERR_ARGUMENT;
  if ((acc_pre == nullptr) != (acc_post == nullptr) || (windows > 1 && !acc_pre)) return MGS_ERR_ARGUMENT;
  const long long runs = static_cast<long long>(n_plans) * n_traces * n_seeds;
  if (runs > 0 && (!plans || !arrivals || !seeds || !out)) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    const int M = pr.t.M, S = pr.t.S, W = windows;
    for (int m = 0; m < M; ++m)
      if (!(slo[m] > 0)) throw PlanFail{MGS_ERR_INPUT_SCENARIO, "latency_full must be positive"};  // workload.hpp:90-92
    for (long long k = 0; k < static_cast<long long>(n_plans) * W * S; ++k)
      if (plans[k] < 0 || plans[k] >= sp.n_opt) throw PlanFail{MGS_ERR_PLAN_INFEASIBLE, "plan names an unknown option"};
    if (runs == 0) return;
    std::vector<double> acc(static_cast<size_t>(W) * 2 * M);  // [W][pre|post][M]
    for (int w = 0; w < W; ++w)
      for (int m = 0; m < M; ++m) {
        acc[(w * 2 + 0) * M + m] = acc_pre ? acc_pre[w * M + m] : p->tables.acc_pre[m];
        acc[(w * 2 + 1) * M + m] = acc_post ? acc_post[w * M + m] : p->tables.acc_post[m];
      }
    const size_t G = static_cast<size_t>(W) * S;
    int32_t* d_plans = c.buf<int32_t>("rp_plans", static_cast<size_t>(n_plans) * G);
    int64_t* d_arr = c.buf<int64_t>("rp_arr", static_cast<size_t>(n_traces) * M * G);
    uint64_t* d_seeds = c.buf<uint64_t>("rp_seeds", n_seeds);
    double* d_acc = c.buf<double>("rp_acc", acc.size());
    mgs_job_metrics* d_out = c.buf<mgs_job_metrics>("rp_out", static_cast<size_t>(runs) * W * M);
    MGS_CUDA_OK(cudaMemcpyAsync(d_plans, plans, static_cast<size_t>(n_plans) * G * 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_arr, arrivals, static_cast<size_t>(n_traces) * M * G * 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_seeds, seeds, static_cast<size_t>(n_seeds) * 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_acc, acc.data(), acc.size() * 8, cudaMemcpyHostToDevice, c.stream));
    uint8_t* d_ov = overrides ? c.buf<uint8_t>("rp_ov", static_cast<size_t>(n_plans) * G * M) : nullptr;
    if (overrides)
      MGS_CUDA_OK(cudaMemcpyAsync(d_ov, overrides, static_cast<size_t>(n_plans) * G * M, cudaMemcpyHostToDevice, c.stream));
    mgs::replay_requests(c, pr, sp, W, d_acc, p->tables.psi, slo, step_seconds, d_plans, d_ov, n_plans, d_arr,
                         n_traces, d_seeds, n_seeds, d_out);
    MGS_CUDA_OK(cudaMemcpyAsync(out, d_out, static_cast<size_t>(runs) * W * M * sizeof(mgs_job_metrics),
                                cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));  // also keeps `acc` alive until its copy has run
  });
}

int mgs_preinit(mgs_ctx* ctx, const mgs_problem* p, const int32_t* plans, int32_t n_plans, uint8_t* overrides,
                uint32_t* fired, mgs_error* err) {
  if (!ctx || !p || n_plans < 0 || (n_plans > 0 && (!plans || !overrides))) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    const int M = pr.t.M, S = pr.t.S;
    for (long long k = 0; k < static_cast<long long>(n_plans) * S; ++k)
      if (plans[k] < 0 || plans[k] >= sp.n_opt) throw PlanFail{MGS_ERR_PLAN_INFEASIBLE, "plan names an unknown option"};
    if (n_plans == 0) return;
    int32_t* d_plans = c.buf<int32_t>("pi_plans", static_cast<size_t>(n_plans) * S);
    uint8_t* d_ov = c.buf<uint8_t>("pi_ov", static_cast<size_t>(n_plans) * S * M);
    uint32_t* d_fired = fired ? c.buf<uint32_t>("pi_fired", static_cast<size_t>(n_plans) * S) : nullptr;
    MGS_CUDA_OK(cudaMemcpyAsync(d_plans, plans, static_cast<size_t>(n_plans) * S * 4, cudaMemcpyHostToDevice, c.stream));
    mgs::preinit_overrides(c, pr, sp, p->lattice, d_plans, n_plans, d_ov, d_fired);
    MGS_CUDA_OK(cudaMemcpyAsync(overrides, d_ov, static_cast<size_t>(n_plans) * S * M, cudaMemcpyDeviceToHost, c.stream));
    if (fired)
      MGS_CUDA_OK(cudaMemcpyAsync(fired, d_fired, static_cast<size_t>(n_plans) * S * 4, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int mgs_solve_window(mgs_ctx* ctx, const mgs_problem* p, int32_t* out_option, int32_t* out_config, int8_t* out_labels,
                     double* out_objective, mgs_stats* stats, mgs_error* err) {
  if (!ctx || !p) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    MGS_CUDA_OK(cudaSetDevice(ctx->c.device));
    solve_one(ctx->c, *p, out_option, out_config, out_labels, out_objective, stats);
  });
}

int mgs_solve_batch(mgs_ctx* ctx, const mgs_problem* problems, int32_t n, int32_t s_max, int32_t* out_option,
                    double* out_objective, int32_t* status, mgs_stats* stats, mgs_error* errs) {
  if (!ctx || (!problems && n > 0) || n < 0) return MGS_ERR_ARGUMENT;
  // every window starts out failed: a call that stops early (CUDA error,
  // capacity growth not converging) never leaves a status unwritten
  for (int i = 0; i < n; ++i) {
    if (status) status[i] = MGS_ERR_CUDA;
    if (errs) fill_err(&errs[i], MGS_ERR_CUDA, "not solved: the batch call failed before this window");
  }
  return guarded(nullptr, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    // Windows of equal shape (S, M <= 2) are solved together: up to
    // MGS_BATCH_LANES of them share every DP kernel launch (grid.y = lane).
    const char* env = std::getenv("MGS_BATCH_LANES");
    const int max_lanes = std::max(1, std::min(mgs::kMaxLanes, env ? std::atoi(env) : 32));
    struct Prep {
      int i;
      mgs::Prepared pr;
      mgs::DevSpace sp;
      double *recv, *ub, *inc;
    };
    std::vector<Prep> group;
    group.reserve(max_lanes);
    auto set_err = [&](int i, int st, const mgs_error& e) {
      if (status) status[i] = st;
      if (errs) errs[i] = e;
    };
    auto flush = [&]() {
      if (group.empty()) return;
      MGS_CUDA_OK(cudaEventRecord(c.ev0, c.stream));
      std::vector<mgs::V2Lane> lanes(group.size());
      for (size_t k = 0; k < group.size(); ++k) {
        mgs::V2Lane& L = lanes[k];
        L.p = &problems[group[k].i];
        L.pr = &group[k].pr;
        L.sp = &group[k].sp;
        L.recv = group[k].recv;
        L.ub = group[k].ub;
        L.incumbent = group[k].inc;
        L.prefix = "L" + std::to_string(k) + "/";
      }
      mgs::solve_dp_v2_lanes(c, lanes);
      MGS_CUDA_OK(cudaEventRecord(c.ev1, c.stream));
      MGS_CUDA_OK(cudaEventSynchronize(c.ev1));
      float ms = 0.f;
      MGS_CUDA_OK(cudaEventElapsedTime(&ms, c.ev0, c.ev1));
      for (size_t k = 0; k < group.size(); ++k) {
        const int i = group[k].i;
        mgs_error e{};
        const mgs::V2Lane& L = lanes[k];
        if (L.status != MGS_OK) {
          fill_err(&e, L.status, L.msg, L.err_step, L.err_count);
          set_err(i, L.status, e);
          continue;
        }
        c.prefix = L.prefix;
        const double total = plan_total(c, group[k].pr, group[k].sp, L.out.options);
        c.prefix.clear();
        const int S = group[k].pr.t.S;
        if (out_option)
          for (int s = 0; s < S; ++s) out_option[static_cast<size_t>(i) * s_max + s] = L.out.options[s];
        if (out_objective) out_objective[i] = total;
        if (stats) {
          stats[i] = L.out.stats;
          stats[i].device_ms = ms;  // the whole batch's device time (shared by its windows)
          for (double& x : stats[i].phase_ms) x = 0.0;
          stats[i].phase_ms[3] = ms;
        }
        set_err(i, MGS_OK, e);
      }
      group.clear();
    };
    for (int i = 0; i < n; ++i) {
      mgs_error e{};
      const int k = static_cast<int>(group.size());
      c.prefix = "L" + std::to_string(k) + "/";
      Prep pp{};
      pp.i = i;
      bool lane_ok = false;
      int st = guarded(&e, [&] {
        const mgs_problem& p = problems[i];
        if (p.tables.steps > s_max) throw PlanFail{MGS_ERR_ARGUMENT, "window longer than s_max"};
        pp.pr = prepare_problem(p);
        mgs::build_space(c, p.lattice, pp.pr, pp.sp);
        mgs::precheck_space(c, p.lattice, pp.pr, pp.sp);
        const int M = pp.pr.t.M, S = pp.pr.t.S;
        if (p.forecast_len != S) throw PlanFail{MGS_ERR_INPUT_FORECAST, "forecast horizon != window size"};
        if (!mgs::solve_dp_v2_supported(pp.pr, pp.sp)) return;
        pp.recv = upload_forecast(c, p, M, S);
        pp.ub = c.buf<double>("ub_suffix", S + 1);
        pp.inc = c.buf<double>("incumbent", 1);
        int32_t* d_greedy = c.buf<int32_t>("greedy", S);
        mgs::goodput_reductions(c, pp.pr, pp.sp, pp.recv, pp.ub, pp.inc, d_greedy);
        lane_ok = true;
      });
      c.prefix.clear();
      if (st != MGS_OK) {
        set_err(i, st, e);
        continue;
      }
      if (!lane_ok) {  // M > 2: the multi-launch engine, one window at a time
        st = guarded(&e, [&] {
          solve_one(c, problems[i], out_option ? out_option + static_cast<size_t>(i) * s_max : nullptr, nullptr,
                    nullptr, out_objective ? out_objective + i : nullptr, stats ? stats + i : nullptr);
        });
        set_err(i, st, e);
        continue;
      }
      if (!group.empty() && (group[0].pr.t.S != pp.pr.t.S || group[0].pr.t.M != pp.pr.t.M)) {
        // shape change: this window was prepared under lane k's prefix, which
        // the current group owns -> flush, then re-prepare it as lane 0
        flush();
        --i;
        continue;
      }
      group.push_back(std::move(pp));
      if (static_cast<int>(group.size()) == max_lanes) flush();
    }
    flush();
  });
}

int mgs_evaluate_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* plans, int32_t n_plans,
                       const uint8_t* overrides, const int64_t* arrivals, int32_t n_traces, double* total,
                       double* throughput, mgs_error* err) {
  if (!ctx || !p || !plans || !arrivals || !total || n_plans < 0 || n_traces < 0) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    mgs::DevSpace sp;
    mgs::build_space(c, p->lattice, pr, sp);
    const int M = pr.t.M, S = pr.t.S;
    for (long long k = 0; k < static_cast<long long>(n_plans) * S; ++k)
      if (plans[k] < 0 || plans[k] >= sp.n_opt) throw PlanFail{MGS_ERR_PLAN_INFEASIBLE, "plan names an unknown option"};
    if (n_plans == 0 || n_traces == 0) return;
    int32_t* d_plans = c.buf<int32_t>("eval_plans", static_cast<size_t>(n_plans) * S);
    int64_t* d_arr = c.buf<int64_t>("eval_arr", static_cast<size_t>(n_traces) * M * S);
    double* d_total = c.buf<double>("eval_total", static_cast<size_t>(n_plans) * n_traces);
    double* d_thr = throughput ? c.buf<double>("eval_thr", static_cast<size_t>(n_plans) * n_traces * S * M) : nullptr;
    uint8_t* d_ov = overrides ? c.buf<uint8_t>("eval_ov", static_cast<size_t>(n_plans) * S * M) : nullptr;
    if (overrides)
      MGS_CUDA_OK(cudaMemcpyAsync(d_ov, overrides, static_cast<size_t>(n_plans) * S * M, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_plans, plans, static_cast<size_t>(n_plans) * S * 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_arr, arrivals, static_cast<size_t>(n_traces) * M * S * 8, cudaMemcpyHostToDevice, c.stream));
    mgs::evaluate_batch(c, pr, sp, d_plans, n_plans, d_arr, n_traces, d_total, d_thr, d_ov);
    MGS_CUDA_OK(cudaMemcpyAsync(total, d_total, static_cast<size_t>(n_plans) * n_traces * 8, cudaMemcpyDeviceToHost, c.stream));
    if (throughput)
      MGS_CUDA_OK(cudaMemcpyAsync(throughput, d_thr, static_cast<size_t>(n_plans) * n_traces * S * M * 8,
                                  cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

namespace {
void table_batch(Ctx& c, const mgs_problem& p, const int32_t* d_arr, int n, double* d_best, double* d_ub,
                 int32_t* n_pareto) {
  // the option space and its Pareto placements depend only on the lattice and
  // the tables: built once per window shape and reused across trace batches
  std::string key(reinterpret_cast<const char*>(&p.tables), sizeof(mgs_tables));
  const int nc = p.lattice.n_configs, ns = nc > 0 ? p.lattice.slot_offset[nc] : 0;
  key.append(reinterpret_cast<const char*>(&p.lattice.n_configs), 8);
  key.append(reinterpret_cast<const char*>(p.lattice.slot_offset), (nc + 1) * 4);
  key.append(reinterpret_cast<const char*>(p.lattice.slot_size), ns * 4);
  key.append(reinterpret_cast<const char*>(p.lattice.slot_start), ns * 4);
  mgs::Prepared pr = prepare_problem(p);
  if (key != c.table_key) {
    const std::string saved = c.prefix;
    c.prefix = "tab/";
    c.table_key.clear();
    mgs::DevSpace sp;
    mgs::build_space(c, p.lattice, pr, sp);
    c.table_np = mgs::table_prepare(c, pr, sp, &c.table_wcp);
    c.prefix = saved;
    c.table_key = key;
  }
  mgs::table_run(c, pr, c.table_wcp, c.table_np, d_arr, n, d_best, d_ub);
  if (n_pareto) *n_pareto = c.table_np;
}
}  // namespace

int mgs_goodput_table_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* arrivals, int32_t n_traces, double* best,
                            double* ub_suffix, int32_t* n_pareto, mgs_error* err) {
  if (!ctx || !p || n_traces < 0 || (n_traces > 0 && (!arrivals || !ub_suffix))) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    const int M = p->tables.models, S = p->tables.steps;
    const size_t n_arr = static_cast<size_t>(n_traces) * M * S;
    int32_t* d_arr = c.buf<int32_t>("tabb_arr", n_arr);
    double* d_best = best ? c.buf<double>("tabb_best", static_cast<size_t>(n_traces) * S) : nullptr;
    double* d_ub = c.buf<double>("tabb_ub", static_cast<size_t>(n_traces) * (S + 1));
    if (n_arr) MGS_CUDA_OK(cudaMemcpyAsync(d_arr, arrivals, n_arr * 4, cudaMemcpyHostToDevice, c.stream));
    table_batch(c, *p, d_arr, n_traces, d_best, d_ub, n_pareto);
    if (n_traces > 0) {
      MGS_CUDA_OK(cudaMemcpyAsync(ub_suffix, d_ub, static_cast<size_t>(n_traces) * (S + 1) * 8, cudaMemcpyDeviceToHost,
                                  c.stream));
      if (best)
        MGS_CUDA_OK(cudaMemcpyAsync(best, d_best, static_cast<size_t>(n_traces) * S * 8, cudaMemcpyDeviceToHost, c.stream));
    }
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int mgs_goodput_table_batch_device(mgs_ctx* ctx, const mgs_problem* p, const int32_t* d_arrivals, int32_t n_traces,
                                   double* d_best, double* d_ub_suffix, int32_t* n_pareto, mgs_error* err) {
  if (!ctx || !p || n_traces < 0 || (n_traces > 0 && (!d_arrivals || !d_ub_suffix))) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    table_batch(c, *p, d_arrivals, n_traces, d_best, d_ub_suffix, n_pareto);
  });
}

// ---------------------------------------------------------------------------
// general per-step allocations (feasible.cu)
int mgs_check_feasible_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* step_config, const uint8_t* slot_tasks,
                             int32_t n_plans, mgs_plan_violation* out, int32_t cap, int32_t* n_out, mgs_error* err) {
  if (!ctx || !p || n_plans < 0 || cap < 0) return MGS_ERR_ARGUMENT;
  if (n_plans > 0 && (!step_config || !slot_tasks || !n_out || (cap > 0 && !out))) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);  // input.scenario / input.catalog as Tables::build
    if (n_plans == 0) return;
    const int S = pr.t.S;
    const mgs::ViewSet v = mgs::upload_views(c, p->lattice, pr, step_config, slot_tasks, static_cast<long long>(n_plans) * S);
    const int cap1 = cap > 0 ? cap : 1;
    mgs_plan_violation* d_out = c.buf<mgs_plan_violation>("cf_out", static_cast<size_t>(n_plans) * cap1);
    int32_t* d_n = c.buf<int32_t>("cf_n", n_plans);
    mgs::check_views(c, pr, v, n_plans, d_out, cap1, d_n);
    if (cap > 0)
      MGS_CUDA_OK(cudaMemcpyAsync(out, d_out, static_cast<size_t>(n_plans) * cap * sizeof(mgs_plan_violation),
                                  cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(n_out, d_n, static_cast<size_t>(n_plans) * 4, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  });
}

int mgs_evaluate_views_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* step_config, const uint8_t* slot_tasks,
                             int32_t n_plans, const double* psi_override, const int64_t* arrivals, int32_t n_traces,
                             int32_t verify, double* total, mgs_score_entry* entries, int32_t* status,
                             mgs_plan_violation* first, mgs_error* err) {
  if (!ctx || !p || n_plans < 0 || n_traces < 0) return MGS_ERR_ARGUMENT;
  if (n_plans > 0 && (!step_config || !slot_tasks || (verify && !status))) return MGS_ERR_ARGUMENT;
  if (static_cast<long long>(n_plans) * n_traces > 0 && (!arrivals || !total)) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    if (n_plans == 0) return;
    const int M = pr.t.M, S = pr.t.S;
    const mgs::ViewSet v = mgs::upload_views(c, p->lattice, pr, step_config, slot_tasks, static_cast<long long>(n_plans) * S);
    std::vector<int32_t> nv;
    std::vector<mgs_plan_violation> fv;
    if (verify) {  // evaluate_plan(verify_feasibility = true): check_feasible first (evaluate.hpp:157-162)
      mgs_plan_violation* d_out = c.buf<mgs_plan_violation>("ev_cf_out", n_plans);
      int32_t* d_n = c.buf<int32_t>("ev_cf_n", n_plans);
      mgs::check_views(c, pr, v, n_plans, d_out, 1, d_n);
      nv.resize(n_plans);
      fv.resize(n_plans);
      MGS_CUDA_OK(cudaMemcpyAsync(nv.data(), d_n, static_cast<size_t>(n_plans) * 4, cudaMemcpyDeviceToHost, c.stream));
      MGS_CUDA_OK(cudaMemcpyAsync(fv.data(), d_out, static_cast<size_t>(n_plans) * sizeof(mgs_plan_violation),
                                  cudaMemcpyDeviceToHost, c.stream));
    }
    const long long n = static_cast<long long>(n_plans) * n_traces;
    double* d_total = c.buf<double>("ev_total", std::max(1ll, n));
    mgs_score_entry* d_ent = entries ? c.buf<mgs_score_entry>("ev_entries", std::max(1ll, n) * S * M) : nullptr;
    double* d_psi = nullptr;
    if (psi_override) {
      d_psi = c.buf<double>("ev_psi", static_cast<size_t>(n_plans) * S * M);
      MGS_CUDA_OK(cudaMemcpyAsync(d_psi, psi_override, static_cast<size_t>(n_plans) * S * M * 8, cudaMemcpyHostToDevice,
                                  c.stream));
    }
    if (n > 0) {
      int64_t* d_arr = c.buf<int64_t>("ev_arr", static_cast<size_t>(n_traces) * M * S);
      MGS_CUDA_OK(cudaMemcpyAsync(d_arr, arrivals, static_cast<size_t>(n_traces) * M * S * 8, cudaMemcpyHostToDevice,
                                  c.stream));
      mgs::evaluate_views(c, pr, v, n_plans, d_psi, d_arr, n_traces, d_total, d_ent);
      MGS_CUDA_OK(cudaMemcpyAsync(total, d_total, n * 8, cudaMemcpyDeviceToHost, c.stream));
      if (entries)
        MGS_CUDA_OK(cudaMemcpyAsync(entries, d_ent, static_cast<size_t>(n) * S * M * sizeof(mgs_score_entry),
                                    cudaMemcpyDeviceToHost, c.stream));
    }
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    if (verify)
      for (int i = 0; i < n_plans; ++i) {
        status[i] = nv[i] ? MGS_ERR_PLAN_INFEASIBLE : MGS_OK;
        if (first) first[i] = nv[i] ? fv[i] : mgs_plan_violation{};
        if (nv[i])
          for (int t = 0; t < n_traces; ++t) total[static_cast<size_t>(i) * n_traces + t] = 0.0;
      }
  });
}

int mgs_run_fluid(mgs_ctx* ctx, const mgs_problem* p, int32_t windows, const double* acc_pre, const double* acc_post,
                  double step_seconds, const int32_t* step_config, const uint8_t* slot_tasks, int32_t n_plans,
                  const double* psi_override, const int64_t* arrivals, int32_t n_traces, mgs_job_metrics* out,
                  mgs_error* err) {
  if (!ctx || !p || windows < 1 || n_plans < 0 || n_traces < 0) return MGS_ERR_ARGUMENT;
  if ((acc_pre == nullptr) != (acc_post == nullptr) || (windows > 1 && !acc_pre)) return MGS_ERR_ARGUMENT;
  const long long runs = static_cast<long long>(n_plans) * n_traces;
  if (n_plans > 0 && (!step_config || !slot_tasks)) return MGS_ERR_ARGUMENT;
  if (runs > 0 && (!arrivals || !out)) return MGS_ERR_ARGUMENT;
  return guarded(err, [&] {
    Ctx& c = ctx->c;
    MGS_CUDA_OK(cudaSetDevice(c.device));
    mgs::Prepared pr = prepare_problem(*p);
    const int M = pr.t.M, S = pr.t.S, W = windows;
    const size_t G = static_cast<size_t>(W) * S;
    if (n_plans == 0) return;
    const mgs::ViewSet v = mgs::upload_views(c, p->lattice, pr, step_config, slot_tasks, static_cast<long long>(n_plans) * G);
    if (runs == 0) return;
    std::vector<double> acc(static_cast<size_t>(W) * 2 * M);  // [W][pre|post][M]
    for (int w = 0; w < W; ++w)
      for (int m = 0; m < M; ++m) {
        acc[(w * 2 + 0) * M + m] = acc_pre ? acc_pre[w * M + m] : p->tables.acc_pre[m];
        acc[(w * 2 + 1) * M + m] = acc_post ? acc_post[w * M + m] : p->tables.acc_post[m];
      }
    double* d_acc = c.buf<double>("fl_acc", acc.size());
    int64_t* d_arr = c.buf<int64_t>("fl_arr", static_cast<size_t>(n_traces) * M * G);
    mgs_job_metrics* d_out = c.buf<mgs_job_metrics>("fl_out", static_cast<size_t>(runs) * W * M);
    double* d_psi = nullptr;
    if (psi_override) {
      d_psi = c.buf<double>("fl_psi", static_cast<size_t>(n_plans) * G * M);
      MGS_CUDA_OK(cudaMemcpyAsync(d_psi, psi_override, static_cast<size_t>(n_plans) * G * M * 8, cudaMemcpyHostToDevice,
                                  c.stream));
    }
    MGS_CUDA_OK(cudaMemcpyAsync(d_acc, acc.data(), acc.size() * 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_arr, arrivals, static_cast<size_t>(n_traces) * M * G * 8, cudaMemcpyHostToDevice, c.stream));
    mgs::fluid_views(c, pr, W, v, n_plans, d_psi, d_acc, d_arr, n_traces, step_seconds, d_out);
    MGS_CUDA_OK(cudaMemcpyAsync(out, d_out, static_cast<size_t>(runs) * W * M * sizeof(mgs_job_metrics),
                                cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));  // keeps `acc` alive until its copy has run
  });
}

}  // extern "C"
