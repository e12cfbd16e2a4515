// Plans given as general per-step allocations ("views"), not option indices:
// the feasibility checker, the Goodput objective and the fluid replay of any
// allocation sequence the reference's resolve_step can read.
//
//   k_views        engine::resolve_step          evaluate.hpp:25-47
//                  per (plan, step): universe inference masks, capability
//                  summed in slot (slice-start) order, retraining size (the
//                  last retraining slot in slot order), retraining slot count,
//                  and the strengthened-floor data of check_feasible
//   k_check        check_feasible families 2-5   evaluate.hpp:82-146
//                  (deployment floor per (step, tenant), step-major; then per
//                  tenant one of retraining-not-launched / -interrupted /
//                  -size / -incomplete / -overrun), records in reference order
//   k_eval_views   evaluate_plan                 evaluate.hpp:153-210
//                  per (plan, trace): the breakdown entries and the total,
//                  step-major / tenant-minor fold; psi overrides as doubles
//   k_fluid        run_fluid + build_series      simulator.hpp:72-131,171-203
//                  per (plan, trace, tenant) over W windows: spill pool,
//                  changed flags across window boundaries, fluid counters
//
// A plan step is (configuration index in lattice order, per-slot task bits):
// bit 2m = inference task of tenant m, bit 2m+1 = its retraining task. One
// slot may carry several tasks (the reference's instance-shared case); its
// string-level validation (unknown ids, second-index) stays in the host
// wrapper, which has the names.
#include <climits>

#include "ctx.cuh"

namespace mgs {
namespace {

struct View {
  uint32_t mask[KM];
  double cap[KM];
  int8_t rsize[KM];   // retraining size, 0 = none
  int8_t anchored[KM];  // some inference slot of size >= floor
  int8_t gpc_ok[KM];    // inference GPC sum >= floor (the weaker check, message only)
  int8_t pad[KM];
};

struct LatticeDev {
  const int32_t* off;   // [n_configs+1]
  const int32_t* size;  // per flat slot
  const int32_t* uid;   // universe id per flat slot
  int n_configs;
};

__global__ void k_views(LatticeDev lat, HostTables t, const int32_t* config, const uint8_t* tasks, long long n, View* out) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int M = t.M;
  View v;
  int gpcs[KM];
  for (int m = 0; m < KM; ++m) {
    v.mask[m] = 0u;
    v.cap[m] = 0.0;
    v.rsize[m] = 0;
    v.anchored[m] = 0;
    v.gpc_ok[m] = 0;
    v.pad[m] = 0;
    gpcs[m] = 0;
  }
  const int c = config[i];
  if (c >= 0 && c < lat.n_configs) {
    const uint8_t* tk = tasks + i * MGS_MAX_SLOTS;
    for (int k = lat.off[c]; k < lat.off[c + 1]; ++k) {  // slots ascend by slice_start
      const uint8_t bits = tk[k - lat.off[c]];
      if (!bits) continue;
      const int sz = lat.size[k];
      for (int m = 0; m < M; ++m) {
        if ((bits >> (2 * m)) & 1u) {
          v.mask[m] |= 1u << lat.uid[k];
          v.cap[m] = dadd(v.cap[m], t.cap[m][sz]);
          gpcs[m] += sz;
          if (sz >= t.floor_[m]) v.anchored[m] = 1;
        }
        if ((bits >> (2 * m + 1)) & 1u) v.rsize[m] = static_cast<int8_t>(sz);
      }
    }
  }
  for (int m = 0; m < M; ++m) v.gpc_ok[m] = gpcs[m] >= t.floor_[m] ? 1 : 0;
  out[i] = v;
}

// one thread per plan: the reference's two loops in its order
__global__ void k_check(HostTables t, const View* views, int n_plans, mgs_plan_violation* out, int cap, int32_t* n_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_plans) return;
  const int S = t.S, M = t.M;
  const View* pv = views + static_cast<size_t>(i) * S;
  mgs_plan_violation* po = out + static_cast<size_t>(i) * cap;
  int n = 0;
  auto put = [&](int code, int step, int m, int d0, int d1, int d2) {
    if (n < cap) {
      po[n].code = code;
      po[n].step = step;
      po[n].model = m;
      po[n].detail[0] = d0;
      po[n].detail[1] = d1;
      po[n].detail[2] = d2;
    }
    ++n;
  };
  for (int s = 0; s < S; ++s)  // strengthened deployment floor (evaluate.hpp:82-109)
    for (int m = 0; m < M; ++m)
      if (!pv[s].anchored[m]) put(MGS_VIOL_DEPLOYMENT_FLOOR, s, m, pv[s].gpc_ok[m], t.floor_[m], 0);
  for (int m = 0; m < M; ++m) {  // retraining run (evaluate.hpp:111-144)
    int first = -1, last = -1, len = 0;
    for (int s = 0; s < S; ++s)
      if (pv[s].rsize[m] > 0) {
        if (first < 0) first = s;
        last = s;
        ++len;
      }
    if (first < 0) {
      put(MGS_VIOL_RETRAINING_NOT_LAUNCHED, -1, m, 0, 0, 0);
      continue;
    }
    const bool contiguous = last - first + 1 == len;
    const int k = pv[first].rsize[m];
    bool constant = true;
    for (int s = first; s <= last; ++s)
      if (pv[s].rsize[m] > 0 && pv[s].rsize[m] != k) constant = false;
    if (!contiguous || !constant) {
      put(MGS_VIOL_RETRAINING_INTERRUPTED, first, m, contiguous ? 1 : 0, 0, 0);
      continue;
    }
    const long long rt = t.rt[m][k];
    if (rt < 1) put(MGS_VIOL_RETRAINING_SIZE, first, m, k, 0, 0);
    else if (len < rt) put(MGS_VIOL_RETRAINING_INCOMPLETE, first, m, len, static_cast<int>(rt), k);
    else if (len > rt) put(MGS_VIOL_RETRAINING_OVERRUN, first, m, len, static_cast<int>(rt), k);
  }
  n_out[i] = n;
}

// evaluate_plan over views: thread per (plan, trace)
__global__ void k_eval_views(HostTables t, const View* views, int n_plans, const double* psi_over,
                             const int64_t* arrivals, int n_traces, int has_initial, uint4 init_lo, double* total,
                             mgs_score_entry* entries) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_plans) * n_traces) return;
  const int i = static_cast<int>(idx / n_traces), j = static_cast<int>(idx % n_traces);
  const int S = t.S, M = t.M;
  const View* pv = views + static_cast<size_t>(i) * S;
  const int64_t* arr = arrivals + static_cast<size_t>(j) * M * S;
  const uint32_t init[KM] = {init_lo.x, init_lo.y, init_lo.z, init_lo.w};
  int finish_after[KM];
  for (int m = 0; m < M; ++m) {  // Eq-12 completion: strictly after the last retraining step
    finish_after[m] = INT_MAX;
    for (int s = S - 1; s >= 0; --s)
      if (pv[s].rsize[m] > 0) {
        finish_after[m] = s + 1;
        break;
      }
  }
  double tot = 0.0;
  for (int s = 0; s < S; ++s)
    for (int m = 0; m < M; ++m) {
      const double raw = pv[s].cap[m];
      const bool changed = s == 0 ? (has_initial && pv[0].mask[m] != init[m]) : pv[s].mask[m] != pv[s - 1].mask[m];
      double loss = 0.0;
      if (changed) {
        double psi = t.psi_raw[m];
        if (psi_over) {
          const double o = psi_over[(static_cast<size_t>(i) * S + s) * M + m];
          if (o == o) psi = o;  // NaN = no override entry
        }
        loss = psi < 1.0 ? psi : 1.0;  // reconfig_loss_fraction
      }
      const double thr = thr_of(static_cast<double>(arr[m * S + s]), eff_cap(raw, loss));
      const bool completion = s >= finish_after[m];
      const double good = dmul(thr, completion ? t.post[m] : t.pre[m]);
      tot = dadd(tot, good);
      if (entries) {
        mgs_score_entry& e = entries[(idx * S + s) * M + m];
        e.throughput = thr;
        e.overhead_loss = dmul(loss, raw);
        e.goodput = good;
        e.completion = completion ? 1 : 0;
        e.pad = 0;
      }
    }
  total[idx] = tot;
}

// run_fluid over W windows: thread per (plan, trace, tenant)
__global__ void k_fluid(HostTables t, int W, const View* views, int n_plans, const double* psi_over, const double* acc,
                        const int64_t* arrivals, int n_traces, double step_seconds, mgs_job_metrics* out) {
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int S = t.S, M = t.M, G = W * S;
  if (tid >= static_cast<long long>(n_plans) * n_traces * M) return;
  const int m = static_cast<int>(tid % M);
  const long long run = tid / M;
  const int ti = static_cast<int>(run % n_traces), pi = static_cast<int>(run / n_traces);
  const int64_t* arr = arrivals + (static_cast<size_t>(ti) * M + m) * G;
  double spill = 0.0;  // one pool for the whole horizon (simulator.hpp:89)
  uint32_t prev_mask = 0u;
  bool have_prev = false;
  for (int w = 0; w < W; ++w) {
    const View* pv = views + (static_cast<size_t>(pi) * W + w) * S;
    int finish_after = INT_MAX;
    for (int s = S - 1; s >= 0; --s)
      if (pv[s].rsize[m] > 0) {
        finish_after = s + 1;
        break;
      }
    const double a_pre = acc[(w * 2 + 0) * M + m], a_post = acc[(w * 2 + 1) * M + m];
    double received = 0.0, served = 0.0, correct = 0.0, overhead = 0.0;
    int reconf = 0;
    for (int s = 0; s < S; ++s) {
      const bool changed = s > 0 ? pv[s].mask[m] != pv[s - 1].mask[m] : (have_prev && pv[s].mask[m] != prev_mask);
      double applied = 0.0;
      if (changed) {
        applied = t.psi_raw[m];
        if (psi_over) {
          const double o = psi_over[((static_cast<size_t>(pi) * W + w) * S + s) * M + m];
          if (o == o) applied = o;
        }
        spill = dadd(spill, applied);
      }
      const double consumed = spill < 1.0 ? spill : 1.0;
      spill = dsub(spill, consumed);
      const double recv = static_cast<double>(arr[w * S + s]);
      const double thr = thr_of(recv, eff_cap(pv[s].cap[m], consumed));
      const double a = s >= finish_after ? a_post : a_pre;
      received = dadd(received, recv);
      served = dadd(served, thr);
      correct = dadd(correct, dmul(thr, a));
      if (changed) {
        ++reconf;
        overhead = dadd(overhead, dmul(applied, step_seconds));
      }
      prev_mask = pv[s].mask[m];
      have_prev = true;
    }
    mgs_job_metrics& r = out[(run * W + w) * M + m];
    r.received = received;
    r.served = served;
    r.timely = served;  // fluid: everything served met its deadline
    r.correct = correct;
    r.valid = correct;
    r.dropped = 0.0;
    r.queued_at_end = 0.0;
    r.reconfigurations = reconf;
    r.overhead_seconds = overhead;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// host side (called from capi.cu with the context's stream)
ViewSet upload_views(Ctx& c, const mgs_lattice& lat, const Prepared& pr, const int32_t* config, const uint8_t* tasks,
                     long long n_steps) {
  const int nc = lat.n_configs, ns = nc > 0 ? lat.slot_offset[nc] : 0;
  for (long long k = 0; k < n_steps; ++k)
    if (config[k] < 0 || config[k] >= nc) throw PlanFail{MGS_ERR_ARGUMENT, "plan step names an unknown configuration"};
  int32_t* d_off = c.buf<int32_t>("vw_off", nc + 1);
  int32_t* d_size = c.buf<int32_t>("vw_size", ns);
  int32_t* d_uid = c.buf<int32_t>("vw_uid", ns);
  int32_t* d_cfg = c.buf<int32_t>("vw_cfg", n_steps);
  uint8_t* d_tk = c.buf<uint8_t>("vw_tasks", n_steps * MGS_MAX_SLOTS);
  MGS_CUDA_OK(cudaMemcpyAsync(d_off, lat.slot_offset, (nc + 1) * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_size, lat.slot_size, ns * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_uid, pr.slot_uid.data(), ns * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_cfg, config, n_steps * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_tk, tasks, n_steps * MGS_MAX_SLOTS, cudaMemcpyHostToDevice, c.stream));
  View* d_v = c.buf<View>("vw_views", n_steps);
  LatticeDev L{d_off, d_size, d_uid, nc};
  if (n_steps > 0) {
    k_views<<<ceil_div(n_steps, 128), 128, 0, c.stream>>>(L, pr.t, d_cfg, d_tk, n_steps, d_v);
    ++c.kernel_launches;
    MGS_CUDA_OK(cudaGetLastError());
  }
  return ViewSet{d_v, n_steps};
}

void check_views(Ctx& c, const Prepared& pr, const ViewSet& v, int n_plans, mgs_plan_violation* d_out, int cap,
                 int32_t* d_n) {
  if (n_plans == 0) return;
  k_check<<<ceil_div(n_plans, 64), 64, 0, c.stream>>>(pr.t, static_cast<const View*>(v.views), n_plans, d_out, cap, d_n);
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

void evaluate_views(Ctx& c, const Prepared& pr, const ViewSet& v, int n_plans, const double* d_psi,
                    const int64_t* d_arr, int n_traces, double* d_total, mgs_score_entry* d_entries) {
  const long long n = static_cast<long long>(n_plans) * n_traces;
  if (n == 0) return;
  const uint4 init{pr.init_mask[0], pr.init_mask[1], pr.init_mask[2], pr.init_mask[3]};
  k_eval_views<<<ceil_div(n, 128), 128, 0, c.stream>>>(pr.t, static_cast<const View*>(v.views), n_plans, d_psi, d_arr,
                                                       n_traces, pr.has_initial, init, d_total, d_entries);
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

void fluid_views(Ctx& c, const Prepared& pr, int W, const ViewSet& v, int n_plans, const double* d_psi,
                 const double* d_acc, const int64_t* d_arr, int n_traces, double step_seconds, mgs_job_metrics* d_out) {
  const long long n = static_cast<long long>(n_plans) * n_traces * pr.t.M;
  if (n == 0) return;
  k_fluid<<<ceil_div(n, 64), 64, 0, c.stream>>>(pr.t, W, static_cast<const View*>(v.views), n_plans, d_psi, d_acc, d_arr,
                                                n_traces, step_seconds, d_out);
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

}  // namespace mgs
