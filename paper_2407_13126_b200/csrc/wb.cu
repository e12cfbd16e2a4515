// Window-boundary planner (the Ekya-like baseline, plan_window_boundary,
// baselines.hpp:139-289) on the GPU: every retraining starts at step 0 on a
// chosen GPC count and the allocation changes only at step 0 and at each
// retraining completion. For every per-tenant GPC-count vector the reference
// runs a phase DP over the options of each phase's signature; here each phase
// is one kernel:
//   k_wb_tail    per candidate: the phase's steps after the first, folded
//                s-major / m-minor with raw capabilities (:205-213)
//   k_wb_first   phase 0: first-step score against the carried-over masks
//                (charged only with an initial placement) + tail (:214-225,
//                :236-238)
//   k_wb_step    phase p > 0: one warp per candidate i, lanes over the previous
//                phase's candidates j; v = (T[j] + first(i | mask_j)) + tail[i]
//                (the reference's association), best by (v desc, option index
//                asc) -- the strict '>' over ascending option indices (:239-245)
//   k_wb_final   first max of the last phase (:249-253)
// Candidates stand for their option groups (same signature and placement =>
// same scores); their representative is the smallest option index, which is
// the option the reference's first-max keeps. The k-vector loop, the 1e-12
// tolerance + encoding tie-break between k-vectors (:268-270) and the
// reconstruction run on the host over at most 7^M tiny results.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kWbMaxPhases = KM + 1;

struct WbPhase {
  int first, end;  // steps [first, end)
  int off, len;    // candidate range (sig_off) of the phase's signature
};

struct WbArgs {
  DevSpace sp;
  HostTables t;
  const double* recv;  // [M][S]
  int phases;
  WbPhase ph[kWbMaxPhases];
  long long done_at[KM];
  int has_initial;
};

__device__ __forceinline__ double wb_acc(const WbArgs& a, int m, int s) {
  return s >= a.done_at[m] ? a.t.post[m] : a.t.pre[m];
}

__device__ __forceinline__ double wb_first(const WbArgs& a, int p, int pid, uint64_t prev_ids, bool charge) {
  const int s = a.ph[p].first;
  const uint64_t ids = a.sp.pl_ids[pid];
  double v = 0.0;
  for (int m = 0; m < a.t.M; ++m) {
    const bool changed = charge && field16(prev_ids, m) != field16(ids, m);
    const double eff = eff_cap(a.sp.pl_cap[pid * KM + m], changed ? a.t.loss[m] : 0.0);
    v = dadd(v, dmul(thr_of(a.recv[m * a.t.S + s], eff), wb_acc(a, m, s)));
  }
  return v;
}

__global__ void k_wb_tail(WbArgs a, double* tail /*[phase][len]*/, int stride) {
  const int p = blockIdx.y;
  const WbPhase ph = a.ph[p];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ph.len; i += gridDim.x * blockDim.x) {
    const int pid = a.sp.cand_pid[ph.off + i];
    double v = 0.0;
    for (int s = ph.first + 1; s < ph.end; ++s)
      for (int m = 0; m < a.t.M; ++m)
        v = dadd(v, dmul(thr_of(a.recv[m * a.t.S + s], a.sp.pl_cap[pid * KM + m]), wb_acc(a, m, s)));
    tail[p * stride + i] = v;
  }
}

__global__ void k_wb_first(WbArgs a, const double* tail, double* T) {
  const WbPhase ph = a.ph[0];
  const uint64_t root = a.sp.pl_ids[a.sp.root_pid];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < ph.len; i += gridDim.x * blockDim.x) {
    const int pid = a.sp.cand_pid[ph.off + i];
    T[i] = dadd(wb_first(a, 0, pid, root, a.has_initial != 0), tail[i]);
  }
}

// (value desc, option index asc)
__device__ __forceinline__ bool wb_better(double va, int oa, double vb, int ob) {
  if (va != vb) return va > vb;
  return oa < ob;
}

__global__ void k_wb_step(WbArgs a, int p, const double* tail_p, const double* Tprev, double* T, int* parent) {
  const WbPhase ph = a.ph[p], pv = a.ph[p - 1];
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int M = a.t.M, s = ph.first;
  for (int i = wid; i < ph.len; i += nw) {
    const int pid = a.sp.cand_pid[ph.off + i];
    const uint64_t ids = a.sp.pl_ids[pid];
    // first-step score per "changed" pattern (it depends on j only through
    // which tenants' inference masks differ)
    double fs[1 << KM];
    for (int bits = 0; bits < (1 << M); ++bits) {
      double v = 0.0;
      for (int m = 0; m < M; ++m) {
        const double eff = eff_cap(a.sp.pl_cap[pid * KM + m], ((bits >> m) & 1) ? a.t.loss[m] : 0.0);
        v = dadd(v, dmul(thr_of(a.recv[m * a.t.S + s], eff), wb_acc(a, m, s)));
      }
      fs[bits] = v;
    }
    const double tl = tail_p[i];
    double bv = -DBL_MAX;
    int bo = INT_MAX, bj = -1;
    for (int j = lane; j < pv.len; j += 32) {
      const uint64_t pids = a.sp.pl_ids[a.sp.cand_pid[pv.off + j]];
      int bits = 0;
      for (int m = 0; m < M; ++m) bits |= field16(pids, m) != field16(ids, m) ? (1 << m) : 0;
      const double v = dadd(dadd(Tprev[j], fs[bits]), tl);
      const int oj = a.sp.cand_oi[pv.off + j];
      if (bj < 0 || wb_better(v, oj, bv, bo)) {
        bv = v;
        bo = oj;
        bj = j;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int oo = __shfl_down_sync(0xffffffffu, bo, o);
      const int oj = __shfl_down_sync(0xffffffffu, bj, o);
      if (oj >= 0 && (bj < 0 || wb_better(ov, oo, bv, bo))) {
        bv = ov;
        bo = oo;
        bj = oj;
      }
    }
    if (lane == 0) {
      T[i] = bv;
      parent[i] = bj;
    }
  }
}

// first max of the last phase: out = {value bits, candidate index}
__global__ void k_wb_final(WbArgs a, const double* T, int p, double* out_v, int* out_i) {
  const WbPhase ph = a.ph[p];
  __shared__ double sv[32];
  __shared__ int so[32], si[32];
  double bv = -DBL_MAX;
  int bo = INT_MAX, bi = -1;
  for (int i = threadIdx.x; i < ph.len; i += blockDim.x) {
    const int oi = a.sp.cand_oi[ph.off + i];
    if (bi < 0 || wb_better(T[i], oi, bv, bo)) {
      bv = T[i];
      bo = oi;
      bi = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, bv, o);
    const int oo = __shfl_down_sync(0xffffffffu, bo, o);
    const int oj = __shfl_down_sync(0xffffffffu, bi, o);
    if (oj >= 0 && (bi < 0 || wb_better(ov, oo, bv, bo))) {
      bv = ov;
      bo = oo;
      bi = oj;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    so[threadIdx.x >> 5] = bo;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (si[w] >= 0 && (bi < 0 || wb_better(sv[w], so[w], bv, bo))) {
        bv = sv[w];
        bo = so[w];
        bi = si[w];
      }
    *out_v = bv;
    *out_i = bi;
  }
}

}  // namespace

// Returns false when no k-vector is realizable (infeasible.window-boundary).
bool window_boundary(Ctx& c, const Prepared& pr, const DevSpace& sp, const mgs_lattice& lat, const double* d_recv,
                     std::vector<int32_t>& plan) {
  const HostTables& t = pr.t;
  const int M = t.M, S = t.S;
  // host copies of the small option tables
  std::vector<int32_t> sig_off(sp.n_sig + 1), cand_pid(sp.n_cand), cand_oi(sp.n_cand), opt_config(sp.n_opt);
  std::vector<int8_t> opt_labels(static_cast<size_t>(sp.n_opt) * MGS_MAX_SLOTS);
  MGS_CUDA_OK(cudaMemcpyAsync(sig_off.data(), sp.sig_off, (sp.n_sig + 1) * 4, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(cand_oi.data(), sp.cand_oi, sp.n_cand * 4, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(opt_config.data(), sp.opt_config, sp.n_opt * 4, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(opt_labels.data(), sp.opt_labels, opt_labels.size(), cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  (void)cand_pid;

  std::vector<std::vector<int>> k_choices(M);  // :158-161
  for (int m = 0; m < M; ++m)
    for (int k = 1; k <= 7; ++k)
      if (t.rt[m][k] >= 1 && t.rt[m][k] <= S) k_choices[m].push_back(k);
  for (int m = 0; m < M; ++m)
    if (k_choices[m].empty()) return false;

  int max_len = 1;
  for (int g = 0; g < sp.n_sig; ++g) max_len = std::max(max_len, sig_off[g + 1] - sig_off[g]);
  double* d_tail = c.buf<double>("wb_tail", static_cast<size_t>(kWbMaxPhases) * max_len);
  double* d_T = c.buf<double>("wb_T", static_cast<size_t>(kWbMaxPhases) * max_len);
  int* d_parent = c.buf<int>("wb_parent", static_cast<size_t>(kWbMaxPhases) * max_len);
  double* d_best_v = c.buf<double>("wb_bv", 1);
  int* d_best_i = c.buf<int>("wb_bi", 1);

  double best_value = -INFINITY;
  std::vector<int> best_encoding;
  std::vector<int32_t> best_plan;
  std::vector<size_t> idx(M, 0);
  std::vector<int> ks(M);
  while (true) {  // for_each_kvec (:166-175): the last tenant varies fastest
    for (int m = 0; m < M; ++m) ks[m] = k_choices[m][idx[m]];
    WbArgs a{};
    a.sp = sp;
    a.t = t;
    a.recv = d_recv;
    a.has_initial = pr.has_initial;
    std::vector<int> bounds{0};  // :178-186
    for (int m = 0; m < M; ++m) {
      a.done_at[m] = t.rt[m][ks[m]];
      if (a.done_at[m] < S) bounds.push_back(static_cast<int>(a.done_at[m]));
    }
    bounds.push_back(S);
    std::sort(bounds.begin(), bounds.end());
    bounds.erase(std::unique(bounds.begin(), bounds.end()), bounds.end());
    a.phases = static_cast<int>(bounds.size()) - 1;
    bool realizable = true;
    for (int p = 0; p < a.phases && realizable; ++p) {  // :189-195
      int sig = 0;
      for (int m = M - 1; m >= 0; --m) sig = sig * 8 + (a.done_at[m] > bounds[p] ? ks[m] : 0);
      a.ph[p] = WbPhase{bounds[p], bounds[p + 1], sig_off[sig], sig_off[sig + 1] - sig_off[sig]};
      realizable = a.ph[p].len > 0;
    }
    if (realizable) {
      dim3 tg(ceil_div(max_len, 128), a.phases);
      k_wb_tail<<<tg, 128, 0, c.stream>>>(a, d_tail, max_len);
      k_wb_first<<<ceil_div(a.ph[0].len, 128), 128, 0, c.stream>>>(a, d_tail, d_T);
      for (int p = 1; p < a.phases; ++p)
        k_wb_step<<<ceil_div(a.ph[p].len * 32ll, 256), 256, 0, c.stream>>>(
            a, p, d_tail + static_cast<size_t>(p) * max_len, d_T + static_cast<size_t>(p - 1) * max_len,
            d_T + static_cast<size_t>(p) * max_len, d_parent + static_cast<size_t>(p) * max_len);
      k_wb_final<<<1, 256, 0, c.stream>>>(a, d_T + static_cast<size_t>(a.phases - 1) * max_len, a.phases - 1,
                                          d_best_v, d_best_i);
      c.kernel_launches += 2 + a.phases;
      MGS_CUDA_OK(cudaGetLastError());
      double value = 0.0;
      int bi = -1;
      MGS_CUDA_OK(cudaMemcpyAsync(&value, d_best_v, 8, cudaMemcpyDeviceToHost, c.stream));
      MGS_CUDA_OK(cudaMemcpyAsync(&bi, d_best_i, 4, cudaMemcpyDeviceToHost, c.stream));
      std::vector<int> par(static_cast<size_t>(a.phases) * max_len);
      if (a.phases > 1)
        MGS_CUDA_OK(cudaMemcpyAsync(par.data(), d_parent, par.size() * 4, cudaMemcpyDeviceToHost, c.stream));
      MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
      // reconstruct per-phase options, then the encoding (:255-265)
      std::vector<int> chosen(a.phases);
      for (int p = a.phases - 1, i = bi; p >= 0; --p) {
        chosen[p] = cand_oi[a.ph[p].off + i];
        if (p > 0) i = par[static_cast<size_t>(p) * max_len + i];
      }
      std::vector<int> encoding;
      std::vector<int32_t> steps;
      for (int p = 0; p < a.phases; ++p) {
        const int o = chosen[p];
        const int cfg = opt_config[o];
        const int nsl = lat.slot_offset[cfg + 1] - lat.slot_offset[cfg];
        for (int s = a.ph[p].first; s < a.ph[p].end; ++s) {
          encoding.push_back(cfg);
          for (int k = 0; k < nsl; ++k) encoding.push_back(opt_labels[static_cast<size_t>(o) * MGS_MAX_SLOTS + k]);
          steps.push_back(o);
        }
      }
      const bool better = value > best_value + 1e-12 ||
                          (std::abs(value - best_value) <= 1e-12 && encoding < best_encoding);  // :268-270
      if (best_encoding.empty() || better) {
        best_value = value;
        best_encoding = std::move(encoding);
        best_plan = std::move(steps);
      }
    }
    int m = M - 1;
    while (m >= 0 && ++idx[m] == k_choices[m].size()) idx[m--] = 0;
    if (m < 0) break;
  }
  if (best_plan.empty()) return false;
  plan = std::move(best_plan);
  return true;
}

}  // namespace mgs
