// The Goodput table: per slot x candidate x tenant SLO-attained counts
// weighted by accuracy, reduced the two ways solve_dp consumes it before the
// search, plus batched plan scoring.
//
//   k_ub_best / k_ub_suffix   ub_suffix (solvers.hpp:258-280): per step the max
//                             over candidates of sum_m acc_max*min(recv, cap),
//                             then a suffix sum in descending step order.
//   k_greedy                  the greedy incumbent (solvers.hpp:282-322): a
//                             sequential walk, each step a block-wide first-max
//                             over the candidates compatible with the status.
//   k_evaluate                evaluate_plan(verify=false) (evaluate.hpp:153-210)
//                             for plans x traces, one thread per pair, folding
//                             step-major / model-minor exactly like the reference.
//
// Candidates are the distinct (signature, placement) pairs: every option of a
// pair has the same capabilities and masks, hence the same cell values, and the
// first-max rule picks its smallest option index — the candidate's index.
#include <cfloat>

#include <cooperative_groups.h>

#include "ctx.cuh"

namespace mgs {
namespace {

struct Recv {
  const double* v;  // [M][S] forecast as double (static_cast in the reference)
  int S;
  __device__ double operator()(int m, int s) const { return v[m * S + s]; }
};

__global__ void k_ub_best(DevSpace sp, HostTables t, Recv recv, double* best_out) {
  const int s = blockIdx.x;
  double acc_max[KM];
  for (int m = 0; m < KM; ++m) acc_max[m] = t.pre[m] > t.post[m] ? t.pre[m] : t.post[m];
  double best = 0.0;  // reference starts at 0.0 and uses std::max
  for (int p = threadIdx.x; p < sp.P; p += blockDim.x) {
    double v = 0.0;
    for (int m = 0; m < t.M; ++m) v = dadd(v, dmul(acc_max[m], thr_of(recv(m, s), sp.pl_cap[p * KM + m])));
    best = v > best ? v : best;
  }
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) {
    double x = __shfl_down_sync(0xffffffffu, best, o);
    best = x > best ? x : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      double x = __shfl_down_sync(0xffffffffu, best, o);
      best = x > best ? x : best;
    }
    if (threadIdx.x == 0) best_out[s] = best;
  }
}

__global__ void k_ub_suffix(const double* best, int S, double* ub) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  ub[S] = 0.0;
  for (int s = S - 1; s >= 0; --s) ub[s] = dadd(ub[s + 1], best[s]);
}

// Sequential greedy walk on one thread-block cluster (kGreedyCluster CTAs of
// 1024 threads): every step each CTA takes a strided slice of the candidates
// and reduces its first-max in shared memory; the CTAs exchange their results
// through distributed shared memory (double-buffered by step parity, so one
// cluster barrier per step suffices) and all of them fold the same winner into
// identical copies of the walk's state.
constexpr int kGreedyCluster = 8;

struct GreedyRes {
  double v;
  int oi, ci;
};

__device__ __forceinline__ bool g_better(double v, int oi, int ci, double bv, int boi, int bci) {
  return ci >= 0 && (bci < 0 || v > bv || (v == bv && oi < boi));
}

__global__ void __launch_bounds__(1024) k_greedy(DevSpace sp, HostTables t, Recv recv, int has_initial,
                                                 double* incumbent, int32_t* greedy) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = static_cast<int>(cluster.block_rank()), nrank = static_cast<int>(cluster.num_blocks());
  __shared__ double s_v[32];
  __shared__ int s_oi[32], s_ci[32];
  __shared__ GreedyRes s_res[2];  // this CTA's first-max, by step parity (read remotely)
  __shared__ int s_state[KM];
  __shared__ uint64_t s_ids;
  __shared__ double s_value;
  __shared__ int s_alive;
  const Codec codec{t.S};
  if (threadIdx.x == 0) {
    for (int m = 0; m < KM; ++m) s_state[m] = 0;
    s_ids = sp.pl_ids[sp.root_pid];
    s_value = 0.0;
    s_alive = 1;
  }
  __syncthreads();
  for (int s = 0; s < t.S; ++s) {
    const bool charge = s > 0 || has_initial;
    const double value = s_value;
    const uint64_t cur_ids = s_ids;
    int st[KM];
    for (int m = 0; m < KM; ++m) st[m] = s_state[m];
    double bv = -DBL_MAX;
    int boi = INT_MAX, bci = -1;
    for (int ci = rank * blockDim.x + threadIdx.x; ci < sp.n_cand; ci += nrank * blockDim.x) {
      const int sig = sp.cand_sig[ci];
      bool ok = true;
      for (int m = 0; m < t.M && ok; ++m) {
        const int ns = codec.advance(t.rt[m], st[m], (sig >> (3 * m)) & 7, s);
        ok = ns >= 0 && !(ns == 0 && (t.min_rt[m] < 0 || s + 1 + t.min_rt[m] > t.S));
      }
      if (!ok) continue;
      const int p = sp.cand_pid[ci];
      const uint64_t ids = sp.pl_ids[p];
      double v = value;
      for (int m = 0; m < t.M; ++m) {
        const double acc = st[m] == Codec::done() ? t.post[m] : t.pre[m];
        const bool changed = charge && field16(cur_ids, m) != field16(ids, m);
        const double eff = eff_cap(sp.pl_cap[p * KM + m], changed ? t.loss[m] : 0.0);
        v = dadd(v, dmul(thr_of(recv(m, s), eff), acc));
      }
      const int oi = sp.cand_oi[ci];
      if (g_better(v, oi, ci, bv, boi, bci)) {
        bv = v;
        boi = oi;
        bci = ci;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int ooi = __shfl_down_sync(0xffffffffu, boi, o);
      const int oci = __shfl_down_sync(0xffffffffu, bci, o);
      if (g_better(ov, ooi, oci, bv, boi, bci)) {
        bv = ov;
        boi = ooi;
        bci = oci;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      s_v[threadIdx.x >> 5] = bv;
      s_oi[threadIdx.x >> 5] = boi;
      s_ci[threadIdx.x >> 5] = bci;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      GreedyRes r{-DBL_MAX, INT_MAX, -1};
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w)
        if (g_better(s_v[w], s_oi[w], s_ci[w], r.v, r.oi, r.ci)) r = GreedyRes{s_v[w], s_oi[w], s_ci[w]};
      s_res[s & 1] = r;
    }
    cluster.sync();  // every CTA's step-s result is published
    if (threadIdx.x == 0) {
      GreedyRes b{-DBL_MAX, INT_MAX, -1};
      for (int q = 0; q < nrank; ++q) {  // same order in every CTA: identical winners
        const GreedyRes r = cluster.map_shared_rank(s_res, q)[s & 1];
        if (g_better(r.v, r.oi, r.ci, b.v, b.oi, b.ci)) b = r;
      }
      if (b.ci < 0) {
        s_alive = 0;
        if (rank == 0) greedy[s] = -1;
      } else {
        if (rank == 0) greedy[s] = b.oi;
        s_value = b.v;
        const int sig = sp.cand_sig[b.ci];
        for (int m = 0; m < t.M; ++m) s_state[m] = codec.advance(t.rt[m], s_state[m], (sig >> (3 * m)) & 7, s);
        s_ids = sp.pl_ids[sp.cand_pid[b.ci]];
      }
    }
    __syncthreads();
    if (!s_alive) break;
  }
  if (threadIdx.x == 0 && rank == 0) {
    bool all_done = s_alive != 0;
    for (int m = 0; m < t.M; ++m) all_done = all_done && s_state[m] == Codec::done();
    *incumbent = all_done ? s_value : -INFINITY;
  }
  cluster.sync();  // no CTA exits while another may still read its shared memory
}

// The same walk on ONE CTA when the candidates and placements fit in shared
// memory (the usual case: thousands of candidates at M <= 2): everything the
// walk reads is staged once, the feasible signatures are flagged once per
// step, and a step costs one first-max over shared memory and two barriers.
constexpr int kGreedyOneThreads = 1024;

__global__ void __launch_bounds__(kGreedyOneThreads) k_greedy_one(DevSpace sp, HostTables t, Recv recv,
                                                                  int has_initial, double* incumbent,
                                                                  int32_t* greedy) {
  extern __shared__ unsigned char smem[];
  const int M = t.M, nc = sp.n_cand, P1 = sp.P1;
  double* s_cap = reinterpret_cast<double*>(smem);                         // [P1][M]
  uint64_t* s_pids = reinterpret_cast<uint64_t*>(s_cap + static_cast<size_t>(P1) * M);  // [P1]
  int32_t* s_oi = reinterpret_cast<int32_t*>(s_pids + P1);                 // [nc]
  int32_t* s_sp = s_oi + nc;                                               // [nc] sig << 20 | pid
  __shared__ double w_v[32];
  __shared__ int w_oi[32], w_ci[32];
  __shared__ uint8_t s_sig_ok[1 << (3 * KM)];
  __shared__ int s_state[KM];
  __shared__ uint64_t s_ids;
  __shared__ double s_value;
  __shared__ int s_alive, s_best;
  const Codec codec{t.S};
  for (int i = threadIdx.x; i < P1; i += blockDim.x) {
    for (int m = 0; m < M; ++m) s_cap[i * M + m] = sp.pl_cap[i * KM + m];
    s_pids[i] = sp.pl_ids[i];
  }
  for (int i = threadIdx.x; i < nc; i += blockDim.x) {
    s_oi[i] = sp.cand_oi[i];
    s_sp[i] = (sp.cand_sig[i] << 20) | sp.cand_pid[i];
  }
  if (threadIdx.x == 0) {
    for (int m = 0; m < KM; ++m) s_state[m] = 0;
    s_ids = sp.pl_ids[sp.root_pid];
    s_value = 0.0;
    s_alive = 1;
  }
  __syncthreads();
  const int n_sig = 1 << (3 * M);
  for (int s = 0; s < t.S; ++s) {
    const bool charge = s > 0 || has_initial;
    for (int g = threadIdx.x; g < n_sig; g += blockDim.x) {  // status feasibility per signature
      bool ok = true;
      for (int m = 0; m < M && ok; ++m) {
        const int ns = codec.advance(t.rt[m], s_state[m], (g >> (3 * m)) & 7, s);
        ok = ns >= 0 && !(ns == 0 && (t.min_rt[m] < 0 || s + 1 + t.min_rt[m] > t.S));
      }
      s_sig_ok[g] = ok ? 1 : 0;
    }
    __syncthreads();
    const double value = s_value;
    const uint64_t cur_ids = s_ids;
    double acc[KM], rv[KM];
    for (int m = 0; m < M; ++m) {
      acc[m] = s_state[m] == Codec::done() ? t.post[m] : t.pre[m];
      rv[m] = recv(m, s);
    }
    double bv = -DBL_MAX;
    int boi = INT_MAX, bci = -1;
    for (int ci = threadIdx.x; ci < nc; ci += blockDim.x) {
      const int spv = s_sp[ci];
      if (!s_sig_ok[spv >> 20]) continue;
      const int p = spv & 0xfffff;
      const uint64_t ids = s_pids[p];
      double v = value;
      for (int m = 0; m < M; ++m) {
        const bool changed = charge && field16(cur_ids, m) != field16(ids, m);
        const double eff = eff_cap(s_cap[p * M + m], changed ? t.loss[m] : 0.0);
        v = dadd(v, dmul(thr_of(rv[m], eff), acc[m]));
      }
      const int oi = s_oi[ci];
      if (g_better(v, oi, ci, bv, boi, bci)) {
        bv = v;
        boi = oi;
        bci = ci;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_down_sync(0xffffffffu, bv, o);
      const int ooi = __shfl_down_sync(0xffffffffu, boi, o);
      const int oci = __shfl_down_sync(0xffffffffu, bci, o);
      if (g_better(ov, ooi, oci, bv, boi, bci)) {
        bv = ov;
        boi = ooi;
        bci = oci;
      }
    }
    if ((threadIdx.x & 31) == 0) {
      w_v[threadIdx.x >> 5] = bv;
      w_oi[threadIdx.x >> 5] = boi;
      w_ci[threadIdx.x >> 5] = bci;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // first-max over the warps, one warp
      const int nw = static_cast<int>(blockDim.x >> 5);
      double v = threadIdx.x < nw ? w_v[threadIdx.x] : -DBL_MAX;
      int oi = threadIdx.x < nw ? w_oi[threadIdx.x] : INT_MAX, ci = threadIdx.x < nw ? w_ci[threadIdx.x] : -1;
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, v, o);
        const int ooi = __shfl_down_sync(0xffffffffu, oi, o);
        const int oci = __shfl_down_sync(0xffffffffu, ci, o);
        if (g_better(ov, ooi, oci, v, oi, ci)) {
          v = ov;
          oi = ooi;
          ci = oci;
        }
      }
      if (threadIdx.x == 0) {
        if (ci < 0) {
          s_alive = 0;
          greedy[s] = -1;
        } else {
          greedy[s] = oi;
          s_value = v;
          s_best = ci;
          const int sig = s_sp[ci] >> 20;
          for (int m = 0; m < M; ++m) s_state[m] = codec.advance(t.rt[m], s_state[m], (sig >> (3 * m)) & 7, s);
          s_ids = s_pids[s_sp[ci] & 0xfffff];
        }
      }
    }
    __syncthreads();
    if (!s_alive) break;
  }
  if (threadIdx.x == 0) {
    bool all_done = s_alive != 0;
    for (int m = 0; m < M; ++m) all_done = all_done && s_state[m] == Codec::done();
    *incumbent = all_done ? s_value : -INFINITY;
  }
}

size_t greedy_one_smem(const DevSpace& sp, int M) {
  return static_cast<size_t>(sp.P1) * (M * 8 + 8) + static_cast<size_t>(sp.n_cand) * 8;
}

}  // namespace

void goodput_reductions(Ctx& c, const Prepared& pr, const DevSpace& sp, const double* d_recv, double* d_ub,
                        double* d_incumbent, int32_t* d_greedy) {
  const HostTables& t = pr.t;
  Recv recv{d_recv, t.S};
  double* best = c.buf<double>("ub_best", t.S);
  k_ub_best<<<t.S, 256, 0, c.stream>>>(sp, t, recv, best);
  ++c.kernel_launches;
  k_ub_suffix<<<1, 32, 0, c.stream>>>(best, t.S, d_ub);
  ++c.kernel_launches;
  const size_t smem = greedy_one_smem(sp, t.M);
  if (smem <= 200 * 1024 && sp.P1 < (1 << 20) && t.M <= 2) {  // placement index in 20 bits, signature above
    static size_t configured = 0;
    if (smem > configured) {
      MGS_CUDA_OK(cudaFuncSetAttribute(k_greedy_one, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      configured = smem;
    }
    k_greedy_one<<<1, kGreedyOneThreads, smem, c.stream>>>(sp, t, recv, pr.has_initial, d_incumbent, d_greedy);
    ++c.kernel_launches;
    MGS_CUDA_OK(cudaGetLastError());
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kGreedyCluster);
  cfg.blockDim = dim3(1024);
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kGreedyCluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  MGS_CUDA_OK(cudaLaunchKernelEx(&cfg, k_greedy, sp, t, recv, pr.has_initial, d_incumbent, d_greedy));
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// evaluate_plan(verify=false) batch: thread per (plan, trace).
__global__ void k_evaluate(DevSpace sp, HostTables t, const int32_t* plans, int n_plans, const uint8_t* overrides,
                           const int64_t* arrivals, int n_traces, int has_initial, uint4 init_lo, double* total,
                           double* thr_out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n_plans * n_traces) return;
  const int i = static_cast<int>(idx / n_traces), j = static_cast<int>(idx % n_traces);
  const int S = t.S, M = t.M;
  const int32_t* plan = plans + (size_t)i * S;
  const int64_t* arr = arrivals + (size_t)j * M * S;
  const uint32_t init[KM] = {init_lo.x, init_lo.y, init_lo.z, init_lo.w};
  int finish_after[KM];
  for (int m = 0; m < M; ++m) {  // Eq-12: finished strictly before step s (evaluate.hpp:174-179)
    finish_after[m] = INT_MAX;
    for (int s = S - 1; s >= 0; --s)
      if (sp.opt_rsize[plan[s] * KM + m] > 0) {
        finish_after[m] = s + 1;
        break;
      }
  }
  double tot = 0.0;
  for (int s = 0; s < S; ++s) {
    const int o = plan[s];
    for (int m = 0; m < M; ++m) {
      const uint32_t mask = sp.opt_mask[o * KM + m];
      const bool changed = s == 0 ? (has_initial && mask != init[m]) : (mask != sp.opt_mask[plan[s - 1] * KM + m]);
      // an override (pre-initialisation, psi_eff = 0) replaces psi (evaluate.hpp:193-197)
      const bool zero_psi = overrides && overrides[(static_cast<size_t>(i) * S + s) * M + m];
      const double eff = eff_cap(sp.opt_cap[o * KM + m], changed && !zero_psi ? t.loss[m] : 0.0);
      const double thr = thr_of(static_cast<double>(arr[m * S + s]), eff);
      const double acc = s >= finish_after[m] ? t.post[m] : t.pre[m];
      tot = dadd(tot, dmul(thr, acc));
      if (thr_out) thr_out[(idx * S + s) * M + m] = thr;
    }
  }
  total[idx] = tot;
}

// Few (plan, trace) pairs (the solve's own objective): one CTA per pair. The
// threads gather every (step, tenant) term in parallel -- option lookups,
// change flags, completion, throughput, goodput -- into shared memory; one
// thread then folds the goodputs in the reference's order (step-major,
// tenant-minor), so the sequential part is S*M dependent adds, not S*M
// dependent global loads.
constexpr int kEvalOneThreads = 256;
__global__ void __launch_bounds__(kEvalOneThreads) k_evaluate_one(DevSpace sp, HostTables t, const int32_t* plans,
                                                                 int n_plans, const uint8_t* overrides,
                                                                 const int64_t* arrivals, int n_traces,
                                                                 int has_initial, uint4 init_lo, double* total,
                                                                 double* thr_out) {
  extern __shared__ double s_good[];  // [S*M]
  __shared__ int s_finish[KM];
  const int pair = blockIdx.x;
  const int i = pair / n_traces, j = pair % n_traces;
  const int S = t.S, M = t.M;
  const int32_t* plan = plans + static_cast<size_t>(i) * S;
  const int64_t* arr = arrivals + static_cast<size_t>(j) * M * S;
  const uint32_t init[KM] = {init_lo.x, init_lo.y, init_lo.z, init_lo.w};
  if (threadIdx.x < KM) s_finish[threadIdx.x] = 0;  // last retraining step + 1 (0: none)
  __syncthreads();
  for (int k = threadIdx.x; k < S * M; k += blockDim.x) {
    const int s = k / M, m = k % M;
    if (sp.opt_rsize[plan[s] * KM + m] > 0) atomicMax(&s_finish[m], s + 1);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < S * M; k += blockDim.x) {
    const int s = k / M, m = k % M;
    const int o = plan[s];
    const uint32_t mask = sp.opt_mask[o * KM + m];
    const bool changed = s == 0 ? (has_initial && mask != init[m]) : (mask != sp.opt_mask[plan[s - 1] * KM + m]);
    const bool zero_psi = overrides && overrides[(static_cast<size_t>(i) * S + s) * M + m];
    const double eff = eff_cap(sp.opt_cap[o * KM + m], changed && !zero_psi ? t.loss[m] : 0.0);
    const double thr = thr_of(static_cast<double>(arr[m * S + s]), eff);
    const bool done = s_finish[m] > 0 && s >= s_finish[m];  // Eq-12 (evaluate.hpp:174-179)
    s_good[k] = dmul(thr, done ? t.post[m] : t.pre[m]);
    if (thr_out) thr_out[(static_cast<size_t>(pair) * S + s) * M + m] = thr;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int k = 0; k < S * M; ++k) tot = dadd(tot, s_good[k]);
    total[pair] = tot;
  }
}

void evaluate_batch(Ctx& c, const Prepared& pr, const DevSpace& sp, const int32_t* d_plans, int n_plans,
                    const int64_t* d_arr, int n_traces, double* d_total, double* d_thr, const uint8_t* d_overrides) {
  const long long n = (long long)n_plans * n_traces;
  uint4 init{pr.init_mask[0], pr.init_mask[1], pr.init_mask[2], pr.init_mask[3]};
  const size_t smem = static_cast<size_t>(pr.t.S) * pr.t.M * 8;
  if (n <= c.sm_count && smem <= 48 * 1024) {
    k_evaluate_one<<<static_cast<unsigned>(n), kEvalOneThreads, smem, c.stream>>>(
        sp, pr.t, d_plans, n_plans, d_overrides, d_arr, n_traces, pr.has_initial, init, d_total, d_thr);
  } else {
    k_evaluate<<<ceil_div(n, 128), 128, 0, c.stream>>>(sp, pr.t, d_plans, n_plans, d_overrides, d_arr, n_traces,
                                                       pr.has_initial, init, d_total, d_thr);
  }
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

}  // namespace mgs
