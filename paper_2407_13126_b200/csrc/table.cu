// Batched Goodput table (configs 2/4: thousands of traces of one window
// shape). For every trace b and slot s, the best accuracy-weighted
// SLO-attained count any candidate allocation can reach,
//   best[b][s] = max(0, max_o sum_m acc_max[m] * min(recv[b][m][s], cap_o[m]))
// and its suffix sum ub[b][s] = best[b][s] + ub[b][s+1], ub[b][S] = 0 -- the
// optimistic bound solve_dp builds before its search (solvers.hpp:258-280),
// for a whole batch of traces in one launch.
//
// Exactness. The reference folds v = 0; v += acc_max[m] * thr(m) (m ascending)
// and keeps std::max. Because rounding is monotone and acc_max >= 0,
//   fl(acc * min(r, c)) == min(fl(acc * r), fl(acc * c)),
// so the kernel pre-scales capabilities (wc = acc_max * cap, per placement) and
// arrivals (wr = acc_max * recv, per slot) and folds min(wr, wc) in the same
// order: bit-identical terms and sums. The same monotonicity means a placement
// whose weighted capabilities are dominated componentwise by another's can
// never exceed it, so the max runs over the Pareto-maximal placements only --
// the maximum (a value, not an index) is unchanged bit for bit.
//
// Layout: arrivals int32 [B][M][S] (coalesced along s), Pareto placements'
// weighted capabilities staged in shared memory in tiles, each thread owns up
// to kSlotsPerThread slots of one trace in registers and reuses every staged
// placement across them; one CTA per trace, the suffix fold by one thread in
// the reference's order.
#include <cub/device/device_select.cuh>

#include <algorithm>

#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kTabThreads = 256;
constexpr int kSlotsPerThread = 4;   // S <= 1024 per pass over the placements
constexpr int kTile = 2048;          // placements per shared-memory tile

// weighted capabilities of every placement: wc[p][m] = acc_max[m] * cap[p][m]
__global__ void k_weight_caps(const double* pl_cap, int P, int M, double4 acc_max, double* wc) {
  const double am[4] = {acc_max.x, acc_max.y, acc_max.z, acc_max.w};
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x)
    for (int m = 0; m < KM; ++m) wc[p * KM + m] = m < M ? dmul(am[m], pl_cap[p * KM + m]) : 0.0;
}

// keep p unless another placement dominates it (>= everywhere, > somewhere),
// or equals it with a smaller index (one representative per vector)
__global__ void k_pareto_flag(const double* wc, int P, int M, uint8_t* keep) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    double c[KM];
    for (int m = 0; m < KM; ++m) c[m] = wc[p * KM + m];
    bool dominated = false;
    for (int q = 0; q < P && !dominated; ++q) {
      if (q == p) continue;
      bool ge = true, gt = false;
      for (int m = 0; m < M; ++m) {
        const double x = wc[q * KM + m];
        ge = ge && x >= c[m];
        gt = gt || x > c[m];
      }
      dominated = ge && (gt || q < p);
    }
    keep[p] = dominated ? 0 : 1;
  }
}

template <int M>
__global__ void __launch_bounds__(kTabThreads) k_table(const double* __restrict__ wcp, int np, int tile_cap,
                                                      const int32_t* __restrict__ arrivals, int S, double4 acc_max,
                                                      double* __restrict__ best_out, double* __restrict__ ub_out) {
  extern __shared__ double smem[];
  double* tile = smem;                    // [tile_cap][M]
  double* best_s = smem + tile_cap * M;   // [S]
  const int nthr = blockDim.x;
  const int b = blockIdx.x;
  const int32_t* arr = arrivals + static_cast<size_t>(b) * M * S;
  const double am[4] = {acc_max.x, acc_max.y, acc_max.z, acc_max.w};
  for (int s0 = 0; s0 < S; s0 += nthr * kSlotsPerThread) {
    double wr[kSlotsPerThread][M], best[kSlotsPerThread];
#pragma unroll
    for (int k = 0; k < kSlotsPerThread; ++k) {
      const int s = s0 + k * nthr + threadIdx.x;  // coalesced along s
      best[k] = 0.0;                                     // the reference starts at 0.0
#pragma unroll
      for (int m = 0; m < M; ++m) wr[k][m] = s < S ? dmul(am[m], static_cast<double>(arr[m * S + s])) : 0.0;
    }
    for (int t0 = 0; t0 < np; t0 += tile_cap) {
      const int nt = min(tile_cap, np - t0);
      __syncthreads();
      for (int i = threadIdx.x; i < nt * M; i += nthr)  // rows are KM wide in global memory
        tile[i] = wcp[static_cast<size_t>(t0 + i / M) * KM + i % M];
      __syncthreads();
      for (int p = 0; p < nt; ++p) {
        double c[M];
#pragma unroll
        for (int m = 0; m < M; ++m) c[m] = tile[p * M + m];  // broadcast
#pragma unroll
        for (int k = 0; k < kSlotsPerThread; ++k) {
          double v = 0.0;
#pragma unroll
          for (int m = 0; m < M; ++m) v = dadd(v, fmin(wr[k][m], c[m]));
          best[k] = best[k] < v ? v : best[k];  // std::max(best, v)
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kSlotsPerThread; ++k) {
      const int s = s0 + k * nthr + threadIdx.x;
      if (s < S) best_s[s] = best[k];
    }
  }
  __syncthreads();
  double* bo = best_out ? best_out + static_cast<size_t>(b) * S : nullptr;
  for (int s = threadIdx.x; s < S && bo; s += nthr) bo[s] = best_s[s];
  if (threadIdx.x == 0) {  // suffix fold in the reference's order (solvers.hpp:278-279)
    double* ub = ub_out + static_cast<size_t>(b) * (S + 1);
    double acc = 0.0;
    ub[S] = 0.0;
    for (int s = S - 1; s >= 0; --s) {
      acc = dadd(acc, best_s[s]);
      ub[s] = acc;
    }
  }
}

}  // namespace

// Pareto-maximal placements' weighted capabilities (rows of KM doubles) for
// one window's tables; returns their count.
int table_prepare(Ctx& c, const Prepared& pr, const DevSpace& sp, double** wcp_out) {
  const HostTables& t = pr.t;
  const int M = t.M, P = sp.P;
  double am[4] = {0, 0, 0, 0};
  for (int m = 0; m < M; ++m) am[m] = t.pre[m] > t.post[m] ? t.pre[m] : t.post[m];  // std::max(pre, post)
  const double4 acc_max{am[0], am[1], am[2], am[3]};
  double* wc = c.buf<double>("tab_wc", static_cast<size_t>(P) * KM + KM);
  uint8_t* keep = c.buf<uint8_t>("tab_keep", P + 1);
  k_weight_caps<<<ceil_div(P, 256), 256, 0, c.stream>>>(sp.pl_cap, P, M, acc_max, wc);
  k_pareto_flag<<<ceil_div(P, 128), 128, 0, c.stream>>>(wc, P, M, keep);
  c.kernel_launches += 2;
  int* d_np = c.buf<int>("tab_np", 1);
  const double4* rows = reinterpret_cast<const double4*>(wc);
  double* wcp = c.buf<double>("tab_wcp", static_cast<size_t>(P) * KM + KM);
  size_t tb = 0;
  MGS_CUDA_OK(cub::DeviceSelect::Flagged(nullptr, tb, rows, keep, reinterpret_cast<double4*>(wcp), d_np, P, c.stream));
  void* tmp = c.buf<char>("tab_cub", tb);
  MGS_CUDA_OK(cub::DeviceSelect::Flagged(tmp, tb, rows, keep, reinterpret_cast<double4*>(wcp), d_np, P, c.stream));
  *wcp_out = wcp;
  return read_scalar(c, d_np);
}

// The table kernel over n_traces device-resident traces (stream-ordered, no sync).
void table_run(Ctx& c, const Prepared& pr, const double* wcp, int np, const int32_t* d_arr, int n_traces,
               double* d_best, double* d_ub) {
  const HostTables& t = pr.t;
  const int M = t.M, S = t.S;
  double am[4] = {0, 0, 0, 0};
  for (int m = 0; m < M; ++m) am[m] = t.pre[m] > t.post[m] ? t.pre[m] : t.post[m];
  const double4 acc_max{am[0], am[1], am[2], am[3]};
  // shared memory: only as many placement rows as exist (up to a tile), so
  // small Pareto sets leave room for more resident CTAs; threads: enough to
  // give every thread kSlotsPerThread slots of the window (warp multiple)
  const int tile_cap = std::max(1, std::min(kTile, np));
  const size_t smem = (static_cast<size_t>(tile_cap) * M + S) * sizeof(double);
  const int want = (S + kSlotsPerThread - 1) / kSlotsPerThread;
  const int threads = std::min(kTabThreads, std::max(32, (want + 31) / 32 * 32));
  if (n_traces <= 0) return;
  auto launch = [&](auto kern) {
    if (smem > 48 * 1024)
      MGS_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<n_traces, threads, smem, c.stream>>>(wcp, np, tile_cap, d_arr, S, acc_max, d_best, d_ub);
  };
  switch (M) {
    case 1: launch(k_table<1>); break;
    case 2: launch(k_table<2>); break;
    case 3: launch(k_table<3>); break;
    default: launch(k_table<4>); break;
  }
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

}  // namespace mgs
