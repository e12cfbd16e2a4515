// Request-mode trace replay (run_requests, simulator.hpp:209-275) over a
// scenario's W windows (queues, psi spill and masks carried across them): the
// literal "replay the arrival trace through each instance's profiled
// throughput and count SLO-attained requests" for a batch of
// (plan, trace, seed) runs, one thread per (run, tenant).
//
// Per tenant, sequentially over the window's steps (the reference's order):
//   build_series (simulator.hpp:72-131): raw capability of the step's option,
//     inference-mask change vs the previous step (never at step 0 of the first
//     window), psi spilled through a pool consumed at most 1 per step,
//     eff = raw - consumed*raw, completion = step >= last retraining step + 1;
//   arrivals enter a FIFO at the step start with deadline now + 2*latency_full;
//   lapsed requests drop; floor(eff + 1e-9) requests are served, the k-th at
//   now + k*g/eff, timely iff <= deadline + 1e-12; each served request draws
//   correctness from the tenant's own mt19937_64 stream
//   (seed*phi + c*(m+1), 64 outputs discarded).
// All requests that arrive in one step share their deadline, so the FIFO is a
// ring of (arrival step, count) batches. The counters are sums of 1.0 (exact)
// except overhead_seconds, folded in step order like the reference.
#include "ctx.cuh"

namespace mgs {
namespace {

// std::mt19937_64 (the C++ standard's parameters), state in local memory.
struct Mt64 {
  static constexpr int N = 312, Mm = 156;
  uint64_t mt[N];
  int idx;
  __device__ void seed(uint64_t s) {
    mt[0] = s;
    for (int i = 1; i < N; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + static_cast<uint64_t>(i);
    idx = N;
  }
  __device__ void twist() {
    constexpr uint64_t kUpper = ~0ull << 31, kLower = ~kUpper, kA = 0xb5026f5aa96619e9ull;
    for (int k = 0; k < N - Mm; ++k) {
      const uint64_t y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
      mt[k] = mt[k + Mm] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
    }
    for (int k = N - Mm; k < N - 1; ++k) {
      const uint64_t y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
      mt[k] = mt[k + (Mm - N)] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
    }
    const uint64_t y = (mt[N - 1] & kUpper) | (mt[0] & kLower);
    mt[N - 1] = mt[Mm - 1] ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
    idx = 0;
  }
  __device__ uint64_t next() {
    if (idx >= N) twist();
    uint64_t z = mt[idx++];
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71d67fffeda60000ull;
    z ^= (z << 37) & 0xfff7eee000000000ull;
    z ^= z >> 43;
    return z;
  }
};

struct ReplayArgs {
  DevSpace sp;
  HostTables t;
  int W;                   // windows: plans are [n_plans][W][S], arrivals span W*S steps
  const double* acc;       // [W][2][M]: acc_pre, acc_post of each window
  const int32_t* plans;    // [n_plans][W][S]
  const uint8_t* overrides;  // [n_plans][W][S][M] psi_eff = 0 (pre-initialisation), or null
  const int64_t* arrivals; // [n_traces][M][W*S]
  const uint64_t* seeds;   // [n_seeds]
  int n_plans, n_traces, n_seeds;
  double slo[KM];          // 2 * latency_full
  double psi[KM];          // reconfiguration overhead in steps (profile psi, not the loss fraction)
  double g_len;            // step seconds
  int32_t* q_step;         // [runs*M][W*S] FIFO batches (arrival step)
  int64_t* q_count;
  mgs_job_metrics* out;    // [run][W][M]
};

__global__ void k_replay(ReplayArgs a) {
  const int M = a.t.M, S = a.t.S, W = a.W, G = W * S;
  const long long runs = static_cast<long long>(a.n_plans) * a.n_traces * a.n_seeds;
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (tid >= runs * M) return;
  const int m = static_cast<int>(tid % M);
  const long long run = tid / M;
  const int si = static_cast<int>(run % a.n_seeds);
  const int ti = static_cast<int>((run / a.n_seeds) % a.n_traces);
  const int pi = static_cast<int>(run / (static_cast<long long>(a.n_seeds) * a.n_traces));
  const int64_t* arr = a.arrivals + (static_cast<size_t>(ti) * M + m) * G;
  int32_t* qs = a.q_step + static_cast<size_t>(tid) * G;
  int64_t* qc = a.q_count + static_cast<size_t>(tid) * G;

  Mt64 rng;
  rng.seed(a.seeds[si] * 0x9e3779b97f4a7c15ull + 0x517cc1b727220a95ull * static_cast<uint64_t>(m + 1));
  for (int i = 0; i < 64; ++i) rng.next();  // discard(64)

  double spill = 0.0;     // carried across windows (build_series keeps one pool)
  uint32_t prev_mask = 0;
  int qh = 0, qt = 0;     // FIFO [qh, qt) of batches, carried across windows
  for (int w = 0; w < W; ++w) {
    const int32_t* plan = a.plans + (static_cast<size_t>(pi) * W + w) * S;
    int finish_after = INT_MAX;  // Eq. 12 (evaluate.hpp:174-179), per window
    for (int s = S - 1; s >= 0; --s)
      if (a.sp.opt_rsize[plan[s] * KM + m] > 0) {
        finish_after = s + 1;
        break;
      }
    const double acc_pre = a.acc[(w * 2 + 0) * M + m], acc_post = a.acc[(w * 2 + 1) * M + m];
    double received = 0.0, served = 0.0, timely = 0.0, correct = 0.0, valid = 0.0, dropped = 0.0, overhead = 0.0;
    int reconf = 0;
    for (int s = 0; s < S; ++s) {
      const int g = w * S + s;
      const int o = plan[s];
      const double raw = a.sp.opt_cap[o * KM + m];
      const uint32_t mask = a.sp.opt_mask[o * KM + m];
      // never at the very first step; across a window boundary against the
      // previous window's last step (simulator.hpp:105-107)
      const bool changed = g > 0 && mask != prev_mask;
      prev_mask = mask;
      double applied = 0.0;
      if (changed) {
        const bool zero = a.overrides && a.overrides[((static_cast<size_t>(pi) * W + w) * S + s) * M + m];
        applied = zero ? 0.0 : a.psi[m];  // EffectivePlan overrides (simulator.hpp:112-114)
        spill = dadd(spill, applied);
      }
      const double consumed = spill < 1.0 ? spill : 1.0;
      spill = dsub(spill, consumed);
      const double cap = eff_cap(raw, consumed);
      const double now = dmul(static_cast<double>(g), a.g_len);
      const long long arriving = arr[g];
      received = dadd(received, static_cast<double>(arriving));
      if (arriving > 0) {
        qs[qt] = g;
        qc[qt] = arriving;
        ++qt;
      }
      while (qh < qt && dadd(dmul(static_cast<double>(qs[qh]), a.g_len), a.slo[m]) < now) {  // lapsed deadlines
        dropped = dadd(dropped, static_cast<double>(qc[qh]));
        ++qh;
      }
      const long long n = static_cast<long long>(dadd(cap, 1e-9));
      const double acc = s >= finish_after ? acc_post : acc_pre;
      for (long long k = 1; k <= n && qh < qt; ++k) {
        const double deadline = dadd(dmul(static_cast<double>(qs[qh]), a.g_len), a.slo[m]);
        if (--qc[qh] == 0) ++qh;
        const double completion = dadd(now, __ddiv_rn(dmul(static_cast<double>(k), a.g_len), cap));
        const bool is_timely = completion <= dadd(deadline, 1e-12);
        const bool is_correct = static_cast<double>(rng.next() >> 11) * 0x1.0p-53 < acc;
        served += 1.0;
        if (is_timely) timely += 1.0;
        if (is_correct) correct += 1.0;
        if (is_timely && is_correct) valid += 1.0;
      }
      if (changed) {
        ++reconf;
        overhead = dadd(overhead, dmul(applied, a.g_len));
      }
    }
    double queued = 0.0;  // the horizon's last window closes with what is still queued
    if (w == W - 1)
      for (int i = qh; i < qt; ++i) queued = dadd(queued, static_cast<double>(qc[i]));
    mgs_job_metrics& r = a.out[(run * W + w) * M + m];
    r.received = received;
    r.served = served;
    r.timely = timely;
    r.correct = correct;
    r.valid = valid;
    r.dropped = dropped;
    r.queued_at_end = queued;
    r.reconfigurations = reconf;
    r.overhead_seconds = overhead;
  }
}

}  // namespace

void replay_requests(Ctx& c, const Prepared& pr, const DevSpace& sp, int W, const double* d_acc, const double* psi,
                     const double* slo, double step_seconds, const int32_t* d_plans, const uint8_t* d_overrides,
                     int n_plans, const int64_t* d_arr, int n_traces, const uint64_t* d_seeds,
                     int n_seeds, mgs_job_metrics* d_out) {
  const HostTables& t = pr.t;
  ReplayArgs a{};
  a.sp = sp;
  a.t = t;
  a.W = W;
  a.acc = d_acc;
  a.plans = d_plans;
  a.overrides = d_overrides;
  a.arrivals = d_arr;
  a.seeds = d_seeds;
  a.n_plans = n_plans;
  a.n_traces = n_traces;
  a.n_seeds = n_seeds;
  for (int m = 0; m < t.M; ++m) {
    a.slo[m] = slo[m];
    a.psi[m] = psi[m];
  }
  a.g_len = step_seconds;
  const long long threads = static_cast<long long>(n_plans) * n_traces * n_seeds * t.M;
  if (threads == 0) return;
  a.q_step = c.buf<int32_t>("rp_qstep", static_cast<size_t>(threads) * W * t.S);
  a.q_count = c.buf<int64_t>("rp_qcount", static_cast<size_t>(threads) * W * t.S);
  a.out = d_out;
  k_replay<<<ceil_div(threads, 64), 64, 0, c.stream>>>(a);
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
}

}  // namespace mgs
