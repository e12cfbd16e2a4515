// solve_bruteforce (solvers.hpp:143-228) on the GPU: every allocation
// sequence of the window is scored by one thread, and the best is taken by a
// deterministic (value desc, sequence asc) reduction.
//
// The reference walks |O|^S sequences depth-first in option-index order and
// keeps the first strictly better complete, all-done leaf -- i.e. the
// lexicographically smallest optimal sequence of option indices. Options that
// share (retraining signature, inference placement) have identical statuses,
// masks and capabilities, so they score identically and the smallest-index one
// (the candidate's representative, DevSpace::cand_oi) always wins the tie. The
// kernel therefore enumerates candidate sequences (n_cand^S <= |O|^S) and
// breaks ties on the option-index sequence packed as a base-|O| integer, which
// orders exactly like the reference's visit order.
//
// Per sequence (thread): statuses advance by StatusCodec::advance, idle
// not-started tenants must remain startable (solvers.hpp:199-203), and the
// value folds step-major / model-minor with the charge rule of :205-214 --
// the same arithmetic as evaluate_plan, with explicit _rn intrinsics.
#include <cfloat>

#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kBfThreads = 256;

struct BfArgs {
  DevSpace sp;
  HostTables t;
  const double* recv;  // [M][S]
  int has_initial;
  uint32_t init[KM];
  unsigned long long n_seq;     // n_cand^S
  unsigned long long top_div;   // n_cand^(S-1)
  unsigned long long n_opt;     // |O| (tie-break radix)
};

// total order on doubles as unsigned keys (larger value -> larger key)
__device__ inline unsigned long long okey(double v) {
  const unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(v));
  return (u >> 63) ? ~u : (u | (1ull << 63));
}

struct Best {
  unsigned long long vkey;  // 0 = none
  unsigned long long lex;   // option-index sequence, base |O|
};

__device__ inline bool bf_better(const Best& a, const Best& b) {
  if (a.vkey != b.vkey) return a.vkey > b.vkey;
  return a.lex < b.lex;
}

__device__ inline Best warp_best(Best b) {
  for (int o = 16; o > 0; o >>= 1) {
    Best x{__shfl_down_sync(0xffffffffu, b.vkey, o), __shfl_down_sync(0xffffffffu, b.lex, o)};
    if (x.vkey && (!b.vkey || bf_better(x, b))) b = x;
  }
  return b;
}

__device__ inline Best block_best(Best b) {
  __shared__ unsigned long long sv[kBfThreads / 32], sl[kBfThreads / 32];
  b = warp_best(b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sv[w] = b.vkey;
    sl[w] = b.lex;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    Best x = threadIdx.x < kBfThreads / 32 ? Best{sv[threadIdx.x], sl[threadIdx.x]} : Best{0ull, 0ull};
    b = warp_best(x);
  }
  return b;
}

__global__ void __launch_bounds__(kBfThreads) k_bruteforce(BfArgs a, unsigned long long* part_v,
                                                          unsigned long long* part_l) {
  const DevSpace& sp = a.sp;
  const HostTables& t = a.t;
  const int M = t.M, S = t.S;
  const Codec codec{S};
  const unsigned long long nc = static_cast<unsigned long long>(sp.n_cand);
  Best best{0ull, 0ull};
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < a.n_seq;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int st[KM] = {0, 0, 0, 0};
    uint32_t mask[KM] = {a.init[0], a.init[1], a.init[2], a.init[3]};
    double v = 0.0;
    unsigned long long lex = 0, div = a.top_div, rest = i;
    bool ok = true;
    for (int s = 0; s < S && ok; ++s) {
      const unsigned long long d = div > 0 ? rest / div : 0;
      rest -= d * div;
      if (nc > 1) div /= nc;
      const int ci = static_cast<int>(d);
      const int sig = sp.cand_sig[ci];
      const int oi = sp.cand_oi[ci];
      int nst[KM];
      for (int m = 0; m < M && ok; ++m) {
        nst[m] = codec.advance(t.rt[m], st[m], (sig >> (3 * m)) & 7, s);
        ok = nst[m] >= 0;
      }
      for (int m = 0; m < M && ok; ++m)
        ok = !(nst[m] == 0 && (t.min_rt[m] < 0 || s + 1 + t.min_rt[m] > S));
      if (!ok) break;
      const bool charge = s > 0 || a.has_initial;
      for (int m = 0; m < M; ++m) {
        const double acc = st[m] == Codec::done() ? t.post[m] : t.pre[m];
        const uint32_t om = sp.opt_mask[oi * KM + m];
        const bool changed = charge && mask[m] != om;
        const double eff = eff_cap(sp.opt_cap[oi * KM + m], changed ? t.loss[m] : 0.0);
        v = dadd(v, dmul(thr_of(a.recv[m * S + s], eff), acc));
        mask[m] = om;
        st[m] = nst[m];
      }
      lex = lex * a.n_opt + static_cast<unsigned long long>(oi);
    }
    if (!ok) continue;
    bool all_done = true;
    for (int m = 0; m < M; ++m) all_done = all_done && st[m] == Codec::done();
    if (!all_done) continue;
    Best c{okey(v), lex};
    if (!best.vkey || bf_better(c, best)) best = c;
  }
  Best b = block_best(best);
  if (threadIdx.x == 0) {
    part_v[blockIdx.x] = b.vkey;
    part_l[blockIdx.x] = b.lex;
  }
}

__global__ void __launch_bounds__(kBfThreads) k_bruteforce_final(const unsigned long long* part_v,
                                                                const unsigned long long* part_l, int n,
                                                                unsigned long long* out) {
  Best b{0ull, 0ull};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    Best x{part_v[i], part_l[i]};
    if (x.vkey && (!b.vkey || bf_better(x, b))) b = x;
  }
  b = block_best(b);
  if (threadIdx.x == 0) {
    out[0] = b.vkey;
    out[1] = b.lex;
  }
}

}  // namespace

// Returns false when no feasible all-done sequence exists (infeasible.joint).
bool bruteforce(Ctx& c, const Prepared& pr, const DevSpace& sp, const double* d_recv, std::vector<int32_t>& plan) {
  const HostTables& t = pr.t;
  BfArgs a{};
  a.sp = sp;
  a.t = t;
  a.recv = d_recv;
  a.has_initial = pr.has_initial;
  for (int m = 0; m < KM; ++m) a.init[m] = pr.init_mask[m];
  a.n_opt = static_cast<unsigned long long>(sp.n_opt);
  // n_cand^S with an overflow guard (the caller has already applied the
  // reference's |O|^S <= bruteforce_cap gate)
  unsigned long long n = 1, top = 1;
  for (int s = 0; s < t.S; ++s) {
    if (sp.n_cand > 1 && n > (1ull << 62) / static_cast<unsigned long long>(sp.n_cand))
      throw PlanFail{MGS_ERR_ARGUMENT, "brute-force space exceeds 2^62 sequences"};
    if (s > 0) top = n;
    n *= static_cast<unsigned long long>(sp.n_cand);
  }
  if (t.S == 1) top = 1;
  a.n_seq = n;
  a.top_div = t.S > 0 ? top : 0;
  // option-index sequences must fit the 64-bit tie-break key: |O|^S < 2^64
  double lex_space = 1.0;
  for (int s = 0; s < t.S; ++s) lex_space *= static_cast<double>(sp.n_opt);
  if (lex_space >= 1.8e19) throw PlanFail{MGS_ERR_ARGUMENT, "brute-force tie-break key exceeds 64 bits"};

  const long long want = static_cast<long long>((n + kBfThreads - 1) / kBfThreads);
  const int blocks = static_cast<int>(std::min<long long>(std::max<long long>(want, 1), 148LL * 8));
  unsigned long long* part_v = c.buf<unsigned long long>("bf_part_v", blocks);
  unsigned long long* part_l = c.buf<unsigned long long>("bf_part_l", blocks);
  unsigned long long* d_out = c.buf<unsigned long long>("bf_out", 2);
  k_bruteforce<<<blocks, kBfThreads, 0, c.stream>>>(a, part_v, part_l);
  ++c.kernel_launches;
  k_bruteforce_final<<<1, kBfThreads, 0, c.stream>>>(part_v, part_l, blocks, d_out);
  ++c.kernel_launches;
  MGS_CUDA_OK(cudaGetLastError());
  unsigned long long* h = c.pinned.get<unsigned long long>(2);
  MGS_CUDA_OK(cudaMemcpyAsync(h, d_out, 16, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  if (h[0] == 0) return false;
  unsigned long long lex = h[1];
  plan.assign(t.S, 0);
  for (int s = t.S - 1; s >= 0; --s) {
    plan[s] = static_cast<int32_t>(lex % a.n_opt);
    lex /= a.n_opt;
  }
  return true;
}

}  // namespace mgs
