// Shared device-side definitions for the B200 Goodput planner.
//
// Arithmetic parity rules: every double op on the
// planner path is written with explicit round-to-nearest intrinsics so no FMA
// contraction can happen regardless of compiler flags (the library is also
// built with --fmad=false), and the fold orders are the reference's.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "migsim_b200.h"

namespace mgs {

constexpr int KM = MGS_MAX_MODELS;
constexpr int kWarp = 32;

// plan_types.hpp:68-72 — loss = min(psi,1); eff = raw - loss*raw; thr = min(recv, cap)
__host__ __device__ inline double eff_cap(double raw, double loss) {
#ifdef __CUDA_ARCH__
  return __dsub_rn(raw, __dmul_rn(loss, raw));
#else
  return raw - loss * raw;
#endif
}
__host__ __device__ inline double thr_of(double recv, double cap) { return recv < cap ? recv : cap; }
__device__ inline double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ inline double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ inline double dsub(double a, double b) { return __dsub_rn(a, b); }

// dp_better (solvers.hpp:123-126): higher value, then smaller lex. Inside one
// frontier a state's dense rank orders exactly like its lex, so the same
// comparator is used with ranks.
__host__ __device__ inline bool better(double va, uint64_t la, double vb, uint64_t lb) {
  if (va != vb) return va > vb;
  return la < lb;
}

// Goodput values are sums of thr*acc with thr >= 0 and acc in [0,1], so they
// are never negative and their IEEE bit patterns order like the values.
__device__ inline unsigned long long vbits(double v) { return static_cast<unsigned long long>(__double_as_longlong(v)); }

// Packed per-tenant fields: 16 bits per tenant in a uint64 (StatusCodec::pack,
// space.hpp:270-274 — kept 64-bit end to end).
__host__ __device__ inline int field16(uint64_t key, int m) { return static_cast<int>((key >> (16 * m)) & 0xffff); }

// engine::StatusCodec (space.hpp:255-298): 0 not started, 1 done, otherwise
// running on k GPCs with rem steps left including this one. The reference
// numbers running statuses 2+(k-1)*S+(rem-1); the codes are only compared for
// equality and decoded, never ordered, so the device packs them as
// 2+((k-1)<<13 | (rem-1)) whenever S <= 8192 (k <= 7 keeps the code in 16
// bits) and decodes with shifts instead of divisions by S. Longer windows use
// the reference numbering.
struct Codec {
  int S;
  int shift;
  __host__ __device__ explicit Codec(int s) : S(s), shift(s <= 8192 ? 13 : 0) {}
  // sh = 0: the reference numbering (compact codes, < 256 for S <= 36)
  __host__ __device__ Codec(int s, int sh) : S(s), shift(sh) {}
  __host__ __device__ static constexpr int done() { return 1; }
  __host__ __device__ int running(int k, long long rem) const {
    return shift ? 2 + (((k - 1) << shift) | static_cast<int>(rem - 1)) : 2 + (k - 1) * S + static_cast<int>(rem - 1);
  }
  __host__ __device__ static bool is_running(int c) { return c >= 2; }
  __host__ __device__ int run_size(int c) const { return shift ? ((c - 2) >> shift) + 1 : (c - 2) / S + 1; }
  __host__ __device__ long long run_rem(int c) const {
    return shift ? ((c - 2) & ((1 << shift) - 1)) + 1 : (c - 2) % S + 1;
  }
  // StatusCodec::advance (space.hpp:286-297); -1 = incompatible
  __host__ __device__ int advance(const long long* rt_row, int status, int size, int s) const {
    if (is_running(status)) {
      if (size != run_size(status)) return -1;
      return run_rem(status) == 1 ? done() : running(size, run_rem(status) - 1);
    }
    if (status == done()) return size == 0 ? done() : -1;
    if (size == 0) return 0;
    const long long rt = rt_row[size];
    if (rt < 1 || s + rt > S) return -1;
    return rt == 1 ? done() : running(size, rt - 1);
  }
};

// status_dominates (solvers.hpp:128-134)
__host__ __device__ inline bool status_dominates(const Codec& c, int x, int y) {
  if (x == y) return true;
  if (x == Codec::done()) return true;
  if (Codec::is_running(x) && Codec::is_running(y) && c.run_size(x) == c.run_size(y)) return c.run_rem(x) <= c.run_rem(y);
  return false;
}

// Successor units of one status group (solvers.hpp:379-411 with allowed_sizes
// :79-97): every per-tenant retraining size the status allows, the cartesian
// product as a signature, kept when every tenant's advance is legal, idle
// not-started tenants can still start, and the signature has options.
// f(sig, packed successor status) is called per unit; returns the count.
template <class F>
__device__ int for_each_unit(int M, int S, const long long (*rt)[8], const long long* min_rt,
                             const int32_t* sig_nopt, uint64_t status, int s, F&& f) {
  const Codec codec{S};
  int st[KM], sizes[KM][9], cnt[KM];
  for (int m = 0; m < M; ++m) {
    st[m] = field16(status, m);
    cnt[m] = 0;
    if (Codec::is_running(st[m])) {
      sizes[m][cnt[m]++] = codec.run_size(st[m]);
    } else if (st[m] == Codec::done()) {
      sizes[m][cnt[m]++] = 0;
    } else {
      if (min_rt[m] >= 0 && s + 1 + min_rt[m] <= S) sizes[m][cnt[m]++] = 0;
      for (int k = 1; k <= 7; ++k)
        if (rt[m][k] >= 1 && s + rt[m][k] <= S) sizes[m][cnt[m]++] = k;
    }
    if (cnt[m] == 0) return 0;
  }
  int pick[KM] = {0, 0, 0, 0};
  int n = 0;
  while (true) {
    int sig = 0;
    uint64_t ns = 0;
    bool ok = true;
    for (int m = M - 1; m >= 0; --m) sig = sig * 8 + sizes[m][pick[m]];
    for (int m = 0; m < M && ok; ++m) {
      const int a = codec.advance(rt[m], st[m], sizes[m][pick[m]], s);
      ok = a >= 0 && !(a == 0 && (min_rt[m] < 0 || s + 1 + min_rt[m] > S));
      ns |= static_cast<uint64_t>(a < 0 ? 0 : a) << (16 * m);
    }
    if (ok && sig_nopt[sig] > 0) {
      f(sig, ns);
      ++n;
    }
    int m = 0;  // odometer over the per-tenant choices
    while (m < M && ++pick[m] == cnt[m]) pick[m++] = 0;
    if (m == M) break;
  }
  return n;
}

// Device-resident, per-solve option space (Space::build output + the derived
// candidate tables the DP consumes).
struct DevSpace {
  int M = 0, S = 0;
  int n_opt = 0;
  int n_sig = 0;       // 8^M
  int P = 0;           // distinct inference placements among options
  int P1 = 0;          // P + 1 (the root's carried-over placement)
  int n_cand = 0;      // distinct (signature, placement) pairs
  int root_pid = 0;    // == P
  int n_mask_ids[KM] = {0, 0, 0, 0};  // per tenant: mask ids in pl_ids (incl. the root's out-of-range id)
  // options (lex order)
  int32_t* opt_config = nullptr;
  int8_t* opt_labels = nullptr;   // [n_opt][MGS_MAX_SLOTS]
  uint32_t* opt_mask = nullptr;   // [n_opt][4]
  double* opt_cap = nullptr;      // [n_opt][4]
  int8_t* opt_rsize = nullptr;    // [n_opt][4]
  int32_t* opt_sig = nullptr;
  int32_t* opt_pid = nullptr;
  // placements
  uint64_t* pl_ids = nullptr;     // [P1] packed per-tenant mask ids
  double* pl_cap = nullptr;       // [P1][4] inference capability (summed in slot order)
  // candidates: (sig, pid) sorted, with the smallest option index
  int32_t* cand_pid = nullptr;
  int32_t* cand_oi = nullptr;
  int32_t* cand_sig = nullptr;
  int32_t* sig_off = nullptr;     // [n_sig+1]
  int32_t* sig_nopt = nullptr;    // [n_sig] reference option count (transitions_ref)
  // subset projections for the dense group tables
  int32_t* proj_id = nullptr;     // [2^M][P1]
  int32_t proj_base[(1 << KM) + 1];
  int32_t proj_total = 0;
};

// Host-side scalar tables (engine::Tables subset the kernels need).
struct HostTables {
  int M, S;
  double cap[KM][8];
  long long rt[KM][8];
  int floor_[KM];
  double loss[KM];
  double psi_raw[KM];  // profile psi in steps (overrides / spill replace it, not the loss fraction)
  double pre[KM], post[KM];
  long long min_rt[KM];
};

}  // namespace mgs

#define MGS_CUDA_OK(expr)                                              \
  do {                                                                 \
    cudaError_t _e = (expr);                                           \
    if (_e != cudaSuccess) throw ::mgs::CudaFail(_e, #expr, __LINE__); \
  } while (0)

namespace mgs {
struct CudaFail {
  cudaError_t err;
  const char* what;
  int line;
  CudaFail(cudaError_t e, const char* w, int l) : err(e), what(w), line(l) {}
};
}  // namespace mgs
