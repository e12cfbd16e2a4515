// The cross-slot max-plus dynamic program (solve_dp, solvers.hpp:242-579) on
// the GPU, reproducing the reference *procedure* bit for bit:
//   * frontier states keyed by (packed retraining status, inference placement);
//   * per status group and tenant subset, the best (value, lex) representative
//     per projected placement (:367-378);
//   * per (group, signature) unit and candidate placement: accuracy-weighted
//     SLO-attained gains, the subset-candidate predecessor choice (:435-447)
//     and the exact fold from that predecessor (:451-458), strict bound test
//     (:459);
//   * equal-key merge by (value desc, lex asc) (:467-468), placement band per
//     status (:499-511), status dominance within equal placements of <= 64
//     states (:514-537), state budget (:539-542), dense lex ranks (:544-548);
//   * best all-done terminal state and parent walk (:552-578).
//
// Frontier layout in HBM (structure of arrays, one entry per state, states of
// one status group contiguous):  status u64 | ids u64 | pid i32 | value f64 |
// lex u64 | rank u32, plus per-step (parent i32, option i32) history for the
// backtrack. Per step the units are ordered by successor status, so every
// successor status owns one contiguous candidate range; candidates land at
// precomputed offsets (no atomics), and are compacted into the next frontier.
//
// Lex ranks: inside one frontier the dense rank orders states exactly like
// their lex keys, so rank replaces lex in every within-frontier comparison.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kSmallGroup = 128;   // groups up to this size use the warp brute-force path
constexpr int kChunkSmall = 64;    // targets per warp work item
constexpr int kChunkBig = 1024;    // targets per CTA work item
constexpr int kBigThreads = 256;

struct Frontier {
  uint64_t* status;
  uint64_t* ids;
  int32_t* pid;
  double* value;
  uint64_t* lex;
  uint32_t* rank;
  int n;
  int32_t* g_start;
  int32_t* g_size;
  uint64_t* g_status;
  int n_groups;
};

struct StepArgs {
  DevSpace sp;
  HostTables t;
  int s;
  int charge;
  const double* recv;  // [M][S]
  const double* ub;    // [S+1]
  const double* incumbent;
  Frontier cur;
  // units (sorted by successor status)
  const int32_t* u_group;
  const int32_t* u_sig;
  const uint64_t* u_ns;
  const int32_t* u_nsid;
  const int32_t* ns_first;  // [n_ns+1]
  const int32_t* cand_off;  // [n_units+1]
  int n_units, n_ns;
  const int32_t* item_unit;
  const int32_t* item_chunk;
  int n_items;
  // candidates
  double* c_value;
  uint64_t* c_lex;
  int32_t* c_parent;
  int32_t* c_pid;
  int32_t* c_unit;
  int8_t* c_ok;
  int32_t* c_live;
  int T;
  int dense;  // big path: dense smem tables fit
};

// ---------------------------------------------------------------------------
// Units: (group, signature) -> successor status (solvers.hpp:379-411 with
// allowed_sizes :79-97 and StatusCodec::advance space.hpp:286-297).
template <bool kWrite>
__device__ int enumerate_units(const HostTables& t, const int32_t* sig_nopt, uint64_t status, int s, int32_t* out_sig,
                               uint64_t* out_ns) {
  const Codec codec{t.S};
  int st[KM], sizes[KM][9], cnt[KM];
  for (int m = 0; m < t.M; ++m) {
    st[m] = field16(status, m);
    cnt[m] = 0;
    if (Codec::is_running(st[m])) {
      sizes[m][cnt[m]++] = codec.run_size(st[m]);
    } else if (st[m] == Codec::done()) {
      sizes[m][cnt[m]++] = 0;
    } else {
      if (t.min_rt[m] >= 0 && s + 1 + t.min_rt[m] <= t.S) sizes[m][cnt[m]++] = 0;
      for (int k = 1; k <= 7; ++k)
        if (t.rt[m][k] >= 1 && s + t.rt[m][k] <= t.S) sizes[m][cnt[m]++] = k;
    }
    if (cnt[m] == 0) return 0;
  }
  int pick[KM] = {0, 0, 0, 0};
  int n = 0;
  while (true) {
    int sig = 0;
    uint64_t ns = 0;
    bool ok = true;
    for (int m = t.M - 1; m >= 0; --m) sig = sig * 8 + sizes[m][pick[m]];
    for (int m = 0; m < t.M && ok; ++m) {
      const int a = codec.advance(t.rt[m], st[m], sizes[m][pick[m]], s);
      ok = a >= 0 && !(a == 0 && (t.min_rt[m] < 0 || s + 1 + t.min_rt[m] > t.S));
      ns |= static_cast<uint64_t>(a < 0 ? 0 : a) << (16 * m);
    }
    if (ok && sig_nopt[sig] > 0) {
      if (kWrite) {
        out_sig[n] = sig;
        out_ns[n] = ns;
      }
      ++n;
    }
    int m = 0;  // odometer over the per-tenant choices
    while (m < t.M && ++pick[m] == cnt[m]) pick[m++] = 0;
    if (m == t.M) break;
  }
  return n;
}

__global__ void k_unit_count(HostTables t, const int32_t* sig_nopt, Frontier f, int s, int32_t* ucount) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < f.n_groups; g += gridDim.x * blockDim.x)
    ucount[g] = enumerate_units<false>(t, sig_nopt, f.g_status[g], s, nullptr, nullptr);
}

__global__ void k_unit_write(HostTables t, const int32_t* sig_nopt, Frontier f, int s, const int32_t* uoff,
                             int32_t* u_group, int32_t* u_sig, uint64_t* u_ns, int32_t* u_iota) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g < f.n_groups; g += gridDim.x * blockDim.x) {
    const int o = uoff[g];
    const int n = enumerate_units<true>(t, sig_nopt, f.g_status[g], s, u_sig + o, u_ns + o);
    for (int k = 0; k < n; ++k) {
      u_group[o + k] = g;
      u_iota[o + k] = o + k;
    }
  }
}

struct Counters {
  unsigned long long tr_ref;
  unsigned long long tr;
};

// Gathers the ns-sorted unit table and its per-unit sizes.
__global__ void k_unit_gather(const int32_t* perm, const uint64_t* ns_sorted, int n, const int32_t* g_in,
                              const int32_t* sig_in, const int32_t* g_size, DevSpace sp, int32_t* su_group,
                              int32_t* su_sig, int32_t* ns_flag, int32_t* L, int32_t* ch_small, int32_t* ch_big,
                              Counters* cnt) {
  unsigned long long ref = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int u = perm[i];
    const int g = g_in[u], sig = sig_in[u];
    su_group[i] = g;
    su_sig[i] = sig;
    ns_flag[i] = (i == 0 || ns_sorted[i] != ns_sorted[i - 1]) ? 1 : 0;
    const int len = sp.sig_off[sig + 1] - sp.sig_off[sig];
    L[i] = len;
    const bool small = g_size[g] <= kSmallGroup;
    ch_small[i] = small ? (len + kChunkSmall - 1) / kChunkSmall : 0;
    ch_big[i] = small ? 0 : (len + kChunkBig - 1) / kChunkBig;
    ref += static_cast<unsigned long long>(sp.sig_nopt[sig]);
  }
  for (int o = 16; o > 0; o >>= 1) ref += __shfl_down_sync(0xffffffffu, ref, o);
  if ((threadIdx.x & 31) == 0 && ref) atomicAdd(&cnt->tr_ref, ref);
}

__global__ void k_ns_index(const int32_t* ns_flag, const int32_t* ns_pos, int n, int32_t* u_nsid, int32_t* ns_first,
                           int n_ns) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int id = ns_pos[i + 1] - 1;
    u_nsid[i] = id;
    if (ns_flag[i]) ns_first[id] = i;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) ns_first[n_ns] = n;
}

__global__ void k_items(const int32_t* ch, const int32_t* item_off, int n, int32_t* item_unit, int32_t* item_chunk) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int o = item_off[i];
    for (int c = 0; c < ch[i]; ++c) {
      item_unit[o + c] = i;
      item_chunk[o + c] = c;
    }
  }
}

// ---------------------------------------------------------------------------
// One transition target: gains, subset-candidate predecessor, exact fold.
template <int M>
struct Best {
  double v[1 << M];
  uint32_t r[1 << M];
  int i[1 << M];
  __device__ void clear() {
#pragma unroll
    for (int k = 0; k < (1 << M); ++k) {
      i[k] = -1;
      v[k] = 0.0;
      r[k] = 0xffffffffu;
    }
  }
};

template <int M>
__device__ void finish_target(const StepArgs& a, int unit, int t_idx, int gstart, const double* acc, int p, int oi,
                              uint64_t ids_p, const Best<M>& b) {
  const HostTables& t = a.t;
  const int s = a.s;
  double cap[M], bonus[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {  // solvers.hpp:426-433
    cap[m] = a.sp.pl_cap[p * KM + m];
    const double recv = a.recv[m * t.S + s];
    const double c_changed = dmul(thr_of(recv, eff_cap(cap[m], a.charge ? t.loss[m] : 0.0)), acc[m]);
    bonus[m] = a.charge ? dsub(dmul(thr_of(recv, cap[m]), acc[m]), c_changed) : 0.0;
  }
  int chosen = -1;  // solvers.hpp:435-447
  double cv = 0.0;
  uint32_t cr = 0;
#pragma unroll
  for (int sub = 0; sub < (1 << M); ++sub) {
    if (b.i[sub] < 0) continue;
    double extra = 0.0;
#pragma unroll
    for (int m = 0; m < M; ++m)
      if ((sub >> m) & 1) extra = dadd(extra, bonus[m]);
    const double cand = dadd(b.v[sub], extra);
    if (chosen < 0 || better(cand, b.r[sub], cv, cr)) {
      chosen = b.i[sub];
      cv = cand;
      cr = b.r[sub];
    }
  }
  const int pred = gstart + chosen;
  const double pv = a.cur.value[pred];
  const uint64_t pids = a.cur.ids[pred];
  const uint32_t prank = a.cur.rank[pred];
  double v = pv;  // exact fold (solvers.hpp:451-458)
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const bool changed = a.charge && field16(pids, m) != field16(ids_p, m);
    const double eff = eff_cap(cap[m], changed ? t.loss[m] : 0.0);
    v = dadd(v, dmul(thr_of(a.recv[m * t.S + s], eff), acc[m]));
  }
  const bool ok = !(dadd(v, a.ub[s + 1]) < *a.incumbent);  // solvers.hpp:459 (strict)
  const int slot = a.cand_off[unit] + t_idx;
  a.c_value[slot] = v;
  a.c_lex[slot] = (static_cast<uint64_t>(prank) << 32) | static_cast<uint32_t>(oi);
  a.c_parent[slot] = pred;
  a.c_pid[slot] = p;
  a.c_unit[slot] = unit;
  a.c_ok[slot] = ok ? 1 : 0;
}

template <int M>
__device__ void group_acc(const StepArgs& a, uint64_t gstat, double* acc) {
#pragma unroll
  for (int m = 0; m < M; ++m) acc[m] = field16(gstat, m) == Codec::done() ? a.t.post[m] : a.t.pre[m];
}

// Small groups: one warp per (unit, chunk); every lane owns a target and scans
// the group's states (broadcast loads) keeping the best state per subset.
template <int M>
__global__ void __launch_bounds__(128) k_trans_small(StepArgs a) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= a.n_items) return;
  const int unit = a.item_unit[w], chunk = a.item_chunk[w];
  const int g = a.u_group[unit], sig = a.u_sig[unit];
  const int gs = a.cur.g_start[g], gn = a.cur.g_size[g];
  double acc[M];
  group_acc<M>(a, a.cur.g_status[g], acc);
  const int sb = a.sp.sig_off[sig], L = a.sp.sig_off[sig + 1] - sb;
  const int t1 = min(L, (chunk + 1) * kChunkSmall);
  for (int ti = chunk * kChunkSmall + lane; ti < t1; ti += 32) {
    const int p = a.sp.cand_pid[sb + ti];
    const int oi = a.sp.cand_oi[sb + ti];
    const uint64_t ids_p = a.sp.pl_ids[p];
    Best<M> b;
    b.clear();
    for (int j = 0; j < gn; ++j) {
      const double vj = a.cur.value[gs + j];
      const uint32_t rj = a.cur.rank[gs + j];
      const uint64_t idj = a.cur.ids[gs + j];
      int mt = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) mt |= (field16(idj, m) == field16(ids_p, m)) << m;
#pragma unroll
      for (int sub = 0; sub < (1 << M); ++sub) {
        if ((sub & ~mt) != 0) continue;
        if (b.i[sub] < 0 || better(vj, rj, b.v[sub], b.r[sub])) {
          b.v[sub] = vj;
          b.r[sub] = rj;
          b.i[sub] = j;
        }
      }
    }
    finish_target<M>(a, unit, ti, gs, acc, p, oi, ids_p, b);
  }
}

struct Ent {
  unsigned long long vb;
  unsigned int rank;
  int idx;
};

// Big groups: one CTA per (unit, chunk). The group's best representative per
// (subset, projected placement) is built in shared memory with a two-phase
// max-value / min-rank atomic reduction, then every thread resolves targets.
template <int M>
__global__ void __launch_bounds__(kBigThreads) k_trans_big(StepArgs a) {
  extern __shared__ Ent tab[];
  const int item = blockIdx.x;
  if (item >= a.n_items) return;
  const int unit = a.item_unit[item], chunk = a.item_chunk[item];
  const int g = a.u_group[unit], sig = a.u_sig[unit];
  const int gs = a.cur.g_start[g], gn = a.cur.g_size[g];
  const int P1 = a.sp.P1;
  double acc[M];
  group_acc<M>(a, a.cur.g_status[g], acc);
  const int sb = a.sp.sig_off[sig], L = a.sp.sig_off[sig + 1] - sb;
  const int t0 = chunk * kChunkBig, t1 = min(L, t0 + kChunkBig);
  if (a.dense) {
    for (int e = threadIdx.x; e < a.sp.proj_total; e += blockDim.x) tab[e] = Ent{0ull, 0xffffffffu, -1};
    __syncthreads();
    for (int j = threadIdx.x; j < gn; j += blockDim.x) {
      const int pj = a.cur.pid[gs + j];
      const unsigned long long vb = vbits(a.cur.value[gs + j]);
#pragma unroll
      for (int sub = 0; sub < (1 << M); ++sub) atomicMax(&tab[a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + pj]].vb, vb);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < gn; j += blockDim.x) {
      const int pj = a.cur.pid[gs + j];
      const unsigned long long vb = vbits(a.cur.value[gs + j]);
      const unsigned rj = a.cur.rank[gs + j];
#pragma unroll
      for (int sub = 0; sub < (1 << M); ++sub) {
        Ent* e = &tab[a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + pj]];
        if (e->vb == vb) atomicMin(&e->rank, rj);
      }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < gn; j += blockDim.x) {
      const int pj = a.cur.pid[gs + j];
      const unsigned long long vb = vbits(a.cur.value[gs + j]);
      const unsigned rj = a.cur.rank[gs + j];
#pragma unroll
      for (int sub = 0; sub < (1 << M); ++sub) {
        Ent* e = &tab[a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + pj]];
        if (e->vb == vb && e->rank == rj) e->idx = j;
      }
    }
    __syncthreads();
    for (int ti = t0 + threadIdx.x; ti < t1; ti += blockDim.x) {
      const int p = a.sp.cand_pid[sb + ti];
      const int oi = a.sp.cand_oi[sb + ti];
      Best<M> b;
#pragma unroll
      for (int sub = 0; sub < (1 << M); ++sub) {
        const Ent e = tab[a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + p]];
        b.i[sub] = e.idx;
        b.v[sub] = __longlong_as_double(static_cast<long long>(e.vb));
        b.r[sub] = e.rank;
      }
      finish_target<M>(a, unit, ti, gs, acc, p, oi, a.sp.pl_ids[p], b);
    }
  } else {  // tables too large for shared memory: per-thread scan
    for (int ti = t0 + threadIdx.x; ti < t1; ti += blockDim.x) {
      const int p = a.sp.cand_pid[sb + ti];
      const int oi = a.sp.cand_oi[sb + ti];
      const uint64_t ids_p = a.sp.pl_ids[p];
      Best<M> b;
      b.clear();
      for (int j = 0; j < gn; ++j) {
        const double vj = a.cur.value[gs + j];
        const uint32_t rj = a.cur.rank[gs + j];
        const uint64_t idj = a.cur.ids[gs + j];
        int mt = 0;
#pragma unroll
        for (int m = 0; m < M; ++m) mt |= (field16(idj, m) == field16(ids_p, m)) << m;
#pragma unroll
        for (int sub = 0; sub < (1 << M); ++sub) {
          if ((sub & ~mt) != 0) continue;
          if (b.i[sub] < 0 || better(vj, rj, b.v[sub], b.r[sub])) {
            b.v[sub] = vj;
            b.r[sub] = rj;
            b.i[sub] = j;
          }
        }
      }
      finish_target<M>(a, unit, ti, gs, acc, p, oi, ids_p, b);
    }
  }
}

// ---------------------------------------------------------------------------
// Equal-key merge across the units of one successor status (solvers.hpp:467-468):
// a candidate survives unless another unit of the same status produced the same
// placement with a better (value, lex). Candidate lists of a unit are sorted by
// placement, so the lookup is a binary search.
__global__ void k_merge(StepArgs a) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x) {
    if (!a.c_ok[k]) {
      a.c_live[k] = 0;
      continue;
    }
    const int unit = a.c_unit[k];
    const int ns = a.u_nsid[unit];
    const int u0 = a.ns_first[ns], u1 = a.ns_first[ns + 1];
    int live = 1;
    if (u1 - u0 > 1) {
      const int p = a.c_pid[k];
      const double v = a.c_value[k];
      const uint64_t lx = a.c_lex[k];
      for (int u = u0; u < u1 && live; ++u) {
        if (u == unit) continue;
        const int sig = a.u_sig[u];
        const int b = a.sp.sig_off[sig], n = a.sp.sig_off[sig + 1] - b;
        int lo = 0, hi = n;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (a.sp.cand_pid[b + mid] < p) lo = mid + 1;
          else hi = mid;
        }
        if (lo < n && a.sp.cand_pid[b + lo] == p) {
          const int k2 = a.cand_off[u] + lo;
          if (a.c_ok[k2] && better(a.c_value[k2], a.c_lex[k2], v, lx)) live = 0;
        }
      }
    }
    a.c_live[k] = live;
  }
}

// Placement band per status (solvers.hpp:499-511).
__global__ void k_band_max(StepArgs a, unsigned long long* ns_best) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x)
    if (a.c_live[k]) atomicMax(&ns_best[a.u_nsid[a.c_unit[k]]], vbits(a.c_value[k]));
}

__global__ void k_band_mark(StepArgs a, const unsigned long long* ns_best, double band) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x) {
    if (!a.c_live[k]) continue;
    const double best = __longlong_as_double(static_cast<long long>(ns_best[a.u_nsid[a.c_unit[k]]]));
    if (!(a.c_value[k] >= dsub(best, band))) a.c_live[k] = 0;
  }
}

// Status dominance within equal placements (solvers.hpp:514-537): buckets of
// 2..64 live states sharing a placement; a state dies iff some other state of
// its bucket dominates it status-wise and is dp_better. (The reference's
// sequential sweep yields exactly the non-dominated set: the kill relation is
// transitive.)
__global__ void k_dom_count(StepArgs a, int32_t* pcount) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x)
    if (a.c_live[k]) atomicAdd(&pcount[a.c_pid[k]], 1);
}

__global__ void k_dom_scatter(StepArgs a, const int32_t* pcount, const int32_t* poff, int32_t* pcursor,
                              int32_t* bucket) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x) {
    if (!a.c_live[k]) continue;
    const int p = a.c_pid[k];
    const int n = pcount[p];
    if (n < 2 || n > 64) continue;
    bucket[poff[p] + atomicAdd(&pcursor[p], 1)] = k;
  }
}

__global__ void k_dom_check(StepArgs a, const int32_t* pcount, const int32_t* poff, const int32_t* bucket, int P1) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= P1) return;
  const int n = pcount[w];
  if (n < 2 || n > 64) return;
  const Codec codec{a.t.S};
  const int* bk = bucket + poff[w];
  int kk[2];
  uint64_t st[2];
  double v[2];
  uint64_t lx[2];
  for (int h = 0; h < 2; ++h) {
    const int j = lane + 32 * h;
    kk[h] = j < n ? bk[j] : -1;
    st[h] = kk[h] >= 0 ? a.u_ns[a.c_unit[kk[h]]] : 0;
    v[h] = kk[h] >= 0 ? a.c_value[kk[h]] : 0.0;
    lx[h] = kk[h] >= 0 ? a.c_lex[kk[h]] : 0;
  }
  bool dead[2] = {false, false};
  for (int j = 0; j < n; ++j) {
    const int h = j >> 5, src = j & 31;
    const uint64_t sa = __shfl_sync(0xffffffffu, st[h], src);
    const double va = __shfl_sync(0xffffffffu, v[h], src);
    const uint64_t la = __shfl_sync(0xffffffffu, lx[h], src);
    for (int hb = 0; hb < 2; ++hb) {
      if (kk[hb] < 0 || lane + 32 * hb == j) continue;
      bool dom = true;
      for (int m = 0; m < a.t.M && dom; ++m) dom = status_dominates(codec, field16(sa, m), field16(st[hb], m));
      if (dom && better(va, la, v[hb], lx[hb])) dead[hb] = true;
    }
  }
  for (int h = 0; h < 2; ++h)
    if (kk[h] >= 0 && dead[h]) a.c_live[kk[h]] = 0;
}

// Compaction into the next frontier + history.
__global__ void k_compact(StepArgs a, const int32_t* pos, Frontier nx, int32_t* h_parent, int32_t* h_option) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < a.T; k += gridDim.x * blockDim.x) {
    if (!a.c_live[k]) continue;
    const int q = pos[k];
    const int p = a.c_pid[k];
    nx.status[q] = a.u_ns[a.c_unit[k]];
    nx.ids[q] = a.sp.pl_ids[p];
    nx.pid[q] = p;
    nx.value[q] = a.c_value[k];
    nx.lex[q] = a.c_lex[k];
    h_parent[q] = a.c_parent[k];
    h_option[q] = static_cast<int32_t>(a.c_lex[k] & 0xffffffffu);
  }
}

__global__ void k_groups(StepArgs a, const int32_t* pos, int32_t* gflag, int32_t* gs_tmp, int32_t* gn_tmp) {
  for (int ns = blockIdx.x * blockDim.x + threadIdx.x; ns < a.n_ns; ns += gridDim.x * blockDim.x) {
    const int i0 = a.ns_first[ns], i1 = a.ns_first[ns + 1];
    const int b = pos[a.cand_off[i0]], e = pos[a.cand_off[i1]];
    gs_tmp[ns] = b;
    gn_tmp[ns] = e - b;
    gflag[ns] = e > b ? 1 : 0;
  }
}

__global__ void k_groups_compact(StepArgs a, const int32_t* gflag, const int32_t* gpos, const int32_t* gs_tmp,
                                 const int32_t* gn_tmp, Frontier nx) {
  for (int ns = blockIdx.x * blockDim.x + threadIdx.x; ns < a.n_ns; ns += gridDim.x * blockDim.x) {
    if (!gflag[ns]) continue;
    const int q = gpos[ns];
    nx.g_start[q] = gs_tmp[ns];
    nx.g_size[q] = gn_tmp[ns];
    nx.g_status[q] = a.u_ns[a.ns_first[ns]];
  }
}

__global__ void k_iota(int32_t* x, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = i;
}

__global__ void k_rank(const int32_t* perm, int n, uint32_t* rank) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) rank[perm[r]] = r;
}

// Terminal: best all-done state (solvers.hpp:552-565), then the parent walk.
__global__ void k_terminal(Frontier f, uint64_t all_done, int* best_idx) {
  __shared__ double sv[32];
  __shared__ unsigned long long sl[32];
  __shared__ int si[32];
  double bv = 0.0;
  unsigned long long bl = ~0ull;
  int bi = -1;
  for (int g = 0; g < f.n_groups; ++g) {
    if (f.g_status[g] != all_done) continue;
    for (int j = threadIdx.x; j < f.g_size[g]; j += blockDim.x) {
      const int k = f.g_start[g] + j;
      if (bi < 0 || better(f.value[k], f.lex[k], bv, bl)) {
        bv = f.value[k];
        bl = f.lex[k];
        bi = k;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_down_sync(0xffffffffu, bv, o);
    const unsigned long long ol = __shfl_down_sync(0xffffffffu, bl, o);
    const int oi = __shfl_down_sync(0xffffffffu, bi, o);
    if (oi >= 0 && (bi < 0 || better(ov, ol, bv, bl))) {
      bv = ov;
      bl = ol;
      bi = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    sl[threadIdx.x >> 5] = bl;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (si[w] >= 0 && (bi < 0 || better(sv[w], sl[w], bv, bl))) {
        bv = sv[w];
        bl = sl[w];
        bi = si[w];
      }
    *best_idx = bi;
  }
}

__global__ void k_backtrack(int32_t* const* h_parent, int32_t* const* h_option, int S, const int* best_idx,
                            int32_t* chosen) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int idx = *best_idx;
  for (int s = S - 1; s >= 0; --s) {
    chosen[s] = idx >= 0 ? h_option[s][idx] : -1;
    idx = idx >= 0 ? h_parent[s][idx] : -1;
  }
}

inline unsigned grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<unsigned>(g);
}

struct FrontierBufs {
  const char* tag;
  Frontier alloc(Ctx& c, int n, int ng) {
    std::string t(tag);
    Frontier f{};
    f.status = c.buf<uint64_t>((t + "_status").c_str(), n);
    f.ids = c.buf<uint64_t>((t + "_ids").c_str(), n);
    f.pid = c.buf<int32_t>((t + "_pid").c_str(), n);
    f.value = c.buf<double>((t + "_value").c_str(), n);
    f.lex = c.buf<uint64_t>((t + "_lex").c_str(), n);
    f.rank = c.buf<uint32_t>((t + "_rank").c_str(), n);
    f.g_start = c.buf<int32_t>((t + "_gstart").c_str(), ng);
    f.g_size = c.buf<int32_t>((t + "_gsize").c_str(), ng);
    f.g_status = c.buf<uint64_t>((t + "_gstatus").c_str(), ng);
    f.n = n;
    f.n_groups = ng;
    return f;
  }
};

}  // namespace

void solve_dp(Ctx& c, const mgs_problem& p, const Prepared& pr, const DevSpace& sp, const double* d_recv,
              const double* d_ub, const double* d_incumbent, SolveOut& out) {
  const HostTables& t = pr.t;
  const int M = t.M, S = t.S;
  const Codec codec{S};
  // band and dominance switch (solvers.hpp:258-267)
  double acc_max[KM] = {0, 0, 0, 0};
  bool dominance_ok = true;
  for (int m = 0; m < M; ++m) {
    acc_max[m] = std::max(t.pre[m], t.post[m]);
    dominance_ok = dominance_ok && t.post[m] >= t.pre[m];
  }
  std::vector<double> cap_max(M, 0.0);
  {
    std::vector<double> pc(static_cast<size_t>(sp.P) * KM);
    MGS_CUDA_OK(cudaMemcpyAsync(pc.data(), sp.pl_cap, pc.size() * 8, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    for (int q = 0; q < sp.P; ++q)
      for (int m = 0; m < M; ++m) cap_max[m] = std::max(cap_max[m], pc[q * KM + m]);
  }
  double band = 1e-9;
  for (int m = 0; m < M; ++m) band += t.loss[m] * cap_max[m] * acc_max[m];

  History& hist = c.history;
  hist.reset();
  FrontierBufs fa{"fa"}, fb{"fb"};
  Frontier cur = fa.alloc(c, 1, 1);
  {
    // root: all not started, carried-over placement, value 0, lex 0, rank 0
    uint64_t zero64 = 0, root_ids = 0;
    MGS_CUDA_OK(cudaMemcpyAsync(&root_ids, sp.pl_ids + sp.root_pid, 8, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    double zd = 0.0;
    uint32_t zr = 0;
    int32_t zi = 0, one = 1, rp = sp.root_pid;
    MGS_CUDA_OK(cudaMemcpyAsync(cur.status, &zero64, 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.ids, &root_ids, 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.pid, &rp, 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.value, &zd, 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.lex, &zero64, 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.rank, &zr, 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.g_start, &zi, 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.g_size, &one, 4, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(cur.g_status, &zero64, 8, cudaMemcpyHostToDevice, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  }
  bool cur_is_a = true;

  Counters* d_cnt = c.buf<Counters>("dp_counters", 1);
  MGS_CUDA_OK(cudaMemsetAsync(d_cnt, 0, sizeof(Counters), c.stream));
  const size_t dense_bytes = static_cast<size_t>(sp.proj_total) * sizeof(Ent);
  const bool dense = dense_bytes <= 200 * 1024;
  auto set_smem = [&](auto kern) {
    if (dense) MGS_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dense_bytes));
  };
  switch (M) {
    case 1: set_smem(k_trans_big<1>); break;
    case 2: set_smem(k_trans_big<2>); break;
    case 3: set_smem(k_trans_big<3>); break;
    default: set_smem(k_trans_big<4>); break;
  }
  uint64_t ftot = 0, fpeak = 0, tr = 0, tbytes = 0;
  int32_t* hcnt = c.pinned.get<int32_t>(8);

  for (int s = 0; s < S; ++s) {
    if (cur.n == 0) throw PlanFail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};
    // 1. units
    c.phase(2);
    const int G = cur.n_groups;
    int32_t* ucount = c.buf<int32_t>("ucount", G);
    int32_t* uoff = c.buf<int32_t>("uoff", G + 1);
    k_unit_count<<<grid_for(G), 256, 0, c.stream>>>(t, sp.sig_nopt, cur, s, ucount);
    ++c.kernel_launches;
    exclusive_scan_i32(c, ucount, uoff, G);
    const int NU = read_scalar(c, uoff + G);
    if (NU == 0) throw PlanFail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};
    int32_t* u_group = c.buf<int32_t>("u_group", NU);
    int32_t* u_sig = c.buf<int32_t>("u_sig", NU);
    uint64_t* u_ns = c.buf<uint64_t>("u_ns", NU);
    int32_t* u_iota = c.buf<int32_t>("u_iota", NU);
    k_unit_write<<<grid_for(G), 256, 0, c.stream>>>(t, sp.sig_nopt, cur, s, uoff, u_group, u_sig, u_ns, u_iota);
    ++c.kernel_launches;
    uint64_t* su_ns = c.buf<uint64_t>("su_ns", NU);
    int32_t* perm = c.buf<int32_t>("u_perm", NU);
    {
      size_t tb = 0;
      const int end_bit = 16 * M;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, u_ns, su_ns, u_iota, perm, NU, 0, end_bit, c.stream);
      void* tmp = c.buf<char>("cub_tmp", tb);
      MGS_CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, tb, u_ns, su_ns, u_iota, perm, NU, 0, end_bit, c.stream));
    }
    int32_t* su_group = c.buf<int32_t>("su_group", NU);
    int32_t* su_sig = c.buf<int32_t>("su_sig", NU);
    int32_t* ns_flag = c.buf<int32_t>("ns_flag", NU);
    int32_t* L = c.buf<int32_t>("u_L", NU);
    int32_t* chs = c.buf<int32_t>("u_chs", NU);
    int32_t* chb = c.buf<int32_t>("u_chb", NU);
    k_unit_gather<<<grid_for(NU), 256, 0, c.stream>>>(perm, su_ns, NU, u_group, u_sig, cur.g_size, sp, su_group,
                                                      su_sig, ns_flag, L, chs, chb, d_cnt);
    int32_t* ns_pos = c.buf<int32_t>("ns_pos", NU + 1);
    int32_t* cand_off = c.buf<int32_t>("cand_off", NU + 1);
    int32_t* ios = c.buf<int32_t>("item_off_s", NU + 1);
    int32_t* iob = c.buf<int32_t>("item_off_b", NU + 1);
    exclusive_scan_i32(c, ns_flag, ns_pos, NU);
    exclusive_scan_i32(c, L, cand_off, NU);
    exclusive_scan_i32(c, chs, ios, NU);
    exclusive_scan_i32(c, chb, iob, NU);
    int32_t* d_tot = c.buf<int32_t>("step_totals", 4);
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 0, ns_pos + NU, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 1, cand_off + NU, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 2, ios + NU, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 3, iob + NU, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(hcnt, d_tot, 16, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    const int n_ns = hcnt[0], T = hcnt[1], nis = hcnt[2], nib = hcnt[3];
    tr += static_cast<uint64_t>(T);

    int32_t* u_nsid = c.buf<int32_t>("u_nsid", NU);
    int32_t* ns_first = c.buf<int32_t>("ns_first", n_ns + 1);
    k_ns_index<<<grid_for(NU), 256, 0, c.stream>>>(ns_flag, ns_pos, NU, u_nsid, ns_first, n_ns);
    ++c.kernel_launches;
    int32_t* its_u = c.buf<int32_t>("item_s_unit", nis);
    int32_t* its_c = c.buf<int32_t>("item_s_chunk", nis);
    int32_t* itb_u = c.buf<int32_t>("item_b_unit", nib);
    int32_t* itb_c = c.buf<int32_t>("item_b_chunk", nib);
    k_items<<<grid_for(NU), 256, 0, c.stream>>>(chs, ios, NU, its_u, its_c);
    ++c.kernel_launches;
    k_items<<<grid_for(NU), 256, 0, c.stream>>>(chb, iob, NU, itb_u, itb_c);
    ++c.kernel_launches;

    StepArgs a{};
    a.sp = sp;
    a.t = t;
    a.s = s;
    a.charge = (s > 0 || pr.has_initial) ? 1 : 0;
    a.recv = d_recv;
    a.ub = d_ub;
    a.incumbent = d_incumbent;
    a.cur = cur;
    a.u_group = su_group;
    a.u_sig = su_sig;
    a.u_ns = su_ns;
    a.u_nsid = u_nsid;
    a.ns_first = ns_first;
    a.cand_off = cand_off;
    a.n_units = NU;
    a.n_ns = n_ns;
    a.T = T;
    a.dense = dense ? 1 : 0;
    a.c_value = c.buf<double>("c_value", T);
    a.c_lex = c.buf<uint64_t>("c_lex", T);
    a.c_parent = c.buf<int32_t>("c_parent", T);
    a.c_pid = c.buf<int32_t>("c_pid", T);
    a.c_unit = c.buf<int32_t>("c_unit", T);
    a.c_ok = c.buf<int8_t>("c_ok", T);
    a.c_live = c.buf<int32_t>("c_live", T);

    // 2. transitions
    c.phase(3);
    tbytes += static_cast<uint64_t>(cur.n) * 20 + static_cast<uint64_t>(T) * (8 + 29);
    if (nis > 0) {
      StepArgs as = a;
      as.item_unit = its_u;
      as.item_chunk = its_c;
      as.n_items = nis;
      const unsigned grid = ceil_div(nis, 4);
      switch (M) {
        case 1: k_trans_small<1><<<grid, 128, 0, c.stream>>>(as); break;
        case 2: k_trans_small<2><<<grid, 128, 0, c.stream>>>(as); break;
        case 3: k_trans_small<3><<<grid, 128, 0, c.stream>>>(as); break;
        default: k_trans_small<4><<<grid, 128, 0, c.stream>>>(as); break;
      }
      ++c.kernel_launches;
    }
    if (nib > 0) {
      StepArgs ab = a;
      ab.item_unit = itb_u;
      ab.item_chunk = itb_c;
      ab.n_items = nib;
      const size_t smem = dense ? dense_bytes : 0;
      switch (M) {
        case 1: k_trans_big<1><<<nib, kBigThreads, smem, c.stream>>>(ab); break;
        case 2: k_trans_big<2><<<nib, kBigThreads, smem, c.stream>>>(ab); break;
        case 3: k_trans_big<3><<<nib, kBigThreads, smem, c.stream>>>(ab); break;
        default: k_trans_big<4><<<nib, kBigThreads, smem, c.stream>>>(ab); break;
      }
      ++c.kernel_launches;
    }
    // 3. merge, band, dominance
    c.phase(4);
    k_merge<<<grid_for(T), 256, 0, c.stream>>>(a);
    ++c.kernel_launches;
    unsigned long long* ns_best = c.buf<unsigned long long>("ns_best", n_ns);
    MGS_CUDA_OK(cudaMemsetAsync(ns_best, 0, static_cast<size_t>(n_ns) * 8, c.stream));
    k_band_max<<<grid_for(T), 256, 0, c.stream>>>(a, ns_best);
    ++c.kernel_launches;
    k_band_mark<<<grid_for(T), 256, 0, c.stream>>>(a, ns_best, band);
    ++c.kernel_launches;
    if (dominance_ok) {
      const int P1 = sp.P1;
      int32_t* pcount = c.buf<int32_t>("dom_count", P1);
      int32_t* poff = c.buf<int32_t>("dom_off", P1 + 1);
      int32_t* pcursor = c.buf<int32_t>("dom_cursor", P1);
      int32_t* bucket = c.buf<int32_t>("dom_bucket", T);
      MGS_CUDA_OK(cudaMemsetAsync(pcount, 0, P1 * 4, c.stream));
      MGS_CUDA_OK(cudaMemsetAsync(pcursor, 0, P1 * 4, c.stream));
      k_dom_count<<<grid_for(T), 256, 0, c.stream>>>(a, pcount);
      ++c.kernel_launches;
      exclusive_scan_i32(c, pcount, poff, P1);
      k_dom_scatter<<<grid_for(T), 256, 0, c.stream>>>(a, pcount, poff, pcursor, bucket);
      ++c.kernel_launches;
      k_dom_check<<<ceil_div(P1, 4), 128, 0, c.stream>>>(a, pcount, poff, bucket, P1);
      ++c.kernel_launches;
    }
    // 4. compaction + groups
    c.phase(5);
    int32_t* pos = c.buf<int32_t>("live_pos", T + 1);
    exclusive_scan_i32(c, a.c_live, pos, T);
    int32_t* gflag = c.buf<int32_t>("gflag", n_ns);
    int32_t* gpos = c.buf<int32_t>("gpos", n_ns + 1);
    int32_t* gs_tmp = c.buf<int32_t>("gs_tmp", n_ns);
    int32_t* gn_tmp = c.buf<int32_t>("gn_tmp", n_ns);
    k_groups<<<grid_for(n_ns), 256, 0, c.stream>>>(a, pos, gflag, gs_tmp, gn_tmp);
    ++c.kernel_launches;
    exclusive_scan_i32(c, gflag, gpos, n_ns);
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 0, pos + T, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(d_tot + 1, gpos + n_ns, 4, cudaMemcpyDeviceToDevice, c.stream));
    MGS_CUDA_OK(cudaMemcpyAsync(hcnt, d_tot, 8, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    const int n_next = hcnt[0], g_next = hcnt[1];
    if (static_cast<uint64_t>(n_next) > p.state_budget)  // solvers.hpp:539-542
      throw PlanFail{MGS_ERR_STATE_BUDGET,
                     "dynamic-program frontier reached " + std::to_string(n_next) + " states at step " +
                         std::to_string(s + 1) + " (budget " + std::to_string(p.state_budget) + ")",
                     s + 1, static_cast<uint64_t>(n_next)};
    Frontier nx = (cur_is_a ? fb : fa).alloc(c, std::max(n_next, 1), std::max(g_next, 1));
    nx.n = n_next;
    nx.n_groups = g_next;
    int32_t *hp, *ho;
    hist.take(std::max(n_next, 1), &hp, &ho);
    k_compact<<<grid_for(T), 256, 0, c.stream>>>(a, pos, nx, hp, ho);
    ++c.kernel_launches;
    k_groups_compact<<<grid_for(n_ns), 256, 0, c.stream>>>(a, gflag, gpos, gs_tmp, gn_tmp, nx);
    ++c.kernel_launches;
    // 5. dense lex ranks (solvers.hpp:544-548)
    c.phase(6);
    if (n_next > 0) {
      uint64_t* lex_sorted = c.buf<uint64_t>("lex_sorted", n_next);
      int32_t* iota = c.buf<int32_t>("rank_iota", n_next);
      int32_t* rperm = c.buf<int32_t>("rank_perm", n_next);
      k_iota<<<grid_for(n_next), 256, 0, c.stream>>>(iota, n_next);
      ++c.kernel_launches;
      int hb = 1;
      while ((1ll << hb) <= cur.n) ++hb;
      const int end_bit = std::min(64, 32 + hb);
      size_t tb = 0;
      cub::DeviceRadixSort::SortPairs(nullptr, tb, nx.lex, lex_sorted, iota, rperm, n_next, 0, end_bit, c.stream);
      void* tmp = c.buf<char>("cub_tmp", tb);
      MGS_CUDA_OK(
          cub::DeviceRadixSort::SortPairs(tmp, tb, nx.lex, lex_sorted, iota, rperm, n_next, 0, end_bit, c.stream));
      k_rank<<<grid_for(n_next), 256, 0, c.stream>>>(rperm, n_next, nx.rank);
      ++c.kernel_launches;
    }
    MGS_CUDA_OK(cudaGetLastError());
    if (std::getenv("MGS_DEBUG_STEPS"))
      std::fprintf(stderr, "v1 step %d units %d ns %d T %d store %d groups %d alive_in %d\n", s, NU, n_ns, T, n_next,
                   g_next, cur.n);
    ftot += n_next;
    fpeak = std::max<uint64_t>(fpeak, n_next);
    cur = nx;
    cur_is_a = !cur_is_a;
  }
  // terminal + backtrack
  c.phase(7);
  uint64_t all_done = 0;
  for (int m = 0; m < M; ++m) all_done |= static_cast<uint64_t>(Codec::done()) << (16 * m);
  int* d_best = c.buf<int>("best_idx", 1);
  k_terminal<<<1, 1024, 0, c.stream>>>(cur, all_done, d_best);
  ++c.kernel_launches;
  int32_t** d_hp = c.buf<int32_t*>("hist_parent_ptrs", S);
  int32_t** d_ho = c.buf<int32_t*>("hist_option_ptrs", S);
  MGS_CUDA_OK(cudaMemcpyAsync(d_hp, hist.parent.data(), S * sizeof(void*), cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_ho, hist.option.data(), S * sizeof(void*), cudaMemcpyHostToDevice, c.stream));
  int32_t* d_chosen = c.buf<int32_t>("chosen", S);
  k_backtrack<<<1, 32, 0, c.stream>>>(d_hp, d_ho, S, d_best, d_chosen);
  ++c.kernel_launches;
  out.options.resize(S);
  MGS_CUDA_OK(cudaMemcpyAsync(out.options.data(), d_chosen, S * 4, cudaMemcpyDeviceToHost, c.stream));
  int best_host = -1;
  MGS_CUDA_OK(cudaMemcpyAsync(&best_host, d_best, 4, cudaMemcpyDeviceToHost, c.stream));
  Counters hc{};
  MGS_CUDA_OK(cudaMemcpyAsync(&hc, d_cnt, sizeof hc, cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  if (best_host < 0) throw PlanFail{MGS_ERR_INFEASIBLE_JOINT, "no feasible allocation sequence exists for this window"};
  out.stats.options = sp.n_opt;
  out.stats.candidates = sp.n_cand;
  out.stats.transitions_ref = hc.tr_ref;
  out.stats.transitions = tr;
  out.stats.frontier_total = ftot;
  out.stats.frontier_peak = fpeak;
  out.stats.transition_bytes = tbytes;
  (void)codec;
}

}  // namespace mgs
