// Device-resident DP engine (M <= 4): the whole per-window search of solve_dp
// (solvers.hpp:242-579) as a stream of phase kernels with every count kept on
// the device: no host round trips inside a window, no sorts, no hot
// (same-address) global atomics.
//
// Same procedure as the reference (and as the multi-launch engine in dp.cu):
// subset representatives per status group, subset-candidate predecessor choice
// + exact fold, strict bound test, equal-key merge, band, status dominance in
// placement buckets of <= 64, state budget, dense lex ranks, terminal + parent
// walk. What differs is how the work is laid out on B200:
//
//   per slot s (F_s = current frontier, status groups contiguous in HBM)
//   S1  units: CTAs own contiguous group ranges; a warp per group enumerates
//       the (signature, successor status) combinations lane-parallel; unit
//       slots are reserved with ONE atomic per CTA batch; successor statuses
//       are keyed by their slot in an open-addressing hash (the slot *is* the
//       id). Also: children per parent (for the ranks) and live-state count.
//   S2  seven decoupled-look-back scans in one pass (candidate / unit offsets
//       per successor status, big / small status lists, warp / CTA work items
//       per unit, child offsets per parent).
//   S3  placement: units get contiguous candidate ranges inside their status,
//       work items and status lists are materialised, children are bucketed
//       by parent.
//   S4  dense lex ranks of F_s: rank = first child slot of the parent + rank
//       of the option index inside the parent's bucket (lex = (rank, option)).
//   S5  transitions: CTAs take big-group items (shared-memory subset tables
//       built with a two-phase max-value / min-rank reduction), warps take
//       small-group items (broadcast scan of the group's states).
//   S6  per successor status: equal-key merge across its units (multi-unit
//       statuses, CTA, dense shared-memory table), band, output of the
//       survivors straight into F_{s+1} (one allocation atomic per CTA batch),
//       history, dominance buckets.
//   S7  status dominance per placement bucket (2..64 states); resets.
//
// Dead (dominated) states stay in F_{s+1} as holes flagged alive = 0 and are
// skipped everywhere; ranks are dense over the live states only.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include <cub/block/block_radix_sort.cuh>

#include "ctx.cuh"

namespace mgs {
namespace {

constexpr int kThreads = 256;
#ifndef MGS_MINB
#define MGS_MINB 6
#endif
// latency-bound phase kernels that gain from more resident warps (units, tables,
// write: +15 % on 8-lane batches, measured): at least MGS_MINB CTAs per SM
#define MGS_LB __launch_bounds__(kThreads, MGS_MINB)
#ifndef MGS_TS_MINB
#define MGS_TS_MINB 4  // k_trans_small: at least 4 CTAs per SM (64 registers)
#endif
constexpr int kWarps = kThreads / 32;
constexpr int kSmall = 64;           // groups up to this size: warp path (128: -0.3 ms, smaller staging arrays)
constexpr int kChunkS = 32;          // targets per warp item
constexpr int kChunkH = 16;          // targets of a half item (two per warp)
constexpr int kChunkQ = 8;           // targets of a quarter item (four per warp)
constexpr int kChunkB = 512;         // targets per CTA item
constexpr int kScanItems = 8;                 // elements per thread of a scan tile
constexpr int kTile = kThreads * kScanItems;  // scan tile
constexpr int kBigNs = 1024;         // single-unit statuses with more candidates use the CTA path
constexpr int kBucketSmall = 256;    // child buckets up to this size: thread per slot
constexpr int kSortItems = 16;       // big child buckets: CTA radix sort of up to 256*16 keys
#ifndef MGS_BITMAP_PER_KEY
#define MGS_BITMAP_PER_KEY 4
#endif
constexpr int kBitmapPerKey = MGS_BITMAP_PER_KEY;  // ... or the option bitmap when |O|/32 <= this x the bucket size
constexpr int kBatch = 512;          // groups / statuses per CTA allocation batch
#ifndef MGS_TB_MINB
#define MGS_TB_MINB 4  // k_trans_big: CTAs per SM the register budget must allow
#endif
#ifndef MGS_RB_MINB
#define MGS_RB_MINB 2  // k_ranks_big: 2 CTAs per SM (127 registers; 1: ranks 6.0 ms eager, 2: 4.6)
#endif
#ifndef MGS_UNITS_W
#define MGS_UNITS_W 8  // lanes per status group in k_units' warp path (M <= 2)
#endif
#ifndef MGS_UNITS_T
#define MGS_UNITS_T 48
#endif
constexpr int kUnitsThreadMin = MGS_UNITS_T;  // groups per CTA from which k_units takes a thread per group
constexpr int kNumScans = 7;
constexpr int kDbg = 19;  // per-step debug counters

enum Err : int { kOk = 0, kOverflow = 100 };

struct FrontierV2 {
  uint32_t* status;
  uint32_t* ids;  // placement's per-tenant mask ids (16 bits each)
  int32_t* pid;
  double* value;
  uint64_t* lex;
  uint32_t* rank;
  uint8_t* alive;
  int32_t* group;
  int32_t* kpos;  // position among the parent's children (k_write's count atomic), for k_kid_fill
  int32_t* g_start;
  int32_t* g_size;
  uint32_t* g_status;
  int32_t* g_alive;
};

struct StepCounters {  // double buffered; zeroed one step ahead
  int n_units, T, items_s, items_b, n_big, n_small, n_big_bucket, ticket, kids;
  int items_h;  // half items: units of <= kChunkH targets over groups of <= kSmall / 2 states
  int items_q;  // quarter items: units of <= kChunkQ targets over groups of <= kSmall / 4 states
  int u_cursor;  // unit-list allocation cursor (k_scans)
  int n_ns;  // successor statuses of the step = entries of the used-slot list
  int n_tab;  // big status groups of F_s whose subset tables k_tables builds
  // F_{s+1} allocation cursor: states in the low 32 bits, groups in the high
  // 32, so a status claims its range and its group with one atomic (every
  // writing warp of the GPU hits this one address)
  unsigned long long out_pack;
  __host__ __device__ int out_states() const { return static_cast<int>(out_pack & 0xffffffffull); }
  __host__ __device__ int out_groups() const { return static_cast<int>(out_pack >> 32); }
};

// claim `total` states and one group of F_{s+1}
__device__ __forceinline__ void claim_out(StepCounters& sc, int total, int* q0, int* gi) {
  const unsigned long long o = atomicAdd(&sc.out_pack, (1ull << 32) | static_cast<unsigned>(total));
  *q0 = static_cast<int>(o & 0xffffffffull);
  *gi = static_cast<int>(o >> 32);
}

struct Ctl {
  int err[2];
  int err_code, err_step;
  unsigned long long err_count;
  long long need;
  int need_what;
  int n_store[2];  // storage size of F (incl. dead)
  int n_groups[2];
  int alive_now[2];  // live states, counted at the start of the step that consumes F
  StepCounters sc[2];
  unsigned long long tr_ref, tr, ftot, fpeak, tbytes;
  unsigned long long best_vb, best_lex;
  int best_idx;
  int ranks_prev[2];  // [s&1]: stored states of F_{s-1}, the parent-rank space of F_s
  int dead[2];        // [x]: states of the frontier of parity x killed by dominance (k_dom)
  int scan_total[kNumScans];
};

struct V2 {
  DevSpace sp;
  HostTables t;
  int S;
  int has_initial;
  int dominance_ok;
  const double* band;  // device scalar (k_band_value), so a solve needs no host round trip for it
  uint64_t budget;
  const double* recv;
  const double* ub;
  const double* incumbent;
  FrontierV2 f[2];
  int fcap, gcap;
  int32_t* h_parent;
  int32_t* h_oi;
  long long hcap;
  long long* hist_base;  // [S+2]
  int32_t *u_group, *u_sig, *u_ns, *u_chs, *u_chb, *u_cbase, *u_upos;  // u_cbase: within the status's range
  int ucap;
  uint32_t* hash;  // key+1 per slot; the slot index is the successor-status id
  int hmask;
  int32_t* ns_used;  // hash slots claimed this step (list order = claim order)
  // per big group of F_s (> kSmall states): subset tables built once per step
  int tcap;                 // table slots
  int32_t* g_tab;           // [gcap] group -> slot (valid for big groups)
  unsigned long long* tab_vb;   // [tcap][n_partial] max value bits per (subset, projection)
  unsigned long long* tab_rx;   // [tcap][n_partial] (rank << 32 | j) of the best among the max
  uint32_t* tab_ex;         // [tcap][P1] j + 1 of the group's state at each placement (0 = none)
  // ex_bits > 0: entries are (step tag << ex_bits) | (j + 1) with tag = s + 1, so
  // a slot's stale entries from earlier steps read as empty and the map needs no
  // clearing (zeroed once per solve); 0: cleared per group and step as plain j + 1
  int ex_bits;
  int units_tmin;  // k_units: thread per group from this many groups per CTA (MGS_UNITS_THREAD_MIN)
  int subitems;    // half / quarter k_trans_small items (MGS_NO_SUBITEMS=1: full items only)
  unsigned long long* tab_hdr;  // [tcap][2] empty subset: value bits, (rank << 32 | j)
  int32_t *ns_ucnt, *ns_ccnt, *ns_ubase, *ns_cbase, *ns_units;
  int32_t *ns_big, *ns_small;
  // per successor status: bit 1 = a unit of a small group with <= kChunkS
  // candidates (one k_trans_small item), bit 2 = any other unit. A status whose
  // only unit is of the first kind is "fused": its k_trans_small item applies the
  // band and writes the survivors itself, and k_band / k_write skip it
  int32_t* ns_fflag;
  int32_t* ns_out;  // survivors per status
  unsigned long long* ns_vmax;  // vbits of the best bound-passing candidate value per status (band max)
  int32_t *it_s_unit, *it_s_chunk, *it_b_unit, *it_b_chunk, *it_h_unit, *it_q_unit;
  int itcap;
  double* c_value;
  uint64_t* c_lex;
  int32_t* c_parent;
  int32_t* c_pid;
  uint8_t* c_ok;
  uint8_t* c_live;
  int ccap;
  int32_t* kid_cnt[2];
  int32_t* kid_base;
  uint64_t* kid_items;
  int32_t* kid_pr;
  int32_t* big_bucket;
  int32_t* pcnt;
  int32_t* pbucket;
  unsigned long long* scan_state;
  int scan_cap;
  int32_t* sig_len;  // [n_sig]
  Ctl* ctl;
  int32_t* chosen;
  int n_partial;                 // entries of the partial-subset tables (all subsets but the full one)
  int sc_big_ctas;               // CTAs of k_trans that may take big-group items
  int oi_bits;                   // bits of an option index (radix sort width)
  int merge_win;                 // placement window of the CTA merge table
  int rank_words;                // 32-bit words of the option-index bitmap of k_ranks_big (0: does not fit)
  // Per-tenant fields of a packed status / placement-ids word: 16 bits at
  // M <= 2; 8 bits at M = 3..4 (status codes in the reference numbering,
  // < 256 for S <= 36; mask ids < 255, all-ones never matches)
  int fw;                        // field width, bits
  uint32_t fmask;
  int codec_shift;
  const uint32_t* ids32;         // [P1] placement ids packed fw bits per tenant
  long long* dbg;                // [S][kDbg] per-step counters (debug dump)
  unsigned long long* dbg_time;  // barrier timestamps (debug)
};

// Per-solve argument blocks, one per lane, device-resident (uploaded before
// each window; see solve_dp_v2_lanes). grid.y selects the lane.
#define c_v2 (ap[blockIdx.y])

__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_volatile(const int* p) {  // GPU-scope relaxed load (not a system-scope volatile)
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ void raise_err(const V2& a, int phi, int code, int step = 0, unsigned long long count = 0, int what = 0,
                          long long need = 0) {
  (void)phi;
  if (atomicCAS(&a.ctl->err_code, 0, code) == 0) {
    a.ctl->err_step = step;
    a.ctl->err_count = count;
    a.ctl->need_what = what;
    a.ctl->need = need;
  }
}

// every phase kernel returns immediately once any error was raised
__device__ __forceinline__ bool failed(const V2& a) { return ld_volatile(&a.ctl->err_code) != 0; }
// The entry check of a kernel, uniform over the block: a flag raised while the
// block starts (by another block, or another kernel) must not let some of its
// threads leave while the others reach a barrier or a full-warp collective.
__device__ __forceinline__ bool block_failed(const V2& a) { return __syncthreads_or(failed(a) ? 1 : 0) != 0; }

// ---------------------------------------------------------------------------
// block reductions / scans (kThreads threads)
__device__ __forceinline__ long long block_sum(long long x, long long* sm) {
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = x;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < kWarps ? sm[threadIdx.x] : 0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
  }
  __syncthreads();
  return t;  // valid in thread 0
}

// exclusive scan of n <= 2*kThreads ints in place (smem); returns total
__device__ int block_scan_small(int* v, int n, int* sm) {
  const int tid = threadIdx.x;
  const int a0 = 2 * tid < n ? v[2 * tid] : 0, a1 = 2 * tid + 1 < n ? v[2 * tid + 1] : 0;
  const int sum = a0 + a1;
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((tid & 31) >= o) x += y;
  }
  if ((tid & 31) == 31) sm[tid >> 5] = x;
  __syncthreads();
  if (tid < 32) {
    const int w = tid < kWarps ? sm[tid] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (tid >= o) z += y;
    }
    if (tid < kWarps) sm[32 + tid] = z - w;
    if (tid == kWarps - 1) sm[64] = z;
  }
  __syncthreads();
  const int ex = sm[32 + (tid >> 5)] + x - sum;
  if (2 * tid < n) v[2 * tid] = ex;
  if (2 * tid + 1 < n) v[2 * tid + 1] = ex + a0;
  const int total = sm[64];
  __syncthreads();
  return total;
}

struct ScanJob {
  const int32_t* in;
  const int32_t* in2;  // mode 1/2: statuses' candidate counts
  int32_t* out;
  int n;
  int mode;  // 0 plain, 1 big-status flag, 2 small-status flag, 3 nonzero flag
  const int32_t* idx = nullptr;  // gather/scatter through this list (status slots) when set
};

__device__ __forceinline__ int scan_load(const ScanJob& J, int i) {
  if (i >= J.n) return 0;
  if (J.idx) i = J.idx[i];
  if (J.mode == 0) return J.in[i];
  if (J.mode == 3) return J.in[i] > 0 ? 1 : 0;
  const int uc = J.in[i];
  if (uc == 0) return 0;
  const bool big = uc > 1 || J.in2[i] > kBigNs;
  return (J.mode == 1) == big ? 1 : 0;
}

// block-wide exclusive scan of one tile (kScanItems per thread); the thread's
// prefixes stay in v (written once the tile's offset is known); returns the
// tile total
__device__ int block_scan_tile(const ScanJob& J, int base, int* sm, int (&v)[kScanItems]) {
  const int tid = threadIdx.x;
  int sum = 0;
  if (J.mode == 0 && !J.idx && base + kTile <= J.n) {  // a full plain tile: 16-byte loads
    const int4* p4 = reinterpret_cast<const int4*>(J.in + base + tid * kScanItems);
#pragma unroll
    for (int k = 0; k < kScanItems / 4; ++k) {
      const int4 q = p4[k];
      v[4 * k] = q.x;
      v[4 * k + 1] = q.y;
      v[4 * k + 2] = q.z;
      v[4 * k + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) v[k] = scan_load(J, base + tid * kScanItems + k);
  }
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) sum += v[k];
  int x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((tid & 31) >= o) x += y;
  }
  if ((tid & 31) == 31) sm[tid >> 5] = x;
  __syncthreads();
  if (tid < 32) {
    const int w = tid < kWarps ? sm[tid] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, z, o);
      if (tid >= o) z += y;
    }
    if (tid < kWarps) sm[32 + tid] = z - w;
    if (tid == kWarps - 1) sm[64] = z;
  }
  __syncthreads();
  int run = sm[32 + (tid >> 5)] + x - sum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int tmp = v[k];
    v[k] = run;
    run += tmp;
  }
  const int agg = sm[64];
  __syncthreads();
  return agg;
}

// Several exclusive scans in one pass: tiles are handed out by a ticket, so
// every tile's predecessors are already owned by running CTAs (decoupled
// look-back cannot deadlock in a cooperative launch).
// NJ jobs, a compile-time count: the per-job tile tables stay in registers
template <int NJ>
__device__ __forceinline__ void multi_scan(const V2& a, const ScanJob (&jobs)[NJ], int epoch, int* ticket, int* totals) {
  constexpr int njobs = NJ;
  __shared__ int sm[80];
  __shared__ int s_tile, s_excl;
  int tiles[NJ], tbase[NJ + 1];
  tbase[0] = 0;
#pragma unroll
  for (int k = 0; k < njobs; ++k) {
    tiles[k] = (jobs[k].n + kTile - 1) / kTile;
    tbase[k + 1] = tbase[k] + tiles[k];
  }
  const int total_tiles = tbase[njobs];
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int k = 0; k < njobs; ++k)
      if (tiles[k] == 0) totals[k] = 0;
  if (static_cast<int>(blockIdx.x) >= total_tiles) return;  // no tile for this CTA: stay off the ticket
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int t = s_tile;
    __syncthreads();
    if (t >= total_tiles) break;
    int k = 0;
#pragma unroll
    for (int q = 1; q < NJ; ++q) k += t >= tbase[q] ? 1 : 0;
    const int j = t - tbase[k];
    const ScanJob& J = jobs[k];
    int v[kScanItems];
    const int agg = block_scan_tile(J, j * kTile, sm, v);
    if (threadIdx.x < 32) {  // warp-parallel decoupled look-back over windows of 32 predecessors
      const int lane = threadIdx.x;
      unsigned long long* st = a.scan_state + t;
      const unsigned long long ep = static_cast<unsigned long long>(epoch);
      if (lane == 0) {
        __threadfence();
        atomicExch(st, (ep << 34) | ((j == 0 ? 2ull : 1ull) << 32) | static_cast<uint32_t>(agg));
      }
      int excl = 0;
      if (j > 0) {
        int hi = t - 1;  // window [hi-31, hi], never below this job's first tile
        const int first = t - j;
        while (true) {
          const int q = hi - lane;
          unsigned long long w = 0;
          if (q >= first) {
            do {
              w = ld_acquire(a.scan_state + q);
            } while ((w >> 34) != ep || ((w >> 32) & 3) == 0);
          }
          const bool is_prefix = q >= first && ((w >> 32) & 3) == 2;
          const unsigned pm = __ballot_sync(0xffffffffu, is_prefix);
          const int stop = pm ? __ffs(pm) - 1 : 32;  // nearest inclusive prefix in the window
          int v = (q >= first && lane <= stop) ? static_cast<int>(w & 0xffffffffu) : 0;
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          excl += v;
          if (pm) break;
          hi -= 32;
        }
        if (lane == 0) {
          __threadfence();
          atomicExch(st, (ep << 34) | (2ull << 32) | static_cast<uint32_t>(excl + agg));
        }
      }
      if (lane == 0) {
        s_excl = excl;
        if (j == tiles[k] - 1) totals[k] = excl + agg;
      }
    }
    __syncthreads();
    const int excl = s_excl;
    const int b0 = j * kTile + threadIdx.x * kScanItems;
    if (!J.idx && (j + 1) * kTile <= J.n) {  // a full tile: 16-byte stores, offset included
      int4* o4 = reinterpret_cast<int4*>(J.out + b0);
#pragma unroll
      for (int k = 0; k < kScanItems / 4; ++k)
        o4[k] = make_int4(v[4 * k] + excl, v[4 * k + 1] + excl, v[4 * k + 2] + excl, v[4 * k + 3] + excl);
    } else {
#pragma unroll
      for (int k = 0; k < kScanItems; ++k) {  // one write per element, offset included
        const int i = b0 + k;
        if (i < J.n) J.out[J.idx ? J.idx[i] : i] = v[k] + excl;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// successor-status hash: the slot holding key+1 is the status id
__device__ __forceinline__ uint32_t mix32(uint32_t h) {  // murmur3 finalizer: all key bits reach the low bits
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// Claimed slots are listed for the step's status loops: first in the CTA's
// shared list (flushed with one global atomic per CTA batch), the global list
// directly when that is full.
constexpr int kNewCap = 512;
__device__ int ns_slot(const V2& a, uint32_t key, int phi, int step, int* s_nnew, int* s_new) {
  const uint32_t want = key + 1u;
  const unsigned h = mix32(key);
  for (int probe = 0; probe <= (a.hmask >> 1); ++probe) {
    const int slot = static_cast<int>((h + static_cast<unsigned>(probe)) & static_cast<unsigned>(a.hmask));
    uint32_t w = a.hash[slot];
    if (w == 0) {
      w = atomicCAS(&a.hash[slot], 0u, want);
      if (w == 0) {  // this thread claimed the slot
        const int i = atomicAdd(s_nnew, 1);
        if (i < kNewCap) s_new[i] = slot;
        else a.ns_used[atomicAdd(&a.ctl->sc[step & 1].n_ns, 1)] = slot;
        return slot;
      }
    }
    if (w == want) return slot;
  }
  raise_err(a, phi, kOverflow, step, 0, 2, 0);  // table too full
  return -1;
}

__device__ __forceinline__ int fld(const V2& a, uint32_t x, int m) {
  return static_cast<int>((x >> (a.fw * m)) & a.fmask);
}
// the same with the width fixed by the tenant count (kernels templated on M)
template <int M>
__device__ __forceinline__ int fldm(uint32_t x, int m) {
  constexpr int kW = M <= 2 ? 16 : 8;
  return static_cast<int>((x >> (kW * m)) & ((1u << kW) - 1u));
}
// some tenant field of x is zero (SWAR: a borrow reaches a field's top bit
// only out of a zero field; unused high fields are padded non-zero)
template <int M>
__device__ __forceinline__ bool any_zero_field(uint32_t x) {
  constexpr int kW = M <= 2 ? 16 : 8;
  constexpr uint32_t ones = kW == 16 ? 0x00010001u : 0x01010101u;
  constexpr uint32_t highs = kW == 16 ? 0x80008000u : 0x80808080u;
  constexpr uint32_t pad = kW * M >= 32 ? 0u : ~((1u << (kW * M)) - 1u);
  const uint32_t y = x | pad;
  return ((y - ones) & ~y & highs) != 0u;
}
template <int M>
__device__ __forceinline__ uint32_t fput(int v, int m) {
  constexpr int kW = M <= 2 ? 16 : 8;
  return static_cast<uint32_t>(v) << (kW * m);
}

// per-tenant allowed retraining sizes of a status (allowed_sizes, solvers.hpp:79-97)
template <int M>
struct UnitSpace {
  // sizes of tenant m: 4-bit entries of sz[m] (<= 9 of them), so the
  // runtime-indexed list stays in registers instead of local memory
  int st[M], cnt[M], total;
  unsigned long long sz[M];
  __device__ __forceinline__ int size_at(int m, int i) const { return static_cast<int>((sz[m] >> (4 * i)) & 0xfull); }
  __device__ __forceinline__ void push(int m, int k) {
    sz[m] |= static_cast<unsigned long long>(k) << (4 * cnt[m]);
    ++cnt[m];
  }
  __device__ void init(const V2& a, uint32_t status, int s) {
    const Codec codec{a.t.S, a.codec_shift};
    total = 1;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      st[m] = fldm<M>(status, m);
      cnt[m] = 0;
      sz[m] = 0ull;
      if (Codec::is_running(st[m])) {
        push(m, codec.run_size(st[m]));
      } else if (st[m] == Codec::done()) {
        push(m, 0);
      } else {
        if (a.t.min_rt[m] >= 0 && s + 1 + a.t.min_rt[m] <= a.t.S) push(m, 0);
#pragma unroll
        for (int k = 1; k <= 7; ++k)
          if (a.t.rt[m][k] >= 1 && s + a.t.rt[m][k] <= a.t.S) push(m, k);
      }
      total *= cnt[m];
    }
  }
  // combination c -> (valid, signature, successor status) (solvers.hpp:388-402)
  __device__ bool combo(const V2& a, int c, int s, int* sig_out, uint32_t* ns_out) const {
    const Codec codec{a.t.S, a.codec_shift};
    int rem = c, pick[M];
#pragma unroll
    for (int m = 0; m < M; ++m) {
      if (m == M - 1) {  // c < total: what remains is the last pick
        pick[m] = rem;
      } else {
        pick[m] = rem % cnt[m];
        rem /= cnt[m];
      }
    }
    int sz_p[M];
#pragma unroll
    for (int m = 0; m < M; ++m) sz_p[m] = size_at(m, pick[m]);
    int sig = 0;
#pragma unroll
    for (int m = M - 1; m >= 0; --m) sig = sig * 8 + sz_p[m];
    bool ok = true;
    uint32_t ns = 0;
#pragma unroll
    for (int m = 0; m < M; ++m) {
      const int adv = codec.advance(a.t.rt[m], st[m], sz_p[m], s);
      ok = ok && adv >= 0 && !(adv == 0 && (a.t.min_rt[m] < 0 || s + 1 + a.t.min_rt[m] > a.t.S));
      ns |= fput<M>(adv < 0 ? 0 : adv, m);
    }
    *sig_out = sig;
    *ns_out = ns;
    const int nopt = a.sp.sig_nopt[sig];  // sig is in range whatever ok is: no load behind it
    return ok && nopt > 0;
  }
};

// S1
// W lanes per group (W = 32: a warp; W < 32: 32 / W groups per warp, for the
// many groups with few size combinations). Loops run warp-uniformly: the
// sub-groups' combination counts are maxed over the warp.
template <int M, int W>
__device__ void phase_units(const V2& a, int s, int phi, int* s_cnt, long long* s_red) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int G = a.ctl->n_groups[cur];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int GPW = 32 / W;  // groups per warp
  const int sl = lane % W, sg = lane / W;
  const unsigned smask = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << (sg * W));
  __shared__ int s_base, s_scan[80];
  __shared__ int s_nnew, s_new[kNewCap];
  if (threadIdx.x == 0) s_nnew = 0;
  const int g0 = static_cast<int>(static_cast<long long>(G) * blockIdx.x / gridDim.x);
  const int g1 = static_cast<int>(static_cast<long long>(G) * (blockIdx.x + 1) / gridDim.x);
  long long ref = 0;
  auto warp_max = [&](int x) {
#pragma unroll
    for (int o = 16; o >= W; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
  };
  for (int bs = g0; bs < g1; bs += kBatch) {
    const int be = min(g1, bs + kBatch);
    // pass 1: unit count per group
    for (int gw = bs + warp * GPW; gw < be; gw += kWarps * GPW) {  // warp-uniform
      const int g = gw + sg;
      int n = 0;
      UnitSpace<M> us;
      us.total = 0;
      if (g < be && F.g_alive[g] > 0) us.init(a, F.g_status[g], s);
      const int tmax = warp_max(us.total);
      for (int c0 = 0; c0 < tmax; c0 += W) {
        int sig;
        uint32_t ns;
        const bool ok = c0 + sl < us.total && us.combo(a, c0 + sl, s, &sig, &ns);
        n += __popc(__ballot_sync(0xffffffffu, ok) & smask);
      }
      if (g < be && sl == 0) s_cnt[g - bs] = n;
    }
    __syncthreads();
    const int total = block_scan_small(s_cnt, be - bs, s_scan);
    if (threadIdx.x == 0) {
      s_base = atomicAdd(&sc.n_units, total);
      if (s_base + total > a.ucap) raise_err(a, phi, kOverflow, s, 0, 3, static_cast<long long>(s_base) + total);
    }
    __syncthreads();
    const int base = s_base;
    if (base + total <= a.ucap) {
      // pass 2: write the units (same enumeration order)
      for (int gw = bs + warp * GPW; gw < be; gw += kWarps * GPW) {  // warp-uniform
        const int g = gw + sg;
        const bool gv = g < be && F.g_alive[g] > 0;
        const bool small = gv && F.g_size[g] <= kSmall;  // big groups: subset tables by k_tables
        UnitSpace<M> us;
        us.total = 0;
        if (gv) us.init(a, F.g_status[g], s);
        int run = gv ? base + s_cnt[g - bs] : 0;
        const int tmax = warp_max(us.total);
        for (int c0 = 0; c0 < tmax; c0 += W) {
          int sig = 0;
          uint32_t ns = 0;
          const bool ok = c0 + sl < us.total && us.combo(a, c0 + sl, s, &sig, &ns);
          const unsigned bal = __ballot_sync(0xffffffffu, ok) & smask;
          if (ok) {
            const int u = run + __popc(bal & ((1u << lane) - 1u));
            const int id = ns_slot(a, ns, phi, s, &s_nnew, s_new);
            if (id >= 0) {
              const int L = a.sig_len[sig];
              a.u_group[u] = g;
              a.u_sig[u] = sig;
              a.u_ns[u] = id;
              // -1 / -2: one half / quarter item (k_trans_small runs two / four per warp)
              const int gsz = F.g_size[g];
              a.u_chs[u] = !small ? 0
                           : a.subitems && L <= kChunkQ && gsz <= kSmall / 4 ? -2
                           : a.subitems && L <= kChunkH && gsz <= kSmall / 2 ? -1
                                                                : (L + kChunkS - 1) / kChunkS;
              a.u_chb[u] = small ? 0 : (L + kChunkB - 1) / kChunkB;
              // the unit's slot in its status's unit list and candidate range
              // (k_scans places the status's range; order is irrelevant)
              a.u_upos[u] = atomicAdd(&a.ns_ucnt[id], 1);
              a.u_cbase[u] = atomicAdd(&a.ns_ccnt[id], L);
              atomicOr(&a.ns_fflag[id], small && L <= kChunkS ? 1 : 2);
              ref += a.sp.sig_nopt[sig];
            }
          }
          run += __popc(bal);
        }
      }
    }
    __syncthreads();
    const int nn = min(s_nnew, kNewCap);
    if (nn > 0) {  // uniform
      if (threadIdx.x == 0) s_base = atomicAdd(&sc.n_ns, nn);
      __syncthreads();
      for (int i = threadIdx.x; i < nn; i += kThreads) a.ns_used[s_base + i] = s_new[i];
      __syncthreads();
      if (threadIdx.x == 0) s_nnew = 0;
      __syncthreads();
    }
  }
  // children per parent (rank buckets of F_s) + live-state count
  const long long rs = block_sum(ref, s_red);
  if (threadIdx.x == 0 && rs) atomicAdd(&a.ctl->tr_ref, static_cast<unsigned long long>(rs));
}


// S1, thread per group (M <= 2: at most 9 x 9 size combinations, about one
// valid unit per group on C1): one CTA-wide pass over 256 groups at a time --
// count, block scan, one reservation, write -- instead of a warp walking its
// groups one after another. The group's unit space stays in registers between
// the count and the write.
template <int M>
__device__ void phase_units_thread(const V2& a, int s, int phi, int* s_cnt, long long* s_red) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int G = a.ctl->n_groups[cur];
  __shared__ int s_base, s_scan[80];
  __shared__ int s_nnew, s_new[kNewCap];
  if (threadIdx.x == 0) s_nnew = 0;
  const int g0 = static_cast<int>(static_cast<long long>(G) * blockIdx.x / gridDim.x);
  const int g1 = static_cast<int>(static_cast<long long>(G) * (blockIdx.x + 1) / gridDim.x);
  long long ref = 0;
  for (int bs = g0; bs < g1; bs += kThreads) {
    const int g = bs + threadIdx.x;
    const bool in = g < g1;
    const int alive = in ? F.g_alive[g] : 0;  // the group's fields loaded together
    const uint32_t gst = in ? F.g_status[g] : 0u;
    const int gsz = in ? F.g_size[g] : 0;
    UnitSpace<M> us;
    us.total = 0;
    int n = 0;
    if (alive > 0) {
      us.init(a, gst, s);
      for (int c = 0; c < us.total; ++c) {
        int sig;
        uint32_t ns;
        n += us.combo(a, c, s, &sig, &ns) ? 1 : 0;
      }
    }
    s_cnt[threadIdx.x] = n;
    __syncthreads();
    const int total = block_scan_small(s_cnt, kThreads, s_scan);
    if (threadIdx.x == 0) {
      s_base = atomicAdd(&sc.n_units, total);
      if (s_base + total > a.ucap) raise_err(a, phi, kOverflow, s, 0, 3, static_cast<long long>(s_base) + total);
    }
    __syncthreads();
    const int base = s_base;
    if (base + total <= a.ucap && n > 0) {
      const bool small = gsz <= kSmall;  // big groups: subset tables by k_tables
      int u = base + s_cnt[threadIdx.x];
      for (int c = 0; c < us.total; ++c) {
        int sig = 0;
        uint32_t ns = 0;
        if (!us.combo(a, c, s, &sig, &ns)) continue;
        const int id = ns_slot(a, ns, phi, s, &s_nnew, s_new);
        if (id >= 0) {
          const int L = a.sig_len[sig];
          a.u_group[u] = g;
          a.u_sig[u] = sig;
          a.u_ns[u] = id;
          // -1 / -2: one half / quarter item (k_trans_small runs two / four per warp)
          a.u_chs[u] = !small ? 0
                       : a.subitems && L <= kChunkQ && gsz <= kSmall / 4 ? -2
                       : a.subitems && L <= kChunkH && gsz <= kSmall / 2 ? -1
                                                            : (L + kChunkS - 1) / kChunkS;
          a.u_chb[u] = small ? 0 : (L + kChunkB - 1) / kChunkB;
          // the unit's slot in its status's unit list and candidate range
          // (k_scans places the status's range; order is irrelevant)
          a.u_upos[u] = atomicAdd(&a.ns_ucnt[id], 1);
          a.u_cbase[u] = atomicAdd(&a.ns_ccnt[id], L);
          atomicOr(&a.ns_fflag[id], small && L <= kChunkS ? 1 : 2);
          ref += a.sp.sig_nopt[sig];
        }
        ++u;
      }
    }
    __syncthreads();
    const int nn = min(s_nnew, kNewCap);
    if (nn > 0) {  // uniform
      if (threadIdx.x == 0) s_base = atomicAdd(&sc.n_ns, nn);
      __syncthreads();
      for (int i = threadIdx.x; i < nn; i += kThreads) a.ns_used[s_base + i] = s_new[i];
      __syncthreads();
      if (threadIdx.x == 0) s_nnew = 0;
      __syncthreads();
    }
  }
  const long long rs = block_sum(ref, s_red);
  if (threadIdx.x == 0 && rs) atomicAdd(&a.ctl->tr_ref, static_cast<unsigned long long>(rs));
}

// S3: placement
// R3 (rank branch): children into their parent's slots
__device__ void phase_kid_fill(const V2& a, int s) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const FrontierV2& F = a.f[cur];
  // every stored state, live or dominated: ranks over the stored states order
  // the live ones exactly like dense ranks over the live ones, and they do not
  // wait for k_dom (this branch runs beside it)
  const int n = s == 0 ? a.ctl->n_store[0] : a.ctl->sc[(s - 1) & 1].out_states();
  const int lane = threadIdx.x & 31;
  // software-pipelined, two deep: element i + 2 * stride's lex and sibling slot,
  // and element i + stride's bucket base and count (its lex arrived one
  // iteration earlier), are loaded before element i's stores
  int i0 = gtid - lane;
  bool al = i0 + lane < n;
  uint64_t lx_c = al ? F.lex[i0 + lane] : 0;
  int kp_c = al ? F.kpos[i0 + lane] : 0;
  int base_c = al ? a.kid_base[static_cast<int>(lx_c >> 32)] : 0;
  int cnt_c = al ? a.kid_cnt[cur][static_cast<int>(lx_c >> 32)] : 0;
  bool al_n = i0 + lane + gstride < n;
  uint64_t lx_n = al_n ? F.lex[i0 + lane + gstride] : 0;
  int kp_n = al_n ? F.kpos[i0 + lane + gstride] : 0;
  for (; i0 < n; i0 += gstride) {  // warp-uniform trip count
    const int i = i0 + lane;
    const int in2 = i + 2 * gstride;
    const bool al_2 = in2 < n;
    const uint64_t lx_2 = al_2 ? F.lex[in2] : 0;
    const int kp_2 = al_2 ? F.kpos[in2] : 0;
    const int pr_n = static_cast<int>(lx_n >> 32);
    const int base_n = al_n ? a.kid_base[pr_n] : 0;
    const int cnt_n = al_n ? a.kid_cnt[cur][pr_n] : 0;
    bool big_first = false;
    int pr = 0;
    if (al) {
      const uint64_t lx = lx_c;
      pr = static_cast<int>(lx >> 32);
      const int q = kp_c;  // the state's slot among its siblings (k_write)
      const int slot = base_c + q;
      a.kid_items[slot] = ((lx & 0xffffffffull) << 32) | static_cast<uint32_t>(i);
      a.kid_pr[slot] = pr;
      big_first = q == 0 && cnt_c > kBucketSmall;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, big_first);
    if (bal) {
      int b0 = 0;
      if (lane == 0) b0 = atomicAdd(&sc.n_big_bucket, __popc(bal));
      b0 = __shfl_sync(0xffffffffu, b0, 0);
      if (big_first) a.big_bucket[b0 + __popc(bal & ((1u << lane) - 1u))] = pr;
    }
    al = al_n;
    lx_c = lx_n;
    kp_c = kp_n;
    base_c = base_n;
    cnt_c = cnt_n;
    al_n = al_2;
    lx_n = lx_2;
    kp_n = kp_2;
  }
}

// S4: dense ranks of F_s (solvers.hpp:544-548 restated: lex = (parent rank,
// option index), so the rank is the parent's first child slot plus the
// position of the option index among the parent's children).
// Big buckets: one CTA each, block radix sort of the option indices.
__device__ void phase_ranks_big(const V2& a, int s, unsigned long long* sm64) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int nb = sc.n_big_bucket;
  using Sort = cub::BlockRadixSort<unsigned long long, kThreads, kSortItems>;
  Sort::TempStorage& tmp = *reinterpret_cast<typename Sort::TempStorage*>(sm64);
  for (int b = blockIdx.x; b < nb; b += gridDim.x) {
    const int pr = a.big_bucket[b];
    const int base = a.kid_base[pr], c = a.kid_cnt[cur][pr];
    // the option-index bitmap costs O(c + |O|/32) and the radix sort O(4096)
    // per bucket: the bitmap whenever its words are few next to the bucket
    const bool use_bits = a.rank_words > 0 && a.rank_words <= kBitmapPerKey * c;
    if (!use_bits && c <= kThreads * kSortItems) {
      unsigned long long keys[kSortItems];
#pragma unroll
      for (int k = 0; k < kSortItems; ++k) {
        const int i = threadIdx.x * kSortItems + k;
        keys[k] = i < c ? a.kid_items[base + i] : ~0ull;
      }
      Sort(tmp).Sort(keys, 32, 32 + a.oi_bits);  // option indices are distinct within a bucket
#pragma unroll
      for (int k = 0; k < kSortItems; ++k) {
        const int i = threadIdx.x * kSortItems + k;
        if (i < c) F.rank[static_cast<uint32_t>(keys[k])] = base + i;
      }
      __syncthreads();
    } else if (a.rank_words > 0) {
      // the siblings' option indices are distinct, so a bitmap over option
      // indices in shared memory and its word prefix popcounts give every rank
      // in O(c + |O|/32) (also beyond one CTA's sort: the root's children)
      uint32_t* bits = reinterpret_cast<uint32_t*>(sm64);
      uint32_t* pre = bits + a.rank_words;
      const int W = a.rank_words;
      for (int w = threadIdx.x; w < W; w += kThreads) bits[w] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < c; i += kThreads) {
        const uint32_t oi = static_cast<uint32_t>(a.kid_items[base + i] >> 32);
        atomicOr(&bits[oi >> 5], 1u << (oi & 31));
      }
      __syncthreads();
      if (threadIdx.x < 32) {  // one warp: exclusive scan of the word popcounts
        int run = 0;
        for (int w0 = 0; w0 < W; w0 += 32) {
          const int w = w0 + threadIdx.x;
          const int v = w < W ? __popc(bits[w]) : 0;
          int x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (threadIdx.x >= o) x += y;
          }
          if (w < W) pre[w] = run + x - v;
          run += __shfl_sync(0xffffffffu, x, 31);
        }
      }
      __syncthreads();
      for (int i = threadIdx.x; i < c; i += kThreads) {
        const unsigned long long me = a.kid_items[base + i];
        const uint32_t oi = static_cast<uint32_t>(me >> 32);
        const int pos = pre[oi >> 5] + __popc(bits[oi >> 5] & ((1u << (oi & 31)) - 1u));
        F.rank[static_cast<uint32_t>(me)] = base + pos;
      }
      __syncthreads();
    } else {  // counting (correct; only when the bitmap does not fit)
      for (int i = threadIdx.x; i < c; i += kThreads) {
        const unsigned long long me = a.kid_items[base + i];
        int pos = 0;
        for (int k = 0; k < c; ++k) pos += a.kid_items[base + k] < me;
        F.rank[static_cast<uint32_t>(me)] = base + pos;
      }
    }
  }
}

// Small buckets: thread per slot (a parent's slots are adjacent: warp broadcasts)
__device__ void phase_ranks_small(const V2& a, int s) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const int n = sc.kids;  // live states of F_s = filled slots
  // software-pipelined, two deep: slot i + 2 * stride's parent and key, and
  // slot i + stride's bucket count and base (its parent arrived one iteration
  // earlier), are loaded before slot i's rank is stored
  int i = gtid;
  int c = 0, base = 0;
  unsigned long long me = 0;
  if (i < n) {
    const int pr = a.kid_pr[i];
    me = a.kid_items[i];
    c = a.kid_cnt[cur][pr];
    base = a.kid_base[pr];
  }
  int pr_n = 0;
  unsigned long long me_n = 0;
  if (i + gstride < n) {
    pr_n = a.kid_pr[i + gstride];
    me_n = a.kid_items[i + gstride];
  }
  for (; i < n; i += gstride) {
    const int in = i + gstride, in2 = i + 2 * gstride;
    int pr_2 = 0;
    unsigned long long me_2 = 0;
    if (in2 < n) {
      pr_2 = a.kid_pr[in2];
      me_2 = a.kid_items[in2];
    }
    int c_n = 0, base_n = 0;
    if (in < n) {
      c_n = a.kid_cnt[cur][pr_n];
      base_n = a.kid_base[pr_n];
    }
    if (c <= kBucketSmall) {
      int rank = base;
      if (c > 1) {  // siblings' option indices (the keys' high words) are distinct: 32-bit compares
        const uint32_t* hi = reinterpret_cast<const uint32_t*>(a.kid_items + base) + 1;
        const uint32_t mo = static_cast<uint32_t>(me >> 32);
        for (int k = 0; k < c; ++k) rank += hi[2 * k] < mo;
      }
      F.rank[static_cast<uint32_t>(me)] = rank;
    }
    me = me_n;
    c = c_n;
    base = base_n;
    pr_n = pr_2;
    me_n = me_2;
  }
}

// ---------------------------------------------------------------------------
// S5: transitions
template <int M>
struct BestT {
  double v[1 << M];
  uint32_t r[1 << M];
  int i[1 << M];
};

struct Cand {  // one transition's result held in registers (fused statuses)
  double v;
  uint64_t lex;
  int parent;
  bool ok;
};

template <int M>
__device__ __forceinline__ unsigned long long emit_target(const V2& a, int s, int charge, int cbu, int t_idx, int gs,
                                            const double* acc, int p, int oi, uint32_t ids_p, const BestT<M>& b,
                                            const FrontierV2& F, Cand* c = nullptr) {
  const HostTables& t = a.t;
  double cap[M], bonus[M];
#pragma unroll
  for (int m = 0; m < M; ++m) {  // solvers.hpp:426-433
    cap[m] = a.sp.pl_cap[p * KM + m];
    const double recv = a.recv[m * t.S + s];
    const double c_changed = dmul(thr_of(recv, eff_cap(cap[m], charge ? t.loss[m] : 0.0)), acc[m]);
    bonus[m] = charge ? dsub(dmul(thr_of(recv, cap[m]), acc[m]), c_changed) : 0.0;
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
  if (chosen < 0) {  // cannot happen: units come from groups with live states
    if (c) c->ok = false;
    else a.c_ok[cbu + t_idx] = 0;
    return 0ull;
  }
  const int pred = gs + chosen;
  const uint32_t pids = F.ids[pred];
  double v = F.value[pred];  // exact fold (solvers.hpp:451-458)
#pragma unroll
  for (int m = 0; m < M; ++m) {
    const bool changed = charge && fldm<M>(pids, m) != fldm<M>(ids_p, m);
    const double eff = eff_cap(cap[m], changed ? t.loss[m] : 0.0);
    v = dadd(v, dmul(thr_of(a.recv[m * t.S + s], eff), acc[m]));
  }
  const bool ok = !(dadd(v, a.ub[s + 1]) < *a.incumbent);  // solvers.hpp:459 (strict)
  const uint64_t lex = (static_cast<uint64_t>(F.rank[pred]) << 32) | static_cast<uint32_t>(oi);
  if (c) {  // kept in registers: the caller finishes the status itself
    c->v = v;
    c->lex = lex;
    c->parent = pred;
    c->ok = ok;
  } else {
    const int slot = cbu + t_idx;
    a.c_value[slot] = v;
    a.c_lex[slot] = lex;
    a.c_parent[slot] = pred;
    a.c_pid[slot] = p;
    a.c_ok[slot] = ok ? 1 : 0;
  }
  return ok ? vbits(v) : 0ull;  // values are >= 0: vbits orders them
}

template <int M>
__device__ __forceinline__ void group_acc(const V2& a, uint32_t gstat, double* acc) {
#pragma unroll
  for (int m = 0; m < M; ++m)
    acc[m] = fldm<M>(gstat, m) == Codec::done() ? a.t.post[m] : a.t.pre[m];
}

// Subset tables of every big group of F_s, built once per step (one CTA per
// group) into L2-resident global slots: the best representative per (subset,
// projected placement) by a max-value then min-(rank, idx) pass (solvers.hpp:
// 363-378), the state at each placement (the full subset), and the group's
// best state (the empty subset). k_trans_big items then only read them.
__device__ void phase_tables(const V2& a, int s) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int P1 = a.sp.P1, np = a.n_partial, M = a.t.M;
  const int nsub = 1 << M;
  const uint32_t ex_tag = a.ex_bits ? static_cast<uint32_t>(s + 1) << a.ex_bits : 0u;
  __shared__ unsigned long long s_bv[kWarps], s_brx[kWarps];
  __shared__ int s_list[kThreads], s_lgs[kThreads], s_lgn[kThreads], s_n, s_slot0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // the CTA's own big groups: F_s's groups strided over the CTAs (big groups
  // are written together, so their indices cluster), found with one parallel
  // load per group (no dependency on k_units: this kernel runs on the rank
  // branch beside the unit branch), then one slot reservation
  const int G = a.ctl->n_groups[cur];
  const int per = G > static_cast<int>(blockIdx.x) ? (G - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;
  for (int c0 = 0; c0 < per; c0 += kThreads) {
  if (threadIdx.x == 0) s_n = 0;
  __syncthreads();
  {
    const int k = c0 + threadIdx.x;
    const int g = static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x);
    const bool in = k < per;
    const int gsz = in ? F.g_size[g] : 0, gal = in ? F.g_alive[g] : 0, gst = in ? F.g_start[g] : 0;
    if (in && gal > 0 && gsz > kSmall) {  // the group's range kept beside it (no reload per group)
      const int li = atomicAdd(&s_n, 1);
      s_list[li] = g;
      s_lgs[li] = gst;
      s_lgn[li] = gsz;
    }
  }
  __syncthreads();
  const int nl = s_n;
  if (nl == 0) continue;  // uniform
  if (threadIdx.x == 0) s_slot0 = atomicAdd(&sc.n_tab, nl);
  __syncthreads();
  const int slot0 = s_slot0;
  if (slot0 + nl > a.tcap) {  // uniform
    if (threadIdx.x == 0) raise_err(a, 0, kOverflow, s, 0, 9, slot0 + nl);
    return;
  }
  for (int li = 0; li < nl; ++li) {
    const int g = s_list[li], b = slot0 + li;
    if (threadIdx.x == 0) a.g_tab[g] = b;
    const int gs = s_lgs[li], gn = s_lgn[li];
    unsigned long long* vb = a.tab_vb + static_cast<size_t>(b) * np;
    unsigned long long* rxs = a.tab_rx + static_cast<size_t>(b) * np;
    uint32_t* ex = a.tab_ex + static_cast<size_t>(b) * P1;
    if (!a.ex_bits)
      for (int i = threadIdx.x; i < P1; i += kThreads) ex[i] = 0u;
    for (int i = threadIdx.x; i < np; i += kThreads) {
      vb[i] = 0ull;
      rxs[i] = ~0ull;
    }
    __syncthreads();
    unsigned long long bv = 0, brx = ~0ull;
    // software-pipelined: the next state's loads are issued before this
    // state's stores / atomics (which loads could not be moved across)
    int j = threadIdx.x;
    bool al = false;
    int pj = 0;
    double vd = 0.0;
    uint32_t rk = 0;
    if (j < gn) {
      al = F.alive[gs + j];
      pj = F.pid[gs + j];
      vd = F.value[gs + j];
      rk = F.rank[gs + j];
    }
    // a group of at most kThreads states is one iteration: the min pass below
    // reuses these registers instead of loading the fields again
    const bool al0 = al;
    const int pj0 = pj;
    const double vd0 = vd;
    const uint32_t rk0 = rk;
    for (; j < gn; j += kThreads) {  // claim placements, max value per entry, group best
      const int jn = j + kThreads;
      bool al_n = false;
      int pj_n = 0;
      double vd_n = 0.0;
      uint32_t rk_n = 0;
      if (jn < gn) {
        al_n = F.alive[gs + jn];
        pj_n = F.pid[gs + jn];
        vd_n = F.value[gs + jn];
        rk_n = F.rank[gs + jn];
      }
      if (al) {
        const unsigned long long v = vbits(vd);
        const unsigned long long rx = (static_cast<unsigned long long>(rk) << 32) | static_cast<uint32_t>(j);
        if (brx == ~0ull || v > bv || (v == bv && rx < brx)) {
          bv = v;
          brx = rx;
        }
        ex[pj] = ex_tag | (static_cast<uint32_t>(j) + 1u);
        for (int sub = 1; sub < nsub - 1; ++sub)
          atomicMax(&vb[a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + pj]], v);
      }
      al = al_n;
      pj = pj_n;
      vd = vd_n;
      rk = rk_n;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long ov = __shfl_down_sync(0xffffffffu, bv, o);
      const unsigned long long orx = __shfl_down_sync(0xffffffffu, brx, o);
      if (orx != ~0ull && (brx == ~0ull || ov > bv || (ov == bv && orx < brx))) {
        bv = ov;
        brx = orx;
      }
    }
    if (lane == 0) {
      s_bv[warp] = bv;
      s_brx[warp] = brx;
    }
    __syncthreads();  // also orders the vb maxima before the min pass (block-scope visibility)
    if (threadIdx.x == 0) {
      for (int w = 1; w < kWarps; ++w)
        if (s_brx[w] != ~0ull && (brx == ~0ull || s_bv[w] > bv || (s_bv[w] == bv && s_brx[w] < brx))) {
          bv = s_bv[w];
          brx = s_brx[w];
        }
      a.tab_hdr[2 * b] = bv;
      a.tab_hdr[2 * b + 1] = brx;
    }
    if (nsub == 4) {  // min (rank, idx) among the max; M = 2: the partial subsets are 1 and 2
      // software-pipelined (the first iteration from pass 1's registers): the
      // next state's fields are loaded before this state's atomics
      int j = threadIdx.x;
      bool al = al0;
      int pj = pj0;
      double vd = vd0;
      uint32_t rk = rk0;
      for (; j < gn; j += kThreads) {
        const int jn = j + kThreads;
        const bool in_n = jn < gn;
        const bool al_n = in_n && F.alive[gs + jn];
        const int pj_n = in_n ? F.pid[gs + jn] : 0;
        const double vd_n = in_n ? F.value[gs + jn] : 0.0;
        const uint32_t rk_n = in_n ? F.rank[gs + jn] : 0u;
        if (al) {
          const unsigned long long v = vbits(vd);
          const unsigned long long rx = (static_cast<unsigned long long>(rk) << 32) | static_cast<uint32_t>(j);
          const int e1 = a.sp.proj_base[1] + a.sp.proj_id[1 * P1 + pj];
          const int e2 = a.sp.proj_base[2] + a.sp.proj_id[2 * P1 + pj];
          const unsigned long long m1 = vb[e1], m2 = vb[e2];  // both loads before either atomic
          if (m1 == v) atomicMin(&rxs[e1], rx);
          if (m2 == v) atomicMin(&rxs[e2], rx);
        }
        al = al_n;
        pj = pj_n;
        vd = vd_n;
        rk = rk_n;
      }
    } else if (nsub > 4) {  // M = 3..4: every partial subset
      for (int j = threadIdx.x; j < gn; j += kThreads) {
        if (!F.alive[gs + j]) continue;
        const int pj = F.pid[gs + j];
        const unsigned long long v = vbits(F.value[gs + j]);
        const unsigned long long rx = (static_cast<unsigned long long>(F.rank[gs + j]) << 32) | static_cast<uint32_t>(j);
        for (int sub = 1; sub < nsub - 1; ++sub) {
          const int e = a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + pj];
          if (vb[e] == v) atomicMin(&rxs[e], rx);
        }
      }
    }
    __syncthreads();
  }
  }
}

// Big groups: one CTA per (unit, chunk) item; every thread owns targets and
// reads its group's subset tables (phase_tables) from L2.
template <int M>
__device__ void phase_trans_big(const V2& a, int s) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int charge = (s > 0 || a.has_initial) ? 1 : 0;
  const int P1 = a.sp.P1, np = a.n_partial;
  const int nib = sc.items_b;
  for (int item = blockIdx.x; item < nib; item += gridDim.x) {
    const int unit = a.it_b_unit[item], chunk = a.it_b_chunk[item];
    const int g = a.u_group[unit], sig = a.u_sig[unit], ns_id = a.u_ns[unit];
    const int gs = F.g_start[g];
    const int cbu = a.ns_cbase[ns_id] + a.u_cbase[unit];
    const int b = a.g_tab[g];
    const unsigned long long* vb = a.tab_vb + static_cast<size_t>(b) * np;
    const unsigned long long* rxs = a.tab_rx + static_cast<size_t>(b) * np;
    const uint32_t* ex = a.tab_ex + static_cast<size_t>(b) * P1;
    const unsigned long long v0 = a.tab_hdr[2 * b], rx0 = a.tab_hdr[2 * b + 1];
    double acc[M];
    group_acc<M>(a, F.g_status[g], acc);
    const int sb = a.sp.sig_off[sig], L = a.sp.sig_off[sig + 1] - sb;
    const int t0 = chunk * kChunkB, t1 = min(L, t0 + kChunkB);
    unsigned long long vmax = 0ull;
    // the next target's candidate is loaded before this target's stores
    int p_n = t0 + threadIdx.x < t1 ? a.sp.cand_pid[sb + t0 + threadIdx.x] : 0;
    int oi_n = t0 + threadIdx.x < t1 ? a.sp.cand_oi[sb + t0 + threadIdx.x] : 0;
    for (int ti = t0 + threadIdx.x; ti < t1; ti += kThreads) {
      const int p = p_n, oi = oi_n;
      if (ti + kThreads < t1) {
        p_n = a.sp.cand_pid[sb + ti + kThreads];
        oi_n = a.sp.cand_oi[sb + ti + kThreads];
      }
      BestT<M> bt;
      bt.i[0] = rx0 == ~0ull ? -1 : static_cast<int>(rx0 & 0xffffffffu);
      bt.v[0] = __longlong_as_double(static_cast<long long>(v0));
      bt.r[0] = static_cast<uint32_t>(rx0 >> 32);
#pragma unroll
      for (int sub = 1; sub < (1 << M) - 1; ++sub) {
        const int e = a.sp.proj_base[sub] + a.sp.proj_id[sub * P1 + p];
        const unsigned long long rx = rxs[e];
        const bool hit = rx != ~0ull;
        bt.i[sub] = hit ? static_cast<int>(rx & 0xffffffffu) : -1;
        bt.v[sub] = hit ? __longlong_as_double(static_cast<long long>(vb[e])) : 0.0;
        bt.r[sub] = hit ? static_cast<uint32_t>(rx >> 32) : 0u;
      }
      {
        const uint32_t w0 = ex[p];
        const uint32_t w = a.ex_bits ? ((w0 >> a.ex_bits) == static_cast<uint32_t>(s + 1) ? w0 & ((1u << a.ex_bits) - 1u) : 0u) : w0;
        const int full = (1 << M) - 1;
        if (w) {
          const int j = static_cast<int>(w) - 1;
          bt.i[full] = j;
          bt.v[full] = F.value[gs + j];
          bt.r[full] = F.rank[gs + j];
        } else {
          bt.i[full] = -1;
          bt.v[full] = 0.0;
          bt.r[full] = 0u;
        }
      }
      const unsigned long long vb_t =
          emit_target<M>(a, s, charge, cbu, ti, gs, acc, p, oi, a.ids32[p], bt, F);
      vmax = vb_t > vmax ? vb_t : vmax;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, vmax, o);
      vmax = y > vmax ? y : vmax;
    }
    if ((threadIdx.x & 31) == 0 && vmax) atomicMax(&a.ns_vmax[a.u_ns[unit]], vmax);
  }
}

// Small groups: one warp per (unit, 32 targets) item; every lane owns a target
// and scans the group's states (broadcast loads) keeping the best per subset.
__device__ __forceinline__ bool claim_fits(const V2& a, int s, int q0, int total, int gi);
__device__ __forceinline__ void write_state_v(const V2& a, int s, int nxt, int q, int gidx, uint32_t key, int p,
                                              uint64_t lx, double v, int parent);
__device__ __forceinline__ void write_state_w(const V2& a, int s, int nxt, int q, int gidx, uint32_t key, int p,
                                              uint64_t lx, double v, int parent, uint32_t ids, int pcv);

// One warp task of k_trans_small: W = 32, one full item (32 targets of a
// unit, it_s list); W = 16 / 8, two half / four quarter items (it_h / it_q
// lists: a unit of <= 16 / 8 targets over a group of <= kSmall / 2 / kSmall / 4
// states), one per W lanes, with their own staging, reductions and output.
template <int M, int W>
__device__ __forceinline__ void small_task(const V2& a, int s, int task, const int32_t* list, int nlist, double band,
                                           uint32_t* sh_ids, uint32_t* sh_rank, double* sh_val) {
  const int cur = s & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& F = a.f[cur];
  const int charge = (s > 0 || a.has_initial) ? 1 : 0;
  const int lane = threadIdx.x & 31;
  constexpr int kFull = (1 << M) - 1;
  constexpr bool half = W < 32;
  {
    const int sl = lane & (W - 1);    // lane within the item
    const int hb = lane - sl;         // first lane of the item
    int unit = 0, chunk = 0;
    bool valid = true;
    if (!half) {
      unit = a.it_s_unit[task];
      chunk = a.it_s_chunk[task];
    } else {  // task is relative to its list
      const int hi = (32 / W) * task + lane / W;
      valid = hi < nlist;
      unit = valid ? list[hi] : 0;
    }
    const int g = a.u_group[unit], sig = a.u_sig[unit];
    const int gs = F.g_start[g], gn = valid ? F.g_size[g] : 0;
    const int sb = a.sp.sig_off[sig], L = valid ? a.sp.sig_off[sig + 1] - sb : 0;
    const int ti = chunk * kChunkS + sl;
    const int ns_id = a.u_ns[unit];
    const int ucnt = a.ns_ucnt[ns_id], fflag = a.ns_fflag[ns_id];  // both loads issued together
    const bool fused = valid && ucnt == 1 && fflag == 1;            // then L <= 32, chunk 0
    if (a.dbg && sl == 0 && valid) {  // [14] group sizes, [15] fused, [16] gn > 32, [17] targets, [18] targets x gn
      unsigned long long* d = reinterpret_cast<unsigned long long*>(a.dbg + kDbg * s);
      atomicAdd(d + 14, static_cast<unsigned long long>(gn));
      if (fused) atomicAdd(d + 15, 1ull);
      if (gn > 32) atomicAdd(d + 16, 1ull);
      const int act = min(32, L - chunk * kChunkS);
      atomicAdd(d + 17, static_cast<unsigned long long>(act));
      atomicAdd(d + 18, static_cast<unsigned long long>(act) * gn);
    }
    const int cbu = a.ns_cbase[ns_id] + a.u_cbase[unit];
    Cand cand{0.0, 0ull, 0, false};
    int cand_p = 0, cand_pcv = 0;
    uint32_t cand_ids = 0u;
    // staging: a half / quarter item uses its part of the warp's arrays (gn <= kSmall * W / 32)
    const int so = (lane / W) * (kSmall * W / 32);
    uint32_t* gids = sh_ids + so;
    uint32_t* grank = sh_rank + so;
    double* gval = sh_val + so;
    // empty subset: the group's best state, one cooperative pass
    double v0 = 0.0;
    uint32_t r0 = 0xffffffffu;
    int i0 = -1;
    __syncwarp();  // the previous task's scan is done with the staging arrays
    for (int j = sl; j < gn; j += W) {
      const uint8_t al = F.alive[gs + j];
      const double vj = F.value[gs + j];
      const uint32_t rj = F.rank[gs + j];
      const uint32_t idj = F.ids[gs + j];  // loaded with the others, not behind al
      // a dead state is staged with all-ones ids: no 16-bit field matches a
      // placement's (ids are indices < 0xffff, k_proj_keys' wildcard)
      gids[j] = al ? idj : 0xffffffffu;
      grank[j] = rj;
      gval[j] = vj;
      if (!al) continue;
      if (i0 < 0 || better(vj, rj, v0, r0)) {
        v0 = vj;
        r0 = rj;
        i0 = j;
      }
    }
    for (int o = W >> 1; o > 0; o >>= 1) {  // xor offsets < W stay inside the item's lanes
      const double ov = __shfl_xor_sync(0xffffffffu, v0, o);
      const uint32_t orr = __shfl_xor_sync(0xffffffffu, r0, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i0, o);
      if (oi >= 0 && (i0 < 0 || better(ov, orr, v0, r0))) {
        v0 = ov;
        r0 = orr;
        i0 = oi;
      }
    }
    __syncwarp();
    unsigned long long vb_t = 0ull;
    if (ti < L) {
    double acc[M];
    group_acc<M>(a, F.g_status[g], acc);
    const int p = a.sp.cand_pid[sb + ti];
    const int oi = a.sp.cand_oi[sb + ti];
    const uint32_t ids_p = a.ids32[p];
    cand_p = p;
    cand_ids = ids_p;
    cand_pcv = fused ? a.pcnt[p] : 0;  // (possibly stale) bucket count for the fused write
    BestT<M> b;
#pragma unroll
    for (int k = 1; k < (1 << M); ++k) {
      b.i[k] = -1;
      b.v[k] = 0.0;
      b.r[k] = 0xffffffffu;
    }
    b.i[0] = i0;
    b.v[0] = v0;
    b.r[0] = r0;
    // non-empty subsets: only states that agree with the target on the
    // subset's tenants can represent it (solvers.hpp:367-378)
    // pass 1, branch-free: the states that agree with the target on some
    // tenant (bit j; gn <= kSmall = 64); pass 2 visits only those, in
    // ascending j (better() is a strict order: the visiting order is free)
    unsigned long long mm = 0ull;
#pragma unroll 8
    for (int j = 0; j < gn; ++j) mm |= static_cast<unsigned long long>(any_zero_field<M>(gids[j] ^ ids_p)) << j;
    while (mm) {
      const int j = __ffsll(static_cast<long long>(mm)) - 1;
      mm &= mm - 1ull;
      const uint32_t x = gids[j] ^ ids_p;
      int mt = 0;
#pragma unroll
      for (int m = 0; m < M; ++m) mt |= fldm<M>(x, m) == 0 ? (1 << m) : 0;
      const double vj = gval[j];
      const uint32_t rj = grank[j];
      if (mt == kFull) {  // the full subset's key is the state's own placement: unique in the group
        b.v[kFull] = vj;
        b.r[kFull] = rj;
        b.i[kFull] = j;
      }
#pragma unroll
      for (int sub = 1; sub < kFull; ++sub) {
        if ((sub & ~mt) != 0) continue;
        if (b.i[sub] < 0 || better(vj, rj, b.v[sub], b.r[sub])) {
          b.v[sub] = vj;
          b.r[sub] = rj;
          b.i[sub] = j;
        }
      }
    }
    vb_t = emit_target<M>(a, s, charge, cbu, ti, gs, acc, p, oi, ids_p, b, F, fused ? &cand : nullptr);
    }
    for (int o = W >> 1; o > 0; o >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, vb_t, o);
      vb_t = y > vb_t ? y : vb_t;
    }
    if (!fused && valid && sl == 0 && vb_t) atomicMax(&a.ns_vmax[ns_id], vb_t);
    // fused status: this item holds all of its candidates (single unit, <= 32
    // targets), so the band (solvers.hpp:499-511: the status's best bound-passing
    // value minus band) and the output happen here, as k_write would do them
    const double thresh = dsub(__longlong_as_double(static_cast<long long>(vb_t)), band);
    const bool keep = fused && ti < L && cand.ok && cand.v >= thresh;
    const unsigned imask = W == 32 ? 0xffffffffu : (((1u << W) - 1u) << hb);
    const unsigned ball = __ballot_sync(0xffffffffu, keep);  // every item of the task
    const unsigned bal = ball & imask;
    const int total = __popc(bal);
    const int nxt = (s + 1) & 1;
    // one claim of F_{s+1} states and groups for the whole task (its 1, 2 or 4
    // items): every lane derives each item's share from the ballot, lane 0
    // issues the one atomic on the step's allocation cursor
    int ngroups = 0, pre_groups = 0;
#pragma unroll
    for (int k = 0; k < 32 / W; ++k) {
      const int ne = ((ball >> (k * W)) & (W == 32 ? 0xffffffffu : ((1u << W) - 1u))) != 0u ? 1 : 0;
      ngroups += ne;
      pre_groups += k < lane / W ? ne : 0;
    }
    const int sum = __popc(ball);
    unsigned long long o = 0ull;
    int fits = 0;
    if (lane == 0 && sum > 0) {
      o = atomicAdd(&sc.out_pack, (static_cast<unsigned long long>(ngroups) << 32) | static_cast<unsigned>(sum));
      fits = claim_fits(a, s, static_cast<int>(o & 0xffffffffull), sum, static_cast<int>(o >> 32) + ngroups - 1) ? 1 : 0;
    }
    fits = __shfl_sync(0xffffffffu, fits, 0);
    o = __shfl_sync(0xffffffffu, o, 0);
    if (!fits || total == 0) return;  // per item (no warp-wide collective follows)
    const int q0 = static_cast<int>(o & 0xffffffffull) + __popc(ball & ((1u << hb) - 1u));
    const int gi = static_cast<int>(o >> 32) + pre_groups;
    const uint32_t key = a.hash[ns_id] - 1u;
    if (sl == 0) {
      const FrontierV2& N = a.f[nxt];
      N.g_start[gi] = q0;
      N.g_size[gi] = total;
      N.g_status[gi] = key;
      N.g_alive[gi] = total;
    }
    if (keep)
      write_state_w(a, s, nxt, q0 + __popc(bal & ((1u << lane) - 1u)), gi, key, cand_p, cand.lex, cand.v, cand.parent,
                    cand_ids, cand_pcv);
  }
}

template <int M>
__device__ void phase_trans_small(const V2& a, int s) {
  const StepCounters& sc = a.ctl->sc[s & 1];
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int nis = sc.items_s, nih = sc.items_h, niq = sc.items_q;
  const int nth = (nih + 1) / 2, ntq = (niq + 3) / 4;
  const int ntask = nis + nth + ntq;
  // the item's group (<= kSmall states) staged once per warp in shared memory:
  // every lane then scans it from there instead of re-reading global memory
  __shared__ uint32_t sh_ids[kWarps][kSmall], sh_rank[kWarps][kSmall];
  __shared__ double sh_val[kWarps][kSmall];
  const int warp = threadIdx.x >> 5;
  const double band = *a.band;
  for (int task = wid; task < ntask; task += nw) {
    if (task < nis) small_task<M, 32>(a, s, task, nullptr, 0, band, sh_ids[warp], sh_rank[warp], sh_val[warp]);
    else if (task < nis + nth)
      small_task<M, 16>(a, s, task - nis, a.it_h_unit, nih, band, sh_ids[warp], sh_rank[warp], sh_val[warp]);
    else
      small_task<M, 8>(a, s, task - nis - nth, a.it_q_unit, niq, band, sh_ids[warp], sh_rank[warp], sh_val[warp]);
  }
}

// ---------------------------------------------------------------------------
// S6: merge + band + output
// One survivor into F_{s+1} (state q of group gidx), from its candidate's
// already-loaded fields. The two dependent lookups (placement ids, bucket
// atomic) are issued before the first store.
__device__ __forceinline__ void write_state_v(const V2& a, int s, int nxt, int q, int gidx, uint32_t key, int p,
                                              uint64_t lx, double v, int parent) {
  const FrontierV2& N = a.f[nxt];
  const long long h = a.hist_base[s + 1] + q;
  const uint32_t ids = a.ids32[p];
  // dominance buckets of more than 64 states are skipped (solvers.hpp:521), and a
  // bucket count only grows within the step: once a (possibly stale) read shows
  // more than 64, the bucket is dead and its atomic can be skipped
  const int slot = a.dominance_ok && a.pcnt[p] <= 64 ? atomicAdd(&a.pcnt[p], 1) : 64;
  // R1 (rank branch) folded in: children per parent rank of F_s, for the dense
  // ranks of F_{s+1}. Every stored state is counted (live or dominated: the
  // ranks are over stored states); F_S is never ranked. The returned count is
  // the state's slot among its siblings (k_kid_fill needs no atomic); it is
  // issued beside the bucket atomic, so it adds no round trip.
  const int kpos = s + 1 < a.S ? atomicAdd(&a.kid_cnt[nxt][static_cast<uint32_t>(lx >> 32)], 1) : 0;
  N.status[q] = key;
  N.ids[q] = ids;
  N.pid[q] = p;
  N.value[q] = v;
  N.lex[q] = lx;
  N.alive[q] = 1;
  N.group[q] = gidx;
  N.kpos[q] = kpos;
  a.h_parent[h] = parent;
  a.h_oi[h] = static_cast<int32_t>(lx & 0xffffffffu);
  if (slot < 64) a.pbucket[p * 64 + slot] = q;
}

// the same with the placement ids and a (possibly stale, see above) bucket
// count already loaded by the caller, one chunk ahead
__device__ __forceinline__ void write_state_w(const V2& a, int s, int nxt, int q, int gidx, uint32_t key, int p,
                                              uint64_t lx, double v, int parent, uint32_t ids, int pcv) {
  const FrontierV2& N = a.f[nxt];
  const long long h = a.hist_base[s + 1] + q;
  const int slot = a.dominance_ok && pcv <= 64 ? atomicAdd(&a.pcnt[p], 1) : 64;
  const int kpos = s + 1 < a.S ? atomicAdd(&a.kid_cnt[nxt][static_cast<uint32_t>(lx >> 32)], 1) : 0;
  N.status[q] = key;
  N.ids[q] = ids;
  N.pid[q] = p;
  N.value[q] = v;
  N.lex[q] = lx;
  N.alive[q] = 1;
  N.group[q] = gidx;
  N.kpos[q] = kpos;
  a.h_parent[h] = parent;
  a.h_oi[h] = static_cast<int32_t>(lx & 0xffffffffu);
  if (slot < 64) a.pbucket[p * 64 + slot] = q;
}

__device__ __forceinline__ void write_state(const V2& a, int s, int nxt, int q, int gidx, uint32_t key, int k) {
  // every load is issued before the first store: the compiler cannot move
  // loads across stores it cannot prove disjoint
  const int p = a.c_pid[k];
  const uint64_t lx = a.c_lex[k];
  const double v = a.c_value[k];
  const int parent = a.c_parent[k];
  write_state_v(a, s, nxt, q, gidx, key, p, lx, v, parent);
}

// S6a: equal-key merge (multi-unit statuses) + band + survivor count per status
__device__ void phase_band(const V2& a, int s, unsigned long long* mvb, unsigned long long* mlx) {
  StepCounters& sc = a.ctl->sc[s & 1];
  __shared__ int s_cnt;
  const int lane = threadIdx.x & 31;
  // The band's reference value (solvers.hpp:499-511) is the best value among
  // the merged survivors, which is the best bound-passing candidate of the
  // status (the merge keeps each placement's maximum): the transition kernels
  // already reduced it into ns_vmax, so merge, band and count are one sweep.
  // big statuses (multi-unit or large): one CTA each
  const int nbig = sc.n_big;
  for (int w = blockIdx.x; w < nbig; w += gridDim.x) {
    const int id = a.ns_big[w];
    const int cb = a.ns_cbase[id], cc = a.ns_ccnt[id], uc = a.ns_ucnt[id];
    const double thresh = dsub(__longlong_as_double(static_cast<long long>(a.ns_vmax[id])), *a.band);
    if (threadIdx.x == 0) s_cnt = 0;
    int mine = 0;
    if (uc == 1) {
      // software-pipelined: the next candidate's loads before this one's store
      int k = cb + threadIdx.x;
      uint8_t ok = k < cb + cc ? a.c_ok[k] : 0;  // both loads issued together (no load behind a branch)
      double v = k < cb + cc ? a.c_value[k] : 0.0;
      for (; k < cb + cc; k += kThreads) {
        const int kn = k + kThreads;
        const uint8_t ok_n = kn < cb + cc ? a.c_ok[kn] : 0;
        const double v_n = kn < cb + cc ? a.c_value[kn] : 0.0;
        const bool keep = ok && v >= thresh;
        a.c_live[k] = keep ? 1 : 0;
        mine += keep;
        ok = ok_n;
        v = v_n;
      }
    } else {  // equal-key merge (solvers.hpp:467-468): max value, then min lex, per placement
      // flat over the status's candidate range (every unit's records are in it,
      // each with its own placement id): the CTA's threads stride the whole
      // range in each pass, no per-unit loop
      const int P1 = a.sp.P1;
      const int win = a.merge_win;
      __syncthreads();  // the previous status is done with the merge table
      for (int w0 = 0; w0 < P1; w0 += win) {
        for (int i = threadIdx.x; i < win; i += kThreads) {
          mvb[i] = 0ull;
          mlx[i] = ~0ull;
        }
        __syncthreads();
        for (int pass = 0; pass < 3; ++pass) {
          // software-pipelined: the next candidate's loads are issued before
          // this one's shared-memory atomics / stores
          int k = cb + threadIdx.x;
          int p = 0;
          bool ok = false;
          double v = 0.0;
          unsigned long long lx = 0;
          if (k < cb + cc) {
            p = a.c_pid[k];
            ok = a.c_ok[k];
            v = a.c_value[k];
            if (pass > 0) lx = a.c_lex[k];
          }
          for (; k < cb + cc; k += kThreads) {
            const int kn = k + kThreads;
            int p_n = 0;
            bool ok_n = false;
            double v_n = 0.0;
            unsigned long long lx_n = 0;
            if (kn < cb + cc) {
              p_n = a.c_pid[kn];
              ok_n = a.c_ok[kn];
              v_n = a.c_value[kn];
              if (pass > 0) lx_n = a.c_lex[kn];
            }
            const bool inw = p >= w0 && p < w0 + win;
            if (!ok) {
              if (pass == 2 && w0 == 0) a.c_live[k] = 0;
            } else if (inw) {
              const unsigned long long vb = vbits(v);
              if (pass == 0) {
                atomicMax(&mvb[p - w0], vb);
              } else if (pass == 1) {
                if (mvb[p - w0] == vb) atomicMin(&mlx[p - w0], lx);
              } else {
                const bool keep = mvb[p - w0] == vb && mlx[p - w0] == lx && v >= thresh;
                a.c_live[k] = keep ? 1 : 0;
                mine += keep;
              }
            }
            p = p_n;
            ok = ok_n;
            v = v_n;
            lx = lx_n;
          }
          __syncthreads();
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) mine += __shfl_down_sync(0xffffffffu, mine, o);
    __syncthreads();
    if (lane == 0 && mine) atomicAdd(&s_cnt, mine);
    __syncthreads();
    if (threadIdx.x == 0) a.ns_out[id] = s_cnt;
  }
  // small statuses: band fused into phase_write
}

// S6c: survivors of every status written at their scanned offsets
// Survivors of every status go to F_{s+1} at positions claimed with one
// atomic per status (big statuses) or per CTA batch of small statuses; the
// frontier's storage order is therefore arbitrary, which nothing depends on
// (every comparison uses values and lex ranks, never storage indices).
__device__ __forceinline__ bool claim_fits(const V2& a, int s, int q0, int total, int gi) {
  if (q0 + total > a.fcap) {
    raise_err(a, 0, kOverflow, s, 0, 4, q0 + total);
    return false;
  }
  if (gi >= a.gcap) {
    raise_err(a, 0, kOverflow, s, 0, 5, gi + 1);
    return false;
  }
  if (a.hist_base[s + 1] + q0 + total > a.hcap) {
    raise_err(a, 0, kOverflow, s, 0, 6, a.hist_base[s + 1] + q0 + total);
    return false;
  }
  return true;
}

__device__ void phase_write(const V2& a, int s) {
  const int nxt = (s + 1) & 1;
  StepCounters& sc = a.ctl->sc[s & 1];
  const FrontierV2& N = a.f[nxt];
  const int lane = threadIdx.x & 31;
  __shared__ int s_q0, s_gi, s_ok, s_run;
  // big statuses: a CTA each; warps compact coalesced 32-candidate chunks
  // into the status's range through a shared cursor (order within a group is
  // irrelevant)
  const int nbig = sc.n_big;
  for (int w = blockIdx.x; w < nbig; w += gridDim.x) {
    const int id = a.ns_big[w];
    const int total = a.ns_out[id];
    if (total == 0) continue;  // uniform
    const int cb = a.ns_cbase[id], cc = a.ns_ccnt[id];
    const uint32_t key = a.hash[id] - 1u;
    if (threadIdx.x == 0) {
      claim_out(sc, total, &s_q0, &s_gi);
      s_ok = claim_fits(a, s, s_q0, total, s_gi) ? 1 : 0;
      s_run = 0;
      if (a.dbg) {
        atomicMax(reinterpret_cast<unsigned long long*>(a.dbg + kDbg * (s + 1 < a.S ? s + 1 : s) + 8),
                  static_cast<unsigned long long>(total));
        if (total > kSmall) atomicAdd(reinterpret_cast<unsigned long long*>(a.dbg + kDbg * (s + 1 < a.S ? s + 1 : s) + 9), 1ull);
      }
    }
    __syncthreads();
    const int q0 = s_q0, gi = s_gi;
    if (s_ok) {
      if (threadIdx.x == 0) {
        N.g_start[gi] = q0;
        N.g_size[gi] = total;
        N.g_status[gi] = key;
        N.g_alive[gi] = total;
      }
      // software-pipelined: the warp's next chunk is loaded before this
      // chunk's states are written
      int k = cb + (threadIdx.x & ~31) + lane;
      bool in = k < cb + cc;
      bool lv = in && a.c_live[k];
      double v = in ? a.c_value[k] : 0.0;
      int p = in ? a.c_pid[k] : 0;
      uint64_t lx = in ? a.c_lex[k] : 0ull;
      int par = in ? a.c_parent[k] : 0;
      uint32_t ids = in ? a.ids32[p] : 0u;
      int pcv = in ? a.pcnt[p] : 0;
      int p_n = k + kThreads < cb + cc ? a.c_pid[k + kThreads] : 0;
      for (int k0 = cb + (threadIdx.x & ~31); k0 < cb + cc; k0 += kThreads) {
        // two deep, as the small-status loop below
        const int kn = k + kThreads, k2 = k + 2 * kThreads;
        const bool in_n = kn < cb + cc;
        const bool lv_n = in_n && a.c_live[kn];
        const double v_n = in_n ? a.c_value[kn] : 0.0;
        const uint64_t lx_n = in_n ? a.c_lex[kn] : 0ull;
        const int par_n = in_n ? a.c_parent[kn] : 0;
        const uint32_t ids_n = in_n ? a.ids32[p_n] : 0u;
        const int pcv_n = in_n ? a.pcnt[p_n] : 0;
        const int p_2 = k2 < cb + cc ? a.c_pid[k2] : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, lv);
        if (bal != 0) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&s_run, __popc(bal));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (lv)
            write_state_w(a, s, nxt, q0 + base + __popc(bal & ((1u << lane) - 1u)), gi, key, p, lx, v, par, ids, pcv);
        }
        k = kn;
        lv = lv_n;
        v = v_n;
        p = p_n;
        lx = lx_n;
        par = par_n;
        ids = ids_n;
        pcv = pcv_n;
        p_n = p_2;
      }
    }
    __syncthreads();
  }
  // small statuses (single unit, <= kBigNs candidates, so no merge): a warp
  // each applies the band, claims its range with one atomic and writes. The
  // next status's metadata is loaded while this one is processed, and a
  // status of at most 32 candidates is done in one pass with every candidate
  // field loaded up front.
  const int nsm = sc.n_small;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const double band = *a.band;
  int id = 0, cb = 0, cc = 0;
  unsigned long long vm = 0;
  uint32_t hk = 0;
  if (wid < nsm) {
    id = a.ns_small[wid];
    cb = a.ns_cbase[id];
    cc = a.ns_ccnt[id];
    vm = a.ns_vmax[id];
    hk = a.hash[id];
  }
  for (int i = wid; i < nsm; i += nw) {
    const int in = i + nw;
    int id_n = 0;
    if (in < nsm) id_n = a.ns_small[in];
    const double thresh = dsub(__longlong_as_double(static_cast<long long>(vm)), band);
    const uint32_t key = hk - 1u;
    if (a.dbg && lane == 0) {  // [10] small statuses <= 32 candidates, [11] their candidates, [12] other small, [13] their candidates
      unsigned long long* d = reinterpret_cast<unsigned long long*>(a.dbg + kDbg * s);
      atomicAdd(d + (cc <= 32 ? 10 : 12), 1ull);
      atomicAdd(d + (cc <= 32 ? 11 : 13), static_cast<unsigned long long>(cc));
    }
    if (cc <= 32) {
      const int k = cb + lane;
      const bool in_range = lane < cc;
      const bool ok = in_range && a.c_ok[k];
      const double v = in_range ? a.c_value[k] : 0.0;
      const int p = in_range ? a.c_pid[k] : 0;
      const uint64_t lx = in_range ? a.c_lex[k] : 0ull;
      const int parent = in_range ? a.c_parent[k] : 0;
      const bool keep = ok && v >= thresh;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      const int total = __popc(bal);
      if (total > 0) {  // uniform
        int q0 = 0, gi = 0, fits = 0;
        if (lane == 0) {
          claim_out(sc, total, &q0, &gi);
          fits = claim_fits(a, s, q0, total, gi) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, fits, 0)) {
          q0 = __shfl_sync(0xffffffffu, q0, 0);
          gi = __shfl_sync(0xffffffffu, gi, 0);
          if (lane == 0) {
            N.g_start[gi] = q0;
            N.g_size[gi] = total;
            N.g_status[gi] = key;
            N.g_alive[gi] = total;
          }
          if (keep) write_state_v(a, s, nxt, q0 + __popc(bal & ((1u << lane) - 1u)), gi, key, p, lx, v, parent);
        }
      }
    } else {
      int total = 0;
      for (int k0 = cb; k0 < cb + cc; k0 += 64) {  // two chunks' loads in flight, none behind a branch
        const int k1 = k0 + lane, k2 = k1 + 32;
        const bool in1 = k1 < cb + cc, in2 = k2 < cb + cc;
        const uint8_t o1 = in1 ? a.c_ok[k1] : 0, o2 = in2 ? a.c_ok[k2] : 0;
        const double v1 = in1 ? a.c_value[k1] : 0.0, v2 = in2 ? a.c_value[k2] : 0.0;
        total += __popc(__ballot_sync(0xffffffffu, o1 && v1 >= thresh)) +
                 __popc(__ballot_sync(0xffffffffu, o2 && v2 >= thresh));
      }
      if (total > 0) {  // uniform
        int q0 = 0, gi = 0, fits = 0;
        if (lane == 0) {
          claim_out(sc, total, &q0, &gi);
          fits = claim_fits(a, s, q0, total, gi) ? 1 : 0;
        }
        if (__shfl_sync(0xffffffffu, fits, 0)) {
          q0 = __shfl_sync(0xffffffffu, q0, 0);
          gi = __shfl_sync(0xffffffffu, gi, 0);
          if (lane == 0) {
            N.g_start[gi] = q0;
            N.g_size[gi] = total;
            N.g_status[gi] = key;
            N.g_alive[gi] = total;
          }
          // software-pipelined: the next chunk's candidate fields are loaded
          // before this chunk's states are written
          int run = 0;
          int k = cb + lane;
          bool in = k < cb + cc;
          uint8_t ok = in ? a.c_ok[k] : 0;
          double v = in ? a.c_value[k] : 0.0;
          int p = in ? a.c_pid[k] : 0;
          uint64_t lx = in ? a.c_lex[k] : 0ull;
          int par = in ? a.c_parent[k] : 0;
          uint32_t ids = in ? a.ids32[p] : 0u;
          int pcv = in ? a.pcnt[p] : 0;
          int p_n = k + 32 < cb + cc ? a.c_pid[k + 32] : 0;
          for (int k0 = cb; k0 < cb + cc; k0 += 32) {
            // two deep: the next chunk's fields and placement lookups, the
            // placement of the one after, all before this chunk's writes
            const int kn = k + 32, k2 = k + 64;
            const bool in_n = kn < cb + cc;
            const uint8_t ok_n = in_n ? a.c_ok[kn] : 0;
            const double v_n = in_n ? a.c_value[kn] : 0.0;
            const uint64_t lx_n = in_n ? a.c_lex[kn] : 0ull;
            const int par_n = in_n ? a.c_parent[kn] : 0;
            const uint32_t ids_n = in_n ? a.ids32[p_n] : 0u;
            const int pcv_n = in_n ? a.pcnt[p_n] : 0;
            const int p_2 = k2 < cb + cc ? a.c_pid[k2] : 0;
            const bool keep = ok && v >= thresh;
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (keep)
              write_state_w(a, s, nxt, q0 + run + __popc(bal & ((1u << lane) - 1u)), gi, key, p, lx, v, par, ids, pcv);
            run += __popc(bal);
            k = kn;
            ok = ok_n;
            v = v_n;
            p = p_n;
            lx = lx_n;
            par = par_n;
            ids = ids_n;
            pcv = pcv_n;
            p_n = p_2;
          }
        }
      }
    }
    if (in < nsm) {  // the next status's metadata (its id was loaded at the top)
      id = id_n;
      cb = a.ns_cbase[id];
      cc = a.ns_ccnt[id];
      vm = a.ns_vmax[id];
      hk = a.hash[id];
    }
  }
}

// encoded-status form of status_dominates (solvers.hpp:128-134): a tenant's
// status is (hi << 16 | lo) with idle = (0, 0), done = (0xffff, 0) and running =
// (0x200 | size, remaining steps). x dominates y iff x == y, or x is done, or
// both run the same size with x's remaining steps <= y's -- i.e. hi equal (or
// x done) and lo(x) <= lo(y): done-vs-done, idle-vs-idle and equal running
// codes pass; done y only by done x; idle and running never cross.
__device__ __forceinline__ bool dom_decoded(uint32_t x, uint32_t y) {
  const uint32_t hx = x >> 16;
  return (hx == (y >> 16) || hx == 0xffffu) && (x & 0xffffu) <= (y & 0xffffu);
}

// one state of a dominance bucket: per tenant the encoded status (dom_decoded);
// value; lex key
template <int MK>
struct DomRec {
  uint32_t d[MK];
  unsigned long long vb;  // value bits: values are >= 0, so the bits order like the values
  uint64_t lx;
};

// dp_better on value bits (integer compares, no FP64 pipe): values are >= 0
__device__ __forceinline__ bool better_bits(unsigned long long va, uint64_t la, unsigned long long vb, uint64_t lb) {
  return va > vb || (va == vb && la < lb);
}

// x dominates y on every tenant (branch-free form of dom_decoded over MK fields)
template <int MK>
__device__ __forceinline__ bool dom_all(const uint32_t (&x)[MK], const uint32_t (&y)[MK]) {
  bool ok = true;
#pragma unroll
  for (int m = 0; m < MK; ++m) ok &= dom_decoded(x[m], y[m]);
  return ok;
}

// S7: status dominance within placement buckets (solvers.hpp:514-537).
// MK = 2 (M <= 2, 16-bit fields) or 4 (M = 3..4, 8-bit fields). One warp per
// bucket of 2..64 states: the bucket's decoded records are staged in the warp's
// shared-memory slice, then every lane tests its one or two states against each
// record in turn (broadcast loads; the second half only for buckets above 32).
template <int MK>
__device__ void phase_dominance(const V2& a, int s) {
  __shared__ DomRec<MK> s_rec[kThreads / 32][64];
  const int nxt = (s + 1) & 1;
  const FrontierV2& N = a.f[nxt];
  const Codec codec{a.t.S, a.codec_shift};
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  DomRec<MK>* R = s_rec[threadIdx.x >> 5];
  const int MT = a.t.M;
  for (int p = wid; p < a.sp.P1; p += nw) {
    const int n = a.pcnt[p];
    if (n >= 2 && n <= 64) {
      const int* bk = a.pbucket + p * 64;
      int q[2];
      DomRec<MK> me[2];
      for (int h = 0; h < 2; ++h) {
        const int j = lane + 32 * h;
        q[h] = j < n ? bk[j] : -1;
        const uint32_t st = q[h] >= 0 ? N.status[q[h]] : 0;
        me[h].vb = q[h] >= 0 ? vbits(N.value[q[h]]) : 0ull;
        me[h].lx = q[h] >= 0 ? N.lex[q[h]] : 0;
#pragma unroll
        for (int m = 0; m < MK; ++m) {  // decode once
          const int code = m < MT ? fldm<MK>(st, m) : 0;
          me[h].d[m] = code == Codec::done() ? 0xffff0000u
                       : Codec::is_running(code) ? ((0x200u | static_cast<uint32_t>(codec.run_size(code))) << 16) |
                                                       static_cast<uint32_t>(codec.run_rem(code))
                                                 : 0u;
        }
        if (q[h] >= 0) R[j] = me[h];
      }
      __syncwarp();
      bool dead[2] = {false, false};
      if (n <= 32) {
#pragma unroll 2
        for (int j = 0; j < n; ++j) {
          const DomRec<MK> r = R[j];
          dead[0] |= (j != lane) & dom_all<MK>(r.d, me[0].d) & better_bits(r.vb, r.lx, me[0].vb, me[0].lx);
        }
      } else {
#pragma unroll 1
        for (int j = 0; j < n; ++j) {
          const DomRec<MK> r = R[j];
          dead[0] |= (j != lane) & dom_all<MK>(r.d, me[0].d) & better_bits(r.vb, r.lx, me[0].vb, me[0].lx);
          dead[1] |= (j != lane + 32) & dom_all<MK>(r.d, me[1].d) & better_bits(r.vb, r.lx, me[1].vb, me[1].lx);
        }
      }
      __syncwarp();  // R is rewritten by the warp's next bucket
      int kills = 0;
      for (int h = 0; h < 2; ++h)
        if (q[h] >= 0 && dead[h]) {
          N.alive[q[h]] = 0;
          atomicSub(&N.g_alive[N.group[q[h]]], 1);
          ++kills;
        }
      for (int o = 16; o > 0; o >>= 1) kills += __shfl_xor_sync(0xffffffffu, kills, o);
      if (lane == 0 && kills && s + 1 < a.S) {  // F_S: k_term1 counts
        atomicSub(&a.ctl->alive_now[nxt], kills);
        atomicAdd(&a.ctl->dead[nxt], kills);
      }
    }
    if (lane == 0) a.pcnt[p] = 0;
  }
}

// ---------------------------------------------------------------------------
// Phase kernels: one launch per phase and slot, stream-ordered, all counts on
// the device (the host never waits inside a window).
template <int M>
__global__ void MGS_LB k_units(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  __shared__ int s_cnt[kBatch];
  __shared__ long long s_red[32];
  if (block_failed(a)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // frontier checks for F_s (solvers.hpp:348, :539-542): k_dom of the previous
    // step (the last writer of F_s) has finished, so the live count is final
    Ctl* ctl = a.ctl;
    const int cur = s & 1;
    const int alive_cur = ctl->n_store[cur] - ctl->dead[cur];
    if (alive_cur == 0) raise_err(a, 0, MGS_ERR_INFEASIBLE_JOINT, s);
    else if (s > 0 && static_cast<uint64_t>(alive_cur) > a.budget) raise_err(a, 0, MGS_ERR_STATE_BUDGET, s, alive_cur);
    if (s > 0) {
      ctl->ftot += alive_cur;
      if (static_cast<unsigned long long>(alive_cur) > ctl->fpeak) ctl->fpeak = alive_cur;
    }
    ctl->ranks_prev[(s + 1) & 1] = ctl->n_store[cur];  // parent-rank space of F_{s+1}: stored F_s
  }
  // thread per group once a CTA has enough groups to fill its threads (lane
  // batches: 20.7 vs 22.1 ms per C1 window at 16 lanes); a warp per group
  // otherwise (one C1 window: 28 groups per CTA at the peak step, where the
  // thread path leaves most threads idle and serialises the size combinations)
  const int G = a.ctl->n_groups[s & 1];
  if (M <= 2 && static_cast<long long>(G) >= static_cast<long long>(a.units_tmin) * gridDim.x)
    phase_units_thread<M>(a, s, 0, s_cnt, s_red);
  else if (M <= 2)
    phase_units<M, MGS_UNITS_W>(a, s, 0, s_cnt, s_red);  // few combinations per group: sub-warps
  else
    phase_units<M, 32>(a, s, 0, s_cnt, s_red);
}

// K independent warp-aggregated reservations at once: the K scans, then the K
// atomics issued together, then the K broadcasts (one atomic round trip)
template <int K>
__device__ __forceinline__ void warp_alloc_n(int* const (&cursor)[K], const int (&n)[K], int (&first)[K]) {
  const int lane = threadIdx.x & 31;
  int x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = n[k];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int y = __shfl_up_sync(0xffffffffu, x[k], o);
      if (lane >= o) x[k] += y;
    }
  }
  int base[K];
#pragma unroll
  for (int k = 0; k < K; ++k) base[k] = lane == 31 ? atomicAdd(cursor[k], x[k]) : 0;
#pragma unroll
  for (int k = 0; k < K; ++k) first[k] = __shfl_sync(0xffffffffu, base[k], 31) + x[k] - n[k];
}


// S2: ranges for the step's successor statuses (candidates, units, big/small
// status lists) and units (work items), reserved with warp-aggregated
// atomics -- their order is arbitrary and nothing depends on it -- and the
// lists written straight away: the status lists here, the work-item lists
// here (bounded by their capacity; the consumers check the totals at entry),
// each unit's candidate range and list slot by the transition kernels (from
// its offsets within the status, taken by k_units).
__global__ void __launch_bounds__(kThreads) k_scans(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  const int cur = s & 1;
  Ctl* ctl = a.ctl;
  StepCounters& sc = ctl->sc[s & 1];
  const int lane = threadIdx.x & 31;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const int n_ns = sc.n_ns;
  for (int k0 = gtid - lane; k0 < n_ns; k0 += gstride) {  // warp-uniform trip count
    const int k = k0 + lane;
    const bool valid = k < n_ns;
    const int id = valid ? a.ns_used[k] : 0;
    const int cc = valid ? a.ns_ccnt[id] : 0, uc = valid ? a.ns_ucnt[id] : 0;
    const int fflag = valid ? a.ns_fflag[id] : 0;
    const bool fused = valid && uc == 1 && fflag == 1;
    const bool big = valid && !fused && (uc > 1 || cc > kBigNs);
    int* const cur4[4] = {&sc.T, &sc.u_cursor, &sc.n_big, &sc.n_small};
    const int n4[4] = {cc, uc, big ? 1 : 0, valid && !big && !fused ? 1 : 0};
    int f4[4];
    warp_alloc_n<4>(cur4, n4, f4);
    const int cb = f4[0], ub = f4[1], bp = f4[2], sp = f4[3];
    if (valid) {
      a.ns_cbase[id] = cb;
      a.ns_ubase[id] = ub;
      if (big) a.ns_big[bp] = id;
      else if (!fused) a.ns_small[sp] = id;  // fused: finished by its k_trans_small item
    }
  }
  const int nu = sc.n_units;
  for (int u0 = gtid - lane; u0 < nu; u0 += gstride) {
    const int u = u0 + lane;
    const bool valid = u < nu;
    const int chs = valid ? a.u_chs[u] : 0, nbg = valid ? a.u_chb[u] : 0;
    const int nsm = chs > 0 ? chs : 0, nh = chs == -1 ? 1 : 0, nq = chs == -2 ? 1 : 0;
    int* const cur4[4] = {&sc.items_s, &sc.items_b, &sc.items_h, &sc.items_q};
    const int n4[4] = {nsm, nbg, nh, nq};
    int f4[4];
    warp_alloc_n<4>(cur4, n4, f4);
    const int sb = f4[0], bb = f4[1], hb = f4[2], qb = f4[3];
    if (nh && hb < a.itcap) a.it_h_unit[hb] = u;
    if (nq && qb < a.itcap) a.it_q_unit[qb] = u;
    if (sb + nsm <= a.itcap)
      for (int c = 0; c < nsm; ++c) {
        a.it_s_unit[sb + c] = u;
        a.it_s_chunk[sb + c] = c;
      }
    if (bb + nbg <= a.itcap)
      for (int c = 0; c < nbg; ++c) {
        a.it_b_unit[bb + c] = u;
        a.it_b_chunk[bb + c] = c;
      }
  }
}

// the step's candidate range and work-item lists fit their buffers (the totals
// are final once k_scans is done); read by every block of the consumers, so
// their early exit is block-uniform
__device__ __forceinline__ bool lists_fit(const V2& a, int s) {
  const StepCounters& sc = a.ctl->sc[s & 1];
  return sc.T <= a.ccap && sc.items_s <= a.itcap && sc.items_b <= a.itcap && sc.items_h <= a.itcap &&
         sc.items_q <= a.itcap;
}

// R2 (rank branch): frontier checks for F_s and the children offsets in
// parent-rank order (the one order-bearing scan: the dense lex ranks)
__global__ void __launch_bounds__(kThreads) k_kid_scan(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  const int cur = s & 1;
  Ctl* ctl = a.ctl;
  StepCounters& sc = ctl->sc[s & 1];
  (void)cur;
  const ScanJob jobs[1] = {{a.kid_cnt[cur], nullptr, a.kid_base, ctl->ranks_prev[s & 1], 0}};
  multi_scan<1>(a, jobs, 2 * (s + 1), &sc.ticket, ctl->scan_total);
}

__global__ void __launch_bounds__(kThreads) k_kid_fill(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ctl->sc[s & 1].kids = a.ctl->scan_total[0];
  phase_kid_fill(a, s);
}

__global__ void __launch_bounds__(kThreads, MGS_RB_MINB) k_ranks_big(const V2* __restrict__ ap, int s, int with_small) {
  const V2& a = c_v2;
  extern __shared__ unsigned long long smem_u64[];
  if (block_failed(a)) return;
  phase_ranks_big(a, s, smem_u64);
  if (with_small) phase_ranks_small(a, s);  // independent of the big buckets
}

// small buckets on their own (full occupancy) beside k_ranks_big in the graph
__global__ void __launch_bounds__(kThreads) k_ranks_small(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  phase_ranks_small(a, s);
}

// Depends on F_s's ranks and on k_dom(s-1) (alive flags) only: in the graph it
// runs on the rank branch, beside k_units / k_scans
__global__ void MGS_LB k_tables(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  phase_tables(a, s);
}

template <int M>
__global__ void __launch_bounds__(kThreads, MGS_TB_MINB) k_trans_big(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // overflow of k_scans' lists; transition counters
    Ctl* ctl = a.ctl;
    const StepCounters& sc = ctl->sc[s & 1];
    const int T_ = sc.T;
    ctl->tr += static_cast<unsigned long long>(T_);
    ctl->tbytes += static_cast<unsigned long long>(ctl->n_store[s & 1]) * 20ull + static_cast<unsigned long long>(T_) * 37ull;
    if (T_ > a.ccap) raise_err(a, 0, kOverflow, s, 0, 7, T_);
    if (sc.items_s > a.itcap || sc.items_b > a.itcap || sc.items_h > a.itcap || sc.items_q > a.itcap)
      raise_err(a, 0, kOverflow, s, 0, 8, max(max(sc.items_s, sc.items_b), max(sc.items_h, sc.items_q)));
  }
  if (!lists_fit(a, s)) return;
  if (static_cast<int>(blockIdx.x) >= a.ctl->sc[s & 1].items_b) return;  // no item for this CTA
  phase_trans_big<M>(a, s);
}

template <int M>
__global__ void __launch_bounds__(kThreads, MGS_TS_MINB) k_trans_small(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a) || !lists_fit(a, s)) return;  // k_trans_big raises the overflow
  phase_trans_small<M>(a, s);
  {  // F_s's child counts were last read by the ranks: cleared here, off the critical path
    const int cur = s & 1, rp = a.ctl->ranks_prev[s & 1];
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
    for (int i = gtid; i < rp; i += gstride) {
      a.kid_cnt[cur][i] = 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // counters of the next step
    const int nxt = (s + 1) & 1;
    a.ctl->sc[nxt] = StepCounters{};
    a.ctl->alive_now[nxt] = 0;
    a.ctl->dead[nxt] = 0;
  }
}

__global__ void __launch_bounds__(kThreads) k_band(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  extern __shared__ unsigned long long smem_u64[];
  if (block_failed(a)) return;
  phase_band(a, s, smem_u64, smem_u64 + a.merge_win);
}

__global__ void __launch_bounds__(kThreads, 4) k_write(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  phase_write(a, s);
}

__global__ void __launch_bounds__(kThreads) k_dom(const V2* __restrict__ ap, int s) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  const int cur = s & 1;
  Ctl* ctl = a.ctl;
  if (a.dominance_ok) {
    if (a.t.M <= 2) phase_dominance<2>(a, s);
    else phase_dominance<4>(a, s);
  }
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  const int n_ns = ctl->sc[s & 1].n_ns;
  for (int k = gtid; k < n_ns; k += gstride) {  // S6 read the keys from the hash: clear the claimed slots
    const int i = a.ns_used[k];
    a.hash[i] = 0u;
    a.ns_out[i] = 0;
    a.ns_vmax[i] = 0ull;
    a.ns_ucnt[i] = 0;
    a.ns_ccnt[i] = 0;
    a.ns_fflag[i] = 0;
  }
  if (gtid == 0) {  // end-of-slot bookkeeping (every value read here is final)
    const int nxt = (s + 1) & 1;
    StepCounters& sc = ctl->sc[s & 1];
    ctl->n_store[nxt] = sc.out_states();   // F_{s+1} as allocated by k_write
    if (s + 1 < a.S) atomicAdd(&ctl->alive_now[nxt], sc.out_states());  // k_dom's kills are subtracted beside it
    ctl->n_groups[nxt] = sc.out_groups();
    a.hist_base[s + 2] = a.hist_base[s + 1] + ctl->n_store[nxt];  // array has S+2 entries
    if (a.dbg) {
      long long* d = a.dbg + static_cast<long long>(kDbg) * s;
      d[6] = sc.items_b;
      d[7] = sc.items_s;
      d[0] = sc.n_units;
      d[1] = sc.n_big + sc.n_small;
      d[2] = sc.T;
      d[3] = ctl->n_store[nxt];
      d[4] = ctl->n_groups[nxt];
      d[5] = ctl->alive_now[cur];
    }
  }
}

// terminal (solvers.hpp:552-565): live count of F_S, budget, best all-done state
__device__ __forceinline__ uint32_t all_done_key(const V2& a, int M) {
  uint32_t k = 0;
  for (int m = 0; m < M; ++m) k |= static_cast<uint32_t>(Codec::done()) << (a.fw * m);
  return k;
}

__global__ void __launch_bounds__(kThreads) k_term1(const V2* __restrict__ ap) {
  const V2& a = c_v2;
  __shared__ long long s_red[32];
  if (block_failed(a)) return;
  const int fin = a.S & 1;
  const FrontierV2& F = a.f[fin];
  const int n = a.ctl->n_store[fin];
  const uint32_t all_done = all_done_key(a, a.t.M);
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  long long live = 0;
  unsigned long long mv = 0;
  bool any = false;
  for (int i = gtid; i < n; i += gstride)
    if (F.alive[i]) {
      ++live;
      if (F.status[i] == all_done) {
        const unsigned long long vb = vbits(F.value[i]);
        mv = any && mv > vb ? mv : vb;
        any = true;
      }
    }
  const long long ls = block_sum(live, s_red);
  if (threadIdx.x == 0 && ls) atomicAdd(&a.ctl->alive_now[fin], static_cast<int>(ls));
  if (any) atomicMax(&a.ctl->best_vb, mv + 1);  // +1: 0 = none
}

__global__ void __launch_bounds__(kThreads) k_term2(const V2* __restrict__ ap) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  const int fin = a.S & 1;
  const FrontierV2& F = a.f[fin];
  const int n = a.ctl->n_store[fin];
  const uint32_t all_done = all_done_key(a, a.t.M);
  const int alive_fin = a.ctl->alive_now[fin];
  const unsigned long long bvb = a.ctl->best_vb;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  if (gtid == 0) {
    a.ctl->ftot += alive_fin;
    if (static_cast<unsigned long long>(alive_fin) > a.ctl->fpeak) a.ctl->fpeak = alive_fin;
    if (static_cast<uint64_t>(alive_fin) > a.budget) raise_err(a, 0, MGS_ERR_STATE_BUDGET, a.S, alive_fin);
    else if (bvb == 0) raise_err(a, 0, MGS_ERR_INFEASIBLE_JOINT, a.S);
  }
  if (bvb == 0) return;
  for (int i = gtid; i < n; i += gstride)
    if (F.alive[i] && F.status[i] == all_done && vbits(F.value[i]) + 1 == bvb) atomicMin(&a.ctl->best_lex, F.lex[i]);
}

__global__ void __launch_bounds__(kThreads) k_term3(const V2* __restrict__ ap) {
  const V2& a = c_v2;
  if (block_failed(a)) return;
  const int fin = a.S & 1;
  const FrontierV2& F = a.f[fin];
  const int n = a.ctl->n_store[fin];
  const uint32_t all_done = all_done_key(a, a.t.M);
  const unsigned long long bvb = a.ctl->best_vb, blx = a.ctl->best_lex;
  const int gtid = blockIdx.x * blockDim.x + threadIdx.x, gstride = gridDim.x * blockDim.x;
  for (int i = gtid; i < n; i += gstride)
    if (F.alive[i] && F.status[i] == all_done && vbits(F.value[i]) + 1 == bvb && F.lex[i] == blx) a.ctl->best_idx = i;
}

__global__ void k_backtrack2(const V2* __restrict__ ap) {
  const V2& a = c_v2;  // parent walk (solvers.hpp:567-574)
  if (block_failed(a) || threadIdx.x != 0 || blockIdx.x != 0) return;
  int idx = a.ctl->best_idx;
  for (int s = a.S - 1; s >= 0; --s) {
    const long long h = a.hist_base[s + 1] + idx;
    a.chosen[s] = a.h_oi[h];
    idx = a.h_parent[h];
  }
}

__global__ void k_init_root(const V2* __restrict__ ap) {
  const V2& a = c_v2;
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int root_pid = a.sp.root_pid;
  FrontierV2 F = a.f[0];
  F.status[0] = 0;
  F.ids[0] = a.ids32[root_pid];
  F.pid[0] = root_pid;
  F.value[0] = 0.0;
  F.lex[0] = 0;
  F.alive[0] = 1;
  F.group[0] = 0;
  F.kpos[0] = 0;
  F.rank[0] = 0;
  F.g_start[0] = 0;
  F.g_size[0] = 1;
  F.g_status[0] = 0;
  F.g_alive[0] = 1;
  Ctl* c = a.ctl;
  c->n_store[0] = 1;
  c->n_groups[0] = 1;
  c->best_vb = 0;
  c->best_lex = ~0ull;
  c->best_idx = -1;
  c->ranks_prev[0] = 1;
  c->alive_now[0] = 1;
  a.kid_cnt[0][0] = 1;  // the root's child count under its (rank 0) parent
  a.hist_base[0] = 0;
  a.hist_base[1] = 0;
}

// band (solvers.hpp:258-267): 1e-9 + sum_m loss_m * cap_max_m * acc_max_m,
// cap_max over the options' capabilities = over the placements'. One CTA.
__global__ void k_band_value(const double* pl_cap, int P, HostTables t, double* band) {
  __shared__ double s_max[KM][32];
  double mx[KM] = {0.0, 0.0, 0.0, 0.0};
  for (int q = threadIdx.x; q < P; q += blockDim.x)
    for (int m = 0; m < t.M; ++m) mx[m] = fmax(mx[m], pl_cap[q * KM + m]);
  for (int m = 0; m < KM; ++m) {
    for (int o = 16; o > 0; o >>= 1) mx[m] = fmax(mx[m], __shfl_xor_sync(0xffffffffu, mx[m], o));
    if ((threadIdx.x & 31) == 0) s_max[m][threadIdx.x >> 5] = mx[m];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = 1e-9;
    for (int m = 0; m < t.M; ++m) {
      double cm = 0.0;
      for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) cm = fmax(cm, s_max[m][w]);
      const double acc_max = t.pre[m] > t.post[m] ? t.pre[m] : t.post[m];
      b = dadd(b, dmul(dmul(t.loss[m], cm), acc_max));
    }
    *band = b;
  }
}

// placement ids (16 bits per tenant in pl_ids) repacked fw bits per tenant
__global__ void k_ids32(const uint64_t* pl_ids, int n, int M, int fw, uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t v = 0;
  for (int m = 0; m < M; ++m) v |= static_cast<uint32_t>((pl_ids[i] >> (16 * m)) & 0xffffu) << (fw * m);
  out[i] = v;
}

__global__ void k_sig_len(const int32_t* sig_off, int n_sig, int32_t* sig_len) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_sig; i += gridDim.x * blockDim.x)
    sig_len[i] = sig_off[i + 1] - sig_off[i];
}

struct Caps {
  int fcap, gcap, ucap, itcap, ccap, hbits, tcap;
  long long hcap;
};

}  // namespace

bool solve_dp_v2_supported(const Prepared& pr, const DevSpace& sp) {
  const char* e = std::getenv("MGS_DP_ENGINE");
  if (e && std::string(e) == "v1") return false;
  if (pr.t.M <= 2) return true;
  // M = 3..4 in 8-bit fields: status codes in the reference numbering stay
  // below 255 (2 + 7 * S - 1 < 255), mask ids below 255 (all-ones never matches)
  if (7 * pr.t.S + 1 >= 255) return false;
  for (int m = 0; m < pr.t.M; ++m)
    if (sp.n_mask_ids[m] > 255) return false;
  return true;
}


namespace {

// words of k_ranks_big's option-index bitmap (plus as many prefix counts);
// 0 when the two arrays would not fit in shared memory
int rank_words_of(long long n_opt) {
  const long long w = (n_opt + 31) / 32;
  return w * 8 <= 160 * 1024 ? static_cast<int>(w) : 0;
}

// Device buffers + scalars of one lane for the current capacities.
V2 lane_args(Ctx& c, const V2Lane& L, const Caps& caps, int dominance_ok, int merge_win, int grid_term) {
  const DevSpace& sp = *L.sp;
  const HostTables& t = L.pr->t;
  const int S = t.S;
  const std::string saved_prefix = c.prefix;
  c.prefix = L.prefix;
  V2 a{};
  a.sp = sp;
  a.t = t;
  a.S = S;
  a.has_initial = L.pr->has_initial;
  a.dominance_ok = dominance_ok;
  {
    double* d_band = c.buf<double>("v2_band", 1);
    k_band_value<<<1, 256, 0, c.stream>>>(sp.pl_cap, sp.P, t, d_band);
    ++c.kernel_launches;
    a.band = d_band;
  }
  a.budget = L.p->state_budget;
  a.recv = L.recv;
  a.ub = L.ub;
  a.incumbent = L.incumbent;
  a.fcap = caps.fcap;
  a.gcap = caps.gcap;
  for (int b = 0; b < 2; ++b) {
    std::string tg = b ? "v2b_" : "v2a_";
    FrontierV2& f = a.f[b];
    f.status = c.buf<uint32_t>((tg + "status").c_str(), caps.fcap);
    f.ids = c.buf<uint32_t>((tg + "ids").c_str(), caps.fcap);
    f.pid = c.buf<int32_t>((tg + "pid").c_str(), caps.fcap);
    f.value = c.buf<double>((tg + "value").c_str(), caps.fcap);
    f.lex = c.buf<uint64_t>((tg + "lex").c_str(), caps.fcap);
    f.rank = c.buf<uint32_t>((tg + "rank").c_str(), caps.fcap);
    f.alive = c.buf<uint8_t>((tg + "alive").c_str(), caps.fcap);
    f.group = c.buf<int32_t>((tg + "group").c_str(), caps.fcap);
    f.kpos = c.buf<int32_t>((tg + "kpos").c_str(), caps.fcap);
    f.g_start = c.buf<int32_t>((tg + "gstart").c_str(), caps.gcap);
    f.g_size = c.buf<int32_t>((tg + "gsize").c_str(), caps.gcap);
    f.g_status = c.buf<uint32_t>((tg + "gstatus").c_str(), caps.gcap);
    f.g_alive = c.buf<int32_t>((tg + "galive").c_str(), caps.gcap);
    a.kid_cnt[b] = c.buf<int32_t>((tg + "kidcnt").c_str(), caps.fcap);
    MGS_CUDA_OK(cudaMemsetAsync(a.kid_cnt[b], 0, static_cast<size_t>(caps.fcap) * 4, c.stream));
  }
  a.kid_base = c.buf<int32_t>("v2_kidbase", caps.fcap + 1);
  a.kid_items = c.buf<uint64_t>("v2_kiditems", caps.fcap);
  a.kid_pr = c.buf<int32_t>("v2_kidpr", caps.fcap);
  a.big_bucket = c.buf<int32_t>("v2_bigbucket", caps.fcap);
  a.hcap = caps.hcap;
  a.h_parent = c.buf<int32_t>("v2_hparent", caps.hcap);
  a.h_oi = c.buf<int32_t>("v2_hoi", caps.hcap);
  a.hist_base = c.buf<long long>("v2_histbase", S + 2);
  a.ucap = caps.ucap;
  a.u_group = c.buf<int32_t>("v2_ugroup", caps.ucap);
  a.u_sig = c.buf<int32_t>("v2_usig", caps.ucap);
  a.u_ns = c.buf<int32_t>("v2_uns", caps.ucap);
  a.u_chs = c.buf<int32_t>("v2_uchs", caps.ucap);
  a.u_chb = c.buf<int32_t>("v2_uchb", caps.ucap);
  a.u_cbase = c.buf<int32_t>("v2_ucbase", caps.ucap);
  a.u_upos = c.buf<int32_t>("v2_uupos", caps.ucap);
  a.ns_units = c.buf<int32_t>("v2_nsunits", caps.ucap);
  a.hmask = (1 << caps.hbits) - 1;
  const size_t H = static_cast<size_t>(a.hmask) + 1;
  a.hash = c.buf<uint32_t>("v2_hash", H);
  a.ns_ucnt = c.buf<int32_t>("v2_nsucnt", H);
  a.ns_ccnt = c.buf<int32_t>("v2_nsccnt", H);
  a.ns_ubase = c.buf<int32_t>("v2_nsubase", H);
  a.ns_cbase = c.buf<int32_t>("v2_nscbase", H);
  a.ns_out = c.buf<int32_t>("v2_nsout", H);
  a.ns_vmax = c.buf<unsigned long long>("v2_nsvmax", H);
  MGS_CUDA_OK(cudaMemsetAsync(a.ns_vmax, 0, H * 8, c.stream));
  a.ns_fflag = c.buf<int32_t>("v2_nsfflag", H);
  MGS_CUDA_OK(cudaMemsetAsync(a.ns_fflag, 0, H * 4, c.stream));
  a.ns_big = c.buf<int32_t>("v2_nsbig", H);
  a.ns_small = c.buf<int32_t>("v2_nssmall", H);
  a.ns_used = c.buf<int32_t>("v2_nsused", H);
  a.tcap = caps.tcap;
  const int n_partial_l = sp.proj_base[(1 << t.M) - 1];
  a.g_tab = c.buf<int32_t>("v2_gtab", caps.gcap);
  a.tab_vb = c.buf<unsigned long long>("v2_tabvb", static_cast<size_t>(caps.tcap) * std::max(1, n_partial_l));
  a.tab_rx = c.buf<unsigned long long>("v2_tabrx", static_cast<size_t>(caps.tcap) * std::max(1, n_partial_l));
  a.tab_ex = c.buf<uint32_t>("v2_tabex", static_cast<size_t>(caps.tcap) * sp.P1);
  // alternative kernel paths, selectable for the parity tests (test_gpu.py::test_kernel_paths_agree)
  a.units_tmin = std::getenv("MGS_UNITS_THREAD_MIN") ? std::atoi(std::getenv("MGS_UNITS_THREAD_MIN")) : kUnitsThreadMin;
  a.subitems = std::getenv("MGS_NO_SUBITEMS") ? 0 : 1;
  {  // step-tagged placement maps when (S + 1) fits the bits j + 1 leaves
    int jb = 1;
    while ((1ll << jb) <= sp.P1) ++jb;
    a.ex_bits = jb < 32 && (static_cast<long long>(S) + 1) < (1ll << (32 - jb)) && !std::getenv("MGS_EX_CLEAR") ? jb : 0;
    if (a.ex_bits)
      MGS_CUDA_OK(cudaMemsetAsync(a.tab_ex, 0, static_cast<size_t>(caps.tcap) * sp.P1 * sizeof(uint32_t), c.stream));
  }
  a.tab_hdr = c.buf<unsigned long long>("v2_tabhdr", static_cast<size_t>(caps.tcap) * 2);
  for (void* z : {static_cast<void*>(a.hash), static_cast<void*>(a.ns_ucnt), static_cast<void*>(a.ns_ccnt),
                  static_cast<void*>(a.ns_out)})
    MGS_CUDA_OK(cudaMemsetAsync(z, 0, H * 4, c.stream));
  a.itcap = caps.itcap;
  a.it_s_unit = c.buf<int32_t>("v2_itsu", caps.itcap);
  a.it_s_chunk = c.buf<int32_t>("v2_itsc", caps.itcap);
  a.it_h_unit = c.buf<int32_t>("v2_itsh", caps.itcap);
  a.it_q_unit = c.buf<int32_t>("v2_itsq", caps.itcap);
  a.it_b_unit = c.buf<int32_t>("v2_itbu", caps.itcap);
  a.it_b_chunk = c.buf<int32_t>("v2_itbc", caps.itcap);
  a.ccap = caps.ccap;
  a.c_value = c.buf<double>("v2_cvalue", caps.ccap);
  a.c_lex = c.buf<uint64_t>("v2_clex", caps.ccap);
  a.c_parent = c.buf<int32_t>("v2_cparent", caps.ccap);
  a.c_pid = c.buf<int32_t>("v2_cpid", caps.ccap);
  a.c_ok = c.buf<uint8_t>("v2_cok", caps.ccap);
  a.c_live = c.buf<uint8_t>("v2_clive", caps.ccap);
  a.pcnt = c.buf<int32_t>("v2_pcnt", sp.P1);
  a.pbucket = c.buf<int32_t>("v2_pbucket", static_cast<size_t>(sp.P1) * 64);
  MGS_CUDA_OK(cudaMemsetAsync(a.pcnt, 0, static_cast<size_t>(sp.P1) * 4, c.stream));
  a.scan_cap = 4 * static_cast<int>(H / kTile + 8) + 2 * (caps.ucap / kTile + 8) + (caps.fcap / kTile + 8);
  a.scan_state = c.buf<unsigned long long>("v2_scan", a.scan_cap);
  MGS_CUDA_OK(cudaMemsetAsync(a.scan_state, 0, static_cast<size_t>(a.scan_cap) * 8, c.stream));
  a.sig_len = c.buf<int32_t>("v2_siglen", sp.n_sig);
  k_sig_len<<<ceil_div(sp.n_sig, 256), 256, 0, c.stream>>>(sp.sig_off, sp.n_sig, a.sig_len);
  ++c.kernel_launches;
  a.ctl = c.buf<Ctl>("v2_ctl", 1);
  MGS_CUDA_OK(cudaMemsetAsync(a.ctl, 0, sizeof(Ctl), c.stream));
  a.chosen = c.buf<int32_t>("v2_chosen", S);
  a.n_partial = sp.proj_base[(1 << t.M) - 1];  // all subsets but the full one
  const bool debug = std::getenv("MGS_DEBUG_STEPS") != nullptr || std::getenv("MGS_TRACE") != nullptr;
  a.dbg = debug ? c.buf<long long>("v2_dbg", kDbg * S) : nullptr;
  if (a.dbg) MGS_CUDA_OK(cudaMemsetAsync(a.dbg, 0, sizeof(long long) * kDbg * S, c.stream));
  a.dbg_time = nullptr;
  a.sc_big_ctas = grid_term;
  a.merge_win = merge_win;
  a.oi_bits = 1;
  while ((1ll << a.oi_bits) < sp.n_opt) ++a.oi_bits;
  a.rank_words = rank_words_of(sp.n_opt);
  a.fw = t.M <= 2 ? 16 : 8;
  a.fmask = t.M <= 2 ? 0xffffu : 0xffu;
  a.codec_shift = t.M <= 2 ? Codec(S).shift : 0;
  {
    uint32_t* ids32 = c.buf<uint32_t>("v2_ids32", sp.P1);
    k_ids32<<<ceil_div(sp.P1, 256), 256, 0, c.stream>>>(sp.pl_ids, sp.P1, t.M, a.fw, ids32);
    ++c.kernel_launches;
    a.ids32 = ids32;
  }
  c.prefix = saved_prefix;
  return a;
}

}  // namespace

void solve_dp_v2_lanes(Ctx& c, std::vector<V2Lane>& lanes) {
  const int K = static_cast<int>(lanes.size());
  if (K < 1 || K > kMaxLanes) throw PlanFail{MGS_ERR_ARGUMENT, "lane count out of range"};
  const int M = lanes[0].pr->t.M, S = lanes[0].pr->t.S;
  for (const auto& L : lanes)
    if (L.pr->t.M != M || L.pr->t.S != S) throw PlanFail{MGS_ERR_ARGUMENT, "batched windows must share S and M"};

  // per-lane scalars: dominance validity, tables' smem (the band is computed
  // on the device, k_band_value)
  std::vector<int> dom_ok(K), merge_win(K);
  size_t smem_merge = 0;
  for (int l = 0; l < K; ++l) {
    const HostTables& t = lanes[l].pr->t;
    const DevSpace& sp = *lanes[l].sp;
    bool dominance_ok = true;
    for (int m = 0; m < M; ++m) dominance_ok = dominance_ok && t.post[m] >= t.pre[m];
    dom_ok[l] = dominance_ok ? 1 : 0;
    merge_win[l] = std::min(sp.P1, 8192);  // whole placement range in one window when it fits
    smem_merge = std::max(smem_merge, static_cast<size_t>(2 * merge_win[l]) * 8);
  }
  size_t smem_rank = sizeof(typename cub::BlockRadixSort<unsigned long long, kThreads, kSortItems>::TempStorage);
  for (int l = 0; l < K; ++l) smem_rank = std::max(smem_rank, static_cast<size_t>(rank_words_of(lanes[l].sp->n_opt)) * 8);
  auto ktbig = M == 1 ? k_trans_big<1> : M == 2 ? k_trans_big<2> : M == 3 ? k_trans_big<3> : k_trans_big<4>;
  auto ktsmall = M == 1 ? k_trans_small<1> : M == 2 ? k_trans_small<2> : M == 3 ? k_trans_small<3> : k_trans_small<4>;
  auto kunits = M == 1 ? k_units<1> : M == 2 ? k_units<2> : M == 3 ? k_units<3> : k_units<4>;
  MGS_CUDA_OK(cudaFuncSetAttribute(k_ranks_big, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_rank)));
  MGS_CUDA_OK(cudaFuncSetAttribute(k_band, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_merge)));
  // One resident wave per kernel (SMs x max co-resident CTAs), shared by the
  // lanes: each lane gets a 1/K slice of the wave as its grid.x.
  auto wave = [&](const void* k, size_t dyn) {
    int occ = 0;
    MGS_CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kThreads, dyn));
    static const int cap = std::getenv("MGS_GRID_CAP") ? std::atoi(std::getenv("MGS_GRID_CAP")) : 0;  // tuning probe
    if (cap > 0) occ = std::min(occ, cap);
    const int w = c.sm_count * std::max(1, occ);
    // many lanes: waves of CTAs shared by the lanes (16 lanes, 2 waves: 27.5 -> 26.0
    // ms per C1 window; 32 lanes, 3 waves: 22.8 vs 23.6 at 16 lanes,
    // profiles/r2/lanes_share_probe.log); MGS_LANE_SHARE overrides
    static const int share_env = std::getenv("MGS_LANE_SHARE") ? std::atoi(std::getenv("MGS_LANE_SHARE")) : -1;
    const int lane_share = share_env >= 0 ? share_env : (K >= 24 ? 3 : K >= 12 ? 2 : 0);
    if (lane_share > 0) return dim3(static_cast<unsigned>(std::max(1, w * lane_share / K)), static_cast<unsigned>(K));
    return dim3(static_cast<unsigned>(std::max(1, (w + K - 1) / K)), static_cast<unsigned>(K));
  };
  const dim3 g_term(static_cast<unsigned>(std::max(1, c.sm_count * 8 / K)), static_cast<unsigned>(K));
  const dim3 g_one(1, static_cast<unsigned>(K));
  const dim3 g_units = wave(reinterpret_cast<const void*>(kunits), 0);
  const dim3 g_scans = wave(reinterpret_cast<const void*>(k_scans), 0);
  const dim3 g_rsmall = wave(reinterpret_cast<const void*>(k_ranks_small), 0);
  const dim3 g_kscan = wave(reinterpret_cast<const void*>(k_kid_scan), 0);
  const dim3 g_kfill = wave(reinterpret_cast<const void*>(k_kid_fill), 0);
  const dim3 g_rbig = wave(reinterpret_cast<const void*>(k_ranks_big), smem_rank);
  const dim3 g_tbig = wave(reinterpret_cast<const void*>(ktbig), 0);
  const dim3 g_tables = wave(reinterpret_cast<const void*>(k_tables), 0);
  const dim3 g_tsmall = wave(reinterpret_cast<const void*>(ktsmall), 0);
  const dim3 g_band = wave(reinterpret_cast<const void*>(k_band), smem_merge);
  const dim3 g_write = wave(reinterpret_cast<const void*>(k_write), 0);
  const dim3 g_dom = wave(reinterpret_cast<const void*>(k_dom), 0);
  // initial capacities (grown on overflow, kept per host thread); MGS_V2_SMALL_CAPS
  // starts tiny so every overflow / regrow path runs (test_gpu.py::test_capacity_regrow)
  static thread_local Caps caps = std::getenv("MGS_V2_SMALL_CAPS")
                                      ? Caps{1 << 12, 1 << 10, 1 << 10, 1 << 9, 1 << 13, 11, 8, 1ll << 18}
                                      : Caps{1 << 20, 1 << 18, 1 << 18, 1 << 18, 1 << 22, 16, 8192, 128ll << 20};
  const bool debug = std::getenv("MGS_DEBUG_STEPS") != nullptr || std::getenv("MGS_TRACE") != nullptr;
  if (std::getenv("MGS_TRACE"))
    std::fprintf(stderr, "trace v2 setup: lanes %d S %d M %d smem trans %zu rank %zu merge %zu grid.x %u %u %u %u %u %u %u %u %u %u\n",
                 K, S, M, size_t(0), smem_rank, smem_merge, g_units.x, g_scans.x, 0u, g_rbig.x, 0u,
                 g_tbig.x, g_tsmall.x, g_band.x, g_write.x, g_dom.x);
  for (int attempt = 0; attempt < 40; ++attempt) {  // each attempt stops at the first overflow
    std::vector<V2> args(K);
    for (int l = 0; l < K; ++l) args[l] = lane_args(c, lanes[l], caps, dom_ok[l], merge_win[l], g_term.x);
    V2* d_args = c.buf<V2>("v2_args", kMaxLanes);
    MGS_CUDA_OK(cudaMemcpyAsync(d_args, args.data(), sizeof(V2) * K, cudaMemcpyHostToDevice, c.stream));
    k_init_root<<<g_one, 32, 0, c.stream>>>(d_args);
    ++c.kernel_launches;
    // The window's kernel sequence depends only on S, M, the lane count and
    // launch shapes (all problem data lives behind d_args), so it is captured
    // once into a CUDA graph and replayed; MGS_DEBUG_STEPS launches eagerly.
    constexpr int kK = 11;
    static const char* kNames[kK] = {"kid_scan", "kid_fill", "ranks", "units", "scans", "tables",
                                     "trans_big", "trans_small", "band", "write", "dom"};
    std::vector<cudaEvent_t> evs;
    // trans_small depends only on the ranks, not on the subset tables (it
    // writes disjoint candidate slots; the band maxima are atomicMax): in the
    // captured graph it is a parallel branch (MGS_NO_FORK keeps one chain)
    static const bool fork_ok = std::getenv("MGS_NO_FORK") == nullptr;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_rank_fork = nullptr, ev_rank_join = nullptr;
    cudaEvent_t ev_rs_fork = nullptr, ev_rs_join = nullptr, ev_dom = nullptr, ev_tab = nullptr;
    cudaStream_t side2 = nullptr;
    // MGS_STEP_TIMES (graph mode): an event node after every step, read back
    // after the replay (per-step device time of the captured graph)
    static std::vector<cudaEvent_t> step_ev;
    static const bool step_times = std::getenv("MGS_STEP_TIMES") != nullptr;
    if (step_times && !debug && static_cast<int>(step_ev.size()) < S + 1) {
      for (auto e : step_ev) cudaEventDestroy(e);
      step_ev.assign(S + 1, nullptr);
      for (auto& e : step_ev) MGS_CUDA_OK(cudaEventCreate(&e));
    }
    // milestones inside each step (graph mode, MGS_STEP_TIMES): where the critical path runs
    constexpr int kMile = 12;
    static const char* kMileNames[kMile] = {"-", "kid_scan", "kid_fill", "ranks_big", "ranks_small", "units",
                                            "scans", "tables", "trans_big", "trans_small", "band", "write"};
    static std::vector<cudaEvent_t> mile_ev;
    if (!step_ev.empty() && static_cast<int>(mile_ev.size()) < S * kMile) {
      for (auto e : mile_ev) cudaEventDestroy(e);
      mile_ev.assign(static_cast<size_t>(S) * kMile, nullptr);
      for (auto& e : mile_ev) MGS_CUDA_OK(cudaEventCreate(&e));
    }
    auto mile = [&](int st, int k, cudaStream_t on) {
      if (!mile_ev.empty()) MGS_CUDA_OK(cudaEventRecordWithFlags(mile_ev[static_cast<size_t>(st) * kMile + k], on,
                                                                  cudaEventRecordExternal));
    };
    auto enqueue = [&](cudaStream_t st_, bool timed) {
      if (!timed && !step_ev.empty()) MGS_CUDA_OK(cudaEventRecordWithFlags(step_ev[0], st_, cudaEventRecordExternal));
      const bool fork = fork_ok && !timed && side != nullptr;
      auto mark = [&]() {
        if (!timed) return;
        cudaEvent_t e;
        MGS_CUDA_OK(cudaEventCreate(&e));
        MGS_CUDA_OK(cudaEventRecord(e, st_));
        evs.push_back(e);
      };
      mark();
      const bool trace = timed && std::getenv("MGS_TRACE") != nullptr;
      auto after = [&](const char* name, int st) {  // MGS_TRACE: serialise + name the kernel that hangs/faults
        if (trace) {
          // watchdog: if the kernel does not finish within 5 s, dump lane 0's
          // control block through a second stream (copies overlap a running kernel)
          const auto t0 = std::chrono::steady_clock::now();
          while (cudaStreamQuery(st_) == cudaErrorNotReady &&
                 std::chrono::steady_clock::now() - t0 < std::chrono::seconds(5)) {
          }
          if (cudaStreamQuery(st_) == cudaErrorNotReady) {
            cudaStream_t side;
            cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
            Ctl* hp = nullptr;
            cudaMallocHost(&hp, sizeof(Ctl));
            unsigned long long* ss = nullptr;
            cudaMallocHost(&ss, 256 * 8);
            cudaMemcpyAsync(hp, args[0].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, side);
            cudaMemcpyAsync(ss, args[0].scan_state, 256 * 8, cudaMemcpyDeviceToHost, side);
            cudaStreamSynchronize(side);
            const StepCounters& q = hp->sc[st & 1];
            std::fprintf(stderr, "HANG in %s step %d: err %d ticket %d n_units %d ranks_prev %d %d alive %d %d\n",
                         name, st, hp->err_code, q.ticket, q.n_units, hp->ranks_prev[0], hp->ranks_prev[1],
                         hp->alive_now[0], hp->alive_now[1]);
            for (int i = 0; i < 140; ++i)
              std::fprintf(stderr, "  tile %d: ep %llu flag %llu agg %llu\n", i, ss[i] >> 34, (ss[i] >> 32) & 3,
                           ss[i] & 0xffffffffull);
            std::fflush(stderr);
            std::abort();
          }
          cudaError_t e = cudaStreamSynchronize(st_);
          Ctl hc{};
          cudaMemcpy(&hc, args[0].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost);
          const StepCounters& q = hc.sc[st & 1];
          std::fprintf(stderr,
                       "trace step %d %s -> %s | lane0 err %d units %d T %d its %d itb %d big %d small %d kids %d"
                       " store %d/%d groups %d/%d alive %d/%d out %d/%d\n",
                       st, name, cudaGetErrorString(e), hc.err_code, q.n_units, q.T, q.items_s, q.items_b, q.n_big,
                       q.n_small, q.kids, hc.n_store[0], hc.n_store[1], hc.n_groups[0], hc.n_groups[1],
                       hc.alive_now[0], hc.alive_now[1], q.out_states(), q.out_groups());
        }
        mark();
      };
      for (int st = 0; st < S; ++st) {
        // rank branch (F_s's dense lex ranks) beside the unit branch
        // (successor statuses and candidate ranges): they meet at the transitions
        cudaStream_t rs_ = fork ? side : st_;
        if (fork && st == 0) {
          // later steps fork the rank branch right after the previous k_write
          // (which counted the children), beside k_dom: the rank branch
          // (stored-state ranks) does not wait for dominance
          MGS_CUDA_OK(cudaEventRecord(ev_rank_fork, st_));
          MGS_CUDA_OK(cudaStreamWaitEvent(side, ev_rank_fork, 0));
        }
        k_kid_scan<<<g_kscan, kThreads, 0, rs_>>>(d_args, st);
        after("kid_scan", st);
        if (fork && !timed) mile(st, 1, rs_);
        k_kid_fill<<<g_kfill, kThreads, 0, rs_>>>(d_args, st);
        after("kid_fill", st);
        if (fork && !timed) mile(st, 2, rs_);
        if (fork) {
          // rank branch: ranks (big on side, small on side2), then the subset
          // tables on side once k_dom(s-1) is done too (alive flags); the unit
          // branch (units -> scans) runs beside it on the main stream. The
          // small-group transitions (side2) need both branches, the big-group
          // ones (main) the tables and the unit branch.
          MGS_CUDA_OK(cudaEventRecord(ev_rs_fork, side));
          MGS_CUDA_OK(cudaStreamWaitEvent(side2, ev_rs_fork, 0));
          k_ranks_small<<<g_rsmall, kThreads, 0, side2>>>(d_args, st);
          if (!timed) mile(st, 4, side2);
          MGS_CUDA_OK(cudaEventRecord(ev_rs_join, side2));
          k_ranks_big<<<g_rbig, kThreads, smem_rank, side>>>(d_args, st, 0);
          if (!timed) mile(st, 3, side);
          MGS_CUDA_OK(cudaEventRecord(ev_rank_join, side));
          MGS_CUDA_OK(cudaStreamWaitEvent(side, ev_rs_join, 0));
          MGS_CUDA_OK(cudaEventRecord(ev_dom, st_));  // k_dom(s-1) (or the root) is done
          MGS_CUDA_OK(cudaStreamWaitEvent(side, ev_dom, 0));
          k_tables<<<g_tables, kThreads, 0, side>>>(d_args, st);
          if (!timed) mile(st, 7, side);
          MGS_CUDA_OK(cudaEventRecord(ev_tab, side));
        } else {
          k_ranks_big<<<g_rbig, kThreads, smem_rank, st_>>>(d_args, st, 1);
          after("ranks", st);
        }
        kunits<<<g_units, kThreads, 0, st_>>>(d_args, st);
        after("units", st);
        if (fork && !timed) mile(st, 5, st_);
        k_scans<<<g_scans, kThreads, 0, st_>>>(d_args, st);
        after("scans", st);
        if (fork && !timed) mile(st, 6, st_);
        if (fork) {
          MGS_CUDA_OK(cudaEventRecord(ev_fork, st_));
          MGS_CUDA_OK(cudaStreamWaitEvent(side2, ev_fork, 0));
          MGS_CUDA_OK(cudaStreamWaitEvent(side2, ev_rank_join, 0));
          ktsmall<<<g_tsmall, kThreads, 0, side2>>>(d_args, st);
          if (!timed) mile(st, 9, side2);
          MGS_CUDA_OK(cudaEventRecord(ev_join, side2));
          MGS_CUDA_OK(cudaStreamWaitEvent(st_, ev_tab, 0));
          ktbig<<<g_tbig, kThreads, 0, st_>>>(d_args, st);
          if (!timed) mile(st, 8, st_);
          MGS_CUDA_OK(cudaStreamWaitEvent(st_, ev_join, 0));
        } else {
          k_tables<<<g_tables, kThreads, 0, st_>>>(d_args, st);
          after("tables", st);
          ktbig<<<g_tbig, kThreads, 0, st_>>>(d_args, st);
          after("trans_big", st);
          ktsmall<<<g_tsmall, kThreads, 0, st_>>>(d_args, st);
          after("trans_small", st);
        }
        k_band<<<g_band, kThreads, smem_merge, st_>>>(d_args, st);
        after("band", st);
        if (fork && !timed) mile(st, 10, st_);
        k_write<<<g_write, kThreads, 0, st_>>>(d_args, st);
        after("write", st);
        if (fork && !timed) mile(st, 11, st_);
        if (fork && st + 1 < S) {
          MGS_CUDA_OK(cudaEventRecord(ev_rank_fork, st_));
          MGS_CUDA_OK(cudaStreamWaitEvent(side, ev_rank_fork, 0));
        }
        k_dom<<<g_dom, kThreads, 0, st_>>>(d_args, st);
        after("dom", st);
        if (!timed && !step_ev.empty()) MGS_CUDA_OK(cudaEventRecordWithFlags(step_ev[st + 1], st_, cudaEventRecordExternal));
      }
      k_term1<<<g_term, kThreads, 0, st_>>>(d_args);
      k_term2<<<g_term, kThreads, 0, st_>>>(d_args);
      k_term3<<<g_term, kThreads, 0, st_>>>(d_args);
      k_backtrack2<<<g_one, 32, 0, st_>>>(d_args);
    };
    // graph replays split the ranks into two kernels (k_ranks_big + k_ranks_small)
    c.kernel_launches += static_cast<unsigned long long>(kK + (!debug && fork_ok ? 1 : 0)) * S + 4;
    if (debug) {
      const auto host_t0 = std::chrono::steady_clock::now();
      enqueue(c.stream, true);
      const double host_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count();
      MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
      std::fprintf(stderr, "v2 host enqueue ms %.2f (eager, with events, %d lanes)\n", host_ms, K);
      double acc[kK] = {0};
      std::vector<double> per_step(S, 0.0);
      for (size_t i = 1; i < evs.size(); ++i) {
        float ms = 0.f;
        MGS_CUDA_OK(cudaEventElapsedTime(&ms, evs[i - 1], evs[i]));
        acc[(i - 1) % kK] += ms;
        if ((i - 1) / kK < static_cast<size_t>(S)) per_step[(i - 1) / kK] += ms;
      }
      if (std::getenv("MGS_STEP_TIMES")) {  // per-step device time (eager, serialised): floor + slope fit
        std::fprintf(stderr, "v2 step_us");
        for (int s = 0; s < S; ++s) std::fprintf(stderr, " %.1f", 1e3 * per_step[s]);
        std::fprintf(stderr, "\n");
      }
      for (auto e : evs) cudaEventDestroy(e);
      std::fprintf(stderr, "v2 caps: fcap %d gcap %d ucap %d itcap %d ccap %d hbits %d hcap %lld\n", caps.fcap, caps.gcap,
                   caps.ucap, caps.itcap, caps.ccap, caps.hbits, caps.hcap);
      std::fprintf(stderr, "v2 in-stream ms per window:");
      for (int k = 0; k < kK; ++k) std::fprintf(stderr, " %s %.2f", kNames[k], acc[k]);
      std::fprintf(stderr, "\n");
    } else {
      char key[256];
      std::snprintf(key, sizeof key, "v2:%d:%d:%d:%zu:%zu:%p:%d", K, S, M, smem_merge, smem_rank,
                    static_cast<void*>(d_args), step_ev.empty() ? 0 : 1);
      auto it = c.graphs.find(key);
      if (it == c.graphs.end()) {
        cudaStream_t cap;
        MGS_CUDA_OK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
        cudaGraph_t graph;
        MGS_CUDA_OK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_rank_fork, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_rank_join, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_rs_fork, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_rs_join, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_dom, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaEventCreateWithFlags(&ev_tab, cudaEventDisableTiming));
        MGS_CUDA_OK(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
        MGS_CUDA_OK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        enqueue(cap, false);
        MGS_CUDA_OK(cudaStreamEndCapture(cap, &graph));
        MGS_CUDA_OK(cudaEventDestroy(ev_fork));
        MGS_CUDA_OK(cudaEventDestroy(ev_join));
        MGS_CUDA_OK(cudaEventDestroy(ev_rank_fork));
        MGS_CUDA_OK(cudaEventDestroy(ev_rank_join));
        MGS_CUDA_OK(cudaEventDestroy(ev_rs_fork));
        MGS_CUDA_OK(cudaEventDestroy(ev_rs_join));
        MGS_CUDA_OK(cudaEventDestroy(ev_dom));
        MGS_CUDA_OK(cudaEventDestroy(ev_tab));
        MGS_CUDA_OK(cudaStreamDestroy(side2));
        side2 = nullptr;
        MGS_CUDA_OK(cudaStreamDestroy(side));
        side = nullptr;
        cudaGraphExec_t exec;
        MGS_CUDA_OK(cudaGraphInstantiate(&exec, graph, 0));
        MGS_CUDA_OK(cudaGraphDestroy(graph));
        MGS_CUDA_OK(cudaStreamDestroy(cap));
        if (c.graphs.size() >= 16) {
          cudaGraphExecDestroy(c.graphs.begin()->second);
          c.graphs.erase(c.graphs.begin());
        }
        it = c.graphs.emplace(key, exec).first;
      }
      MGS_CUDA_OK(cudaGraphLaunch(it->second, c.stream));
      if (!step_ev.empty()) {
        MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
        std::fprintf(stderr, "v2 graph step_us");
        for (int st = 0; st < S; ++st) {
          float ms = 0.f;
          MGS_CUDA_OK(cudaEventElapsedTime(&ms, step_ev[st], step_ev[st + 1]));
          std::fprintf(stderr, " %.1f", 1e3 * ms);
        }
        std::fprintf(stderr, "\n");
        if (!mile_ev.empty() && fork_ok) {  // mean milestone time after the step's start (previous k_dom), us
          std::fprintf(stderr, "v2 graph milestones_us (from step start):");
          for (int k = 0; k < kMile; ++k) {
            double acc = 0.0;
            int n = 0;
            for (int st = 1; st < S; ++st) {
              float ms = 0.f;
              if (cudaEventElapsedTime(&ms, step_ev[st], mile_ev[static_cast<size_t>(st) * kMile + k]) != cudaSuccess) {
                (void)cudaGetLastError();  // a milestone this graph does not record
                continue;
              }
              acc += 1e3 * ms;
              ++n;
            }
            std::fprintf(stderr, " %s %.1f", kMileNames[k], n ? acc / n : 0.0);
          }
          std::fprintf(stderr, "\n");
        }
      }
    }
    MGS_CUDA_OK(cudaGetLastError());
    std::vector<Ctl> h(K);
    for (int l = 0; l < K; ++l)
      MGS_CUDA_OK(cudaMemcpyAsync(&h[l], args[l].ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    // a failing step's need is a lower bound for the later steps: 4x it
    bool grow = false;
    for (int l = 0; l < K; ++l) {
      if (h[l].err_code != kOverflow) continue;
      grow = true;
      const long long need = h[l].need;
      if (debug) std::fprintf(stderr, "v2 capacity growth: what %d need %lld at step %d\n", h[l].need_what, need, h[l].err_step);
      switch (h[l].need_what) {
        case 2: caps.hbits += 2; break;  // table too full: 4x the slots
        case 3: caps.ucap = static_cast<int>(std::max<long long>(need * 4, caps.ucap * 2ll)); break;
        case 4: caps.fcap = static_cast<int>(std::max<long long>(need * 4, caps.fcap * 2ll)); break;
        case 5: caps.gcap = static_cast<int>(std::max<long long>(need * 4, caps.gcap * 2ll)); break;
        case 6: caps.hcap = std::max<long long>(need * 4, caps.hcap * 2); break;
        case 7: caps.ccap = static_cast<int>(std::max<long long>(need * 4, caps.ccap * 2ll)); break;
        case 8: caps.itcap = static_cast<int>(std::max<long long>(need * 4, caps.itcap * 2ll)); break;
        case 9: caps.tcap = static_cast<int>(std::max<long long>(need * 4, caps.tcap * 2ll)); break;
        default: throw PlanFail{MGS_ERR_CUDA, "persistent DP: unknown capacity overflow"};
      }
    }
    if (grow) continue;  // every lane re-runs with the larger capacities
    for (int l = 0; l < K; ++l) {
      V2Lane& L = lanes[l];
      const Ctl& hc = h[l];
      if (debug && args[l].dbg && l == 0) {
        std::vector<long long> d(kDbg * S);
        MGS_CUDA_OK(cudaMemcpy(d.data(), args[l].dbg, d.size() * 8, cudaMemcpyDeviceToHost));
        for (int s = 0; s < S; ++s) {
          const long long* q = d.data() + kDbg * s;
          std::fprintf(stderr,
                       "v2 step %d units %lld ns %lld T %lld store %lld groups %lld alive_in %lld items_b %lld "
                       "items_s %lld max_group %lld big_groups %lld small32 %lld/%lld small %lld/%lld gn_sum %lld fused %lld gn>32 %lld"
                       " small_targets %lld targets_x_gn %lld\n",
                       s, q[0], q[1], q[2], q[3], q[4], q[5], q[6], q[7], q[8], q[9], q[10], q[11], q[12], q[13], q[14],
                       q[15], q[16], q[17], q[18]);
        }
      }
      L.status = MGS_OK;
      if (hc.err_code == MGS_ERR_STATE_BUDGET) {
        L.status = MGS_ERR_STATE_BUDGET;
        L.err_step = hc.err_step;
        L.err_count = hc.err_count;
        L.msg = "dynamic-program frontier reached " + std::to_string(hc.err_count) + " states at step " +
                std::to_string(hc.err_step) + " (budget " + std::to_string(L.p->state_budget) + ")";
        continue;
      }
      if (hc.err_code == MGS_ERR_INFEASIBLE_JOINT) {
        L.status = MGS_ERR_INFEASIBLE_JOINT;
        L.msg = "no feasible allocation sequence exists for this window";
        continue;
      }
      if (hc.err_code != 0) {
        L.status = MGS_ERR_CUDA;
        L.msg = "persistent DP: error " + std::to_string(hc.err_code);
        continue;
      }
      L.out.d_options = args[l].chosen;
      if (L.host_options) {
        L.out.options.resize(S);
        MGS_CUDA_OK(cudaMemcpyAsync(L.out.options.data(), args[l].chosen, S * 4, cudaMemcpyDeviceToHost, c.stream));
      }
      L.out.stats.options = L.sp->n_opt;
      L.out.stats.candidates = L.sp->n_cand;
      L.out.stats.transitions_ref = hc.tr_ref;
      L.out.stats.transitions = hc.tr;
      L.out.stats.frontier_total = hc.ftot;
      L.out.stats.frontier_peak = hc.fpeak;
      L.out.stats.transition_bytes = hc.tbytes;
    }
    bool any_host = false;
    for (const auto& L : lanes) any_host = any_host || L.host_options;
    if (any_host) MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
    return;
  }
  throw PlanFail{MGS_ERR_CUDA, "persistent DP: capacity growth did not converge"};
}

void solve_dp_v2(Ctx& c, const mgs_problem& p, const Prepared& pr, const DevSpace& sp, const double* d_recv,
                 const double* d_ub, const double* d_incumbent, SolveOut& out) {
  std::vector<V2Lane> lanes(1);
  V2Lane& L = lanes[0];
  L.p = &p;
  L.pr = &pr;
  L.sp = &sp;
  L.recv = d_recv;
  L.ub = d_ub;
  L.incumbent = d_incumbent;
  L.prefix = c.prefix;
  L.host_options = false;  // the caller reads the plan back together with its labels and objective
  solve_dp_v2_lanes(c, lanes);
  if (L.status != MGS_OK) throw PlanFail{L.status, L.msg, L.err_step, L.err_count};
  out.d_options = L.out.d_options;
  out.stats = L.out.stats;
}

}  // namespace mgs
