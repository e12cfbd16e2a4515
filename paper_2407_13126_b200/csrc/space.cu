// Candidate enumeration over the MIG partition lattice on the GPU.
//
// Reference: engine::Space::build (proj/include/migsim/space.hpp:126-210) walks,
// per configuration in catalog order, every per-slot label vector in ascending
// lexicographic order (slot 0 most significant) and keeps the admissible,
// anchored ones. Here each label vector is one thread: the vector's mixed-radix
// index *is* its lexicographic rank inside the configuration, so a flag pass +
// an exclusive scan reproduces the reference option indices exactly (the index
// is part of the tie-break, solvers.hpp:466).
//
// On top of the option list the planner needs derived tables, all built here
// on the device with sort/unique passes:
//   * per-tenant inference-mask ids (dense ranks of distinct masks);
//   * placements = distinct per-tenant mask-id tuples (the DP state key's
//     mask part, solvers.hpp:99-103), with their inference capability;
//   * candidates = distinct (signature, placement) pairs with the smallest
//     option index. All options of one (signature, placement) yield identical
//     successor keys and values inside one DP unit, so only the smallest index
//     can survive the equal-key merge (solvers.hpp:467-468);
//   * projection ids of every placement onto every tenant subset, used by
//     the dense predecessor tables (solvers.hpp:367-378).
#include <algorithm>
#include <cub/cub.cuh>

#include "ctx.cuh"

namespace mgs {

Prepared prepare_tables(const mgs_lattice& lat, const mgs_tables& tab) {
  Prepared pr;
  if (tab.models > KM) throw PlanFail{MGS_ERR_INPUT_SCENARIO, "at most 4 models are supported"};  // space.hpp:49-50
  if (tab.models < 1 || tab.steps < 1 || lat.n_configs < 1 || !lat.slot_offset || !lat.slot_size || !lat.slot_start)
    throw PlanFail{MGS_ERR_ARGUMENT, "empty lattice or tables"};
  std::map<std::pair<int, int>, int> uid;  // universe: first-appearance order (space.hpp:56-64)
  const int nslots = lat.slot_offset[lat.n_configs];
  pr.slot_uid.resize(nslots);
  for (int c = 0; c < lat.n_configs; ++c) {
    if (lat.slot_offset[c + 1] - lat.slot_offset[c] > MGS_MAX_SLOTS)
      throw PlanFail{MGS_ERR_ARGUMENT, "configuration has more slots than MGS_MAX_SLOTS"};
    for (int i = lat.slot_offset[c]; i < lat.slot_offset[c + 1]; ++i) {
      std::pair<int, int> r{lat.slot_start[i], lat.slot_size[i]};
      auto it = uid.find(r);
      int u;
      if (it == uid.end()) {
        u = static_cast<int>(uid.size());
        uid[r] = u;
      } else {
        u = it->second;
      }
      pr.slot_uid[i] = u;
    }
  }
  if (uid.size() > 30) throw PlanFail{MGS_ERR_INPUT_CATALOG, "catalog has more than 30 distinct instances"};  // :65
  pr.n_universe = static_cast<int>(uid.size());
  HostTables& t = pr.t;
  std::memset(&t, 0, sizeof t);
  t.M = tab.models;
  t.S = tab.steps;
  for (int m = 0; m < t.M; ++m) {
    for (int k = 0; k < 8; ++k) {
      t.cap[m][k] = tab.cap_by_size[m][k];
      t.rt[m][k] = tab.rt_by_size[m][k];
    }
    t.floor_[m] = tab.floor_gpcs[m];
    t.loss[m] = tab.psi[m] < 1.0 ? tab.psi[m] : 1.0;  // reconfig_loss_fraction, plan_types.hpp:68
    t.psi_raw[m] = tab.psi[m];
    t.pre[m] = tab.acc_pre[m];
    t.post[m] = tab.acc_post[m];
    t.min_rt[m] = -1;  // space.hpp:79-83
    for (int k = 1; k <= 7; ++k) {
      long long r = t.rt[m][k];
      if (r >= 1 && r <= t.S && (t.min_rt[m] < 0 || r < t.min_rt[m])) t.min_rt[m] = r;
    }
  }
  return pr;
}

namespace {

struct LatticeDev {
  int n_configs;
  const unsigned long long* vprefix;  // [n_configs+1] prefix of (2M+1)^n_slots
  const int* slot_off;
  const int* slot_size;
  const int* slot_uid;
};

__device__ inline int find_config(const unsigned long long* vprefix, int n, unsigned long long i) {
  int lo = 0, hi = n;  // largest c with vprefix[c] <= i
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (vprefix[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Decodes label vector i of its configuration; returns false when the vector
// is not an option (space.hpp:178-192 admissibility, :162-163 anchoring).
__device__ bool decode_option(const LatticeDev& L, const HostTables& t, unsigned long long i, int* cfg, int8_t* labels,
                              int* n_out) {
  const int c = find_config(L.vprefix, L.n_configs, i);
  unsigned long long v = i - L.vprefix[c];
  const int base = L.slot_off[c], n = L.slot_off[c + 1] - base;
  const int B = 2 * t.M + 1;
  for (int k = n - 1; k >= 0; --k) {
    labels[k] = static_cast<int8_t>(v % B);
    v /= B;
  }
  *cfg = c;
  *n_out = n;
  unsigned anchored = 0, retrain_seen = 0;
  for (int k = 0; k < n; ++k) {
    const int lab = labels[k];
    if (lab == 0) continue;
    const int m = (lab - 1) >> 1, size = L.slot_size[base + k];
    if (((lab - 1) & 1) == 0) {
      if (!(t.cap[m][size] > 0.0)) return false;  // zero-capability slots never help
      if (size >= t.floor_[m]) anchored |= 1u << m;
    } else {
      const long long rt = t.rt[m][size];
      if (!(rt >= 1 && rt <= t.S)) return false;  // must finish in-window
      if (retrain_seen & (1u << m)) return false;  // one instance per retraining task
      retrain_seen |= 1u << m;
    }
  }
  return anchored == (1u << t.M) - 1u;
}

__global__ void k_enum_flags(LatticeDev L, HostTables t, unsigned long long total, int32_t* flag) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    int8_t labels[MGS_MAX_SLOTS];
    int c, n;
    flag[i] = decode_option(L, t, i, &c, labels, &n) ? 1 : 0;
  }
}

__global__ void k_enum_write(LatticeDev L, HostTables t, unsigned long long total, const int32_t* flag,
                             const int32_t* pos, DevSpace sp) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < total;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    int8_t labels[MGS_MAX_SLOTS] = {0, 0, 0, 0, 0, 0, 0, 0};
    int c, n;
    decode_option(L, t, i, &c, labels, &n);
    const int o = pos[i];
    const int base = L.slot_off[c];
    uint32_t mask[KM] = {0, 0, 0, 0};
    double cap[KM] = {0.0, 0.0, 0.0, 0.0};
    int8_t rs[KM] = {0, 0, 0, 0};
    for (int k = 0; k < n; ++k) {  // slot (slice_start) order: capability sums fold identically (space.hpp:147-160)
      const int lab = labels[k];
      if (lab == 0) continue;
      const int m = (lab - 1) >> 1, size = L.slot_size[base + k];
      if (((lab - 1) & 1) == 0) {
        mask[m] |= 1u << L.slot_uid[base + k];
        cap[m] = dadd(cap[m], t.cap[m][size]);
      } else {
        rs[m] = static_cast<int8_t>(size);
      }
    }
    int sig = 0;
    for (int m = t.M - 1; m >= 0; --m) sig = sig * 8 + rs[m];  // Option::signature (space.hpp:109-113)
    sp.opt_config[o] = c;
    for (int k = 0; k < MGS_MAX_SLOTS; ++k) sp.opt_labels[o * MGS_MAX_SLOTS + k] = labels[k];
    for (int m = 0; m < KM; ++m) {
      sp.opt_mask[o * KM + m] = mask[m];
      sp.opt_cap[o * KM + m] = cap[m];
      sp.opt_rsize[o * KM + m] = rs[m];
    }
    sp.opt_sig[o] = sig;
  }
}

template <class T>
__device__ inline int lower_bound_dev(const T* a, int n, T x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void k_copy_mask_col(const uint32_t* opt_mask, int n, int m, uint32_t* out) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) out[o] = opt_mask[o * KM + m];
}

__global__ void k_assign_ids(const uint32_t* opt_mask, int n, int M, const uint32_t* vals, const int* val_off,
                             uint64_t* opt_ids) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    uint64_t key = 0;
    for (int m = 0; m < M; ++m) {
      const int lo = val_off[m], cnt = val_off[m + 1] - lo;
      const int id = lower_bound_dev(vals + lo, cnt, opt_mask[o * KM + m]);
      key |= static_cast<uint64_t>(id) << (16 * m);
    }
    opt_ids[o] = key;
  }
}

__global__ void k_assign_pid(const uint64_t* opt_ids, int n, const uint64_t* pl_keys, int P, int32_t* opt_pid,
                             const double* opt_cap, double* pl_cap, const int32_t* opt_sig, uint64_t* cand_key,
                             int32_t* iota, int32_t* sig_nopt) {
  for (int o = blockIdx.x * blockDim.x + threadIdx.x; o < n; o += gridDim.x * blockDim.x) {
    const int pid = lower_bound_dev(pl_keys, P, opt_ids[o]);
    opt_pid[o] = pid;
    for (int m = 0; m < KM; ++m) pl_cap[pid * KM + m] = opt_cap[o * KM + m];  // identical for every option of pid
    cand_key[o] = (static_cast<uint64_t>(opt_sig[o]) << 32) | static_cast<uint32_t>(pid);
    iota[o] = o;
    atomicAdd(&sig_nopt[opt_sig[o]], 1);
  }
}

__global__ void k_first_of_run(const uint64_t* keys, int n, int32_t* flag) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void k_scatter_cands(const uint64_t* keys, const int32_t* vals, const int32_t* flag, const int32_t* pos,
                                int n, int32_t* cand_pid, int32_t* cand_oi, int32_t* cand_sig) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    if (!flag[i]) continue;
    const int q = pos[i];
    cand_pid[q] = static_cast<int32_t>(keys[i] & 0xffffffffu);
    cand_sig[q] = static_cast<int32_t>(keys[i] >> 32);
    cand_oi[q] = vals[i];  // radix sort is stable: first of the run = smallest option index
  }
}

__global__ void k_sig_off(const int32_t* cand_sig, int n_cand, int n_sig, int32_t* sig_off) {
  for (int g = blockIdx.x * blockDim.x + threadIdx.x; g <= n_sig; g += gridDim.x * blockDim.x)
    sig_off[g] = lower_bound_dev(cand_sig, n_cand, static_cast<int32_t>(g));
}

__global__ void k_proj_keys(const uint64_t* pl_ids, int P1, int M, int sub, uint64_t* out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P1; p += gridDim.x * blockDim.x) {
    uint64_t k = 0;
    for (int m = 0; m < M; ++m) {
      const uint64_t f = (sub >> m) & 1 ? static_cast<uint64_t>(field16(pl_ids[p], m)) : 0xffffull;
      k |= f << (16 * m);
    }
    out[p] = k;
  }
}

__global__ void k_proj_assign(const uint64_t* keys, int P1, const uint64_t* uniq, int nu, int32_t* out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P1; p += gridDim.x * blockDim.x)
    out[p] = lower_bound_dev(uniq, nu, keys[p]);
}

// sort + unique of n 64-bit (or 32-bit) keys; returns the unique count
template <class K>
int sort_unique(Ctx& c, const K* in, K* sorted, K* uniq, int n) {
  size_t tb1 = 0, tb2 = 0;
  int* d_nu = c.buf<int>("su_n", 1);
  cub::DeviceRadixSort::SortKeys(nullptr, tb1, in, sorted, n, 0, sizeof(K) * 8, c.stream);
  cub::DeviceSelect::Unique(nullptr, tb2, sorted, uniq, d_nu, n, c.stream);
  size_t tb = std::max(tb1, tb2);
  void* tmp = c.buf<char>("cub_tmp", tb);
  MGS_CUDA_OK(cub::DeviceRadixSort::SortKeys(tmp, tb, in, sorted, n, 0, sizeof(K) * 8, c.stream));
  MGS_CUDA_OK(cub::DeviceSelect::Unique(tmp, tb, sorted, uniq, d_nu, n, c.stream));
  return read_scalar(c, d_nu);
}

inline unsigned grid_for(long long n, int threads = 256) {
  long long g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<unsigned>(g);
}

}  // namespace

void build_space(Ctx& c, const mgs_lattice& lat, const Prepared& pr, DevSpace& sp) {
  const HostTables& t = pr.t;
  const int M = t.M;
  sp.M = M;
  sp.S = t.S;
  // lattice upload
  const int nc = lat.n_configs, nslots = lat.slot_offset[nc];
  std::vector<unsigned long long> vprefix(nc + 1, 0);
  for (int i = 0; i < nc; ++i) {
    unsigned long long v = 1;
    for (int k = lat.slot_offset[i]; k < lat.slot_offset[i + 1]; ++k) v *= static_cast<unsigned long long>(2 * M + 1);
    vprefix[i + 1] = vprefix[i] + v;
  }
  const unsigned long long total = vprefix[nc];
  auto* d_vprefix = c.buf<unsigned long long>("lat_vprefix", nc + 1);
  auto* d_soff = c.buf<int>("lat_soff", nc + 1);
  auto* d_ssize = c.buf<int>("lat_ssize", nslots);
  auto* d_suid = c.buf<int>("lat_suid", nslots);
  MGS_CUDA_OK(cudaMemcpyAsync(d_vprefix, vprefix.data(), (nc + 1) * 8, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_soff, lat.slot_offset, (nc + 1) * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_ssize, lat.slot_size, nslots * 4, cudaMemcpyHostToDevice, c.stream));
  MGS_CUDA_OK(cudaMemcpyAsync(d_suid, pr.slot_uid.data(), nslots * 4, cudaMemcpyHostToDevice, c.stream));
  LatticeDev L{nc, d_vprefix, d_soff, d_ssize, d_suid};

  // 1. flags + scan + write (Space::build)
  auto* flag = c.buf<int32_t>("enum_flag", total);
  auto* pos = c.buf<int32_t>("enum_pos", total + 1);
  k_enum_flags<<<grid_for(total), 256, 0, c.stream>>>(L, t, total, flag);
  ++c.kernel_launches;
  exclusive_scan_i32(c, flag, pos, static_cast<int>(total));
  const int n_opt = read_scalar(c, pos + total);
  sp.n_opt = n_opt;
  if (n_opt == 0) {
    sp.P = 0;
    sp.P1 = 1;
    sp.n_cand = 0;
    sp.n_sig = 1 << (3 * M);
    sp.sig_nopt = c.buf<int32_t>("sig_nopt", sp.n_sig);
    MGS_CUDA_OK(cudaMemsetAsync(sp.sig_nopt, 0, sp.n_sig * 4, c.stream));
    return;
  }
  sp.opt_config = c.buf<int32_t>("opt_config", n_opt);
  sp.opt_labels = c.buf<int8_t>("opt_labels", static_cast<size_t>(n_opt) * MGS_MAX_SLOTS);
  sp.opt_mask = c.buf<uint32_t>("opt_mask", static_cast<size_t>(n_opt) * KM);
  sp.opt_cap = c.buf<double>("opt_cap", static_cast<size_t>(n_opt) * KM);
  sp.opt_rsize = c.buf<int8_t>("opt_rsize", static_cast<size_t>(n_opt) * KM);
  sp.opt_sig = c.buf<int32_t>("opt_sig", n_opt);
  sp.opt_pid = c.buf<int32_t>("opt_pid", n_opt);
  k_enum_write<<<grid_for(total), 256, 0, c.stream>>>(L, t, total, flag, pos, sp);
  ++c.kernel_launches;

  // 2. per-tenant mask ids
  auto* col = c.buf<uint32_t>("col", n_opt);
  auto* col_sorted = c.buf<uint32_t>("col_sorted", n_opt);
  auto* vals = c.buf<uint32_t>("mask_vals", static_cast<size_t>(n_opt) * KM);
  std::vector<int> val_off(M + 1, 0);
  std::vector<std::vector<uint32_t>> host_vals(M);
  for (int m = 0; m < M; ++m) {
    k_copy_mask_col<<<grid_for(n_opt), 256, 0, c.stream>>>(sp.opt_mask, n_opt, m, col);
    ++c.kernel_launches;
    int nu = sort_unique(c, col, col_sorted, vals + val_off[m], n_opt);
    val_off[m + 1] = val_off[m] + nu;
    host_vals[m].resize(nu);
    MGS_CUDA_OK(cudaMemcpyAsync(host_vals[m].data(), vals + val_off[m], nu * 4, cudaMemcpyDeviceToHost, c.stream));
  }
  auto* d_val_off = c.buf<int>("mask_val_off", M + 1);
  MGS_CUDA_OK(cudaMemcpyAsync(d_val_off, val_off.data(), (M + 1) * 4, cudaMemcpyHostToDevice, c.stream));
  auto* opt_ids = c.buf<uint64_t>("opt_ids", n_opt);
  k_assign_ids<<<grid_for(n_opt), 256, 0, c.stream>>>(sp.opt_mask, n_opt, M, vals, d_val_off, opt_ids);
  ++c.kernel_launches;

  // 3. placements (+ the root's carried-over placement at index P)
  auto* ids_sorted = c.buf<uint64_t>("ids_sorted", n_opt);
  sp.pl_ids = c.buf<uint64_t>("pl_ids", n_opt + 1);
  const int P = sort_unique(c, opt_ids, ids_sorted, sp.pl_ids, n_opt);
  sp.P = P;
  sp.P1 = P + 1;
  sp.root_pid = P;
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));  // host_vals ready
  uint64_t root = 0;
  for (int m = 0; m < M; ++m) {
    // initial_masks (space.hpp:305-323): a mask that no option uses gets the
    // out-of-range id, so it never matches (kForeignMask included).
    const uint32_t want = pr.has_initial ? pr.init_mask[m] : 0u;
    auto it = std::lower_bound(host_vals[m].begin(), host_vals[m].end(), want);
    int id = (it != host_vals[m].end() && *it == want) ? static_cast<int>(it - host_vals[m].begin())
                                                       : static_cast<int>(host_vals[m].size());
    root |= static_cast<uint64_t>(id) << (16 * m);
  }
  MGS_CUDA_OK(cudaMemcpyAsync(sp.pl_ids + P, &root, 8, cudaMemcpyHostToDevice, c.stream));
  for (int m = 0; m < M; ++m) sp.n_mask_ids[m] = static_cast<int>(host_vals[m].size()) + 1;
  sp.pl_cap = c.buf<double>("pl_cap", static_cast<size_t>(P + 1) * KM);
  MGS_CUDA_OK(cudaMemsetAsync(sp.pl_cap, 0, static_cast<size_t>(P + 1) * KM * 8, c.stream));

  // 4. candidates: distinct (sig, pid), smallest option index
  sp.n_sig = 1 << (3 * M);
  sp.sig_nopt = c.buf<int32_t>("sig_nopt", sp.n_sig);
  MGS_CUDA_OK(cudaMemsetAsync(sp.sig_nopt, 0, sp.n_sig * 4, c.stream));
  auto* ckey = c.buf<uint64_t>("cand_key", n_opt);
  auto* ckey_sorted = c.buf<uint64_t>("cand_key_sorted", n_opt);
  auto* iota = c.buf<int32_t>("cand_iota", n_opt);
  auto* iota_sorted = c.buf<int32_t>("cand_iota_sorted", n_opt);
  k_assign_pid<<<grid_for(n_opt), 256, 0, c.stream>>>(opt_ids, n_opt, sp.pl_ids, P, sp.opt_pid, sp.opt_cap,
                                                      sp.pl_cap, sp.opt_sig, ckey, iota, sp.sig_nopt);
  {
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, ckey, ckey_sorted, iota, iota_sorted, n_opt, 0, 64, c.stream);
    void* tmp = c.buf<char>("cub_tmp", tb);
    MGS_CUDA_OK(cub::DeviceRadixSort::SortPairs(tmp, tb, ckey, ckey_sorted, iota, iota_sorted, n_opt, 0, 64, c.stream));
  }
  auto* fl = c.buf<int32_t>("cand_flag", n_opt);
  auto* fpos = c.buf<int32_t>("cand_fpos", n_opt + 1);
  k_first_of_run<<<grid_for(n_opt), 256, 0, c.stream>>>(ckey_sorted, n_opt, fl);
  ++c.kernel_launches;
  exclusive_scan_i32(c, fl, fpos, n_opt);
  sp.n_cand = read_scalar(c, fpos + n_opt);
  sp.cand_pid = c.buf<int32_t>("cand_pid", sp.n_cand);
  sp.cand_oi = c.buf<int32_t>("cand_oi", sp.n_cand);
  sp.cand_sig = c.buf<int32_t>("cand_sig", sp.n_cand);
  k_scatter_cands<<<grid_for(n_opt), 256, 0, c.stream>>>(ckey_sorted, iota_sorted, fl, fpos, n_opt, sp.cand_pid,
                                                         sp.cand_oi, sp.cand_sig);
  sp.sig_off = c.buf<int32_t>("sig_off", sp.n_sig + 1);
  k_sig_off<<<grid_for(sp.n_sig + 1), 256, 0, c.stream>>>(sp.cand_sig, sp.n_cand, sp.n_sig, sp.sig_off);
  ++c.kernel_launches;

  // 5. subset projections of every placement (incl. the root)
  const int n_sub = 1 << M;
  const int P1 = P + 1;
  sp.proj_id = c.buf<int32_t>("proj_id", static_cast<size_t>(n_sub) * P1);
  auto* pk = c.buf<uint64_t>("proj_keys", P1);
  auto* pk_sorted = c.buf<uint64_t>("proj_keys_sorted", P1);
  auto* pk_uniq = c.buf<uint64_t>("proj_keys_uniq", P1);
  sp.proj_base[0] = 0;
  for (int sub = 0; sub < n_sub; ++sub) {
    k_proj_keys<<<grid_for(P1), 256, 0, c.stream>>>(sp.pl_ids, P1, M, sub, pk);
    ++c.kernel_launches;
    const int nu = sort_unique(c, pk, pk_sorted, pk_uniq, P1);
    k_proj_assign<<<grid_for(P1), 256, 0, c.stream>>>(pk, P1, pk_uniq, nu, sp.proj_id + static_cast<size_t>(sub) * P1);
    ++c.kernel_launches;
    sp.proj_base[sub + 1] = sp.proj_base[sub] + nu;
  }
  sp.proj_total = sp.proj_base[n_sub];
  MGS_CUDA_OK(cudaGetLastError());
}

// precheck_scenario (solvers.hpp:27-69) over the device-built signature
// histogram. Messages follow the reference text with "<m>" standing in for
// the model name (the C++ drop-in re-renders them with names).
// precheck_scenario (solvers.hpp:27-69): every violation in the reference's
// order as (status code, model or -1).
std::vector<std::pair<int, int>> collect_violations(Ctx& c, const mgs_lattice& lat, const Prepared& pr,
                                                    const DevSpace& sp) {
  const HostTables& t = pr.t;
  std::vector<std::pair<int, int>> out;
  for (int m = 0; m < t.M; ++m) {
    bool anchor = false;
    for (int i = 0; i < lat.slot_offset[lat.n_configs]; ++i)
      if (lat.slot_size[i] >= t.floor_[m]) anchor = true;
    if (!anchor) {
      out.push_back({MGS_ERR_DEPLOYMENT_FLOOR, m});
      continue;
    }
    if (t.min_rt[m] < 0) out.push_back({MGS_ERR_RETRAINING_WINDOW, m});
  }
  if (!out.empty()) return out;
  std::vector<int32_t> nopt(sp.n_sig, 0);
  if (sp.n_opt > 0) {
    MGS_CUDA_OK(cudaMemcpyAsync(nopt.data(), sp.sig_nopt, sp.n_sig * 4, cudaMemcpyDeviceToHost, c.stream));
    MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  }
  if (nopt[0] == 0) {
    out.push_back({MGS_ERR_DEPLOYMENT_FLOOR, -1});
    return out;
  }
  for (int m = 0; m < t.M; ++m) {
    bool co = false;
    for (int s = 0; s < sp.n_sig; ++s)
      if (nopt[s] > 0 && ((s >> (3 * m)) & 7)) co = true;
    if (!co) out.push_back({MGS_ERR_NO_COEXISTENCE, m});
  }
  return out;
}

void precheck_space(Ctx& c, const mgs_lattice& lat, const Prepared& pr, const DevSpace& sp) {
  const auto v = collect_violations(c, lat, pr, sp);
  if (v.empty()) return;
  const int code = v.front().first, m = v.front().second;
  const std::string who = "<" + std::to_string(m) + ">";
  std::string msg;
  if (code == MGS_ERR_DEPLOYMENT_FLOOR && m >= 0)
    msg = "deployment-floor unsatisfiable: no catalog instance reaches " + std::to_string(pr.t.floor_[m]) +
          " GPCs for model " + who;
  else if (code == MGS_ERR_DEPLOYMENT_FLOOR)
    msg = "deployment-floor unsatisfiable: no configuration deploys every inference task simultaneously";
  else if (code == MGS_ERR_RETRAINING_WINDOW)
    msg = "model " + who + ": every retraining time exceeds the window (" + std::to_string(pr.t.S) + " steps)";
  else
    msg = "no-coexistence-configuration: no configuration runs " + who + ":r alongside every inference task";
  throw PlanFail{code, msg, 0, 0, m};
}

}  // namespace mgs
