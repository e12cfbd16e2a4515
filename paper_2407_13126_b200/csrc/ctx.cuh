// Library context: one device, one stream, grow-only scratch pools.
#pragma once

#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "common.cuh"

namespace mgs {

// Grow-only device allocation; contents are NOT preserved on growth.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    size_t bytes = n * sizeof(T);
    if (bytes == 0) bytes = sizeof(T);
    if (bytes > cap) {
      if (p) MGS_CUDA_OK(cudaFree(p));
      size_t want = bytes + bytes / 4 + 256;
      MGS_CUDA_OK(cudaMalloc(&p, want));
      cap = want;
    }
    return static_cast<T*>(p);
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

// Pinned host staging for small device->host reads.
struct HostPinned {
  void* p = nullptr;
  size_t cap = 0;
  template <class T>
  T* get(size_t n) {
    size_t bytes = n * sizeof(T);
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      MGS_CUDA_OK(cudaMallocHost(&p, bytes));
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
};

// Planner failure carrying the reference's error code (mgs_status) and text.
struct PlanFail {
  int code;
  std::string msg;
  int step = 0;
  uint64_t frontier = 0;
  int model = -1;
};

// History arena: per-step (parent, option) arrays kept for the backtrack;
// chunks are reused across solves.
struct History {
  std::vector<void*> chunks;
  std::vector<size_t> chunk_cap;  // int32 entries
  size_t cur = 0, used = 0;
  std::vector<int32_t*> parent, option;
  void reset() {
    cur = 0;
    used = 0;
    parent.clear();
    option.clear();
  }
  void take(size_t n, int32_t** p, int32_t** o) {
    const size_t need = 2 * n + 64;
    while (cur < chunks.size() && used + need > chunk_cap[cur]) {
      ++cur;
      used = 0;
    }
    if (cur == chunks.size()) {
      const size_t cap = need > (size_t(64) << 20) ? need : (size_t(64) << 20);
      void* ptr = nullptr;
      MGS_CUDA_OK(cudaMalloc(&ptr, cap * 4));
      chunks.push_back(ptr);
      chunk_cap.push_back(cap);
      used = 0;
    }
    int32_t* base = static_cast<int32_t*>(chunks[cur]) + used;
    *p = base;
    *o = base + n;
    used += need;
    parent.push_back(*p);
    option.push_back(*o);
  }
  void release() {
    for (void* q : chunks) cudaFree(q);
    chunks.clear();
    chunk_cap.clear();
    reset();
  }
};

// Per-phase device timing: event pairs recorded on the solve stream, summed
// after the solve (no extra synchronisation inside the step loop).
struct PhaseTimer {
  std::vector<cudaEvent_t> pool;
  size_t next = 0;
  struct Rec {
    int phase;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  cudaEvent_t get() {
    if (next == pool.size()) {
      cudaEvent_t e;
      MGS_CUDA_OK(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[next++];
  }
  void reset() {
    next = 0;
    recs.clear();
  }
  void release() {
    for (auto e : pool) cudaEventDestroy(e);
    pool.clear();
    reset();
  }
};

struct Ctx;
void shard_release(Ctx& c);  // shard.cu: destroys an owned NCCL communicator

struct Ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;      // the stream all work goes to
  cudaStream_t own_stream = nullptr;  // created by mgs_open
  PhaseTimer timer;
  int open_phase = -1;
  cudaEvent_t open_ev = nullptr;
  void phase(int p) {  // closes the open phase (if any) and opens p (-1: none)
    if (open_phase >= 0) {
      cudaEvent_t e = timer.get();
      MGS_CUDA_OK(cudaEventRecord(e, stream));
      timer.recs.push_back({open_phase, open_ev, e});
    }
    open_phase = p;
    if (p >= 0) {
      open_ev = timer.get();
      MGS_CUDA_OK(cudaEventRecord(open_ev, stream));
    }
  }
  void phase_totals(double* out8) {
    for (int i = 0; i < 8; ++i) out8[i] = 0.0;
    for (auto& r : timer.recs) {
      float ms = 0.f;
      MGS_CUDA_OK(cudaEventElapsedTime(&ms, r.a, r.b));
      out8[r.phase] += ms;
    }
  }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::map<std::string, DevBuf> bufs;
  HostPinned pinned;
  uint64_t kernel_launches = 0;
  History history;
  std::map<std::string, cudaGraphExec_t> graphs;  // cached per-window kernel sequences
  // batched-table cache: the option space and Pareto rows of the last window
  // shape (lattice + tables bytes), kept under the "tab/" buffer prefix
  std::string table_key;
  int table_np = 0;
  double* table_wcp = nullptr;

  // Buffer names are looked up under `prefix`: a batched solve sets a
  // per-lane prefix so every lane owns a disjoint set of scratch buffers.
  std::string prefix;
  template <class T>
  T* buf(const char* name, size_t n) {
    return bufs[prefix + name].get<T>(n);
  }
  // multi-GPU sharding (shard.cu): this rank's NCCL communicator
  void* nccl_comm = nullptr;
  bool own_comm = false;
  int world = 1, rank = 0;
  ~Ctx() {
    shard_release(*this);
    for (auto& kv : bufs) kv.second.release();
    history.release();
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    if (pinned.p) cudaFreeHost(pinned.p);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    timer.release();
    if (own_stream) cudaStreamDestroy(own_stream);
  }
};

}  // namespace mgs

// the opaque handle of the C ABI
struct mgs_ctx {
  mgs::Ctx c;
};

namespace mgs {

// Host-side derived inputs of one window (engine::Tables + initial masks).
struct Prepared {
  HostTables t;
  std::vector<int> slot_uid;        // universe id per flat slot
  int n_universe = 0;
  int has_initial = 0;
  uint32_t init_mask[KM] = {0, 0, 0, 0};
};

// space.cu
Prepared prepare_tables(const mgs_lattice& lat, const mgs_tables& tab);
void build_space(Ctx& c, const mgs_lattice& lat, const Prepared& pr, DevSpace& sp);
void precheck_space(Ctx& c, const mgs_lattice& lat, const Prepared& pr, const DevSpace& sp);
std::vector<std::pair<int, int>> collect_violations(Ctx& c, const mgs_lattice& lat, const Prepared& pr,
                                                    const DevSpace& sp);
// bruteforce.cu: solve_bruteforce; false when no feasible all-done sequence
bool bruteforce(Ctx& c, const Prepared& pr, const DevSpace& sp, const double* d_recv, std::vector<int32_t>& plan);
// wb.cu: plan_window_boundary; false when no k-vector is realizable
bool window_boundary(Ctx& c, const Prepared& pr, const DevSpace& sp, const mgs_lattice& lat, const double* d_recv,
                     std::vector<int32_t>& plan);
// replay.cu: run_requests for plans x traces x seeds
void replay_requests(Ctx& c, const Prepared& pr, const DevSpace& sp, int W, const double* d_acc, const double* psi,
                     const double* slo, double step_seconds, const int32_t* d_plans, const uint8_t* d_overrides,
                     int n_plans,
                     const int64_t* d_arr, int n_traces, const uint64_t* d_seeds, int n_seeds, mgs_job_metrics* d_out);
// preinit.cu: plan_preinit + apply_preinit overrides [n_plans][S][M], fired [n_plans][S]
void preinit_overrides(Ctx& c, const Prepared& pr, const DevSpace& sp, const mgs_lattice& lat, const int32_t* d_plans,
                       int n_plans, uint8_t* d_overrides, uint32_t* d_fired);
// feasible.cu: plans as general per-step allocations (config + per-slot task bits)
struct ViewSet {
  void* views;  // device [n_steps] resolved steps
  long long n;
};
ViewSet upload_views(Ctx& c, const mgs_lattice& lat, const Prepared& pr, const int32_t* config, const uint8_t* tasks,
                     long long n_steps);
void check_views(Ctx& c, const Prepared& pr, const ViewSet& v, int n_plans, mgs_plan_violation* d_out, int cap,
                 int32_t* d_n);
void evaluate_views(Ctx& c, const Prepared& pr, const ViewSet& v, int n_plans, const double* d_psi,
                    const int64_t* d_arr, int n_traces, double* d_total, mgs_score_entry* d_entries);
void fluid_views(Ctx& c, const Prepared& pr, int W, const ViewSet& v, int n_plans, const double* d_psi,
                 const double* d_acc, const int64_t* d_arr, int n_traces, double step_seconds, mgs_job_metrics* d_out);
// table.cu: batched ub table (Pareto placements prepared once per window shape)
int table_prepare(Ctx& c, const Prepared& pr, const DevSpace& sp, double** wcp_out);
void table_run(Ctx& c, const Prepared& pr, const double* wcp, int np, const int32_t* d_arr, int n_traces,
               double* d_best, double* d_ub);
// goodput.cu
void goodput_reductions(Ctx& c, const Prepared& pr, const DevSpace& sp, const double* d_recv, double* d_ub,
                        double* d_incumbent, int32_t* d_greedy);
// dp.cu
struct SolveOut {
  std::vector<int32_t> options;        // host copy (batched / multi-launch paths)
  const int32_t* d_options = nullptr;  // device copy of the chosen options (device-resident engine)
  mgs_stats stats{};
};
void solve_dp(Ctx& c, const mgs_problem& p, const Prepared& pr, const DevSpace& sp, const double* d_recv,
              const double* d_ub, const double* d_incumbent, SolveOut& out);
// dp2.cu: the device-resident engine (M <= 2); several independent windows of
// equal shape ("lanes") run in the same kernels (grid.y = lane).
constexpr int kMaxLanes = 32;
struct V2Lane {
  const mgs_problem* p = nullptr;
  const Prepared* pr = nullptr;
  const DevSpace* sp = nullptr;
  const double* recv = nullptr;
  const double* ub = nullptr;
  const double* incumbent = nullptr;
  std::string prefix;  // the lane's buffer-name prefix
  bool host_options = true;  // copy the chosen options to out.options (else only out.d_options)
  SolveOut out;
  int status = 0;      // mgs_status of this lane
  std::string msg;
  int err_step = 0;
  uint64_t err_count = 0;
};
bool solve_dp_v2_supported(const Prepared& pr, const DevSpace& sp);
void solve_dp_v2_lanes(Ctx& c, std::vector<V2Lane>& lanes);

// small device helpers (scan.cu)
void exclusive_scan_i32(Ctx& c, const int32_t* in, int32_t* out, int n);  // out has n+1 entries
void exclusive_scan_u32(Ctx& c, const uint32_t* in, uint32_t* out, int n);

template <class T>
inline T read_scalar(Ctx& c, const T* dptr) {
  T* h = c.pinned.get<T>(1);
  MGS_CUDA_OK(cudaMemcpyAsync(h, dptr, sizeof(T), cudaMemcpyDeviceToHost, c.stream));
  MGS_CUDA_OK(cudaStreamSynchronize(c.stream));
  return *h;
}

inline unsigned ceil_div(long long a, long long b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace mgs
