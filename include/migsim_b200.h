/* migsim_b200.h — C ABI of the B200 Goodput-planner hot path.
 *
 * Plain C, POD structs, caller-owned host buffers, library-owned device state.
 * This is the thin layer under the unchanged C++ planner API: the C++ drop-in
 * (paper_2407_13126_b200/csrc/host/migsim/*.hpp) marshals a
 * migsim::PlanContext into an mgs_problem and rethrows mgs_error as
 * migsim::Error(code, message). Python (ctypes) and any other FFI bind the same
 * symbols; see INTEGRATION.md.
 *
 * Reference interfaces each entry point replaces (paths relative to the
 * reference root, proj/include/migsim/):
 *   mgs_enumerate      engine::Space::build            space.hpp:126-210
 *   mgs_precheck       precheck_scenario               solvers.hpp:27-69
 *   mgs_goodput_table  solve_dp ub_suffix + incumbent  solvers.hpp:258-322
 *   mgs_solve_window   solve_dp                        solvers.hpp:242-579
 *   mgs_bruteforce     solve_bruteforce                solvers.hpp:143-228
 *   mgs_precheck       precheck_scenario (all violations, reference order)
 *   mgs_solve_batch    solve_dp over independent windows (the reference's
 *                      per-scenario call in a host loop)
 *   mgs_evaluate_batch evaluate_plan(verify=false)     evaluate.hpp:153-210
 *   mgs_window_boundary plan_window_boundary         baselines.hpp:139-289
 *   mgs_replay_requests run_requests                   simulator.hpp:209-275
 *   mgs_preinit        plan_preinit + apply_preinit    preinit.hpp:41-114
 *   mgs_goodput_table_batch  solve_dp's ub_suffix table  solvers.hpp:258-280
 *                      for a batch of traces sharing one window's tables
 *   mgs_check_feasible_batch check_feasible            evaluate.hpp:55-146
 *   mgs_evaluate_views_batch evaluate_plan (any allocation, verify optional)
 *                                                      evaluate.hpp:25-47,153-210
 *   mgs_run_fluid      run_fluid (+ build_series)      simulator.hpp:72-131,171-203
 *   mgs_shard_*, mgs_solve_batch_sharded: one process per GPU over NCCL
 *                      (no reference analogue: the reference is single-node,
 *                      single-process)
 */
#ifndef MIGSIM_B200_H
#define MIGSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define MGS_API __attribute__((visibility("default")))
#else
#define MGS_API
#endif

#define MGS_MAX_MODELS 4  /* engine::kMaxModels, space.hpp:17 */
#define MGS_MAX_SLOTS 8   /* slots per configuration (gpc_count <= 8) */
#define MGS_SIZES 8       /* tables indexed by instance size 0..7 (space.hpp:39-40) */
#define MGS_FOREIGN_MASK 0xffffffffu /* engine::kForeignMask, space.hpp:303 */

/* Status codes map 1:1 onto the reference's migsim::Error code strings
 * (mgs_status_code() returns the string). */
typedef enum {
  MGS_OK = 0,
  MGS_ERR_INPUT_SCENARIO = 1,          /* "input.scenario"   space.hpp:49-50 */
  MGS_ERR_INPUT_CATALOG = 2,           /* "input.catalog"    space.hpp:65 */
  MGS_ERR_INPUT_FORECAST = 3,          /* "input.forecast"   solvers.hpp:250-252 */
  MGS_ERR_INPUT_ARRIVALS = 4,          /* "input.arrivals"   evaluate.hpp:166-167 */
  MGS_ERR_DEPLOYMENT_FLOOR = 5,        /* "infeasible.deployment-floor" solvers.hpp:38,51 */
  MGS_ERR_RETRAINING_WINDOW = 6,       /* "infeasible.retraining-window" solvers.hpp:44 */
  MGS_ERR_NO_COEXISTENCE = 7,          /* "infeasible.no-coexistence-configuration" :62 */
  MGS_ERR_INFEASIBLE_JOINT = 8,        /* "infeasible.joint" solvers.hpp:348,565 */
  MGS_ERR_STATE_BUDGET = 9,            /* "planner.state-budget" solvers.hpp:539-542 */
  MGS_ERR_PLAN_INFEASIBLE = 10,        /* "plan.infeasible" evaluate.hpp:165 */
  MGS_ERR_CUDA = 11,                   /* device failure (no reference analogue) */
  MGS_ERR_ARGUMENT = 12,               /* null pointer / size out of range */
  MGS_ERR_BRUTEFORCE_CAP = 13,         /* "planner.bruteforce-cap" solvers.hpp:153-158 */
  MGS_ERR_WINDOW_BOUNDARY = 14         /* "infeasible.window-boundary" baselines.hpp:280-281 */
} mgs_status;

typedef struct {
  int32_t code;        /* mgs_status */
  int32_t step;        /* planner.state-budget: step s+1 of the overflow */
  uint64_t frontier;   /* planner.state-budget: frontier size at that step */
  int32_t model;       /* precheck: offending model index, -1 if none */
  char message[320];   /* same text the reference puts in Error::what() */
} mgs_error;

/* The partition lattice: catalog configurations in file order, slots of each
 * configuration sorted by slice_start (catalog.hpp:141-142). */
typedef struct {
  int32_t n_configs;
  int32_t gpc_count;
  const int32_t* slot_offset; /* [n_configs+1] */
  const int32_t* slot_size;   /* [slot_offset[n_configs]] */
  const int32_t* slot_start;  /* [slot_offset[n_configs]] */
} mgs_lattice;

/* Per-window tables (engine::Tables, space.hpp:32-86). cap 0 = no capability,
 * rt -1 = undefined, exactly as Tables::build fills them. */
typedef struct {
  int32_t models; /* M, 1..4 */
  int32_t steps;  /* S */
  double cap_by_size[MGS_MAX_MODELS][MGS_SIZES];
  int64_t rt_by_size[MGS_MAX_MODELS][MGS_SIZES];
  int32_t floor_gpcs[MGS_MAX_MODELS];
  double psi[MGS_MAX_MODELS];       /* loss fraction = min(psi, 1), plan_types.hpp:68 */
  double acc_pre[MGS_MAX_MODELS];   /* accuracy of window w (PlanContext::accuracy_pre) */
  double acc_post[MGS_MAX_MODELS];
} mgs_tables;

/* One planning window (PlanContext + ArrivalForecast + SolveOptions). */
typedef struct {
  mgs_lattice lattice;
  mgs_tables tables;
  const int64_t* forecast;            /* [models][forecast_len] row-major */
  int32_t forecast_len;               /* must equal steps (input.forecast otherwise) */
  int32_t has_initial;                /* PlanContext::initial present */
  uint32_t init_mask[MGS_MAX_MODELS]; /* initial_masks(): universe bit masks */
  uint64_t state_budget;              /* SolveOptions::state_budget (4,000,000) */
  int32_t workers;                    /* accepted; results never depend on it */
} mgs_problem;

typedef struct {
  uint64_t options;          /* |O|, Space::options.size() */
  uint64_t candidates;       /* distinct (signature, inference-placement) pairs */
  uint64_t transitions_ref;  /* reference inner-loop trips, solvers.hpp:424-469 */
  uint64_t transitions;      /* (unit, candidate) pairs the GPU evaluated */
  uint64_t frontier_total;   /* sum over steps of surviving states */
  uint64_t frontier_peak;
  double device_ms;          /* device time of the solve (CUDA events) */
  uint64_t kernel_launches;  /* launches of this library's own kernels */
  /* per-phase device time (CUDA events on the solve stream), ms:
   * [0] enumeration + tables  [1] Goodput reductions  [2] unit expansion
   * [3] transitions           [4] merge/band/dominance [5] compaction
   * [6] lex ranks             [7] terminal + backtrack + objective */
  double phase_ms[8];
  /* algorithmic bytes of the transition kernels over the solve: every
   * frontier state read once (value, rank, ids: 20 B), every candidate
   * descriptor read once (8 B) and every candidate record written (29 B) */
  uint64_t transition_bytes;
} mgs_stats;

/* One precheck_scenario violation (solvers.hpp:27-69): code is
 * MGS_ERR_DEPLOYMENT_FLOOR / MGS_ERR_RETRAINING_WINDOW / MGS_ERR_NO_COEXISTENCE,
 * model the offending tenant or -1 (the "no configuration deploys every
 * inference task" case). The host wrapper formats the reference's message. */
typedef struct {
  int32_t code;
  int32_t model;
} mgs_violation;

/* JobMetrics counters of one tenant (simulator.hpp:17-32); the fractions
 * (goodput, slo_attainment, accuracy) follow from them (finalize_fractions). */
typedef struct {
  double received, served, timely, correct, valid, dropped, queued_at_end;
  int32_t reconfigurations;
  double overhead_seconds;
} mgs_job_metrics;

/* check_feasible violation families (evaluate.hpp:82-144); the host wrapper
 * formats the reference's message from code/step/model/detail. */
typedef enum {
  MGS_VIOL_DEPLOYMENT_FLOOR = 1,        /* "deployment-floor": detail[0] = GPC-sum check satisfied, detail[1] = L */
  MGS_VIOL_RETRAINING_NOT_LAUNCHED = 2, /* "retraining-not-launched" (step -1) */
  MGS_VIOL_RETRAINING_INTERRUPTED = 3,  /* "retraining-interrupted": detail[0] = run contiguous (size changed) */
  MGS_VIOL_RETRAINING_SIZE = 4,         /* "retraining-size": detail[0] = k */
  MGS_VIOL_RETRAINING_INCOMPLETE = 5,   /* "retraining-incomplete": detail = run length, RT, k */
  MGS_VIOL_RETRAINING_OVERRUN = 6       /* "retraining-overrun": detail = run length, RT, k */
} mgs_violation_family;

typedef struct {
  int32_t code;    /* mgs_violation_family */
  int32_t step;    /* Violation::second (-1 for not-launched) */
  int32_t model;   /* tenant index */
  int32_t detail[3];
} mgs_plan_violation;

/* One evaluate_plan breakdown entry (plan_types.hpp:38-45). */
typedef struct {
  double throughput;     /* SLO-attained requests of the step */
  double overhead_loss;  /* loss_frac * raw capability */
  double goodput;        /* throughput * accuracy */
  int32_t completion;    /* retraining finished strictly before the step */
  int32_t pad;
} mgs_score_entry;

typedef struct mgs_ctx mgs_ctx;

MGS_API int mgs_open(int device, mgs_ctx** out);
MGS_API void mgs_close(mgs_ctx* ctx);
MGS_API const char* mgs_status_code(int status);
MGS_API const char* mgs_version(void);
/* Run this context's work on a caller-provided cudaStream_t (e.g. a framework's
 * current stream, so the caller's events time it). NULL restores the
 * context's own stream. */
MGS_API int mgs_set_stream(mgs_ctx* ctx, void* stream);

/* Candidate enumeration (Space::build). *n_options receives |O|. Optional
 * host copies (pass NULL to skip) hold min(cap, |O|) options in lex order:
 * config[i], labels[i*MGS_MAX_SLOTS + slot], infer_mask[i*4+m],
 * infer_cap[i*4+m], retrain_size[i*4+m]. */
MGS_API int mgs_enumerate(mgs_ctx* ctx, const mgs_lattice* lattice, const mgs_tables* tables, int64_t* n_options,
                  int64_t cap, int32_t* config, int8_t* labels, uint32_t* infer_mask, double* infer_cap,
                  int8_t* retrain_size, mgs_error* err);

/* Goodput table reductions used by solve_dp before the search: the
 * optimistic per-step bound ub_suffix[0..S] (solvers.hpp:270-280) and the
 * greedy incumbent (solvers.hpp:283-322; -inf when the greedy walk does not
 * finish every retraining). greedy_option[s] = chosen option or -1. */
MGS_API int mgs_goodput_table(mgs_ctx* ctx, const mgs_problem* p, double* ub_suffix, double* incumbent,
                      int32_t* greedy_option, mgs_error* err);

/* solve_dp on one window. out_option[s] = option index (lex rank) chosen at
 * step s; out_config[s] / out_labels[s*MGS_MAX_SLOTS+slot] its configuration
 * and per-slot labels (0 unused, 1+2m inference m, 2+2m retraining m);
 * *out_objective = evaluate_plan(...).total of that plan. Any output pointer
 * may be NULL. */
MGS_API int mgs_solve_window(mgs_ctx* ctx, const mgs_problem* p, int32_t* out_option, int32_t* out_config,
                     int8_t* out_labels, double* out_objective, mgs_stats* stats, mgs_error* err);

/* precheck_scenario: writes up to cap violations (reference order) and the
 * total count to *n_out. Returns MGS_OK even when violations exist; input
 * errors (input.scenario / input.catalog) are returned as status codes. */
MGS_API int mgs_precheck(mgs_ctx* ctx, const mgs_lattice* lattice, const mgs_tables* tables, mgs_violation* out,
                         int32_t cap, int32_t* n_out, mgs_error* err);

/* solve_bruteforce on one window: every allocation sequence scored on the
 * device, best by (objective desc, option-index sequence asc). Gated like the
 * reference by |O|^S <= bruteforce_cap (MGS_ERR_BRUTEFORCE_CAP otherwise).
 * Outputs as for mgs_solve_window. */
MGS_API int mgs_bruteforce(mgs_ctx* ctx, const mgs_problem* p, double bruteforce_cap, int32_t* out_option,
                           int32_t* out_config, int8_t* out_labels, double* out_objective, mgs_error* err);

/* n independent windows (different scenarios / traces) solved back to back on
 * the device; per-problem outputs at out_option[i*S_max...], status[i],
 * objective[i]. Returns MGS_OK if the call itself ran (per-problem errors are
 * in status[]/errs[]). */
MGS_API int mgs_solve_batch(mgs_ctx* ctx, const mgs_problem* problems, int32_t n, int32_t s_max, int32_t* out_option,
                    double* out_objective, int32_t* status, mgs_stats* stats, mgs_error* errs);

/* evaluate_plan(verify_feasibility=false) for n_plans plans x n_traces traces
 * sharing one window's tables: plans[i*S+s] = option index,
 * arrivals[t*M*S + m*S + s]. total[i*n_traces+t] = objective;
 * throughput (optional, [i][t][s][m]) = SLO-attained counts. overrides
 * (optional, [i][s][m], nonzero = psi_eff 0) are OverheadOverrides, e.g. the
 * pre-initialisation result of mgs_preinit. */
MGS_API int mgs_evaluate_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* plans, int32_t n_plans,
                       const uint8_t* overrides, const int64_t* arrivals, int32_t n_traces, double* total,
                       double* throughput, mgs_error* err);

/* Pre-initialisation (plan_preinit + apply_preinit, preinit.hpp:41-114) of
 * n_plans plans: overrides[i*S*M + s*M + m] = 1 where tenant m's overhead at
 * step s drops to 0 (every instance it acquires was created early on unused
 * slices during s-1); fired (optional) [i*S+s] = universe-id bitmask
 * (instances in first-appearance order over the lattice) created early during
 * step s. */
MGS_API int mgs_preinit(mgs_ctx* ctx, const mgs_problem* p, const int32_t* plans, int32_t n_plans, uint8_t* overrides,
                        uint32_t* fired, mgs_error* err);

/* plan_window_boundary (the Ekya-like comparison planner): retraining starts
 * at step 0, the allocation changes only at step 0 and at retraining
 * completions; exhaustive over per-tenant GPC counts with a phase DP on the
 * device. Outputs as for mgs_solve_window (objective = evaluate_plan total). */
MGS_API int mgs_window_boundary(mgs_ctx* ctx, const mgs_problem* p, int32_t* out_option, int32_t* out_config,
                                int8_t* out_labels, double* out_objective, mgs_error* err);

/* Request-mode replay (run_requests, simulator.hpp:209-275) of a scenario's
 * `windows` consecutive windows (one window's tables in p; queues, psi spill
 * and inference masks carry across windows) for n_plans x n_traces x n_seeds
 * runs on the device. plans[(i*windows + w)*S + s] option indices;
 * arrivals[t*M*windows*S + m*windows*S + g] (g = w*S + s); seeds[k];
 * acc_pre/acc_post [w*M + m] per-window accuracies (NULL with windows == 1:
 * p's tables); slo[m] = 2*latency_full (seconds); step_seconds =
 * Scenario::step_seconds; overrides [(i*windows + w)*S + s][m] as for
 * mgs_evaluate_batch (EffectivePlan::overrides) or NULL.
 * out[((run*windows + w)*M + m)], run = (i*n_traces + t)*n_seeds + k: the
 * per-window JobMetrics (totals = their sums in window order). */
MGS_API int mgs_replay_requests(mgs_ctx* ctx, const mgs_problem* p, int32_t windows, const double* acc_pre,
                                const double* acc_post, const double* slo, double step_seconds, const int32_t* plans,
                                int32_t n_plans, const uint8_t* overrides, const int64_t* arrivals, int32_t n_traces,
                                const uint64_t* seeds, int32_t n_seeds, mgs_job_metrics* out, mgs_error* err);

/* The Goodput table for n_traces traces that share one window's lattice and
 * tables (configs 2/4): best[b*S+s] = max(0, max over candidates of
 * sum_m acc_max[m]*min(recv, cap)) and ub_suffix[b*(S+1)+s] its suffix sums
 * (solvers.hpp:270-280), bit-identical to the per-window solve.
 * arrivals[b*M*S + m*S + s] are int32 counts. mgs_goodput_table_batch takes
 * host buffers; the _device variant takes device pointers on the context's
 * stream (inputs already resident in HBM) and does not synchronise.
 * *n_pareto (optional) receives the number of Pareto-maximal placements the
 * table kernel scanned. best may be NULL. */
MGS_API int mgs_goodput_table_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* arrivals, int32_t n_traces,
                                    double* best, double* ub_suffix, int32_t* n_pareto, mgs_error* err);
MGS_API int mgs_goodput_table_batch_device(mgs_ctx* ctx, const mgs_problem* p, const int32_t* d_arrivals,
                                           int32_t n_traces, double* d_best, double* d_ub_suffix, int32_t* n_pareto,
                                           mgs_error* err);

/* Plans as general per-step allocations (any sequence resolve_step reads,
 * evaluate.hpp:25-47): step_config[i*S+s] = configuration index (lattice
 * order); slot_tasks[(i*S+s)*MGS_MAX_SLOTS + k] = task bits of slot k of that
 * configuration: bit 2m = inference task of tenant m, bit 2m+1 = its
 * retraining task (several bits = a shared instance). String-level checks
 * (unknown ids, second-index, validate_allocation) belong to the caller.
 *
 * check_feasible's constraint families for n_plans plans: up to cap records
 * per plan at out[i*cap...] in the reference's order, n_out[i] = total count
 * (0 = feasible). */
MGS_API int mgs_check_feasible_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* step_config,
                                     const uint8_t* slot_tasks, int32_t n_plans, mgs_plan_violation* out, int32_t cap,
                                     int32_t* n_out, mgs_error* err);

/* evaluate_plan of n_plans general plans x n_traces traces (arrivals
 * [t][M][S]); psi_override (optional) [i][s][m] replaces the profile psi where
 * it is not NaN (OverheadOverrides). total[i*n_traces+t]; entries (optional)
 * [i][t][s][m]. verify != 0 runs check_feasible first: status[i] (required
 * then) = MGS_ERR_PLAN_INFEASIBLE and first[i] (optional) = the first
 * violation for infeasible plans, whose totals are left 0. */
MGS_API int mgs_evaluate_views_batch(mgs_ctx* ctx, const mgs_problem* p, const int32_t* step_config,
                                     const uint8_t* slot_tasks, int32_t n_plans, const double* psi_override,
                                     const int64_t* arrivals, int32_t n_traces, int32_t verify, double* total,
                                     mgs_score_entry* entries, int32_t* status, mgs_plan_violation* first,
                                     mgs_error* err);

/* run_fluid: fluid-mode replay of `windows` consecutive windows of n_plans
 * general plans (step_config / slot_tasks [i][w][s], psi_override
 * [i][w][s][m] or NULL) against n_traces traces (arrivals [t][M][windows*S]);
 * acc_pre/acc_post [w*M+m] (NULL with windows == 1: p's tables).
 * out[((i*n_traces + t)*windows + w)*M + m] = per-window JobMetrics. */
MGS_API int mgs_run_fluid(mgs_ctx* ctx, const mgs_problem* p, int32_t windows, const double* acc_pre,
                          const double* acc_post, double step_seconds, const int32_t* step_config,
                          const uint8_t* slot_tasks, int32_t n_plans, const double* psi_override,
                          const int64_t* arrivals, int32_t n_traces, mgs_job_metrics* out, mgs_error* err);

/* ---- multi-GPU sharding over NCCL (one process per GPU) ----------------
 * NCCL is loaded at run time (libnccl.so.2). A context holds one
 * communicator: create it with mgs_shard_init (rank 0 calls
 * mgs_nccl_unique_id and shares the bytes with the other ranks out of band),
 * or attach a caller-owned ncclComm_t with mgs_shard_attach. Collectives run
 * on the context's stream. */
#define MGS_NCCL_ID_BYTES 128
MGS_API int mgs_nccl_unique_id(uint8_t* id /* [MGS_NCCL_ID_BYTES] */);
MGS_API int mgs_shard_init(mgs_ctx* ctx, int32_t world, int32_t rank, const uint8_t* id, mgs_error* err);
MGS_API int mgs_shard_attach(mgs_ctx* ctx, void* nccl_comm, int32_t world, int32_t rank);
/* recv[world*n] = every rank's n values, rank-major */
MGS_API int mgs_shard_allgather_i64(mgs_ctx* ctx, const int64_t* send, int64_t n, int64_t* recv, mgs_error* err);
/* per-shard best: *best = max objective over the ranks (objective >= 0),
 * *owner = lowest rank holding it (all-reduce(max) of the order-preserving
 * bits, then all-reduce(min) of the owner) */
MGS_API int mgs_shard_best(mgs_ctx* ctx, double objective, double* best, int32_t* owner, mgs_error* err);
/* mgs_solve_batch over the ranks: every rank passes all n windows; rank r
 * solves [n*r/world, n*(r+1)/world) and the (status, objective, plan) rows are
 * all-gathered, so every rank returns all n results. Without a communicator
 * it solves all n windows locally. */
MGS_API int mgs_solve_batch_sharded(mgs_ctx* ctx, const mgs_problem* problems, int32_t n, int32_t s_max,
                                    int32_t* out_option, double* out_objective, int32_t* status, mgs_error* err);

#ifdef __cplusplus
}
#endif
#endif
