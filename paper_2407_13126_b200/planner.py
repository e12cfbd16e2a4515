"""Python host API over the C ABI — the same operations as the reference's C++
planner API (solve_dp, evaluate_plan, Space::build, ...), on B200.

Every call goes through lib/libmigsim_b200.so (CUDA). There is no CPU path: if
the library or a GPU is missing the calls raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi
from .scenario import Problem


class Planner:
    """One device context (mgs_open). Not shared across threads."""

    def __init__(self, device: int = 0):
        self.lib = capi.load()
        h = C.c_void_p()
        st = self.lib.mgs_open(device, C.byref(h))
        if st != 0:
            raise capi.PlannerError(st)
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.mgs_close(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- engine::Space::build -------------------------------------------------
    def enumerate(self, problem: Problem):
        n = C.c_int64()
        err = capi.empty_error()
        lat, tab = C.byref(problem.c.lattice), C.byref(problem.c.tables)
        st = self.lib.mgs_enumerate(self.h, lat, tab, C.byref(n), 0, None, None, None, None, None, C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        N = n.value
        out = dict(config=np.zeros(N, np.int32), labels=np.zeros((N, capi.MAX_SLOTS), np.int8),
                   mask=np.zeros((N, 4), np.uint32), cap=np.zeros((N, 4), np.float64),
                   rsize=np.zeros((N, 4), np.int8))
        st = self.lib.mgs_enumerate(self.h, lat, tab, C.byref(n), N, capi.ptr(out["config"], C.c_int32),
                                    capi.ptr(out["labels"], C.c_int8), capi.ptr(out["mask"], C.c_uint32),
                                    capi.ptr(out["cap"], C.c_double), capi.ptr(out["rsize"], C.c_int8), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return out

    # -- ub_suffix + greedy incumbent ------------------------------------------
    def goodput_table(self, problem: Problem):
        ub = np.zeros(problem.S + 1, np.float64)
        inc = C.c_double()
        greedy = np.zeros(problem.S, np.int32)
        err = capi.empty_error()
        st = self.lib.mgs_goodput_table(self.h, problem.byref(), capi.ptr(ub, C.c_double), C.byref(inc),
                                        capi.ptr(greedy, C.c_int32), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return ub, inc.value, greedy

    # -- solve_dp ---------------------------------------------------------------
    def solve_window(self, problem: Problem):
        """Returns (options[S], config[S], labels[S][8], objective, stats)."""
        S = problem.S
        opt = np.zeros(S, np.int32)
        cfg = np.zeros(S, np.int32)
        lab = np.zeros((S, capi.MAX_SLOTS), np.int8)
        obj = C.c_double()
        stats = capi.mgs_stats()
        err = capi.empty_error()
        st = self.lib.mgs_solve_window(self.h, problem.byref(), capi.ptr(opt, C.c_int32), capi.ptr(cfg, C.c_int32),
                                       capi.ptr(lab, C.c_int8), C.byref(obj), C.byref(stats), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return opt, cfg, lab, obj.value, stats.as_dict()

    # -- precheck_scenario -------------------------------------------------------
    def precheck(self, problem: Problem):
        """All violations as [(code string, model or -1)], reference order."""
        out = (capi.mgs_violation * 16)()
        n = C.c_int32()
        err = capi.empty_error()
        st = self.lib.mgs_precheck(self.h, C.byref(problem.c.lattice), C.byref(problem.c.tables), out, 16,
                                   C.byref(n), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return [(capi.STATUS_CODES[out[i].code], out[i].model) for i in range(min(n.value, 16))]

    # -- solve_bruteforce -------------------------------------------------------
    def solve_bruteforce(self, problem: Problem, bruteforce_cap: float = 5e7):
        """Returns (options[S], config[S], labels[S][8], objective)."""
        S = problem.S
        opt = np.zeros(S, np.int32)
        cfg = np.zeros(S, np.int32)
        lab = np.zeros((S, capi.MAX_SLOTS), np.int8)
        obj = C.c_double()
        err = capi.empty_error()
        st = self.lib.mgs_bruteforce(self.h, problem.byref(), float(bruteforce_cap), capi.ptr(opt, C.c_int32),
                                     capi.ptr(cfg, C.c_int32), capi.ptr(lab, C.c_int8), C.byref(obj), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return opt, cfg, lab, obj.value

    # -- plan_window_boundary (baselines.hpp:139-289) ----------------------------
    def window_boundary(self, problem: Problem):
        """Returns (options[S], config[S], labels[S][8], objective)."""
        S = problem.S
        opt = np.zeros(S, np.int32)
        cfg = np.zeros(S, np.int32)
        lab = np.zeros((S, capi.MAX_SLOTS), np.int8)
        obj = C.c_double()
        err = capi.empty_error()
        st = self.lib.mgs_window_boundary(self.h, problem.byref(), capi.ptr(opt, C.c_int32), capi.ptr(cfg, C.c_int32),
                                          capi.ptr(lab, C.c_int8), C.byref(obj), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return opt, cfg, lab, obj.value

    # -- run_requests (simulator.hpp:209-275) ---------------------------------------
    def replay_requests(self, problem: Problem, plans, arrivals, seeds, step_seconds=1.0, overrides=None,
                        windows=1):
        """Request-mode replay of `windows` consecutive windows (queues, psi spill
        and masks carry across them). plans [n_p][W*S] option indices (window
        after window), arrivals [n_t][M][W*S], seeds [n_s], overrides (optional)
        [n_p][W*S][M] psi_eff-zero flags (mgs_preinit). Per-window accuracies
        come from problem.scenario. Returns mgs_job_metrics as a structured
        numpy array [n_p][n_t][n_s][M] (W = 1) or [n_p][n_t][n_s][W][M]."""
        W, S, M = windows, problem.S, problem.M
        plans = np.ascontiguousarray(plans, dtype=np.int32).reshape(-1, W * S)
        ov = None if overrides is None else np.ascontiguousarray(overrides, dtype=np.uint8).reshape(
            plans.shape[0], W * S, M)
        arrivals = np.ascontiguousarray(arrivals, dtype=np.int64).reshape(-1, M, W * S)
        seeds = np.ascontiguousarray(seeds, dtype=np.uint64).reshape(-1)
        models = problem.scenario.models
        slo = np.asarray([2.0 * m.latency_full for m in models], dtype=np.float64)  # slo_target
        w0 = problem.window
        acc_pre = np.asarray([[m.acc_pre[w0 + w] for m in models] for w in range(W)], np.float64)
        acc_post = np.asarray([[m.acc_post[w0 + w] for m in models] for w in range(W)], np.float64)
        n = plans.shape[0] * arrivals.shape[0] * seeds.shape[0] * W * M
        out = (capi.mgs_job_metrics * max(1, n))()
        err = capi.empty_error()
        st = self.lib.mgs_replay_requests(self.h, problem.byref(), W, capi.ptr(acc_pre, C.c_double),
                                          capi.ptr(acc_post, C.c_double), capi.ptr(slo, C.c_double),
                                          float(step_seconds), capi.ptr(plans, C.c_int32), plans.shape[0],
                                          capi.ptr(ov, C.c_uint8) if ov is not None else None,
                                          capi.ptr(arrivals, C.c_int64), arrivals.shape[0],
                                          capi.ptr(seeds, C.c_uint64), seeds.shape[0], out, C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        arr = np.ctypeslib.as_array(out)[:n].reshape(plans.shape[0], arrivals.shape[0], seeds.shape[0], W, M)
        return arr[:, :, :, 0, :] if W == 1 else arr

    # -- plan_preinit + apply_preinit (preinit.hpp:41-114) ------------------------
    def preinit(self, problem: Problem, plans):
        """Returns (overrides uint8 [n][S][M], fired uint32 [n][S] universe masks)."""
        plans = np.ascontiguousarray(plans, dtype=np.int32).reshape(-1, problem.S)
        n = plans.shape[0]
        ov = np.zeros((n, problem.S, problem.M), np.uint8)
        fired = np.zeros((n, problem.S), np.uint32)
        err = capi.empty_error()
        st = self.lib.mgs_preinit(self.h, problem.byref(), capi.ptr(plans, C.c_int32), n, capi.ptr(ov, C.c_uint8),
                                  capi.ptr(fired, C.c_uint32), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return ov, fired

    def solve_batch(self, problems):
        n = len(problems)
        s_max = max(p.S for p in problems)
        arr = (capi.mgs_problem * n)(*[p.c for p in problems])
        opts = np.full((n, s_max), -1, np.int32)
        obj = np.zeros(n, np.float64)
        status = np.zeros(n, np.int32)
        stats = (capi.mgs_stats * n)()
        errs = (capi.mgs_error * n)()
        st = self.lib.mgs_solve_batch(self.h, arr, n, s_max, capi.ptr(opts, C.c_int32), capi.ptr(obj, C.c_double),
                                      capi.ptr(status, C.c_int32), stats, errs)
        if st:
            raise capi.PlannerError(st)
        return opts, obj, status, [s.as_dict() for s in stats], errs

    # -- multi-GPU sharding over NCCL (C ABI, one process per GPU) --------------
    def shard_init(self, world: int, rank: int, nccl_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(nccl_id)
        err = capi.empty_error()
        st = self.lib.mgs_shard_init(self.h, world, rank, buf, C.byref(err))
        if st:
            raise capi.PlannerError(st, err)

    def nccl_unique_id(self) -> bytes:
        buf = (C.c_uint8 * 128)()
        st = self.lib.mgs_nccl_unique_id(buf)
        if st:
            raise capi.PlannerError(st)
        return bytes(buf)

    def shard_allgather(self, values, world: int):
        v = np.ascontiguousarray(values, np.int64)
        out = np.zeros(v.size * world, np.int64)
        err = capi.empty_error()
        st = self.lib.mgs_shard_allgather_i64(self.h, capi.ptr(v, C.c_int64), v.size, capi.ptr(out, C.c_int64),
                                              C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return out.reshape(world, v.size)

    def shard_best(self, objective: float):
        best, owner = C.c_double(), C.c_int32()
        err = capi.empty_error()
        st = self.lib.mgs_shard_best(self.h, objective, C.byref(best), C.byref(owner), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return best.value, owner.value

    def solve_batch_sharded(self, problems):
        n = len(problems)
        s_max = max(p.S for p in problems)
        arr = (capi.mgs_problem * n)(*[p.c for p in problems])
        opts = np.full((n, s_max), -1, np.int32)
        obj = np.zeros(n, np.float64)
        status = np.zeros(n, np.int32)
        err = capi.empty_error()
        st = self.lib.mgs_solve_batch_sharded(self.h, arr, n, s_max, capi.ptr(opts, C.c_int32),
                                              capi.ptr(obj, C.c_double), capi.ptr(status, C.c_int32), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return opts, obj, status

    # -- ub_suffix table for a batch of traces (configs 2/4) ---------------------
    def goodput_table_batch(self, problem: Problem, arrivals, with_best=False):
        """arrivals int32 [n][M][S] (host). Returns ub [n][S+1] (and best [n][S])
        plus the number of Pareto placements scanned."""
        arr = np.ascontiguousarray(arrivals, dtype=np.int32).reshape(-1, problem.M, problem.S)
        n = arr.shape[0]
        ub = np.zeros((n, problem.S + 1), np.float64)
        best = np.zeros((n, problem.S), np.float64) if with_best else None
        npar = C.c_int32()
        err = capi.empty_error()
        st = self.lib.mgs_goodput_table_batch(self.h, problem.byref(), capi.ptr(arr, C.c_int32), n,
                                              capi.ptr(best, C.c_double) if best is not None else None,
                                              capi.ptr(ub, C.c_double), C.byref(npar), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return (ub, best, npar.value) if with_best else (ub, npar.value)

    def goodput_table_batch_device(self, problem: Problem, d_arrivals, n, d_best, d_ub):
        """Device-pointer variant (ints): enqueues on the context's stream, no sync."""
        npar = C.c_int32()
        err = capi.empty_error()
        st = self.lib.mgs_goodput_table_batch_device(self.h, problem.byref(), C.c_void_p(d_arrivals), n,
                                                     C.c_void_p(d_best) if d_best else None, C.c_void_p(d_ub),
                                                     C.byref(npar), C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return npar.value

    # -- evaluate_plan(verify=false) batch ---------------------------------------
    def evaluate_batch(self, problem: Problem, plans, arrivals, with_throughput=False, overrides=None):
        plans = np.ascontiguousarray(plans, dtype=np.int32).reshape(-1, problem.S)
        ov = None if overrides is None else np.ascontiguousarray(overrides, dtype=np.uint8).reshape(
            plans.shape[0], problem.S, problem.M)
        arrivals = np.ascontiguousarray(arrivals, dtype=np.int64).reshape(-1, problem.M, problem.S)
        n_p, n_t = plans.shape[0], arrivals.shape[0]
        total = np.zeros((n_p, n_t), np.float64)
        thr = np.zeros((n_p, n_t, problem.S, problem.M), np.float64) if with_throughput else None
        err = capi.empty_error()
        st = self.lib.mgs_evaluate_batch(self.h, problem.byref(), capi.ptr(plans, C.c_int32), n_p,
                                         capi.ptr(ov, C.c_uint8) if ov is not None else None,
                                         capi.ptr(arrivals, C.c_int64), n_t, capi.ptr(total, C.c_double),
                                         capi.ptr(thr, C.c_double) if thr is not None else None, C.byref(err))
        if st:
            raise capi.PlannerError(st, err)
        return (total, thr) if with_throughput else total


def encode(config, labels, nslots):
    """Space::encode (space.hpp:231-251): per step the configuration index then
    that configuration's per-slot labels."""
    out = []
    for c, lab in zip(config, labels):
        out.append(int(c))
        out += [int(x) for x in lab[:nslots[int(c)]]]
    return out
