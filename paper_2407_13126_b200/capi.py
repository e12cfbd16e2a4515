"""ctypes mirror of include/migsim_b200.h (the C ABI) and the product library loader.

The product path is the CUDA library `lib/libmigsim_b200.so`; `load()` raises if it
is missing — there is deliberately no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

MAX_MODELS = 4
MAX_SLOTS = 8
SIZES = 8
FOREIGN_MASK = 0xFFFFFFFF

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(PKG_DIR, "lib")
LIB_PATH = os.path.join(LIB_DIR, "libmigsim_b200.so")

STATUS_CODES = {
    0: "ok",
    1: "input.scenario",
    2: "input.catalog",
    3: "input.forecast",
    4: "input.arrivals",
    5: "infeasible.deployment-floor",
    6: "infeasible.retraining-window",
    7: "infeasible.no-coexistence-configuration",
    8: "infeasible.joint",
    9: "planner.state-budget",
    10: "plan.infeasible",
    11: "device.cuda",
    12: "input.argument",
    13: "planner.bruteforce-cap",
    14: "infeasible.window-boundary",
}


class mgs_error(C.Structure):
    _fields_ = [("code", C.c_int32), ("step", C.c_int32), ("frontier", C.c_uint64), ("model", C.c_int32),
                ("message", C.c_char * 320)]


class mgs_lattice(C.Structure):
    _fields_ = [("n_configs", C.c_int32), ("gpc_count", C.c_int32), ("slot_offset", C.POINTER(C.c_int32)),
                ("slot_size", C.POINTER(C.c_int32)), ("slot_start", C.POINTER(C.c_int32))]


class mgs_tables(C.Structure):
    _fields_ = [("models", C.c_int32), ("steps", C.c_int32),
                ("cap_by_size", (C.c_double * SIZES) * MAX_MODELS),
                ("rt_by_size", (C.c_int64 * SIZES) * MAX_MODELS),
                ("floor_gpcs", C.c_int32 * MAX_MODELS), ("psi", C.c_double * MAX_MODELS),
                ("acc_pre", C.c_double * MAX_MODELS), ("acc_post", C.c_double * MAX_MODELS)]


class mgs_problem(C.Structure):
    _fields_ = [("lattice", mgs_lattice), ("tables", mgs_tables), ("forecast", C.POINTER(C.c_int64)),
                ("forecast_len", C.c_int32), ("has_initial", C.c_int32), ("init_mask", C.c_uint32 * MAX_MODELS),
                ("state_budget", C.c_uint64), ("workers", C.c_int32)]


class mgs_violation(C.Structure):
    _fields_ = [("code", C.c_int32), ("model", C.c_int32)]


class mgs_job_metrics(C.Structure):
    _fields_ = [("received", C.c_double), ("served", C.c_double), ("timely", C.c_double), ("correct", C.c_double),
                ("valid", C.c_double), ("dropped", C.c_double), ("queued_at_end", C.c_double),
                ("reconfigurations", C.c_int32), ("overhead_seconds", C.c_double)]


class mgs_plan_violation(C.Structure):
    _fields_ = [("code", C.c_int32), ("step", C.c_int32), ("model", C.c_int32), ("detail", C.c_int32 * 3)]


class mgs_score_entry(C.Structure):
    _fields_ = [("throughput", C.c_double), ("overhead_loss", C.c_double), ("goodput", C.c_double),
                ("completion", C.c_int32), ("pad", C.c_int32)]


VIOLATION_FAMILIES = {1: "deployment-floor", 2: "retraining-not-launched", 3: "retraining-interrupted",
                      4: "retraining-size", 5: "retraining-incomplete", 6: "retraining-overrun"}


class mgs_stats(C.Structure):
    _fields_ = [("options", C.c_uint64), ("candidates", C.c_uint64), ("transitions_ref", C.c_uint64),
                ("transitions", C.c_uint64), ("frontier_total", C.c_uint64), ("frontier_peak", C.c_uint64),
                ("device_ms", C.c_double), ("kernel_launches", C.c_uint64), ("phase_ms", C.c_double * 8),
                ("transition_bytes", C.c_uint64)]

    PHASES = ("enumerate", "goodput", "units", "transitions", "merge_band_dominance", "compaction", "ranks",
              "terminal")

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "phase_ms"}
        d["phase_ms"] = dict(zip(self.PHASES, list(self.phase_ms)))
        return d


class PlannerError(RuntimeError):
    """Mirror of migsim::Error: `.code` is the reference's stable code string."""

    def __init__(self, status: int, err: mgs_error | None = None):
        self.status = status
        self.code = STATUS_CODES.get(status, "unknown")
        self.message = err.message.decode(errors="replace") if err is not None else ""
        self.step = err.step if err is not None else 0
        self.frontier = err.frontier if err is not None else 0
        super().__init__("%s: %s" % (self.code, self.message))


def ptr(arr, ctype):
    return arr.ctypes.data_as(C.POINTER(ctype))


_LIB = None


def load():
    """Loads the CUDA product library; fails loudly when it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("MGS_LIB_PATH", LIB_PATH)  # A/B builds of the same library
    if not os.path.exists(path):
        raise RuntimeError("CUDA extension %s is missing: run __graft_entry__.build() (no CPU fallback exists)"
                           % path)
    lib = C.CDLL(path)
    P = C.POINTER
    lib.mgs_open.argtypes = [C.c_int, P(C.c_void_p)]
    lib.mgs_close.argtypes = [C.c_void_p]
    lib.mgs_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    lib.mgs_version.restype = C.c_char_p
    lib.mgs_status_code.restype = C.c_char_p
    lib.mgs_enumerate.argtypes = [C.c_void_p, P(mgs_lattice), P(mgs_tables), P(C.c_int64), C.c_int64,
                                  P(C.c_int32), P(C.c_int8), P(C.c_uint32), P(C.c_double), P(C.c_int8),
                                  P(mgs_error)]
    lib.mgs_goodput_table.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_double), P(C.c_double), P(C.c_int32),
                                      P(mgs_error)]
    lib.mgs_solve_window.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), P(C.c_int32), P(C.c_int8),
                                     P(C.c_double), P(mgs_stats), P(mgs_error)]
    lib.mgs_solve_batch.argtypes = [C.c_void_p, P(mgs_problem), C.c_int32, C.c_int32, P(C.c_int32),
                                    P(C.c_double), P(C.c_int32), P(mgs_stats), P(mgs_error)]
    lib.mgs_evaluate_batch.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), C.c_int32, P(C.c_uint8),
                                       P(C.c_int64), C.c_int32, P(C.c_double), P(C.c_double), P(mgs_error)]
    lib.mgs_preinit.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), C.c_int32, P(C.c_uint8), P(C.c_uint32),
                                P(mgs_error)]
    lib.mgs_precheck.argtypes = [C.c_void_p, P(mgs_lattice), P(mgs_tables), P(mgs_violation), C.c_int32,
                                 P(C.c_int32), P(mgs_error)]
    lib.mgs_bruteforce.argtypes = [C.c_void_p, P(mgs_problem), C.c_double, P(C.c_int32), P(C.c_int32), P(C.c_int8),
                                   P(C.c_double), P(mgs_error)]
    lib.mgs_goodput_table_batch.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), C.c_int32, P(C.c_double),
                                            P(C.c_double), P(C.c_int32), P(mgs_error)]
    lib.mgs_goodput_table_batch_device.argtypes = [C.c_void_p, P(mgs_problem), C.c_void_p, C.c_int32, C.c_void_p,
                                                   C.c_void_p, P(C.c_int32), P(mgs_error)]
    lib.mgs_window_boundary.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), P(C.c_int32), P(C.c_int8),
                                        P(C.c_double), P(mgs_error)]
    lib.mgs_replay_requests.argtypes = [C.c_void_p, P(mgs_problem), C.c_int32, P(C.c_double), P(C.c_double),
                                        P(C.c_double), C.c_double, P(C.c_int32),
                                        C.c_int32, P(C.c_uint8), P(C.c_int64), C.c_int32, P(C.c_uint64), C.c_int32,
                                        P(mgs_job_metrics), P(mgs_error)]
    lib.mgs_check_feasible_batch.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), P(C.c_uint8), C.c_int32,
                                             P(mgs_plan_violation), C.c_int32, P(C.c_int32), P(mgs_error)]
    lib.mgs_evaluate_views_batch.argtypes = [C.c_void_p, P(mgs_problem), P(C.c_int32), P(C.c_uint8), C.c_int32,
                                             P(C.c_double), P(C.c_int64), C.c_int32, C.c_int32, P(C.c_double),
                                             P(mgs_score_entry), P(C.c_int32), P(mgs_plan_violation), P(mgs_error)]
    lib.mgs_run_fluid.argtypes = [C.c_void_p, P(mgs_problem), C.c_int32, P(C.c_double), P(C.c_double), C.c_double,
                                  P(C.c_int32), P(C.c_uint8), C.c_int32, P(C.c_double), P(C.c_int64), C.c_int32,
                                  P(mgs_job_metrics), P(mgs_error)]
    lib.mgs_nccl_unique_id.argtypes = [P(C.c_uint8)]
    lib.mgs_shard_init.argtypes = [C.c_void_p, C.c_int32, C.c_int32, P(C.c_uint8), P(mgs_error)]
    lib.mgs_shard_attach.argtypes = [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32]
    lib.mgs_shard_allgather_i64.argtypes = [C.c_void_p, P(C.c_int64), C.c_int64, P(C.c_int64), P(mgs_error)]
    lib.mgs_shard_best.argtypes = [C.c_void_p, C.c_double, P(C.c_double), P(C.c_int32), P(mgs_error)]
    lib.mgs_solve_batch_sharded.argtypes = [C.c_void_p, P(mgs_problem), C.c_int32, C.c_int32, P(C.c_int32),
                                            P(C.c_double), P(C.c_int32), P(mgs_error)]
    _LIB = lib
    return lib


EXPORTED_SYMBOLS = ["mgs_open", "mgs_close", "mgs_status_code", "mgs_version", "mgs_set_stream", "mgs_enumerate",
                    "mgs_goodput_table", "mgs_solve_window", "mgs_solve_batch", "mgs_evaluate_batch",
                    "mgs_precheck", "mgs_bruteforce", "mgs_goodput_table_batch", "mgs_goodput_table_batch_device",
                    "mgs_window_boundary", "mgs_replay_requests", "mgs_preinit", "mgs_check_feasible_batch",
                    "mgs_evaluate_views_batch", "mgs_run_fluid", "mgs_nccl_unique_id", "mgs_shard_init",
                    "mgs_shard_attach", "mgs_shard_allgather_i64", "mgs_shard_best", "mgs_solve_batch_sharded"]


def empty_error():
    e = mgs_error()
    e.code = 0
    return e
