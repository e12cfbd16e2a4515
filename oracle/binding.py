"""TEST INFRASTRUCTURE ONLY: ctypes bindings for the CPU checkers.

  liboracle.so        our CPU restatement (oracle/restate.cpp)
  _ref/migref(.so)    the unmodified reference planner (oracle/ref_driver.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

from paper_2407_13126_b200 import capi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "liboracle.so")
REF_BIN = os.path.join(HERE, "_ref", "migref")
REF_LIB = os.path.join(HERE, "_ref", "libmigref.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError("oracle not built: make -C oracle restate")
        L = C.CDLL(ORACLE_LIB)
        P = C.POINTER
        L.oracle_enumerate.argtypes = [P(capi.mgs_lattice), P(capi.mgs_tables), P(C.c_int64), C.c_int64,
                                       P(C.c_int32), P(C.c_int8), P(C.c_uint32), P(C.c_double), P(C.c_int8),
                                       P(capi.mgs_error)]
        L.oracle_goodput_table.argtypes = [P(capi.mgs_problem), P(C.c_double), P(C.c_double), P(C.c_int32),
                                           P(capi.mgs_error)]
        L.oracle_solve_window.argtypes = [P(capi.mgs_problem), P(C.c_int32), P(C.c_double), P(capi.mgs_stats),
                                          P(capi.mgs_error)]
        L.oracle_evaluate.argtypes = [P(capi.mgs_problem), P(C.c_int32), P(C.c_int64), C.c_int32, P(C.c_double),
                                      P(C.c_double), P(capi.mgs_error)]
        _lib = L
    return _lib


def enumerate_options(problem):
    L = lib()
    n = C.c_int64()
    err = capi.empty_error()
    st = L.oracle_enumerate(C.byref(problem.c.lattice), C.byref(problem.c.tables), C.byref(n), 0, None, None,
                            None, None, None, C.byref(err))
    if st:
        raise capi.PlannerError(st, err)
    N = n.value
    out = dict(config=np.zeros(N, np.int32), labels=np.zeros((N, capi.MAX_SLOTS), np.int8),
               mask=np.zeros((N, 4), np.uint32), cap=np.zeros((N, 4), np.float64), rsize=np.zeros((N, 4), np.int8))
    st = L.oracle_enumerate(C.byref(problem.c.lattice), C.byref(problem.c.tables), C.byref(n), N,
                            capi.ptr(out["config"], C.c_int32), capi.ptr(out["labels"], C.c_int8),
                            capi.ptr(out["mask"], C.c_uint32), capi.ptr(out["cap"], C.c_double),
                            capi.ptr(out["rsize"], C.c_int8), C.byref(err))
    if st:
        raise capi.PlannerError(st, err)
    return out


def goodput_table(problem):
    L = lib()
    ub = np.zeros(problem.S + 1, np.float64)
    inc = C.c_double()
    greedy = np.zeros(problem.S, np.int32)
    err = capi.empty_error()
    st = L.oracle_goodput_table(problem.byref(), capi.ptr(ub, C.c_double), C.byref(inc),
                                capi.ptr(greedy, C.c_int32), C.byref(err))
    if st:
        raise capi.PlannerError(st, err)
    return ub, inc.value, greedy


def solve_window(problem):
    """Returns (options[S], objective, stats dict)."""
    L = lib()
    out = np.zeros(problem.S, np.int32)
    obj = C.c_double()
    stats = capi.mgs_stats()
    err = capi.empty_error()
    st = L.oracle_solve_window(problem.byref(), capi.ptr(out, C.c_int32), C.byref(obj), C.byref(stats),
                               C.byref(err))
    if st:
        raise capi.PlannerError(st, err)
    return out, obj.value, stats.as_dict()


def evaluate(problem, plan, arrivals):
    L = lib()
    plan = np.ascontiguousarray(plan, dtype=np.int32)
    arrivals = np.ascontiguousarray(arrivals, dtype=np.int64)
    total = C.c_double()
    thr = np.zeros(problem.S * problem.M, np.float64)
    err = capi.empty_error()
    st = L.oracle_evaluate(problem.byref(), capi.ptr(plan, C.c_int32), capi.ptr(arrivals, C.c_int64),
                           arrivals.shape[1], C.byref(total), capi.ptr(thr, C.c_double), C.byref(err))
    if st:
        raise capi.PlannerError(st, err)
    return total.value, thr


def ref_solve(scn_path, window=0, chain=False, bf=False, budget=None, timeout=None):
    """Runs the unmodified reference on a scenario file; returns its JSON."""
    cmd = [REF_BIN, "solve", scn_path, str(window)]
    if chain:
        cmd.append("--chain")
    if bf:
        cmd.append("--bf")
    if budget is not None:
        cmd += ["--budget", str(budget)]
    out = subprocess.run(cmd, check=True, capture_output=True, text=True, timeout=timeout)
    return json.loads(out.stdout)


def encode_plan(options, plan):
    """Space::encode (space.hpp:231-251) of a plan given as option indices:
    per step the configuration index followed by that configuration's labels."""
    out = []
    for oi in plan:
        c = int(options["config"][oi])
        out.append(c)
        n = options["nslots"][c]
        out += [int(x) for x in options["labels"][oi][:n]]
    return out


def ref_solve_inproc(scn_path, window=0, workers=1):
    """In-process reference solve (bench CPU baseline). Returns (seconds, objective, encode)."""
    L = C.CDLL(REF_LIB)
    enc = np.zeros(1 << 16, np.int32)
    n = C.c_int()
    secs = C.c_double()
    obj = C.c_double()
    code = C.create_string_buffer(128)
    st = L.migref_solve_file(scn_path.encode(), window, workers, C.byref(secs), C.byref(obj),
                             enc.ctypes.data_as(C.POINTER(C.c_int)), enc.size, C.byref(n), code, 128)
    if st:
        raise RuntimeError("reference error %s" % code.value.decode())
    return secs.value, obj.value, enc[:n.value].tolist()
