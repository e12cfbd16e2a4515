"""Runs every device entry point once on small inputs (ncu target for the
kernels outside the DP step loop): enumeration, Goodput reductions, greedy,
brute force, evaluate (options and general views), check_feasible, fluid and
request replay, pre-initialisation, window boundary, the C4 table batch."""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2407_13126_b200 import planner  # noqa: E402
from paper_2407_13126_b200 import scenario as SC  # noqa: E402
from paper_2407_13126_b200 import workloads as W  # noqa: E402

c1 = SC.Problem(SC.load_scenario(os.path.join(ROOT, "tests", "golden", "c1", "c1_S200_100001.scn")), 0)
small = SC.Problem(SC.load_scenario(os.path.join(ROOT, "tests", "golden", "kat", "worked_example.scn")), 0)
with planner.Planner(0) as pl:
    opt, cfg, lab, obj, st = pl.solve_window(c1)  # enumeration, reductions, greedy, DP, evaluate
    pl.evaluate_batch(c1, np.stack([opt] * 64), np.stack([c1.forecast] * 16))
    pl.preinit(c1, opt[None])
    pl.window_boundary(c1)
    pl.replay_requests(c1, opt[None], c1.forecast[None], [1, 2])
    pl.solve_bruteforce(small)
    d = tempfile.mkdtemp()
    p4 = SC.Problem(SC.load_scenario(W.write_scenario(W.c2_spec(400000, steps=600, windows=1), d, "c4")), 0)
    tr = np.stack([W.mmpp_trace([40.0, 120.0, 12.0, 10.0], p4.S, 400000 + k) for k in range(4096)]).astype(np.int32)
    pl.goodput_table_batch(p4, tr)
    # plans as general allocations: check_feasible, evaluate_plan(verify), run_fluid
    import ctypes as C
    from paper_2407_13126_b200 import capi
    S, M = c1.S, c1.M
    tasks = np.zeros((S, capi.MAX_SLOTS), np.uint8)
    for s in range(S):
        for k, l in enumerate(lab[s]):
            if l > 0:
                tasks[s, k] = 1 << (int(l) - 1)
    cfg32 = np.ascontiguousarray(cfg, np.int32)
    out = (capi.mgs_plan_violation * (S * M + M))()
    n = np.zeros(1, np.int32)
    err = capi.empty_error()
    L = pl.lib
    assert L.mgs_check_feasible_batch(pl.h, C.byref(c1.c), capi.ptr(cfg32, C.c_int32), capi.ptr(tasks, C.c_uint8), 1,
                                      out, S * M + M, capi.ptr(n, C.c_int32), C.byref(err)) == 0 and n[0] == 0
    tot = np.zeros(1, np.float64)
    stat = np.zeros(1, np.int32)
    arr = np.ascontiguousarray(c1.forecast, np.int64)
    assert L.mgs_evaluate_views_batch(pl.h, C.byref(c1.c), capi.ptr(cfg32, C.c_int32), capi.ptr(tasks, C.c_uint8), 1,
                                      None, capi.ptr(arr, C.c_int64), 1, 1, capi.ptr(tot, C.c_double), None,
                                      capi.ptr(stat, C.c_int32), None, C.byref(err)) == 0 and tot[0] == obj
    jm = (capi.mgs_job_metrics * M)()
    assert L.mgs_run_fluid(pl.h, C.byref(c1.c), 1, None, None, 1.0, capi.ptr(cfg32, C.c_int32),
                           capi.ptr(tasks, C.c_uint8), 1, None, capi.ptr(arr, C.c_int64), 1, jm, C.byref(err)) == 0
print("ok")
