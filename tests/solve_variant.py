"""Helper for test_gpu.py::test_launch_modes_agree / test_capacity_regrow: solves
golden windows in a fresh process (the launch mode and the initial capacities
are read from the environment once per process: MGS_NO_FORK = one chain instead
of the graph's parallel branches, MGS_DEBUG_STEPS = eager launches,
MGS_V2_SMALL_CAPS = tiny initial buffers, grown on overflow) and prints plan,
objective bits and counters. With --batch the same windows are also solved as
one lane batch (mgs_solve_batch)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import bits  # noqa: E402
from paper_2407_13126_b200 import planner  # noqa: E402
from paper_2407_13126_b200 import scenario as SC  # noqa: E402

args = sys.argv[1:]
batch = "--batch" in args
paths = [a for a in args if a != "--batch"]
out = {}
with planner.Planner(0) as pl:
    if batch:
        probs = [SC.Problem(SC.load_scenario(path), 0) for path in paths]
        opt, obj, st, _, _ = pl.solve_batch(probs)
        for i, path in enumerate(paths):
            out["batch:" + os.path.basename(path)] = {"status": int(st[i]), "obj": bits(obj[i]),
                                                      "opt": [int(x) for x in opt[i][: probs[i].S]]}
    for path in paths:
        p = SC.Problem(SC.load_scenario(path), 0)
        opt, cfg, lab, obj, st = pl.solve_window(p)
        out[os.path.basename(path)] = {
            "opt": [int(x) for x in opt],
            "obj": bits(obj),
            "counters": [st[k] for k in ("transitions_ref", "transitions", "frontier_total", "frontier_peak")],
        }
print(json.dumps(out))
