"""Helper for test_gpu.py::test_launch_modes_agree: solves the config-1 golden
windows in a fresh process (the launch mode is read from the environment once
per process: MGS_NO_FORK = one chain instead of the graph's parallel branches,
MGS_DEBUG_STEPS = eager launches) and prints plan, objective bits and counters."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import bits  # noqa: E402
from paper_2407_13126_b200 import planner  # noqa: E402
from paper_2407_13126_b200 import scenario as SC  # noqa: E402

out = {}
with planner.Planner(0) as pl:
    for path in sys.argv[1:]:
        p = SC.Problem(SC.load_scenario(path), 0)
        opt, cfg, lab, obj, st = pl.solve_window(p)
        out[os.path.basename(path)] = {
            "opt": [int(x) for x in opt],
            "obj": bits(obj),
            "counters": [st[k] for k in ("transitions_ref", "transitions", "frontier_total", "frontier_peak")],
        }
print(json.dumps(out))
