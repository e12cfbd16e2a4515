"""Solves one config-1 window once (profiling target for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import planner  # noqa: E402
from paper_2407_13126_b200 import scenario as SC  # noqa: E402

path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden", "c1", "c1_S200_100001.scn")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
p = SC.Problem(SC.load_scenario(path), 0)
with planner.Planner(0) as pl:
    for _ in range(reps):
        opt, cfg, lab, obj, st = pl.solve_window(p)
print("objective", obj, "device_ms", st["device_ms"], "launches", st["kernel_launches"])
print("phases", st["phase_ms"])
