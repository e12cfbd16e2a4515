"""Per-step device time of the captured DP graph (MGS_STEP_TIMES=1) for the C1
window and for a one-tenant S=200 window (tiny frontier: the per-step floor)."""
import os
import sys
import tempfile

os.environ["MGS_STEP_TIMES"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import planner  # noqa: E402
from paper_2407_13126_b200 import scenario as SC  # noqa: E402
from paper_2407_13126_b200 import workloads as W  # noqa: E402

d = tempfile.mkdtemp()
spec = W.c1_spec(100001)
spec.tenants = spec.tenants[:1]
spec.counts = spec.counts[:1]
one = W.write_scenario(spec, d, "m1")
c1 = os.path.join(ROOT, "tests", "golden", "c1", "c1_S200_100001.scn")
with planner.Planner(0) as pl:
    for name, path in (("m1", one), ("c1", c1)):
        p = SC.Problem(SC.load_scenario(path), 0)
        for _ in range(3):
            opt, cfg, lab, obj, st = pl.solve_window(p)
        print(name, "device_ms", st["device_ms"], "peak", st["frontier_peak"], "total", st["frontier_total"], flush=True)
