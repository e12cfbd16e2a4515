"""Throughput of batched C1 windows (lanes) vs single windows."""
import os, sys, time, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import planner, scenario as SC, workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
work = tempfile.mkdtemp()
probs = []
for k in range(n):
    path = W.write_scenario(W.c1_spec(100001 + k), work, "c1_%d" % k)
    probs.append(SC.Problem(SC.load_scenario(path), 0))
with planner.Planner(0) as pl:
    pl.solve_batch(probs)  # warm (capacity growth, graph capture)
    t = time.perf_counter(); opts, obj, st, stats, errs = pl.solve_batch(probs); dt = time.perf_counter() - t
    tr = sum(s["transitions_ref"] for s in stats)
    print("lanes=%s windows %d: %.1f ms total, %.2f ms/window, %.3g plans/s, status %s" % (
        os.environ.get("MGS_BATCH_LANES", "8"), n, dt * 1e3, dt * 1e3 / n, tr / dt, set(st.tolist())))
