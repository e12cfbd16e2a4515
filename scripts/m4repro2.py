"""Reproducer of the flaky M=4 failure: the test order (C1 lanes in one context,
then the M=3/4 corpus and the C2-shaped windows in a fresh context)."""
import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0, '/root/repo/oracle')
import tempfile
import golden_util
from paper_2407_13126_b200 import planner, capi, scenario as SC
budget = int(sys.argv[1]) if len(sys.argv) > 1 else 4000000
skip_corpus = len(sys.argv) > 2 and sys.argv[2] == "nocorpus"
c1a = SC.Problem(SC.load_scenario('tests/golden/c1/c1_S200_100001.scn'), 0)
c1b = SC.Problem(SC.load_scenario('tests/golden/c1/c1_S200_100002.scn'), 0)
with planner.Planner(0) as pl:
    pl.solve_batch([c1a, c1b, c1a, c1b])
cases = golden_util.materialize(tempfile.mkdtemp())
with planner.Planner(0) as pl:
    if not skip_corpus:
        for stem, path, g in cases["multi"]:
            try:
                pl.solve_window(SC.Problem(SC.load_scenario(path), 0))
            except capi.PlannerError as e:
                if e.code == "device.cuda":
                    print("corpus", stem, e.message, flush=True)
                    sys.exit(1)
    for stem in ('c2_m3_S20_v6_200003', 'c2_m4_S12_v2_200004', 'c2_m4_S12_v3_200004'):
        try:
            pl.solve_window(SC.Problem(SC.load_scenario('tests/golden/multi/%s.scn' % stem), 0, state_budget=budget))
            print(stem, 'ok', flush=True)
        except capi.PlannerError as e:
            print(stem, e.code, e.message[:120], flush=True)
