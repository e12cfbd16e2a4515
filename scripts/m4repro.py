"""Reproducer: four C1 windows as lanes, then the M=4 / S=12 state-budget window."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2407_13126_b200 import planner, capi, scenario as SC
c1a = SC.Problem(SC.load_scenario('tests/golden/c1/c1_S200_100001.scn'), 0)
c1b = SC.Problem(SC.load_scenario('tests/golden/c1/c1_S200_100002.scn'), 0)
with planner.Planner(0) as pl:
    opts, obj, status, stats, errs = pl.solve_batch([c1a, c1b, c1a, c1b])
    print('batch', list(status), flush=True)
    for stem in ('c2_m3_S20_v6_200003', 'c2_m4_S12_v2_200004'):
        try:
            pl.solve_window(SC.Problem(SC.load_scenario('tests/golden/multi/%s.scn' % stem), 0))
            print(stem, 'ok', flush=True)
        except capi.PlannerError as e:
            print(stem, e.code, e.message, flush=True)
