import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests'); sys.path.insert(0,'/root/repo/oracle')
from paper_2407_13126_b200 import planner, capi, scenario as SC
import torch
def mem():
    f, t = torch.cuda.mem_get_info(0)
    return "free %.1f GB" % (f / 1e9)
c1 = SC.Problem(SC.load_scenario('tests/golden/c1/c1_S200_100001.scn'), 0)
with planner.Planner(0) as pl:
    pl.solve_window(c1); print('c1 done', mem(), flush=True)
    pl.solve_batch([c1] * 8); print('batch done', mem(), flush=True)
    for stem in ('c2_m3_S20_v6_200003', 'c2_m4_S12_v2_200004', 'c2_m4_S12_v3_200004'):
        try:
            pl.solve_window(SC.Problem(SC.load_scenario('tests/golden/multi/%s.scn' % stem), 0)); print(stem, 'ok', mem(), flush=True)
        except capi.PlannerError as e:
            print(stem, e.code, e.message, mem(), flush=True)
