"""Config 5 (8 physical MIG GPUs x 7 slices, 16 tenants, 1800 slots): the box
is decomposed into 8 independent two-tenant subproblems, one per MIG GPU
(workloads.c5_specs). Each subproblem's per-window loop
on the GPU (batched lanes, carried final ranges) must equal the UNMODIFIED
reference's loop (`migref drive <scn> oracle <max_windows>`, goldens by
oracle/make_c5_goldens.py) bit for bit, at the full S = 200."""
import json
import os

import pytest

from golden_util import bits, nslots
from paper_2407_13126_b200 import driver, planner
from paper_2407_13126_b200 import scenario as SC
from paper_2407_13126_b200 import workloads as W

D = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c5")


def test_c5_fixtures_are_the_generator():
    """CPU: the committed fixtures are exactly workloads.c5_specs (8 GPUs,
    2 tenants each, 9 windows x 200 slots, seeds 500001..500008)."""
    import tempfile
    specs = W.c5_specs()
    assert len(specs) == 8
    d = tempfile.mkdtemp()
    for k, spec in enumerate(specs):
        assert spec.window_size == 200 and spec.window_count == 9 and len(spec.tenants) == 2
        W.write_scenario(spec, d, "c5_gpu%d" % k)
        for ext in (".csv",):
            assert open(os.path.join(d, "c5_gpu%d" % k + ext)).read() == open(os.path.join(D, "c5_gpu%d" % k + ext)).read()
    names = {t.name for s in specs for t in s.tenants}
    assert len(names) == 16


@pytest.mark.gpu
@pytest.mark.slow
def test_c5_subproblems_match_reference():
    path = os.path.join(D, "c5_golden.json")
    if not os.path.exists(path):
        pytest.skip("c5 goldens not generated (oracle/make_c5_goldens.py)")
    g = json.load(open(path))
    stems = sorted(g["golden"])
    assert len(stems) == 8  # every MIG-GPU subproblem of the box
    scs = [SC.load_scenario(os.path.join(D, stem + ".scn")) for stem in stems]
    with planner.Planner(0) as pl:
        plans = driver.plan_scenarios(pl, scs, "oracle", max_windows=g["max_windows"])
    for stem, sc, wins in zip(stems, scs, plans):
        want = g["golden"][stem]["windows"]
        assert len(wins) == len(want) == g["max_windows"]
        for wp, w in zip(wins, want):
            assert planner.encode(wp.config, wp.labels, nslots(sc)) == w["encode"], (stem, wp.window)
            assert bits(wp.objective) == w["obj"] and bits(wp.realized) == w["realized"], (stem, wp.window)
