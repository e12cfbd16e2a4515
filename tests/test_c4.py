"""Config 4 (4096 MMPP traces x 4 tenants x 600 slots): the per-trace DP is
outside the reference's reach at M = 4 (truncation bug; state budget), so
SURVEY.md §8(d) pins the batched Goodput table per trace (tests/test_gpu.py)
and an M = 2 / S = 200 variant of the same generator for DP parity on a sampled
subset: the first two tenants (ResNet-50, MobileNetV2) of traces 400000..400003,
one 200-slot window each, solved as one lane batch on the GPU and compared with
the UNMODIFIED reference's solve_dp (goldens by `migref solve`, committed)."""
import json
import os
import tempfile

import numpy as np
import pytest

from golden_util import bits, nslots
from paper_2407_13126_b200 import planner
from paper_2407_13126_b200 import scenario as SC
from paper_2407_13126_b200 import workloads as W

D = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c4")
SEEDS = [400000, 400001, 400002, 400003]


def test_c4_variant_fixtures_are_the_generator():
    """CPU: the fixtures are the C4 generator's traces restricted to the first two
    tenants (the same PCG64 draws), 200 slots."""
    d = tempfile.mkdtemp()
    for seed in SEEDS:
        spec = W.c2_spec(seed, steps=200, windows=1, tenants=2)
        W.write_scenario(spec, d, "x")
        assert open(os.path.join(d, "x.csv")).read() == open(os.path.join(D, "c4_m2_S200_%d.csv" % seed)).read()
        full = W.mmpp_trace([40.0, 120.0, 12.0, 10.0], 200, seed)
        assert np.array_equal(full[:2], spec.counts)


@pytest.mark.gpu
def test_c4_variant_lane_batch_matches_reference():
    gold = json.load(open(os.path.join(D, "c4_golden.json")))
    stems = ["c4_m2_S200_%d" % s for s in SEEDS]
    scs = [SC.load_scenario(os.path.join(D, st + ".scn")) for st in stems]
    probs = [SC.Problem(sc, 0) for sc in scs]
    with planner.Planner(0) as pl:
        opts, obj, status, stats, errs = pl.solve_batch(probs)
        for i, (st, sc, p) in enumerate(zip(stems, scs, probs)):
            want = gold[st]["dp"]
            assert status[i] == 0, st
            en = pl.enumerate(p)
            o = opts[i, :p.S]
            assert planner.encode(en["config"][o], en["labels"][o], nslots(sc)) == want["encode"], st
            assert bits(obj[i]) == want["obj"], st
            total, thr = pl.evaluate_batch(p, o[None], p.forecast[None], with_throughput=True)
            assert [bits(x) for x in thr[0, 0].reshape(-1)] == want["thr"], st
