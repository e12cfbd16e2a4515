"""CPU: pins the CPU restatement (oracle/restate.cpp) to the unmodified reference.

The goldens under tests/golden/ were produced by the reference planner itself
(oracle/make_goldens.py -> oracle/_ref/migref). Here the restatement must
reproduce every plan encoding, objective bits and per-(s,m) throughput bits,
cold and chained, plus the reference tests' known answers.
"""
import os

import numpy as np
import pytest

import binding as B
from golden_util import bits, nslots
from paper_2407_13126_b200 import capi
from paper_2407_13126_b200 import scenario as SC


def solve_and_encode(path, initial=None, budget=4_000_000):
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0, initial=initial, state_budget=budget)
    plan, obj, stats = B.solve_window(p)
    opts = B.enumerate_options(p)
    opts["nslots"] = nslots(sc)
    total, thr = B.evaluate(p, plan, p.forecast)
    assert bits(total) == bits(obj)
    return B.encode_plan(opts, plan), obj, thr, stats


def check_against(golden_plan, enc, obj, thr):
    assert enc == golden_plan["encode"]
    assert bits(obj) == golden_plan["obj"]
    assert [bits(x) for x in thr] == golden_plan["thr"]


def test_random_corpus_matches_reference(golden_dir):
    n = 0
    for stem, path, g in golden_dir["random"]:
        enc, obj, thr, _ = solve_and_encode(path)
        check_against(g["dp"], enc, obj, thr)
        # the reference's DP and brute force agree on value (solver_test.cpp:110-128)
        if "encode" in g.get("bf", {}):
            assert g["bf"]["obj"] == g["dp"]["obj"] or abs(
                float(g["bf"]["objective"]) - float(g["dp"]["objective"])) < 1e-9
        n += 1
    assert n >= 150


def test_random_corpus_chained_matches_reference(golden_dir):
    n = 0
    for stem, path, g in golden_dir["random"]:
        ch = g["chain"]
        init = [tuple(x) for x in ch["initial"]]
        if "error" in ch["dp"]:
            with pytest.raises(capi.PlannerError) as e:
                solve_and_encode(path, initial=init)
            assert e.value.code == ch["dp"]["error"]
            continue
        enc, obj, thr, _ = solve_and_encode(path, initial=init)
        check_against(ch["dp"], enc, obj, thr)
        n += 1
    assert n >= 100


def test_c1_fixtures_match_reference(golden_dir):
    for stem, path, g in golden_dir["c1"]:
        if int(stem.split("_")[1][1:]) > 60:
            continue  # full-size windows: checked on the GPU only (2 min of CPU each)
        enc, obj, thr, stats = solve_and_encode(path)
        check_against(g["dp"], enc, obj, thr)
        assert stats["options"] == g["options"]


def test_known_answers(golden_dir):
    kat = {stem: (path, g) for stem, path, g in golden_dir["kat"]}
    # worked example optimum 12.5 (solver_test.cpp:34-47, eval_test.cpp:16-29)
    enc, obj, thr, _ = solve_and_encode(kat["worked_example"][0])
    assert obj == 12.5 and enc == kat["worked_example"][1]["dp"]["encode"]
    # zero trace scores zero (solver_test.cpp:72-79)
    _, obj, _, _ = solve_and_encode(kat["zero_trace"][0])
    assert obj == 0.0
    # forced plan (solver_test.cpp:49-70)
    enc, _, _, _ = solve_and_encode(kat["forced"][0])
    assert enc == kat["forced"][1]["dp"]["encode"]
    for name in ("no_coexistence", "deployment_floor"):
        with pytest.raises(capi.PlannerError) as e:
            solve_and_encode(kat[name][0])
        assert e.value.code == kat[name][1]["expect_error"]
    # state budget: code and the 'states' message (solver_test.cpp:194-207)
    with pytest.raises(capi.PlannerError) as e:
        solve_and_encode(kat["small_two_model"][0], budget=1)
    assert e.value.code == "planner.state-budget"
    assert e.value.message == kat["small_two_model"][1]["budget1"]["message"]


def test_worked_example_breakdown():
    """eval_test.cpp:16-29: the worked plan scores 2.5 / 5 / 5 = 12.5."""
    path = os.path.join(os.path.dirname(__file__), "golden", "kat", "worked_example.scn")
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0)
    opts = B.enumerate_options(p)
    # plan: step 0 retrain on 4@0 with inference on 3@4, then inference on 4@0
    want = [[2, 1], [1, 0], [1, 0]]  # labels per slot (4@0, 3@4): 1 = m0:i, 2 = m0:r
    plan = []
    for lab in want:
        hit = [i for i in range(len(opts["config"])) if list(opts["labels"][i][:2]) == lab]
        plan.append(hit[0])
    total, thr = B.evaluate(p, np.array(plan), p.forecast)
    assert total == 12.5
    assert [t * a for t, a in zip(thr, [0.5, 1.0, 1.0])] == [2.5, 5.0, 5.0]
