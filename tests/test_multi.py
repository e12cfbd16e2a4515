"""M = 3..4 tenants: the planner against "reference + 1-line fix".

The shipped reference cannot solve any window with three or more tenants: it
narrows the packed per-tenant status to `int` (solvers.hpp:359,401,414), so
tenants >= 2 never start and every such window ends in infeasible.joint
(the goldens record that answer under "unpatched"). The M >= 3
goldens therefore come from oracle/_ref/migref_patched, the reference headers
with only that widening (oracle/Makefile ref-patched), and, where |O|^S is
small, from the reference's own exhaustive solve_bruteforce as well.

CPU tests pin the restatement (oracle/restate.cpp) to those goldens; GPU tests
pin the sm_100a planner through the C ABI (plans, objective bits, per-(s, m)
SLO-attained counts, brute force, error codes and the state-budget message).
"""
import pytest

import binding as B
from golden_util import bits, nslots
from paper_2407_13126_b200 import capi, planner
from paper_2407_13126_b200 import scenario as SC


def _init(g):
    return [tuple(x) for x in g["chain"]["initial"]]


def _check(want, enc, obj, thr):
    assert enc == want["encode"]
    assert bits(obj) == want["obj"]
    assert [bits(x) for x in thr] == want["thr"]


# ---------------------------------------------------------------- CPU (oracle)
def test_goldens_show_the_reference_truncation(golden_dir):
    """The unmodified reference answers infeasible.joint on every M >= 3 window
    the patched build solves: the bug the widening fixes."""
    n = 0
    for stem, path, g in golden_dir["multi"] + golden_dir["multi_c2"]:
        if "dp" in g:
            assert g["unpatched"]["error"] == "infeasible.joint", stem
            n += 1
    assert n >= 40


def test_patched_dp_equals_reference_bruteforce(golden_dir):
    """Plan identity DP == BF (the reference's solve_bruteforce) where |O|^S allows."""
    n = 0
    for stem, path, g in golden_dir["multi"]:
        for gg in (g, g.get("chain", {})):
            if "bf" in gg and "encode" in gg["bf"] and "encode" in gg.get("dp", {}):
                assert gg["bf"]["obj"] == gg["dp"]["obj"], stem
                n += 1
    assert n >= 20


def test_restatement_matches_patched_reference(golden_dir):
    for stem, path, g in golden_dir["multi"]:
        sc = SC.load_scenario(path)
        for initial, want in ((None, g["dp"]), (_init(g), g["chain"]["dp"])):
            p = SC.Problem(sc, 0, initial=initial)
            if "error" in want:
                with pytest.raises(capi.PlannerError) as e:
                    B.solve_window(p)
                assert e.value.code == want["error"], stem
                continue
            plan, obj, _ = B.solve_window(p)
            opts = B.enumerate_options(p)
            opts["nslots"] = nslots(sc)
            _, thr = B.evaluate(p, plan, p.forecast)
            _check(want, B.encode_plan(opts, plan), obj, thr)


# ---------------------------------------------------------------- GPU
@pytest.fixture(scope="module")
def gpu():
    with planner.Planner(0) as pl:
        yield pl


def _gpu_solve(pl, path, initial=None, budget=4_000_000):
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0, initial=initial, state_budget=budget)
    opt, cfg, lab, obj, stats = pl.solve_window(p)
    total, thr = pl.evaluate_batch(p, opt[None, :], p.forecast[None], with_throughput=True)
    assert bits(total[0, 0]) == bits(obj)
    return planner.encode(cfg, lab, nslots(sc)), obj, thr[0, 0].reshape(-1), stats


@pytest.mark.gpu
def test_gpu_enumeration_m3_m4(gpu, golden_dir):
    import numpy as np
    for stem, path, g in golden_dir["multi"] + golden_dir["multi_c2"][:1]:
        p = SC.Problem(SC.load_scenario(path), 0)
        want = B.enumerate_options(p)
        got = gpu.enumerate(p)
        for k in ("config", "labels", "mask", "rsize"):
            assert np.array_equal(got[k], want[k]), (stem, k)
        assert got["cap"].tobytes() == want["cap"].tobytes(), stem


@pytest.mark.gpu
def test_gpu_solve_m3_m4_cold_and_chained(gpu, golden_dir):
    n = 0
    for stem, path, g in golden_dir["multi"]:
        for initial, want in ((None, g["dp"]), (_init(g), g["chain"]["dp"])):
            if "error" in want:
                with pytest.raises(capi.PlannerError) as e:
                    _gpu_solve(gpu, path, initial)
                assert e.value.code == want["error"], stem
                continue
            enc, obj, thr, _ = _gpu_solve(gpu, path, initial)
            _check(want, enc, obj, thr)
            n += 1
    assert n >= 60


@pytest.mark.gpu
def test_gpu_bruteforce_m3(gpu, golden_dir):
    n = 0
    for stem, path, g in golden_dir["multi"]:
        if "bf" not in g:
            continue
        sc = SC.load_scenario(path)
        for initial, want in ((None, g["bf"]), (_init(g), g["chain"]["bf"])):
            p = SC.Problem(sc, 0, initial=initial)
            if "error" in want:
                with pytest.raises(capi.PlannerError) as e:
                    gpu.solve_bruteforce(p)
                assert e.value.code == want["error"], stem
                continue
            opt, cfg, lab, obj = gpu.solve_bruteforce(p)
            assert planner.encode(cfg, lab, nslots(sc)) == want["encode"], stem
            assert bits(obj) == want["obj"], stem
            n += 1
    assert n >= 20


@pytest.mark.gpu
def test_gpu_c2_shaped_windows(gpu, golden_dir):
    """C2-shaped (workloads.c2_spec, shortened) M = 3 / S = 20 and M = 4 / S = 12
    windows: the plan bit-exact, or planner.state-budget with the reference's
    exact message (same frontier count, same step)."""
    seen = set()
    for stem, path, g in golden_dir["multi_c2"]:
        if "error" in g:
            with pytest.raises(capi.PlannerError) as e:
                _gpu_solve(gpu, path)
            assert e.value.code == g["error"], (stem, e.value.message)
            assert e.value.message == g["message"], stem
            seen.add(g["error"])
            continue
        enc, obj, thr, stats = _gpu_solve(gpu, path)
        _check(g["dp"], enc, obj, thr)
        assert stats["options"] == g["options"]
        seen.add("solved")
    assert seen == {"solved", "planner.state-budget"}


@pytest.mark.gpu
def test_gpu_multi_launch_engine_fallback(gpu, golden_dir, monkeypatch):
    """The multi-launch engine (csrc/dp.cu) stays the fallback for M = 3..4 windows
    the graph engine's 8-bit fields cannot hold (S > 36): pinned on the same
    goldens by forcing it (MGS_DP_ENGINE=v1)."""
    monkeypatch.setenv("MGS_DP_ENGINE", "v1")
    n = 0
    for stem, path, g in golden_dir["multi"][:20]:
        want = g["dp"]
        if "error" in want:
            continue
        enc, obj, thr, _ = _gpu_solve(gpu, path, None)
        _check(want, enc, obj, thr)
        n += 1
    assert n >= 10


@pytest.mark.gpu
def test_gpu_budget_error_mid_kernel_is_clean(golden_dir):
    """Regression: planner.state-budget is raised by one block of k_units while
    the other blocks (and the rank branch beside it) are starting. Every kernel's
    entry check is block-uniform (__syncthreads_or), so no block can lose some of
    its threads before a barrier or a full-warp collective. Before the fix this
    sequence (a 4-lane C1 batch, then the M = 4 budget window in a fresh context)
    faulted with an illegal address in about half the runs."""
    c1 = {stem: path for stem, path, g in golden_dir["c1"]}
    probs = [SC.Problem(SC.load_scenario(c1[s]), 0) for s in ("c1_S200_100001", "c1_S200_100002") * 2]
    with planner.Planner(0) as pl:
        assert (pl.solve_batch(probs)[2] == 0).all()
    budget = dict((stem, (path, g)) for stem, path, g in golden_dir["multi_c2"])["c2_m4_S12_v2_200004"]
    with planner.Planner(0) as pl:
        for _ in range(4):
            with pytest.raises(capi.PlannerError) as e:
                _gpu_solve(pl, budget[0])
            assert e.value.code == "planner.state-budget" and e.value.message == budget[1]["message"]
        enc, obj, thr, _ = _gpu_solve(pl, c1["c1_S200_100001"])  # the context is still healthy
