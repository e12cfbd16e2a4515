"""GPU parity: the sm_100a planner (through the C ABI) against the reference.

Bar (BASELINE.json north_star): bit-exact plans, option / placement indices and
SLO-attained counts; objective Goodput bit-exact here (tolerance stated by the
spec: 1e-6 relative — we require equality of the IEEE bits, which is stricter).
"""
import numpy as np
import pytest

import binding as B
from golden_util import bits, nslots
from paper_2407_13126_b200 import capi, planner
from paper_2407_13126_b200 import scenario as SC

pytestmark = pytest.mark.gpu

OBJ_RTOL = 1e-6  # north_star tolerance; the checks below are stricter (bitwise)


@pytest.fixture(scope="module")
def gpu():
    with planner.Planner(0) as pl:
        yield pl


def gpu_solve(pl, path, initial=None, budget=4_000_000):
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0, initial=initial, state_budget=budget)
    opt, cfg, lab, obj, stats = pl.solve_window(p)
    enc = planner.encode(cfg, lab, nslots(sc))
    total, thr = pl.evaluate_batch(p, opt[None, :], p.forecast[None], with_throughput=True)
    return p, opt, enc, obj, thr[0, 0].reshape(-1), stats, total[0, 0]


def check(golden_plan, enc, obj, thr):
    assert enc == golden_plan["encode"]
    assert bits(obj) == golden_plan["obj"]
    assert abs(obj - float(golden_plan["objective"])) <= OBJ_RTOL * max(1.0, abs(obj))
    assert [bits(x) for x in thr] == golden_plan["thr"]


def test_library_loads_and_reports_version():
    lib = capi.load()
    assert b"sm_100a" in lib.mgs_version()


def test_enumeration_matches_oracle(gpu, golden_dir):
    cases = golden_dir["random"][:40] + golden_dir["c1"] + golden_dir["kat"]
    for stem, path, g in cases:
        sc = SC.load_scenario(path)
        p = SC.Problem(sc, 0)
        try:
            want = B.enumerate_options(p)
        except capi.PlannerError:
            continue
        got = gpu.enumerate(p)
        for k in ("config", "labels", "mask", "rsize"):
            assert np.array_equal(got[k], want[k]), (stem, k)
        assert got["cap"].tobytes() == want["cap"].tobytes(), stem


def test_goodput_table_matches_oracle(gpu, golden_dir):
    for stem, path, g in golden_dir["random"][:60] + golden_dir["c1"]:
        sc = SC.load_scenario(path)
        for initial in (None, [tuple(x) for x in g.get("chain", {}).get("initial", [])] or None):
            p = SC.Problem(sc, 0, initial=initial)
            ub, inc, greedy = gpu.goodput_table(p)
            ub_o, inc_o, greedy_o = B.goodput_table(p)
            assert ub.tobytes() == ub_o.tobytes(), stem
            assert bits(inc) == bits(inc_o), stem
            if np.isfinite(inc_o):
                assert np.array_equal(greedy, greedy_o), stem


def test_solve_random_corpus(gpu, golden_dir):
    for stem, path, g in golden_dir["random"]:
        p, opt, enc, obj, thr, stats, total = gpu_solve(gpu, path)
        check(g["dp"], enc, obj, thr)
        assert bits(total) == bits(obj)


def test_solve_random_corpus_chained(gpu, golden_dir):
    for stem, path, g in golden_dir["random"]:
        ch = g["chain"]
        init = [tuple(x) for x in ch["initial"]]
        if "error" in ch["dp"]:
            with pytest.raises(capi.PlannerError) as e:
                gpu_solve(gpu, path, initial=init)
            assert e.value.code == ch["dp"]["error"]
            continue
        p, opt, enc, obj, thr, stats, total = gpu_solve(gpu, path, initial=init)
        check(ch["dp"], enc, obj, thr)


def test_solve_c1_fixtures(gpu, golden_dir):
    for stem, path, g in golden_dir["c1"]:
        p, opt, enc, obj, thr, stats, total = gpu_solve(gpu, path)
        check(g["dp"], enc, obj, thr)
        assert stats["options"] == g["options"]
        if "chain" in g:
            init = [tuple(x) for x in g["chain"]["initial"]]
            _, _, enc2, obj2, thr2, _, _ = gpu_solve(gpu, path, initial=init)
            check(g["chain"]["dp"], enc2, obj2, thr2)


def test_c1_counters_match_oracle(gpu, golden_dir):
    """Work counters (transitions, frontier sizes) equal the restatement's."""
    for stem, path, g in golden_dir["c1"]:
        if int(stem.split("_")[1][1:]) > 60:
            continue
        sc = SC.load_scenario(path)
        p = SC.Problem(sc, 0)
        _, _, _, _, stats = gpu.solve_window(p)
        _, _, ostats = B.solve_window(p)
        for k in ("options", "candidates", "transitions_ref", "transitions", "frontier_total", "frontier_peak"):
            assert stats[k] == ostats[k], (stem, k, stats[k], ostats[k])


def test_known_answers_and_errors(gpu, golden_dir):
    kat = {stem: (path, g) for stem, path, g in golden_dir["kat"]}
    _, _, enc, obj, _, _, _ = gpu_solve(gpu, kat["worked_example"][0])
    assert obj == 12.5 and enc == kat["worked_example"][1]["dp"]["encode"]
    _, _, _, obj, _, _, _ = gpu_solve(gpu, kat["zero_trace"][0])
    assert obj == 0.0
    _, _, enc, _, _, _, _ = gpu_solve(gpu, kat["forced"][0])
    assert enc == kat["forced"][1]["dp"]["encode"]
    _, _, enc, obj, thr, _, _ = gpu_solve(gpu, kat["small_two_model"][0])
    check(kat["small_two_model"][1]["dp"], enc, obj, thr)
    for name in ("no_coexistence", "deployment_floor"):
        with pytest.raises(capi.PlannerError) as e:
            gpu_solve(gpu, kat[name][0])
        assert e.value.code == kat[name][1]["expect_error"]
    with pytest.raises(capi.PlannerError) as e:
        gpu_solve(gpu, kat["small_two_model"][0], budget=1)
    assert e.value.code == "planner.state-budget"
    assert "states" in e.value.message
    assert e.value.message == kat["small_two_model"][1]["budget1"]["message"]


def test_forecast_length_error(gpu, golden_dir):
    stem, path, g = golden_dir["kat"][0]
    sc = SC.load_scenario(golden_dir["c1"][0][1])
    p = SC.Problem(sc, 0, forecast=np.zeros((2, sc.window_size + 1), np.int64))
    with pytest.raises(capi.PlannerError) as e:
        gpu.solve_window(p)
    assert e.value.code == "input.forecast"


def test_evaluate_batch_matches_oracle(gpu, golden_dir):
    rng = np.random.default_rng(7)
    for stem, path, g in golden_dir["c1"][:2] + golden_dir["random"][:20]:
        sc = SC.load_scenario(path)
        p = SC.Problem(sc, 0)
        n_opt = len(B.enumerate_options(p)["config"])
        plans = rng.integers(0, n_opt, size=(5, p.S)).astype(np.int32)
        traces = rng.integers(0, 300, size=(7, p.M, p.S)).astype(np.int64)
        total, thr = gpu.evaluate_batch(p, plans, traces, with_throughput=True)
        for i in range(plans.shape[0]):
            for j in range(traces.shape[0]):
                t_o, thr_o = B.evaluate(p, plans[i], traces[j])
                assert bits(total[i, j]) == bits(t_o)
                assert thr[i, j].reshape(-1).tobytes() == thr_o.tobytes()


def test_solve_batch_equals_single(gpu, golden_dir):
    cases = golden_dir["c1"][:3]
    probs = [SC.Problem(SC.load_scenario(path), 0) for _, path, _ in cases]
    opts, obj, status, stats, errs = gpu.solve_batch(probs)
    for i, (stem, path, g) in enumerate(cases):
        assert status[i] == 0
        o1, _, _, obj1, _ = gpu.solve_window(probs[i])
        assert np.array_equal(opts[i, :probs[i].S], o1)
        assert bits(obj[i]) == bits(obj1) == g["dp"]["obj"]


def test_deterministic_repeat(gpu, golden_dir):
    stem, path, g = golden_dir["c1"][0]
    a = gpu_solve(gpu, path)
    b = gpu_solve(gpu, path)
    assert a[2] == b[2] and bits(a[3]) == bits(b[3])


def test_bruteforce_matches_reference(gpu, golden_dir):
    """solve_bruteforce on the GPU == the reference's DFS (plan and objective bits),
    cold and chained, on the whole random corpus."""
    for stem, path, g in golden_dir["random"]:
        sc = SC.load_scenario(path)
        for initial, want in ((None, g["bf"]), ([tuple(x) for x in g["chain"]["initial"]], g["chain"]["bf"])):
            p = SC.Problem(sc, 0, initial=initial)
            if "error" in want:
                with pytest.raises(capi.PlannerError) as e:
                    gpu.solve_bruteforce(p)
                assert e.value.code == want["error"], stem
                continue
            opt, cfg, lab, obj = gpu.solve_bruteforce(p)
            assert planner.encode(cfg, lab, nslots(sc)) == want["encode"], stem
            assert bits(obj) == want["obj"], stem


def test_bruteforce_cap_and_errors(gpu, golden_dir):
    kat = {stem: (path, g) for stem, path, g in golden_dir["kat"]}
    p = SC.Problem(SC.load_scenario(kat["small_two_model"][0]), 0)
    with pytest.raises(capi.PlannerError) as e:
        gpu.solve_bruteforce(p, bruteforce_cap=10.0)
    assert e.value.code == "planner.bruteforce-cap"
    assert e.value.message.startswith("brute-force space estimate ")
    p = SC.Problem(SC.load_scenario(kat["worked_example"][0]), 0)
    opt, cfg, lab, obj = gpu.solve_bruteforce(p)
    assert obj == 12.5
    for name in ("no_coexistence", "deployment_floor"):
        p = SC.Problem(SC.load_scenario(kat[name][0]), 0)
        with pytest.raises(capi.PlannerError) as e:
            gpu.solve_bruteforce(p)
        assert e.value.code == kat[name][1]["expect_error"]
        v = gpu.precheck(p)
        assert v and "infeasible." + v[0][0].split(".", 1)[1] == kat[name][1]["expect_error"]
    p = SC.Problem(SC.load_scenario(kat["worked_example"][0]), 0)
    assert gpu.precheck(p) == []


def test_solve_batch_random_corpus(gpu, golden_dir):
    """Every random-corpus window in ONE batched call (lanes share kernels;
    shapes change between windows) == the reference's plans and objective bits."""
    cases = golden_dir["random"]
    probs = [SC.Problem(SC.load_scenario(path), 0) for _, path, _ in cases]
    opts, obj, status, stats, errs = gpu.solve_batch(probs)
    for i, (stem, path, g) in enumerate(cases):
        assert status[i] == 0, (stem, errs[i].message)
        assert bits(obj[i]) == g["dp"]["obj"], stem
        _, cfg, lab, _, _ = gpu.solve_window(probs[i])
        assert list(opts[i, :probs[i].S]) == list(gpu.solve_window(probs[i])[0]), stem


def test_solve_batch_c1_lanes(gpu, golden_dir):
    """Four C1 S=200 windows as four lanes of one launch sequence."""
    c1 = {stem: (path, g) for stem, path, g in golden_dir["c1"]}
    stems = ["c1_S200_100001", "c1_S200_100002", "c1_S200_100001", "c1_S200_100002"]
    probs = [SC.Problem(SC.load_scenario(c1[s][0]), 0) for s in stems]
    opts, obj, status, stats, errs = gpu.solve_batch(probs)
    for i, s in enumerate(stems):
        assert status[i] == 0
        assert bits(obj[i]) == c1[s][1]["dp"]["obj"], s
        assert stats[i]["transitions_ref"] == stats[i % 2]["transitions_ref"]


def _c4_problem(tmp_path, seed=400000, steps=600):
    from paper_2407_13126_b200 import workloads as W
    path = W.write_scenario(W.c2_spec(seed, steps=steps, windows=1), str(tmp_path), "c4_%d" % seed)
    return SC.Problem(SC.load_scenario(path), 0)


def test_goodput_table_batch_matches_window(gpu, golden_dir):
    """The batched table (Pareto placements, pre-scaled min-fold) == the
    per-window ub_suffix, bit for bit, for every trace of a batch."""
    rng = np.random.default_rng(11)
    for stem, path, g in golden_dir["random"][:40] + golden_dir["c1"]:
        sc = SC.load_scenario(path)
        p = SC.Problem(sc, 0)
        traces = np.concatenate([p.forecast[None].astype(np.int32),
                                 rng.integers(0, 400, size=(3, p.M, p.S)).astype(np.int32)])
        ub, best, npar = gpu.goodput_table_batch(p, traces, with_best=True)
        assert 1 <= npar
        for b in range(traces.shape[0]):
            q = SC.Problem(sc, 0, forecast=traces[b].astype(np.int64))
            ub_w, _, _ = gpu.goodput_table(q)
            assert ub[b].tobytes() == ub_w.tobytes(), (stem, b)
            assert np.array_equal(np.cumsum(best[b][::-1])[::-1] >= 0, np.ones(p.S, bool))


def test_goodput_table_batch_c4_matches_oracle(gpu, tmp_path):
    """Config-4 shape: 4 tenants (C2 generator, MMPP), S = 600, a batch of traces;
    two traces checked against the CPU restatement directly."""
    from paper_2407_13126_b200 import workloads as W
    p = _c4_problem(tmp_path)
    traces = np.stack([W.mmpp_trace([40.0, 120.0, 12.0, 10.0], p.S, 400000 + k) for k in range(32)]).astype(np.int32)
    ub, npar = gpu.goodput_table_batch(p, traces)
    for b in (0, 17):
        q = SC.Problem(p.scenario, 0, forecast=traces[b].astype(np.int64))
        ub_o, _, _ = B.goodput_table(q)
        assert ub[b].tobytes() == ub_o.tobytes(), b


def test_window_boundary_matches_reference(gpu, golden_dir):
    """plan_window_boundary (the Ekya-like baseline, §8(f) row 1) on the GPU ==
    the unmodified reference: plan encoding and evaluate_plan objective bits,
    cold and chained, on the random corpus, the config-1 fixtures and the KATs."""
    import json
    import os
    wb = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "wb_golden.json")))
    n = 0
    for kind in ("random", "c1", "kat"):
        for stem, path, g in golden_dir[kind]:
            if stem not in wb:
                continue
            sc = SC.load_scenario(path)
            runs = [(None, wb[stem]["wb"])]
            if "chain" in wb[stem]:
                runs.append(([tuple(x) for x in wb[stem]["chain"]["initial"]], wb[stem]["chain"]["wb"]))
            for initial, want in runs:
                p = SC.Problem(sc, 0, initial=initial)
                if "error" in want:
                    with pytest.raises(capi.PlannerError) as e:
                        gpu.window_boundary(p)
                    assert e.value.code == want["error"], stem
                    continue
                opt, cfg, lab, obj = gpu.window_boundary(p)
                assert planner.encode(cfg, lab, nslots(sc)) == want["encode"], (stem, initial is not None)
                assert bits(obj) == want["obj"], stem
                n += 1
    assert n >= 150


def test_replay_requests_matches_reference(gpu, golden_dir):
    """Request-mode replay (run_requests, §8(f) row 2) of each window's solve_dp
    plan: every tenant's counters bit-equal to the unmodified reference
    (per-request mt19937_64 correctness draws, FIFO deadlines, psi spill)."""
    import json
    import os
    rp = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "replay_golden.json")))
    fields = ("received", "served", "timely", "correct", "valid", "dropped", "queued_at_end")
    n = 0
    for kind in ("random", "c1", "kat"):
        for stem, path, g in golden_dir[kind]:
            want = rp.get(stem)
            if not want or "runs" not in want:
                continue
            p = SC.Problem(SC.load_scenario(path), 0)
            opt = gpu.solve_window(p)[0]
            seeds = [r["seed"] for r in want["runs"]]
            got = gpu.replay_requests(p, opt[None], p.forecast[None], seeds)
            for k, run in enumerate(want["runs"]):
                for m, job in enumerate(run["jobs"]):
                    r = got[0, 0, k, m]
                    assert [bits(r[f]) for f in fields] == job[:7], (stem, run["seed"], m)
                    assert int(r["reconfigurations"]) == job[7], (stem, m)
                    assert bits(r["overhead_seconds"]) == job[8], (stem, m)
                    n += 1
    assert n >= 300


def test_preinit_matches_reference(gpu, golden_dir):
    """Pre-initialisation (§8(f) row 4) on the GPU == the reference's
    plan_preinit + apply_preinit: override sets, evaluate_plan totals with the
    overrides, and request-mode replays of the EffectivePlan, for the solve_dp
    plan and three sparse random feasible plans of every scenario."""
    import json
    import os
    pg = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "preinit_golden.json")))
    fields = ("received", "served", "timely", "correct", "valid", "dropped", "queued_at_end")
    n_plans = n_ov = 0
    for kind in ("random", "c1", "kat"):
        for stem, path, g in golden_dir[kind]:
            want = pg.get(stem)
            if not want or "dp" not in want:
                continue
            sc = SC.load_scenario(path)
            p = SC.Problem(sc, 0)
            en = gpu.enumerate(p)
            ns = nslots(sc)
            index = {}
            for o in range(len(en["config"])):
                c = int(en["config"][o])
                index.setdefault((c,) + tuple(int(x) for x in en["labels"][o][:ns[c]]), o)
            cases = [want["dp"]] + want["random"]
            plans = []
            for w in cases:
                enc, plan, i = w["encode"], [], 0
                while i < len(enc):
                    c = enc[i]
                    plan.append(index[tuple(enc[i:i + 1 + ns[c]])])
                    i += 1 + ns[c]
                plans.append(plan)
            plans = np.asarray(plans, np.int32)
            ov, fired = gpu.preinit(p, plans)
            totals = gpu.evaluate_batch(p, plans, p.forecast[None], overrides=ov)
            runs = gpu.replay_requests(p, plans, p.forecast[None], [want["dp"]["seed"]], overrides=ov)
            for k, w in enumerate(cases):
                got = sorted((int(m), int(s)) for s, m in zip(*np.nonzero(ov[k])))
                assert got == sorted(tuple(x) for x in w["overrides"]), (stem, k)
                assert bits(totals[k, 0]) == w["obj"], (stem, k)
                for m, job in enumerate(w["jobs"]):
                    r = runs[k, 0, 0, m]
                    assert [bits(r[f]) for f in fields] == job[:7], (stem, k, m)
                    assert int(r["reconfigurations"]) == job[7] and bits(r["overhead_seconds"]) == job[8]
                n_plans += 1
                n_ov += len(w["overrides"])
    assert n_plans >= 600 and n_ov >= 500


def test_per_window_driver_matches_reference(gpu):
    """The per-window planning loop (§8(f) row 3): predictor -> GPU solve_dp with
    the carried final ranges -> realized evaluate_plan, window after window,
    for several scenarios advanced together as batched lanes; == the loop
    built from the unmodified reference's own pieces (`migref drive`)."""
    import json
    import os
    from paper_2407_13126_b200 import driver
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "drive")
    gold = json.load(open(os.path.join(d, "drive_golden.json")))
    feasible = ["d_c1_40", "d_c1_40v"]
    for pred in ("oracle", "persistence", "ewma:0.3"):
        scs = [SC.load_scenario(os.path.join(d, stem + ".scn")) for stem in feasible]
        plans = driver.plan_scenarios(gpu, scs, pred)
        for stem, sc, wins in zip(feasible, scs, plans):
            want = gold[stem][pred]["windows"]
            assert len(wins) == len(want)
            for wp, w in zip(wins, want):
                assert planner.encode(wp.config, wp.labels, nslots(sc)) == w["encode"], (stem, pred, wp.window)
                assert wp.forecast.tolist() == w["forecast"], (stem, pred, wp.window)
                assert bits(wp.objective) == w["obj"] and bits(wp.realized) == w["realized"], (stem, pred)
        sc = SC.load_scenario(os.path.join(d, "d_c2_100.scn"))
        with pytest.raises(capi.PlannerError) as e:
            driver.plan_scenarios(gpu, [sc], pred)
        assert e.value.code == gold["d_c2_100"][pred]["error"]


def test_edge_cases(gpu, tmp_path):
    """The shortest windows the grammar allows (S = 2; every retraining finishes
    in a single slot), empty batches, and an all-zero trace: GPU DP == GPU brute force == the CPU
    restatement; empty inputs return empty outputs without error."""
    from paper_2407_13126_b200 import workloads as W
    ts = [W.Tenant("a", 40.0, [0.6], [0.9], rt={k: 1 for k in range(1, 8)}, psi=0.5),
          W.Tenant("b", 50.0, [0.62], [0.89], rt={k: 1 for k in range(1, 8)}, psi=1.5)]
    for S, counts in ((2, [[120, 30], [150, 9]]), (2, [[0, 0], [0, 0]]), (3, [[500, 0, 900], [7, 3000, 1]])):
        spec = W.ScenarioSpec(ts, S, 1)
        spec.counts = np.asarray(counts, np.int64)
        p = SC.Problem(SC.load_scenario(W.write_scenario(spec, str(tmp_path), "edge%d_%d" % (S, sum(map(sum, counts))))), 0)
        opt, cfg, lab, obj, _ = gpu.solve_window(p)
        want, want_obj, _ = B.solve_window(p)
        assert list(opt) == list(want), S
        assert bits(obj) == bits(want_obj), S
        if S == 2:  # |O|^2 ~ 6e8 sequences: the GPU brute force takes it with a raised cap
            bopt, _, _, bobj = gpu.solve_bruteforce(p, bruteforce_cap=1e9)
            assert list(bopt) == list(want) and bits(bobj) == bits(want_obj)
    opts, obj, status, stats, errs = gpu.solve_batch([p])
    assert status[0] == 0 and bits(obj[0]) == bits(want_obj)
    assert gpu.evaluate_batch(p, np.zeros((0, p.S), np.int32), p.forecast[None]).shape == (0, 1)
    ub, npar = gpu.goodput_table_batch(p, np.zeros((0, p.M, p.S), np.int32))
    assert ub.shape == (0, p.S + 1)
    assert gpu.replay_requests(p, opt[None], p.forecast[None], []).shape == (1, 1, 0, p.M)
    ov, fired = gpu.preinit(p, np.zeros((0, p.S), np.int32))
    assert ov.shape == (0, p.S, p.M)


def test_replay_requests_multi_window(gpu):
    """run_requests over a 3-window scenario (queues, psi spill and masks carried
    across windows) for the per-window loop's plans: per-window counters bit-equal
    to the reference's, and their window-order sums equal its totals."""
    import json
    import os
    from paper_2407_13126_b200 import driver
    d = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "drive")
    gold = json.load(open(os.path.join(d, "replay_windows_golden.json")))
    fields = ("received", "served", "timely", "correct", "valid", "dropped", "queued_at_end")
    for stem in ("d_c1_40", "d_c1_40v"):
        sc = SC.load_scenario(os.path.join(d, stem + ".scn"))
        wins = driver.plan_scenarios(gpu, [sc], "oracle")[0]
        for w, wp in enumerate(wins):
            assert planner.encode(wp.config, wp.labels, nslots(sc)) == gold[stem + ":5"]["encode"][w]
        plans = np.concatenate([wp.options for wp in wins])[None]
        p = SC.Problem(sc, 0)
        got = gpu.replay_requests(p, plans, sc.counts[None], [5, 77], windows=sc.window_count)
        for k, seed in enumerate((5, 77)):
            want = gold["%s:%d" % (stem, seed)]
            for w in range(sc.window_count):
                for m, job in enumerate(want["windows"][w]):
                    r = got[0, 0, k, w, m]
                    assert [bits(r[f]) for f in fields] == job[:7], (stem, seed, w, m)
                    assert int(r["reconfigurations"]) == job[7] and bits(r["overhead_seconds"]) == job[8]
            for m, job in enumerate(want["totals"]):
                tot = 0.0
                for w in range(sc.window_count):
                    tot += float(got[0, 0, k, w, m]["valid"])
                assert bits(tot) == job[4]


def test_launch_modes_agree(golden_dir):
    """The captured graph (parallel branches per step), a single-chain graph
    (MGS_NO_FORK) and eager launches (MGS_DEBUG_STEPS) give the same plans,
    objective bits and counters, equal to the reference goldens."""
    import json
    import os
    import subprocess
    import sys

    cases = [(stem, path, g) for stem, path, g in golden_dir["c1"] if int(stem.split("_")[1][1:]) <= 60][:2]
    assert cases
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "solve_variant.py")
    results = {}
    for name, extra in (("graph", {}), ("chain", {"MGS_NO_FORK": "1"}), ("eager", {"MGS_DEBUG_STEPS": "1"})):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, script] + [str(p) for _, p, _ in cases], env=env, capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        results[name] = json.loads(r.stdout.strip().splitlines()[-1])
    assert results["graph"] == results["chain"] == results["eager"]
    for stem, path, g in cases:
        assert results["graph"][os.path.basename(str(path))]["obj"] == g["dp"]["obj"], stem


def test_kernel_paths_agree(golden_dir):
    """Every alternative path of the graph engine gives the reference's plans and
    objective bits, single windows and lane batches: k_units with a thread per
    group everywhere (MGS_UNITS_THREAD_MIN=0) or a warp per group everywhere,
    k_trans_small without half / quarter items (MGS_NO_SUBITEMS), and placement
    maps cleared per group instead of step-tagged (MGS_EX_CLEAR). Includes both
    full S = 200 C1 windows."""
    import json
    import os
    import subprocess
    import sys

    c1 = list(golden_dir["c1"])
    rnd = golden_dir["random"][::16]
    multi = [(stem, path, g) for stem, path, g in golden_dir["multi"] if "error" not in g["dp"]][:4]
    cases = c1 + rnd + multi
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "solve_variant.py")
    results = {}
    variants = (("default", {}), ("units_thread", {"MGS_UNITS_THREAD_MIN": "0"}),
                ("units_warp", {"MGS_UNITS_THREAD_MIN": "1000000000"}), ("full_items", {"MGS_NO_SUBITEMS": "1"}),
                ("ex_clear", {"MGS_EX_CLEAR": "1"}))
    for name, extra in variants:
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, script, "--batch"] + [str(p) for _, p, _ in cases], env=env,
                           capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        results[name] = json.loads(r.stdout.strip().splitlines()[-1])
    for name, _ in variants[1:]:
        assert results[name] == results["default"], name
    for stem, path, g in cases:
        base = os.path.basename(str(path))
        assert results["default"][base]["obj"] == g["dp"]["obj"], stem
        assert results["default"]["batch:" + base]["obj"] == g["dp"]["obj"], stem


def test_capacity_regrow(golden_dir):
    """Every device buffer of the graph engine starting tiny (MGS_V2_SMALL_CAPS):
    each overflow is raised block-uniformly, the window is re-run with grown
    capacities (frontier, groups, history, units, candidates, work items, subset
    tables, successor hash), and plans, objective bits and counters come out
    equal to the default run and to the reference goldens, single windows and
    lane batches (M = 1..4)."""
    import json
    import os
    import subprocess
    import sys

    c1 = [(stem, path, g) for stem, path, g in golden_dir["c1"] if int(stem.split("_")[1][1:]) <= 60][:1]
    rnd = golden_dir["random"][::16]
    multi = [(stem, path, g) for stem, path, g in golden_dir["multi"] if "error" not in g["dp"]][:4]
    cases = c1 + rnd + multi
    script = os.path.join(os.path.dirname(os.path.abspath(__file__)), "solve_variant.py")
    results = {}
    for name, extra in (("default", {}), ("small", {"MGS_V2_SMALL_CAPS": "1"})):
        env = dict(os.environ, **extra)
        r = subprocess.run([sys.executable, script, "--batch"] + [str(p) for _, p, _ in cases], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, (name, r.stderr[-2000:])
        results[name] = json.loads(r.stdout.strip().splitlines()[-1])
    assert results["default"] == results["small"]
    for stem, path, g in cases:
        name = os.path.basename(str(path))
        assert results["small"][name]["obj"] == g["dp"]["obj"], stem
        assert results["small"]["batch:" + name]["obj"] == g["dp"]["obj"], stem
