"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs /root/reference and oracle/_ref/migref):

    python oracle/make_goldens.py [--c1-full]

Outputs (all small, committed):
  tests/golden/random_<seed>.json  the reference's own randomized oracle corpus
        (tests/test_util.hpp:104-181 via `migref gen-random`), each scenario's
        catalog / scenario / trace text plus the reference's solve_dp and
        solve_bruteforce plans, objective bits and per-(s,m) throughput bits,
        cold and chained (initial = final_ranges of the cold plan).
  tests/golden/c1/*.scn|csv + c1_golden.json   config-1 fixtures (paper_2407_13126_b200
        .workloads.c1_spec) with the reference's plans; --c1-full adds the S=200
        windows (about two minutes of reference CPU time each).
  tests/golden/kat/*  hand-written known-answer scenarios whose expected values
        come from the reference's own tests (eval_test.cpp, solver_test.cpp).
  tests/golden/multi_m<M>_<seed>.json, tests/golden/multi/*  M = 3..4 windows
        solved by "reference + 1-line fix" (oracle/_ref/migref_patched: only the
        packed-status widening at solvers.hpp:359,401,414), with brute force
        where |O|^S is small, plus the unmodified reference's answer
        (infeasible.joint, the truncation bug).
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import workloads as W  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
MIGREF = os.path.join(HERE, "_ref", "migref")
MIGREF_PATCHED = os.path.join(HERE, "_ref", "migref_patched")

# (seed, count, allow_accuracy_drop): the seeds of the reference's solver /
# baseline suites (solver_test.cpp:110-178, baseline_test.cpp:139-180) plus
# extra seeds for breadth.
RANDOM_SEEDS = [(20250101, 25, True), (424242, 10, True), (777, 4, True), (1312, 8, False), (5150, 20, True),
                (31337, 20, True), (1, 25, True), (2, 25, False), (3, 25, True)]


def ref_solve(path, *extra, binary=MIGREF):
    out = subprocess.run([binary, "solve", path] + list(extra), check=True, capture_output=True, text=True)
    return json.loads(out.stdout)


# M = 3..4 corpora: "reference + 1-line fix" (oracle/Makefile ref-patched), the
# only reference build that can solve them. Each entry:
# (M, seed, count, S_lo, S_hi, brute-force estimate cap or None for DP only).
MULTI_SEEDS = [(3, 31, 24, 3, 4, 2e6), (3, 32, 12, 5, 8, None), (4, 41, 12, 4, 6, None)]
# C2-shaped windows (workloads.c2_spec, shortened): (tenants, S, vol_per_gpc, seed)
MULTI_C2 = [(3, 20, 6, 200003), (4, 12, 2, 200004), (4, 12, 3, 200004)]


def make_multi():
    for M, seed, count, s_lo, s_hi, cap in MULTI_SEEDS:
        with tempfile.TemporaryDirectory() as td:
            cmd = [MIGREF_PATCHED, "gen-multi", str(seed), str(count), td, str(M), str(s_lo), str(s_hi),
                   "%g" % (cap or 1e300)]
            paths = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout.split()
            bundle = {}
            for p in paths:
                stem = os.path.basename(p)[:-4]
                files = {ext: open(os.path.join(td, stem + "." + ext)).read() for ext in ("scn", "catalog", "csv")}
                extra = ["--chain"] + (["--bf"] if cap else [])
                files["golden"] = ref_solve(p, *extra, binary=MIGREF_PATCHED)
                files["golden"]["unpatched"] = ref_solve(p)  # the shipped reference: infeasible.joint
                bundle[stem] = files
        out = os.path.join(GOLD, "multi_m%d_%d.json" % (M, seed))
        with open(out, "w") as f:
            json.dump(bundle, f, indent=0, sort_keys=True)
        print(out, len(bundle))
    d = os.path.join(GOLD, "multi")
    os.makedirs(d, exist_ok=True)
    golden = {}
    for M, S, vol, seed in MULTI_C2:
        stem = "c2_m%d_S%d_v%d_%d" % (M, S, vol, seed)
        spec = W.c2_spec(seed, steps=S, windows=1, tenants=M, vol_per_gpc=vol)
        spec.catalog_path = os.path.join(GOLD, "lattice_a100.catalog")
        scn = W.write_scenario(spec, d, stem)
        golden[stem] = ref_solve(scn, binary=MIGREF_PATCHED)
        golden[stem]["unpatched"] = ref_solve(scn)
        print(stem, json.dumps(golden[stem])[:200])
    with open(os.path.join(d, "multi_golden.json"), "w") as f:
        json.dump(golden, f, indent=0, sort_keys=True)


def make_random():
    for seed, count, drop in RANDOM_SEEDS:
        with tempfile.TemporaryDirectory() as td:
            cmd = [MIGREF, "gen-random", str(seed), str(count), td] + ([] if drop else ["--no-drop"])
            paths = subprocess.run(cmd, check=True, capture_output=True, text=True).stdout.split()
            bundle = {}
            for p in paths:
                stem = os.path.basename(p)[:-4]
                files = {ext: open(os.path.join(td, stem + "." + ext)).read() for ext in ("scn", "catalog", "csv")}
                files["golden"] = ref_solve(p, "--chain", "--bf")
                bundle[stem] = files
        out = os.path.join(GOLD, "random_%d.json" % seed)
        with open(out, "w") as f:
            json.dump(bundle, f, indent=0, sort_keys=True)
        print(out, len(bundle))


C1_MINI = [(100001, 40, 600), (100002, 40, 600), (100003, 60, 900), (100004, 24, 360)]
C1_FULL = [(100001, 200, 3000), (100002, 200, 3000)]


def make_c1(full):
    d = os.path.join(GOLD, "c1")
    os.makedirs(d, exist_ok=True)
    gpath = os.path.join(d, "c1_golden.json")
    golden = json.load(open(gpath)) if os.path.exists(gpath) else {}
    todo = C1_MINI + (C1_FULL if full else [])
    for seed, S, vol in todo:
        stem = "c1_S%d_%d" % (S, seed)
        spec = W.c1_spec(seed, steps=S, data_volume=vol)
        spec.catalog_path = os.path.join(GOLD, "lattice_a100.catalog")
        scn = W.write_scenario(spec, d, stem)
        if stem in golden:
            continue
        golden[stem] = ref_solve(scn, "--chain") if S <= 60 else ref_solve(scn)
        print(stem, golden[stem]["seconds"], golden[stem]["dp"]["objective"])
        with open(gpath, "w") as f:
            json.dump(golden, f, indent=0, sort_keys=True)


KAT_CATALOG_43 = "config 4_3 4@0 3@4\n"


def kat_files():
    """Known-answer scenarios transcribed from the reference tests; the expected
    numbers are the reference tests' assertions."""
    return {
        # test_util.hpp:71-99 worked example: optimum exactly 12.5 (solver_test.cpp:34-47)
        "worked_example": dict(catalog=KAT_CATALOG_43, S=3, models=[
            dict(name="m0", cap={3: 6, 4: 8}, rt={3: 2, 4: 1}, psi=0.0, floor=1, pre=0.5, post=1.0)],
            trace=[[5, 5, 5]], expect_objective=12.5),
        # solver_test.cpp:49-70 forced scenario: inference 4@0, retraining 3@4 every step
        "forced": dict(catalog=KAT_CATALOG_43, S=4, models=[
            dict(name="m0", cap={4: 40}, rt={3: 4}, psi=0.0, floor=4, pre=0.5, post=1.0)],
            trace=[[10, 10, 10, 10]]),
        # solver_test.cpp:72-79: zero arrivals score zero
        "zero_trace": dict(catalog=KAT_CATALOG_43, S=3, models=[
            dict(name="m0", cap={3: 6, 4: 8}, rt={3: 2, 4: 1}, psi=0.0, floor=1, pre=0.5, post=1.0)],
            trace=[[0, 0, 0]], expect_objective=0.0),
        # solver_test.cpp:81-94: single 7-slot configuration cannot co-locate retraining
        "no_coexistence": dict(catalog="config 7 7@0\n", S=3, models=[
            dict(name="m0", cap={7: 70}, rt={7: 1}, psi=0.0, floor=1, pre=0.5, post=1.0)],
            trace=[[10, 10, 10]], expect_error="infeasible.no-coexistence-configuration"),
        # solver_test.cpp:96-108: deployment floor above the largest instance
        "deployment_floor": dict(catalog=KAT_CATALOG_43, S=3, models=[
            dict(name="m0", cap={5: 50, 6: 60, 7: 70}, rt={3: 1}, psi=0.0, floor=5, pre=0.5, post=1.0)],
            trace=[[10, 10, 10]], expect_error="infeasible.deployment-floor"),
        # test_util.hpp:43-69 small two-model scenario (solver_test.cpp:180-207 guards)
        "small_two_model": dict(catalog="config 4_3 4@0 3@4\nconfig 4_2_1 4@0 2@4 1@6\nconfig 2_2_2_1 2@0 2@2 2@4 1@6\n",
                                S=6, models=[
            dict(name="alpha", cap={1: 10, 2: 20, 3: 30, 4: 40, 7: 70}, rt={1: 3, 2: 2, 3: 2, 4: 1, 7: 1}, psi=0.5,
                 floor=1, pre=0.5, post=0.9, gflops=10.0, latency=0.02),
            dict(name="beta", cap={1: 8, 2: 16, 3: 24, 4: 32, 7: 56}, rt={1: 3, 2: 2, 3: 1, 4: 1, 7: 1}, psi=0.5,
                 floor=1, pre=0.6, post=0.8, gflops=5.0, latency=0.05)],
            trace=[[12] * 6, [9] * 6]),
    }


def write_kat(name, k, d):
    with open(os.path.join(d, name + ".catalog"), "w") as f:
        f.write(k["catalog"])
    with open(os.path.join(d, name + ".csv"), "w") as f:
        f.write("second,model,count\n")
        for s in range(k["S"]):
            for m, mod in enumerate(k["models"]):
                f.write("%d,%s,%d\n" % (s, mod["name"], k["trace"][m][s]))
    lines = ["[windows]", "size %d" % k["S"], "count 1", "[catalog]", "file %s.catalog" % name, "[models]"]
    for mod in k["models"]:
        lines += ["model %s" % mod["name"], "gflops %s" % W.fmt_real(mod.get("gflops", 1.0)),
                  "min_deploy_gpcs %d" % mod["floor"], "latency_full %s" % W.fmt_real(mod.get("latency", 0.01)),
                  "reconfig_overhead %s" % W.fmt_real(mod["psi"]),
                  "capability " + " ".join("%d:%s" % (kk, W.fmt_real(v)) for kk, v in sorted(mod["cap"].items())),
                  "rt_table " + " ".join("%d:%d" % (kk, v) for kk, v in sorted(mod["rt"].items())),
                  "accuracy_pre %s" % W.fmt_real(mod["pre"]), "accuracy_post %s" % W.fmt_real(mod["post"])]
    lines += ["[trace]", "file %s.csv" % name, ""]
    path = os.path.join(d, name + ".scn")
    with open(path, "w") as f:
        f.write("\n".join(lines))
    return path


def make_kat():
    d = os.path.join(GOLD, "kat")
    os.makedirs(d, exist_ok=True)
    golden = {}
    for name, k in kat_files().items():
        p = write_kat(name, k, d)
        g = ref_solve(p, "--bf")
        for key in ("expect_objective", "expect_error"):
            if key in k:
                g[key] = k[key]
        golden[name] = g
        budget = ref_solve(p, "--budget", "1") if name == "small_two_model" else None
        if budget:
            golden[name]["budget1"] = budget
    with open(os.path.join(d, "kat_golden.json"), "w") as f:
        json.dump(golden, f, indent=0, sort_keys=True)
    print("kat", sorted(golden))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--c1-full", action="store_true")
    ap.add_argument("--only", choices=["random", "c1", "kat", "multi"])
    a = ap.parse_args()
    if not os.path.exists(MIGREF):
        sys.exit("build the reference first: make -C oracle ref")
    if a.only in (None, "kat"):
        make_kat()
    if a.only in (None, "random"):
        make_random()
    if a.only in (None, "c1"):
        make_c1(a.c1_full)
    if a.only in (None, "multi"):
        make_multi()
