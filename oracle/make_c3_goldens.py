"""TEST INFRASTRUCTURE ONLY: config-3 fixtures (tests/golden/c3/: three
two-tenant pairs on the H100 lattice, 18 x 200 slots, MMPP) and the per-window
loop's results from the UNMODIFIED reference
(`migref drive <scn> <predictor> <max_windows> <lookback> <psi>`: the
reference's predict_arrivals over a sliding history of the last `lookback`
windows, solve_dp with the carried final_ranges, evaluate_plan on forecast and
actual counts, every tenant's reconfig_overhead set to psi).

    python oracle/make_c3_goldens.py   (~70 s of reference CPU per window; cases in parallel)
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c3")
# (pair, predictor, windows, lookback, psi): the sweep's extremes, both history
# predictors, and a lookahead that slides (window 2 sees only window 1)
CASES = [(0, "ewma:0.3", 3, 1, 0.5), (1, "persistence", 2, 1, 6.0), (2, "oracle", 2, 1, 0.0),
         (0, "persistence", 2, 1, 1.0), (1, "ewma:0.5", 3, 2, 0.25), (2, "ewma:0.3", 3, 1, 6.0)]


def main():
    os.makedirs(OUT, exist_ok=True)
    for k, spec in enumerate(W.c3_specs()):
        W.write_scenario(spec, OUT, "c3_pair%d" % k)
    procs = {}
    for case in CASES:
        pair, pred, nw, lb, psi = case
        path = os.path.join(OUT, "c3_pair%d.scn" % pair)
        procs[case] = subprocess.Popen([os.path.join(HERE, "_ref", "migref"), "drive", path, pred, str(nw), str(lb),
                                        repr(psi)], stdout=subprocess.PIPE, text=True)
    gold = []
    for case, p in procs.items():
        out, _ = p.communicate(timeout=7200)
        pair, pred, nw, lb, psi = case
        gold.append({"pair": pair, "predictor": pred, "windows": nw, "lookback": lb, "psi": psi,
                     "result": json.loads(out)})
        print(case, [w.get("obj") for w in gold[-1]["result"].get("windows", [])], flush=True)
    json.dump(gold, open(os.path.join(OUT, "c3_golden.json"), "w"), sort_keys=True)


if __name__ == "__main__":
    main()
