"""TEST INFRASTRUCTURE ONLY: multi-window scenarios (tests/golden/drive/) and the
per-window planning loop's results from the UNMODIFIED reference's pieces
(`migref drive`: predict_arrivals -> solve_dp with carried final_ranges ->
evaluate_plan), for the oracle, persistence and ewma:0.3 predictors.

    python oracle/make_drive_goldens.py   -> tests/golden/drive/*

Also the multi-window request replay of the loop's plans (`migref replay-windows`,
run_requests over all windows with queues and psi spill carried across them).
"""
import dataclasses
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "drive")
PREDICTORS = ["oracle", "persistence", "ewma:0.3"]


def fixtures():
    specs = {"d_c2_100": W.c2_spec(500001, steps=100, windows=3, tenants=2)}
    for stem, seed, vol in (("d_c1_40", 500003, 1000), ("d_c1_40v", 500004, 800)):
        c1 = W.c1_spec(seed, steps=40 * 3, data_volume=vol)
        specs[stem] = dataclasses.replace(c1, window_size=40, window_count=3)
    return specs


def main():
    os.makedirs(OUT, exist_ok=True)
    gold = {}
    for stem, spec in fixtures().items():
        path = W.write_scenario(spec, OUT, stem)
        gold[stem] = {}
        for pred in PREDICTORS:
            r = subprocess.run([os.path.join(HERE, "_ref", "migref"), "drive", path, pred], capture_output=True,
                               text=True, timeout=900)
            gold[stem][pred] = json.loads(r.stdout)
            print(stem, pred, list(gold[stem][pred].keys()), flush=True)
    json.dump(gold, open(os.path.join(OUT, "drive_golden.json"), "w"), sort_keys=True)
    # multi-window request replay of the loop's plans (run_requests over all windows)
    rw = {}
    for stem in ("d_c1_40", "d_c1_40v"):
        for seed in ("5", "77"):
            r = subprocess.run([os.path.join(HERE, "_ref", "migref"), "replay-windows", os.path.join(OUT, stem + ".scn"),
                                seed], capture_output=True, text=True, timeout=900)
            rw["%s:%s" % (stem, seed)] = json.loads(r.stdout)
    json.dump(rw, open(os.path.join(OUT, "replay_windows_golden.json"), "w"), sort_keys=True)


if __name__ == "__main__":
    main()
