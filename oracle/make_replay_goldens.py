"""TEST INFRASTRUCTURE ONLY: request-mode replay goldens from the UNMODIFIED
reference (run_requests, simulator.hpp:209-275) of each scenario's window-0
solve_dp plan, seeds 1 and 20240607, for the random corpus and the config-1
fixtures up to S = 60.

    python oracle/make_replay_goldens.py   -> tests/golden/replay_golden.json
"""
import json
import os
import subprocess
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_util  # noqa: E402

SEEDS = ["1", "20240607"]


def main():
    cases = golden_util.materialize(tempfile.mkdtemp())
    out = {}
    for kind in ("random", "c1", "kat"):
        for stem, path, _ in cases[kind]:
            if kind == "c1" and int(stem.split("_")[1][1:]) > 60:
                continue
            r = subprocess.run([os.path.join(HERE, "_ref", "migref"), "replay", path] + SEEDS,
                               capture_output=True, text=True, timeout=600)
            out[stem] = json.loads(r.stdout)
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "replay_golden.json"), "w"), sort_keys=True)
    print(len(out), "scenarios")


if __name__ == "__main__":
    main()
