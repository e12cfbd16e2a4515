"""TEST INFRASTRUCTURE ONLY: the config-4 M = 2 / S = 200 variant (tests/golden/c4/):
the first two tenants of the C4 generator's traces 400000..400003, one window
each, and the UNMODIFIED reference's solve_dp on them (`migref solve`).

    python oracle/make_c4_goldens.py   (~1 min of reference CPU per window; in parallel)
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c4")
SEEDS = [400000, 400001, 400002, 400003]


def main():
    os.makedirs(OUT, exist_ok=True)
    procs = {}
    for seed in SEEDS:
        stem = "c4_m2_S200_%d" % seed
        path = W.write_scenario(W.c2_spec(seed, steps=200, windows=1, tenants=2), OUT, stem)
        procs[stem] = subprocess.Popen([os.path.join(HERE, "_ref", "migref"), "solve", path, "0"], stdout=subprocess.PIPE,
                                       text=True)
    gold = {stem: json.loads(p.communicate(timeout=3600)[0]) for stem, p in procs.items()}
    json.dump(gold, open(os.path.join(OUT, "c4_golden.json"), "w"), sort_keys=True)


if __name__ == "__main__":
    main()
