"""TEST INFRASTRUCTURE ONLY: config-5 subproblems (tests/golden/c5/) and the
per-window planning loop's results for their first windows from the UNMODIFIED
reference (`migref drive <scn> oracle <max_windows>`: solve_dp with the carried
final_ranges, evaluate_plan on forecast and actual counts).

    python oracle/make_c5_goldens.py [n_subproblems=2] [max_windows=2]

Each window is a full S=200 config-1-style solve (~2 min of reference CPU time);
the subproblems run in parallel processes.
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
from paper_2407_13126_b200 import workloads as W  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "c5")


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wmax = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    os.makedirs(OUT, exist_ok=True)
    specs = W.c5_specs()
    procs = {}
    for k, spec in enumerate(specs):
        path = W.write_scenario(spec, OUT, "c5_gpu%d" % k)
        if k < n:
            procs[k] = subprocess.Popen([os.path.join(HERE, "_ref", "migref"), "drive", path, "oracle", str(wmax)],
                                        stdout=subprocess.PIPE, text=True)
    gold = {}
    for k, p in procs.items():
        out, _ = p.communicate(timeout=7200)
        gold["c5_gpu%d" % k] = json.loads(out)
        print(k, [w["obj"] for w in gold["c5_gpu%d" % k]["windows"]], flush=True)
    json.dump({"max_windows": wmax, "golden": gold}, open(os.path.join(OUT, "c5_golden.json"), "w"), sort_keys=True)


if __name__ == "__main__":
    main()
