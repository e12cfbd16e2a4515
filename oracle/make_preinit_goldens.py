"""TEST INFRASTRUCTURE ONLY: pre-initialisation goldens from the UNMODIFIED
reference (plan_preinit + apply_preinit, preinit.hpp:41-114; evaluate_plan
with the overrides; overhead_summary; run_requests of the EffectivePlan) for
each scenario's window-0 solve_dp plan.

    python oracle/make_preinit_goldens.py   -> tests/golden/preinit_golden.json
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


def main():
    cases = golden_util.materialize(tempfile.mkdtemp())
    out = {}
    for kind in ("random", "c1", "kat"):
        for stem, path, _ in cases[kind]:
            if kind == "c1" and int(stem.split("_")[1][1:]) > 60:
                continue
            r = subprocess.run([os.path.join(HERE, "_ref", "migref"), "preinit", path, "99", "3"],
                               capture_output=True, text=True, timeout=600)
            out[stem] = json.loads(r.stdout)
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "preinit_golden.json"), "w"), sort_keys=True)
    n_ov = sum(len(p["overrides"]) for v in out.values() if "dp" in v for p in [v["dp"]] + v["random"])
    print(len(out), "scenarios,", n_ov, "overrides")


if __name__ == "__main__":
    main()
