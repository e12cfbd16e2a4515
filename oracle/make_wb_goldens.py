"""TEST INFRASTRUCTURE ONLY: window-boundary (Ekya) goldens from the UNMODIFIED
reference (plan_window_boundary, baselines.hpp:139-289), cold and chained, for
every scenario of the committed corpus (random corpus, config-1 fixtures,
known-answer scenarios) plus config-1 S=200 windows.

    python oracle/make_wb_goldens.py        -> tests/golden/wb_golden.json
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

MIGREF = os.path.join(HERE, "_ref", "migref")


def main():
    tmp = tempfile.mkdtemp()
    cases = golden_util.materialize(tmp)
    out = {}
    for kind in ("random", "c1", "kat"):
        for stem, path, _ in cases[kind]:
            r = subprocess.run([MIGREF, "solve", path, "--wb", "--chain"], capture_output=True, text=True, timeout=600)
            d = json.loads(r.stdout)
            if "error" in d:  # the DP itself fails: no chained window to plan
                out[stem] = {"wb": d}
                continue
            out[stem] = {"wb": d["wb"], "chain": {"initial": d["chain"]["initial"], "wb": d["chain"]["wb"]}}
            print(stem, "ok" if "encode" in d["wb"] else d["wb"].get("error"), flush=True)
    json.dump(out, open(os.path.join(ROOT, "tests", "golden", "wb_golden.json"), "w"), sort_keys=True)


if __name__ == "__main__":
    main()
