"""Runs one golden corpus case through the GPU engines with per-step dumps."""
import os, sys, json, subprocess
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import golden_util, tempfile
from paper_2407_13126_b200 import planner, scenario as SC
cases = golden_util.materialize(tempfile.mkdtemp())
want = sys.argv[1] if len(sys.argv) > 1 else None
for stem, path, g in cases["random"]:
    if want and stem != want:
        continue
    sc = SC.load_scenario(path)
    p = SC.Problem(sc, 0)
    with planner.Planner(0) as pl:
        opt, cfg, lab, obj, st = pl.solve_window(p)
    enc = planner.encode(cfg, lab, golden_util.nslots(sc))
    ok = enc == g["dp"]["encode"]
    print(stem, "OK" if ok else "MISMATCH", obj, g["dp"]["objective"], list(opt), flush=True)
    if not want and not ok:
        print("first mismatch:", stem)
        break
