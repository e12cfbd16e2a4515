"""Loads the committed golden corpus (tests/golden/, produced from the unmodified
reference by oracle/make_goldens.py) into scenario files on disk."""
import glob
import json
import os
import struct

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def bits(x):
    return "%016x" % struct.unpack("<Q", struct.pack("<d", float(x)))[0]


def materialize(tmp):
    """Writes every random-corpus scenario to tmp; returns a dict of case lists."""
    cases = {"random": [], "c1": [], "kat": [], "multi": [], "multi_c2": []}
    for path in sorted(glob.glob(os.path.join(GOLD, "random_*.json"))):
        bundle = json.load(open(path))
        for stem, files in sorted(bundle.items()):
            for ext in ("scn", "catalog", "csv"):
                with open(os.path.join(tmp, stem + "." + ext), "w") as f:
                    f.write(files[ext])
            cases["random"].append((stem, os.path.join(tmp, stem + ".scn"), files["golden"]))
    for path in sorted(glob.glob(os.path.join(GOLD, "multi_m*.json"))):
        bundle = json.load(open(path))
        for stem, files in sorted(bundle.items()):
            for ext in ("scn", "catalog", "csv"):
                with open(os.path.join(tmp, stem + "." + ext), "w") as f:
                    f.write(files[ext])
            cases["multi"].append((stem, os.path.join(tmp, stem + ".scn"), files["golden"]))
    mpath = os.path.join(GOLD, "multi", "multi_golden.json")
    if os.path.exists(mpath):
        for stem, g in sorted(json.load(open(mpath)).items()):
            cases["multi_c2"].append((stem, os.path.join(GOLD, "multi", stem + ".scn"), g))
    c1 = json.load(open(os.path.join(GOLD, "c1", "c1_golden.json")))
    for stem, g in sorted(c1.items()):
        cases["c1"].append((stem, os.path.join(GOLD, "c1", stem + ".scn"), g))
    kat = json.load(open(os.path.join(GOLD, "kat", "kat_golden.json")))
    for stem, g in sorted(kat.items()):
        cases["kat"].append((stem, os.path.join(GOLD, "kat", stem + ".scn"), g))
    return cases


def nslots(sc):
    return [len(c.slots) for c in sc.catalog.configs]
