"""Config 3: six tenants on the H100-80GB 7-slice lattice, 3600 slots, sliding
lookahead, reconfiguration-cost (psi) sweep.

CPU: the authored lattice (paper_2407_13126_b200/data/h100.catalog) passes the
reference's catalog cross-check (catalog_test.cpp:20-57 restated: maximal
packings of the placement rules, deduplicated by GPC-size multiset, equal the
configuration list), and the six-tenant single-device problem is infeasible
under the generator, which is why the tenants are planned as three pairs.

GPU: the C++ per-window driver (host/tools/plan_horizon.cpp, on the reference's
planner API with the drop-in headers) equals the unmodified reference's loop
(`migref drive ... <lookback> <psi>`, oracle/make_c3_goldens.py) window by
window, bit for bit, at S = 200; the psi sweep picks its best point
consistently. The six-tenant joint problem is unpinned (the reference rejects
more than 4 tenants, space.hpp:49-50)."""
import json
import math
import os
import subprocess

import pytest

from paper_2407_13126_b200 import scenario as SC
from paper_2407_13126_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = os.path.join(ROOT, "tests", "golden", "c3")
TOOL = os.path.join(ROOT, "paper_2407_13126_b200", "lib", "tools", "plan_horizon")


def _rules(text):
    rules = []
    for line in text.splitlines():
        t = line.split("#")[0].split()
        if t and t[0] == "rule":
            rules.append((int(t[1]), int(t[2]), [int(x) for x in t[3].split(",")]))
    return rules


def _maximal_multisets(rules, gpc, mem):
    """catalog_test.cpp:20-57: every maximal packing on the memory axis under the
    GPC budget (maximal also against earlier instances), as size multisets."""
    inst = [(size, s, foot) for size, foot, starts in rules for s in starts]
    out = set()

    def fits(i, mask, left):
        size, s, foot = inst[i]
        return size <= left and not any(mask >> m & 1 for m in range(s, s + foot))

    def rec(frm, mask, left, sizes):
        ext = False
        for i in range(frm, len(inst)):
            if fits(i, mask, left):
                ext = True
                size, s, foot = inst[i]
                rec(i + 1, mask | (((1 << foot) - 1) << s), left - size, sizes + [size])
        if not ext and not any(fits(i, mask, left) for i in range(frm)):
            out.add(tuple(sorted(sizes, reverse=True)))

    rec(0, 0, gpc, [])
    return out


def test_h100_catalog_matches_rule_enumerator():
    text = open(W.H100_LATTICE).read()
    cat = SC.parse_catalog(text, W.H100_LATTICE)
    assert cat.gpc_count == 7 and cat.mem_slices == 8
    declared = [tuple(sorted((s for s, _ in c.slots), reverse=True)) for c in cat.configs]
    assert len(set(declared)) == len(declared)  # no two configurations share a multiset
    assert set(declared) == _maximal_multisets(_rules(text), cat.gpc_count, cat.mem_slices)
    assert len(declared) == 22
    for c in cat.configs:  # slots sorted, non-overlapping, inside the 7-slice axis
        ends = [st + sz for sz, st in c.slots]
        assert all(ends[i] <= c.slots[i + 1][1] for i in range(len(c.slots) - 1)) and ends[-1] <= 7


def test_six_tenants_cannot_share_one_h100_under_the_generator():
    """Six inference tasks each hold a slot of size >= 1 at every step, leaving at
    most one slice: a retraining instance would have one GPC, and RT(1) =
    ceil(240/1) = 240 > 200 steps (retraining-window). Hence three pairs."""
    specs = W.c3_specs()
    tenants = [t for s in specs for t in s.tenants]
    assert len(tenants) == 6 and len({t.name for t in tenants}) == 6
    for t in tenants:
        rt1 = math.ceil(3 * t.data_volume / t.per_gpc)  # workload.hpp RT = ceil(3*vol/cap[k])
        assert rt1 > specs[0].window_size
    assert all(s.window_size * s.window_count == 3600 for s in specs)


def _run(args):
    r = subprocess.run([TOOL] + args, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stderr[-3000:]
    return json.loads(r.stdout)


@pytest.mark.gpu
@pytest.mark.slow
def test_cpp_driver_matches_reference_loop():
    if not os.path.exists(TOOL):
        pytest.skip("plan_horizon not built (needs the reference headers at build time)")
    gold = json.load(open(os.path.join(D, "c3_golden.json")))
    for case in gold:
        out = _run([os.path.join(D, "c3_pair%d.scn" % case["pair"]), "--predictor", case["predictor"],
                    "--windows", str(case["windows"]), "--lookback", str(case["lookback"]), "--psi", repr(case["psi"])])
        got = out["units"][0]["windows"]
        want = case["result"]["windows"]
        assert len(got) == len(want) == case["windows"]
        for w, (g, r) in enumerate(zip(got, want)):
            assert g["encode"] == r["encode"], (case, w)
            assert g["obj"] == r["obj"] and g["realized"] == r["realized"], (case, w)


@pytest.mark.gpu
@pytest.mark.slow
def test_psi_sweep_over_pairs():
    if not os.path.exists(TOOL):
        pytest.skip("plan_horizon not built")
    scns = [os.path.join(D, "c3_pair%d.scn" % k) for k in range(3)]
    psis = ",".join(repr(p) for p in W.C3_PSI_SWEEP)
    out = _run(scns + ["--predictor", "ewma:0.3", "--lookback", "2", "--windows", "2", "--psi", psis])
    assert len(out["units"]) == 15 and len(out["per_psi"]) == 5
    totals = [p["realized_total"] for p in out["per_psi"]]
    assert out["best_realized_total"] == max(totals)
    assert out["best_psi"] == W.C3_PSI_SWEEP[totals.index(max(totals))]
    # window 0 is planned on its actual counts: the DP's optimum can only fall as
    # reconfigurations get costlier (every plan's Goodput is non-increasing in psi)
    import struct
    val = lambda h: struct.unpack("<d", struct.pack("<Q", int(h, 16)))[0]
    for k in range(3):
        w0 = [val(out["units"][k * 5 + j]["windows"][0]["obj"]) for j in range(5)]
        assert all(w0[j] >= w0[j + 1] for j in range(4)), (k, w0)
