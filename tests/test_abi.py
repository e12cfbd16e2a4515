"""CPU: the C-ABI library loads and exports every entry point the header
declares, status codes map onto the reference's error-code strings, and the
C++ drop-in header compiles against the reference's own headers."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2407_13126_b200 import capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "migsim_b200.h")
REF = "/root/reference/proj"


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"MGS_API\s+[\w\s\*]+?\b(mgs_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(capi.LIB_PATH)  # no GPU needed to load (cudart is static)
    names = declared()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(capi.EXPORTED_SYMBOLS) == names


def test_status_codes_are_the_reference_strings():
    lib = capi.load()
    for st, code in capi.STATUS_CODES.items():
        assert lib.mgs_status_code(st).decode() == code
    # every code string the reference's planner path can raise
    for code in ("input.scenario", "input.catalog", "input.forecast", "infeasible.deployment-floor",
                 "infeasible.retraining-window", "infeasible.no-coexistence-configuration", "infeasible.joint",
                 "planner.state-budget", "planner.bruteforce-cap", "plan.infeasible"):
        assert code in capi.STATUS_CODES.values()
    assert b"sm_100a" in lib.mgs_version()


def test_open_without_gpu_fails_loudly():
    """No CPU fallback: on a box without a GPU, opening a context is an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = capi.load()
    h = C.c_void_p()
    assert lib.mgs_open(0, C.byref(h)) != 0


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference headers not mounted")
def test_dropin_header_compiles_against_reference(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text('#include "migsim/solvers.hpp"\n#include "migsim/baselines.hpp"\n#include "migsim/simulator.hpp"\n'
                   '#include "migsim_b200/extras.hpp"\n'
                   "static_assert(sizeof(migsim::b200::PlanSteps) > 0);\n"
                   "int main() { migsim::SolveOptions o; return o.workers - 1; }\n")
    host = os.path.join(ROOT, "paper_2407_13126_b200", "host")
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(host, "dropin"), "-I", host,
                        "-I", os.path.join(ROOT, "include"), "-I", REF + "/include", str(src)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
