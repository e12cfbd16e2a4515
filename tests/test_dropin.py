"""The reference's OWN Catch2 suites (plus our extras_test of the widened C++ API
against the reference functions), compiled unchanged against the B200
drop-in header (paper_2407_13126_b200/host/migsim/solvers.hpp) and run on the
GPU: solve_dp / solve_bruteforce / precheck_scenario go through the C ABI to
the sm_100a kernels. Binaries are built by tests/dropin/Makefile (from
__graft_entry__.build(), where /root/reference exists) into the git-ignored
paper_2407_13126_b200/lib/dropin/ and travel to the GPU box with the snapshot.
"""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2407_13126_b200", "lib", "dropin")
SUITES = ["solver_test", "eval_test", "baseline_test", "simulator_test", "preinit_test", "extras_test"]


@pytest.fixture(scope="module")
def data_dir(tmp_path_factory):
    d = tmp_path_factory.mktemp("migsim_data")
    # the reference's default lattice (data/a100.catalog), same configurations in file order
    shutil.copy(os.path.join(ROOT, "tests", "golden", "lattice_a100.catalog"), d / "a100.catalog")
    return str(d)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_b200(suite, data_dir):
    exe = os.path.join(BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("drop-in suite binaries not built (needs /root/reference at build time)")
    env = dict(os.environ, MIGSIM_DATA_DIR=data_dir)
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=900)
    print(r.stdout[-4000:])
    print(r.stderr[-4000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    last = [l for l in r.stdout.splitlines() if l.startswith("summary:")][-1]
    assert " 0 failed" in last, last
