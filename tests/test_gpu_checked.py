"""GPU: the bounds-checked build (compute-sanitizer is closed on this pool)
runs every kernel path -- sweeps, solves (static and dynamic schedules, both
arithmetics, split rows), batched solves, row_rhs, both interpolation modes,
the reduction hook and the failure path, the pairs arithmetic and the
finite-mu kernels (direct and moments mode) -- with zero index violations."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_checked_build_has_no_index_violations():
    lib = os.path.join(ROOT, "build", "libdse_checked.so")
    if not os.path.exists(lib):
        pytest.fail("build/libdse_checked.so missing: run __graft_entry__.build()")
    env = dict(os.environ, DSE_LIB=lib)
    res = subprocess.run([sys.executable, "scripts/checked_probe.py"], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "CHECK_FLAGS 0" in res.stdout, res.stdout
