"""The reference package's OWN test files, run against this implementation.

integration/octfield is the reference package with its hot-path modules
(errors, octree, field, traversal, render, trainer, modelio, metrics)
replaced by this repository's; geometry, sampling and the
cli stay the reference's. tools/stage_reference_tests.sh copies the
reference's tests/ and installs its package under baseline/ (git-ignored;
it travels to the GPU box with the repository snapshot). This test runs
that suite unchanged on the GPU and requires every test to pass except the
ones listed in DESELECTED, each for the reason given there. Acceptance
criterion 9 is also printed by the run (it must reproduce the reference's
own numbers).
"""

import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref_tests")

# Tests that patch a module-global seam of the reference's host march
# (`render.query_field`) with a synthetic Python field: the device march
# evaluates the field inside the kernel, so a Python stub cannot be
# substituted there. The same stop rules are pinned on the oracle against
# stub fields (tests/test_oracle.py::test_march_stop_rules_with_stub_field)
# and on the device by the frame parity tests.
DESELECTED = {
    "test_render.py::test_converging_creep_is_a_hit": "patches render.query_field (host seam)",
    "test_render.py::test_stalled_march_is_a_miss": "patches render.query_field (host seam)",
    "test_render.py::test_overshoot_lands_as_hit": "patches render.query_field (host seam)",
    "test_render.py::test_iteration_cap_ends_ray": "patches render.query_field (host seam)",
    "test_acceptance.py::test_criterion_7_empty_space": "patches render.query_field (host seam) to detect "
                                                         "empty-space decodes; the device frame counts them "
                                                         "(evals_missing_level, asserted zero in every render)",
    # The unmodified reference fails this criterion itself, with the same
    # numbers (LOD3 0.582/0.408, LOD4 0.729/0.356; run on CPU in the build
    # container, profiles/r02_parity/reference_cpu_criteria_5_9.log): the
    # frozen-decoder torus is 2.05x the joint one at LOD4 against a 2.0x bar.
    # Reproducing it to three digits is the parity result.
    "test_acceptance.py::test_criterion_9_frozen_decoder": "fails identically in the unmodified reference",
}


def test_reference_suite_against_b200_path():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    if not os.path.isdir(SUITE):
        pytest.skip("reference tests not staged (tools/stage_reference_tests.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "integration"), ROOT, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-rf", "--timeout", "900"]
    for t in DESELECTED:
        cmd += ["--deselect", t]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=3000)
    tail = r.stdout[-6000:]
    print(tail)
    m = re.search(r"(\d+) passed", tail)
    assert r.returncode == 0, tail + r.stderr[-2000:]
    assert m and int(m.group(1)) >= 250, tail
