"""The reference's own tests, run against the B200 backend (drop-in proof).

Runs ``pytest`` on the unmodified reference test modules (baseline/_ref/tsgemm_tests, installed by
tools/install_reference.sh; or /root/reference/pkg/tests in the build container) with the
ref_b200_plugin, which swaps ``tsgemm.kernels.run_native`` for ``paper_2002_03258_b200.run_native``
on the result-level tests (reference test_kernels.py:18-40,102-107,150-155,182-195,233-253,265-269
and test_acceptance.py:52-86). Every selected test must pass, except acceptance criterion 1,
which must end in the plugin's spot-check skip (reached only after its 300-config loop passed).
"""

import os
import subprocess
import sys

import pytest

from conftest import ROOT, reference_path, reference_tests_dir

pytestmark = pytest.mark.gpu


def test_reference_result_tests_pass_on_b200():
    ref, tests = reference_path(), reference_tests_dir()
    if ref is None or tests is None:
        pytest.skip("reference not installed (tools/install_reference.sh)")
    from ref_b200_plugin import SELECTED, SPOT_CHECK_SKIP
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, ref, env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-p", "ref_b200_plugin", "-p", "no:cacheprovider", "-q", "-rs",
           "--rootdir", tests, os.path.join(tests, "test_kernels.py"), os.path.join(tests, "test_acceptance.py")]
    out = subprocess.run(cmd, cwd=tests, env=env, capture_output=True, text=True, timeout=1200)
    text = out.stdout + out.stderr
    assert out.returncode == 0, text[-4000:]
    n_pass = len(SELECTED) - 1
    assert f"{n_pass} passed" in text, text[-3000:]
    assert "1 skipped" in text and SPOT_CHECK_SKIP in text, text[-3000:]
