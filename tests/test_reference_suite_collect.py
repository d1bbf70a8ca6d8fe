"""CPU: the reference's own test suite imports and collects against the drop-in.

``tools/run_reference_suite.py`` aliases ``fftlasso`` to this package and runs
the reference's unmodified suite on a B200 (187 of 188 pass,
``profiles/r02_reference_suite_final2.txt``).  Here, without a GPU, the same
alias must let pytest import every reference test module and collect all 188
tests in place (nothing copied) -- i.e. every name, signature default and
exception the suite imports exists in the drop-in.  Skipped where the
reference is absent (the GPU box).
"""
import os
import subprocess
import sys

import pytest

from conftest import REPO

REF_TESTS = "/root/reference/pkg/tests"


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference not present (GPU box)")
def test_reference_suite_collects_against_drop_in():
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "run_reference_suite.py"), "collect-in-place"], capture_output=True, text=True, cwd="/tmp", timeout=600)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "188 tests collected" in out.stdout, out.stdout[-2000:]
