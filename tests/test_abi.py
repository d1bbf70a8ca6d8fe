"""CPU: the C-ABI library loads and exports exactly what include/*.h declares.

No compute calls here (no GPU in the CPU suite); the ctypes table in
paper_2502_04217_b200/_lib.py must cover every declared entry point.
"""

import ctypes
import os
import re

import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "fftlasso_b200.h")
LIB = os.path.join(REPO, "paper_2502_04217_b200", "libfftlasso_b200.so")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^FL_API\s+[\w\s\*]+?\b(fl_\w+)\(", src, flags=re.M)))


def test_header_declares_entry_points():
    names = declared()
    assert len(names) >= 30
    for must in ("fl_plan_create", "fl_synthesize", "fl_analyze", "fl_gram", "fl_kkt_apply",
                 "fl_precond_apply", "fl_pcg_kkt", "fl_ipm_assess", "fl_ipm_update"):
        assert must in names


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built (run __graft_entry__.build())")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_ctypes_table_matches_header():
    from paper_2502_04217_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared()
    lib = _lib.load_library()
    assert lib.fl_version() == 1


@pytest.mark.skipif(not os.path.exists(LIB), reason="library not built")
def test_library_targets_sm100a():
    """The fatbinary carries sm_100a SASS (cuobjdump lists the ELF arch)."""
    import shutil
    import subprocess

    tool = shutil.which("cuobjdump")
    if tool is None:
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
