"""Run the reference's own test suite against the B200 drop-in (test tooling).

SURVEY.md §4: the reference's pytest suite (``/root/reference/pkg/tests``,
188 tests) run unmodified with ``fftlasso`` resolved to this repository's
GPU package.  The reference's files are never committed here (the task
forbids copying reference sources); instead

    python tools/run_reference_suite.py fetch     # build container only

copies the test files and the reference's ``diagnostics.py`` into
``reference_suite/`` (git-ignored; it travels to the GPU box with the gpurun
snapshot), and

    python tools/run_reference_suite.py run [pytest args]   # on a B200

installs the alias and runs pytest on that directory in-process:

* ``fftlasso`` and ``fftlasso.{fourier, masking, newton_system, pcg, ipm,
  synthetic, errors, dataio, cli}`` are the GPU package's modules -- every
  numeric call the tests make goes through ``libfftlasso_b200.so``;
* ``fftlasso.diagnostics`` is the reference's diagnostics module loaded by
  path (its dense O(n^2)-O(n^3) probes are out of scope) with its
  own ``fftlasso.*`` imports resolved to the GPU package -- so ``densify``
  and ``dense_gram_matrix`` densify the GPU ``gram`` -- and the in-scope
  names (``soft_threshold``, ``ista_solve``, ``classify_support``,
  ``scaling_trajectory_check``, rows f2/f3 of SURVEY §8) replaced by the GPU
  implementations.

The product package never imports this file or ``reference_suite/``.
"""
from __future__ import annotations

import importlib.util
import os
import shutil
import sys
import types

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(REPO, "reference_suite")
REF_TESTS = "/root/reference/pkg/tests"
REF_DIAG = "/root/reference/pkg/src/fftlasso/diagnostics.py"

GPU_MODULES = ["fourier", "masking", "newton_system", "pcg", "ipm", "synthetic", "errors", "dataio", "cli"]
GPU_DIAGNOSTICS = ["soft_threshold", "ista_solve", "classify_support", "SupportClassification",
                   "scaling_trajectory_check", "ScalingReport", "ISTA_DIM_GUARD", "ISTA_ITER_CAP"]


def fetch() -> None:
    if not os.path.isdir(REF_TESTS):
        raise SystemExit(f"{REF_TESTS} not found (the reference exists only in the build container)")
    os.makedirs(SUITE, exist_ok=True)
    for name in sorted(os.listdir(REF_TESTS)):
        if name.endswith(".py"):
            shutil.copy(os.path.join(REF_TESTS, name), os.path.join(SUITE, name))
    shutil.copy(REF_DIAG, os.path.join(SUITE, "_ref_diagnostics.py"))
    print(f"copied {len(os.listdir(SUITE))} files into {SUITE} (git-ignored)")


def install_alias(diag_path: str | None = None) -> None:
    sys.path.insert(0, REPO)
    import paper_2502_04217_b200 as gpu

    sys.modules["fftlasso"] = gpu
    for name in GPU_MODULES:
        mod = importlib.import_module(f"paper_2502_04217_b200.{name}")
        sys.modules[f"fftlasso.{name}"] = mod
        setattr(gpu, name, mod)
    spec = importlib.util.spec_from_file_location("fftlasso.diagnostics",
                                                  diag_path or os.path.join(SUITE, "_ref_diagnostics.py"))
    diag = importlib.util.module_from_spec(spec)
    sys.modules["fftlasso.diagnostics"] = diag
    spec.loader.exec_module(diag)
    gpu_diag = importlib.import_module("paper_2502_04217_b200.diagnostics")
    for name in GPU_DIAGNOSTICS:
        if hasattr(gpu_diag, name):
            setattr(diag, name, getattr(gpu_diag, name))
    gpu.diagnostics = diag
    assert isinstance(sys.modules["fftlasso"], types.ModuleType)


def run(args, suite: str = SUITE, diag_path: str | None = None) -> int:
    if not os.path.isdir(suite):
        raise SystemExit(f"{suite} missing: run `python tools/run_reference_suite.py fetch` in the build container")
    install_alias(diag_path)
    import pytest

    sys.path.insert(0, suite)  # the suite's `from conftest import ...`
    return pytest.main([suite, "-p", "no:cacheprovider", "-o", "addopts=", "--rootdir", suite] + list(args))


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "fetch":
        fetch()
    elif cmd == "collect-in-place":  # build container: collect /root/reference's suite without copying it
        sys.exit(run(["--collect-only", "-q"] + sys.argv[2:], suite=REF_TESTS, diag_path=REF_DIAG))
    else:
        sys.exit(run(sys.argv[2:]))
