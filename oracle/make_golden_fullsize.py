"""Record converged solve summaries at the BASELINE sizes -- TEST INFRASTRUCTURE.

The GPU parity suite (``tests/test_gpu_fullsize_parity.py``) compares the
drop-in ``solve`` with these records at C2 2048^2, C3 256^3 and C4 512^3.
A full solution vector is 32 MB / 128 MB / 1 GB there, so the record is a
compact summary of the reference's answer (``ipm.py:474-486`` return value
and ``ipm.py:143-158`` / ``:185-197`` records):

* lambda, status, IPM iterations, per-iteration records (wall time dropped),
  final objective / KKT / mu;
* the support (``diagnostics.py:129-142`` classes at threshold
  1e-6 * max|beta|): positive and negative index sets, beta on the support,
  ||beta||_2 and ||beta off the support||_2;
* the SHA-256 of the observed samples ``b``, so the test can prove that it
  rebuilt bitwise the same input on the GPU box (``workloads`` recipe +
  the oracle's ``observe``, which is bitwise equal to the reference's).

Engines:

``--engine reference`` (default; build container only) imports the real
    reference read-only from ``/root/reference/pkg/src``.  Used for C2 and
    C3 (80 s and ~9 min on 8 cores).
``--engine oracle`` runs ``oracle/fftlasso_oracle.py`` (bitwise-pinned to the
    reference by ``tests/test_oracle_golden.py``).  Used for C4: the reference
    needs ~660 B/voxel (89 GB at 512^3), more than the build container's
    62 GB, so C4 is recorded once on the GPU box's host (``gpurun``).

    python oracle/make_golden_fullsize.py c2 c3
    python oracle/make_golden_fullsize.py --engine oracle c4
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, REPO)

from oracle import fftlasso_oracle as orc  # noqa: E402
from paper_2502_04217_b200 import workloads  # noqa: E402

CASES = {
    # name: (recipe, description) -- SURVEY.md Appendix A
    "c2": (lambda: workloads.c2_2d(seed=0, n_side=2048), "C2 2D 2048^2 block-punched, default lambda"),
    "c3": (lambda: workloads.c3_bragg(256, seed=0), "C3 3D 256^3 Bragg-punched, default lambda"),
    "c4": (lambda: workloads.c4_const(512), "C4 3D 512^3 Bragg-punched, lambda = 0.5"),
}
FILES = {"c2": "solve_c2_2048.json", "c3": "solve_c3_256.json", "c4": "solve_c4_512.json"}


def b_digest(b: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(b, dtype="<f8").tobytes()).hexdigest()


def summarize(beta: np.ndarray, report: dict) -> dict:
    pos, neg, _, thr = orc.support(beta)
    sup = np.concatenate([pos, neg])
    off = np.ones(beta.size, bool)
    off[sup] = False
    return dict(
        report,
        support_threshold=thr,
        support_pos=pos.tolist(),
        support_neg=neg.tolist(),
        beta_on_support={"index": sup.tolist(), "value": beta[sup].tolist()},
        beta_norm=float(np.linalg.norm(beta)),
        beta_off_support_norm=float(np.linalg.norm(beta[off])),
    )


def run(name: str, engine: str) -> dict:
    recipe, desc = CASES[name]
    inst = recipe()
    dims = inst.dims
    t0 = time.perf_counter()
    if engine == "reference":
        sys.path.insert(0, "/root/reference/pkg/src")
        import fftlasso as ref  # the reference, read-only
        from fftlasso import ipm as ref_ipm

        g = ref.GridShape(dims)
        mask = ref.Mask.from_bool(inst.flags, g)
        b = ref.observe(inst.beta_true, mask) + inst.noise
        beta, rep = ref.solve(b, mask, ref_ipm.IpmConfig(lam=inst.lam, tol=1e-8))
        records = [r.to_dict() for r in rep.records]
        head = dict(lam=rep.lam, status=rep.status, iterations=rep.iterations,
                    final_objective=rep.final_objective, final_kkt=rep.final_kkt,
                    final_mu=rep.final_mu)
        engine_desc = f"reference fftlasso ({'/root/reference/pkg/src'})"
    else:
        om = orc.make_mask(dims, flags=inst.flags)
        b = orc.observe(inst.beta_true, om) + inst.noise
        beta, rep = orc.solve(b, om, orc.OConfig(lam=inst.lam, tol=1e-8))
        records = [dict(r) for r in rep.records]
        head = dict(lam=rep.lam, status=rep.status, iterations=rep.iterations,
                    final_objective=rep.final_objective, final_kkt=rep.final_kkt,
                    final_mu=rep.final_mu)
        engine_desc = "oracle/fftlasso_oracle.py (bitwise-pinned restatement)"
    seconds = time.perf_counter() - t0
    for r in records:
        r.pop("wall_time", None)
    out = summarize(np.asarray(beta), dict(
        case=name, description=desc, dims=list(dims), engine=engine_desc,
        b_sha256=b_digest(b), n_observed=int(b.size), **head,
        krylov=[int(r["krylov_iters"]) for r in records], records=records,
        cpu_seconds=round(seconds, 1), cpu_threads=orc._workers()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="+", choices=sorted(CASES))
    ap.add_argument("--engine", choices=("reference", "oracle"), default="reference")
    ap.add_argument("--out-dir", default=OUT)
    args = ap.parse_args()
    os.makedirs(args.out_dir, exist_ok=True)
    for name in args.cases:
        rec = run(name, args.engine)
        path = os.path.join(args.out_dir, FILES[name])
        with open(path, "w") as fh:
            json.dump(rec, fh, separators=(",", ":"), sort_keys=True)
        print(f"{name}: {rec['status']} {rec['iterations']} IPM, krylov {rec['krylov']}, "
              f"obj {rec['final_objective']!r}, support {len(rec['beta_on_support']['index'])}, "
              f"{rec['cpu_seconds']} s -> {os.path.relpath(path, REPO)}", flush=True)


if __name__ == "__main__":
    main()
