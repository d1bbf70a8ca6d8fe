"""Record golden vectors from the REAL reference package -- test infrastructure.

Run in the build container (the only place ``/root/reference`` exists):

    python oracle/make_golden.py

It imports ``fftlasso`` read-only from ``/root/reference/pkg/src``, evaluates
the hot-path functions on seeded inputs and writes ``tests/golden/*.npz``.
It also evaluates ``oracle/fftlasso_oracle.py`` on the same inputs and prints
the worst deviation, so a drifting restatement is caught at generation time;
``tests/test_oracle_golden.py`` repeats that check on every CPU test run.
The GPU parity tests compare the CUDA path against these fixtures and the
oracle.  Nothing here runs on the GPU box.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(REPO, "tests", "golden")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import fftlasso as ref  # noqa: E402  (the reference, read-only)
from fftlasso import ipm as ref_ipm  # noqa: E402
from fftlasso import newton_system as ref_ns  # noqa: E402
from fftlasso.pcg import PcgConfig, pcg_solve  # noqa: E402

from oracle import fftlasso_oracle as orc  # noqa: E402
from paper_2502_04217_b200 import workloads  # noqa: E402

WORST = {}


def note(tag, a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(1.0, float(np.max(np.abs(a))) if a.size else 1.0)
    err = float(np.max(np.abs(a - b))) / scale if a.size else 0.0
    WORST[tag] = max(WORST.get(tag, 0.0), err)


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {os.path.relpath(path, REPO)} ({os.path.getsize(path) // 1024} KiB)")


TRANSFORM_DIMS = [(2,), (4,), (6,), (10,), (16,), (64,), (96,), (4096,), (16384,),
                  (8, 6), (8, 8), (6, 10), (64, 64), (4, 2, 6), (6, 4, 10),
                  (16, 16, 16), (8, 12, 6), (32, 32, 32)]


def transforms():
    rng = np.random.default_rng(7001)
    arrays = {}
    for dims in TRANSFORM_DIMS:
        g = ref.GridShape(dims)
        beta = rng.standard_normal(g.n)
        x = rng.standard_normal(g.n)
        key = "x".join(map(str, dims))
        arrays[f"{key}__beta"] = beta
        arrays[f"{key}__synth"] = ref.synthesize(beta, g)
        arrays[f"{key}__x"] = x
        arrays[f"{key}__analyze"] = ref.analyze(x, g)
        note("synthesize", arrays[f"{key}__synth"], orc.synthesize(beta, dims))
        note("analyze", arrays[f"{key}__analyze"], orc.analyze(x, dims))
    arrays["dims_json"] = np.array(json.dumps([list(d) for d in TRANSFORM_DIMS]))
    save("transforms", **arrays)


MASK_CASES = [((64,), 9), ((4096,), 410), ((16, 24), 60), ((8, 12, 16), 200),
              ((32, 32, 32), 4900)]


def masking():
    rng = np.random.default_rng(7002)
    arrays = {}
    for dims, k in MASK_CASES:
        g = ref.GridShape(dims)
        miss = np.sort(rng.choice(g.n, k, replace=False))
        mask = ref.Mask(miss, g)
        beta = rng.standard_normal(g.n)
        vals = rng.standard_normal(mask.n_observed)
        key = "x".join(map(str, dims))
        arrays[f"{key}__missing"] = miss
        arrays[f"{key}__beta"] = beta
        arrays[f"{key}__vals"] = vals
        arrays[f"{key}__observe"] = ref.observe(beta, mask)
        arrays[f"{key}__embed"] = ref.embed(vals, mask)
        arrays[f"{key}__adjoint"] = ref.observe_adjoint(vals, mask)
        arrays[f"{key}__gram"] = ref.gram(beta, mask)
        om = orc.make_mask(dims, missing=miss)
        note("observe", arrays[f"{key}__observe"], orc.observe(beta, om))
        note("embed", arrays[f"{key}__embed"], orc.embed(vals, om))
        note("adjoint", arrays[f"{key}__adjoint"], orc.observe_adjoint(vals, om))
        note("gram", arrays[f"{key}__gram"], orc.gram(beta, om))
    arrays["cases_json"] = np.array(json.dumps([[list(d), k] for d, k in MASK_CASES]))
    save("masking", **arrays)


def interior_state(rng, n, mu=0.05):
    """Same distribution as the reference's random_interior_state fixture."""
    return dict(beta=rng.standard_normal(n) * 0.4, z=rng.random(n) + 0.8,
                s1=rng.random(n) + 0.4, s2=rng.random(n) + 0.4,
                y1=rng.random(n) + 0.3, y2=rng.random(n) + 0.3,
                nu1=rng.random(n) + 0.3, nu2=rng.random(n) + 0.3, mu=mu)


NEWTON_CASES = [((64,), 8), ((4, 6, 8), 30), ((32, 32), 150)]


def newton():
    rng = np.random.default_rng(7003)
    arrays = {}
    for dims, k in NEWTON_CASES:
        g = ref.GridShape(dims)
        n = g.n
        miss = np.sort(rng.choice(n, k, replace=False))
        mask = ref.Mask(miss, g)
        st = interior_state(rng, n)
        b = rng.standard_normal(mask.n_observed)
        lam = 0.4
        rst = ref_ipm.IpmState(**st)
        d = ref_ns.barrier_diagonals(st["s1"], st["s2"], st["nu1"], st["nu2"])
        rhs = ref_ns.newton_rhs(rst, b, mask, lam)
        db = rng.standard_normal(n)
        dz = rng.standard_normal(n)
        top, bot = ref_ns.apply_kkt(db, dz, d, mask)
        ptop, pbot = ref_ns.apply_precond_inverse(db, dz, d)
        rec = ref_ns.recover_eliminated(db, dz, rhs, d)
        key = "x".join(map(str, dims))
        for f in ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2"):
            arrays[f"{key}__st_{f}"] = st[f]
        arrays[f"{key}__mu"] = np.array(st["mu"])
        arrays[f"{key}__lam"] = np.array(lam)
        arrays[f"{key}__missing"] = miss
        arrays[f"{key}__b"] = b
        arrays[f"{key}__db"] = db
        arrays[f"{key}__dz"] = dz
        for f in ("sigma1", "sigma2", "lambda1", "lambda2", "dvec", "bvec"):
            arrays[f"{key}__diag_{f}"] = getattr(d, f)
        for f in ("r1", "r2", "r3", "r4", "r5", "r6", "r_beta", "r_c"):
            arrays[f"{key}__rhs_{f}"] = getattr(rhs, f)
        arrays[f"{key}__kkt_top"] = top
        arrays[f"{key}__kkt_bottom"] = bot
        arrays[f"{key}__pinv_top"] = ptop
        arrays[f"{key}__pinv_bottom"] = pbot
        for f in ("d_s1", "d_s2", "d_y1", "d_y2"):
            arrays[f"{key}__rec_{f}"] = getattr(rec, f)
        # condensed PCG solve at this state (the inner hot loop)
        res = pcg_solve(lambda v: np.concatenate(ref_ns.apply_kkt(v[:n], v[n:], d, mask)),
                        lambda v: np.concatenate(ref_ns.apply_precond_inverse(v[:n], v[n:], d)),
                        np.concatenate([rhs.r_beta, rhs.r_c]),
                        PcgConfig(abs_tol=1e-12, record_history=True))
        arrays[f"{key}__pcg_x"] = res.solution
        arrays[f"{key}__pcg_iters"] = np.array(res.iterations)
        arrays[f"{key}__pcg_hist"] = np.array(res.residual_history)
        # oracle cross-check
        om = orc.make_mask(dims, missing=miss)
        ost = orc.OState(**{f: st[f].copy() for f in st if f != "mu"}, mu=st["mu"])
        od = orc.diagonals(st["s1"], st["s2"], st["nu1"], st["nu2"])
        orhs = orc.newton_rhs(ost, b, om, lam)
        for i, f in enumerate(("sigma1", "sigma2", "lambda1", "lambda2", "dvec", "bvec")):
            note("diag(bitwise)", getattr(d, f), od[i])
        for f in ("r1", "r_beta", "r_c"):
            note("rhs", getattr(rhs, f), orhs[f])
        otop, obot = orc.kkt_apply(db, dz, od, om)
        note("kkt", top, otop)
        note("kkt", bot, obot)
        optop, opbot = orc.precond_apply(db, dz, od)
        note("pinv(bitwise)", ptop, optop)
        note("pinv(bitwise)", pbot, opbot)
        ores = orc.pcg(lambda v: np.concatenate(orc.kkt_apply(v[:n], v[n:], od, om)),
                       lambda v: np.concatenate(orc.precond_apply(v[:n], v[n:], od)),
                       np.concatenate([orhs["r_beta"], orhs["r_c"]]), history=True)
        note("pcg", res.solution, ores.solution)
        assert ores.iterations == res.iterations, (ores.iterations, res.iterations)
    arrays["cases_json"] = np.array(json.dumps([[list(d), k] for d, k in NEWTON_CASES]))
    save("newton", **arrays)


def _record_solve(name, dims, flags, b, lam, beta_true=None, max_iters=200):
    g = ref.GridShape(dims)
    mask = ref.Mask.from_bool(flags, g)
    cfg = ref_ipm.IpmConfig(lam=lam, tol=1e-8, max_iters=max_iters)
    beta, rep = ref.solve(b, mask, cfg)
    om = orc.make_mask(dims, flags=flags)
    obeta, orep = orc.solve(b, om, orc.OConfig(lam=lam, tol=1e-8, max_iters=max_iters))
    note("solve beta", beta, obeta)
    assert orep.krylov_counts == rep.krylov_counts, (name, orep.krylov_counts, rep.krylov_counts)
    recs = [r.to_dict() for r in rep.records]
    arrays = dict(dims=np.array(dims), missing=mask.missing, b=b, beta=beta,
                  lam=np.array(rep.lam), status=np.array(rep.status),
                  iterations=np.array(rep.iterations),
                  final_objective=np.array(rep.final_objective),
                  final_kkt=np.array(rep.final_kkt), final_mu=np.array(rep.final_mu),
                  records_json=np.array(json.dumps(recs)))
    if beta_true is not None:
        arrays["beta_true"] = beta_true
    save("solve_" + name, **arrays)
    print(f"    {name}: {rep.status} {rep.iterations} IPM, krylov {rep.krylov_counts}, "
          f"obj {rep.final_objective:.12e}, lam {rep.lam:.6g}")


def _observed(inst):
    g = ref.GridShape(inst.dims)
    mask = ref.Mask.from_bool(inst.flags, g)
    return ref.observe(inst.beta_true, mask) + inst.noise


def solves():
    # C1 at its full size (1D 4096, lambda 0.3) -- SURVEY Appendix A
    inst = workloads.c1_1d(seed=0)
    _record_solve("c1_4096", inst.dims, inst.flags, _observed(inst), inst.lam, inst.beta_true)
    # C2 recipe scaled to 256^2 (same block sizes/density law)
    inst = workloads.c2_2d(seed=0, n_side=256)
    _record_solve("c2_256", inst.dims, inst.flags, _observed(inst), inst.lam, inst.beta_true)
    # C3 recipe at 32^3 and C4/C5 recipe at 32^3
    inst = workloads.c3_bragg(32, seed=0)
    _record_solve("c3_32", inst.dims, inst.flags, _observed(inst), inst.lam, inst.beta_true)
    inst = workloads.c4_const(32)
    _record_solve("c4_32", inst.dims, inst.flags, _observed(inst), inst.lam, inst.beta_true)
    # reference's own generator (Appendix B rows 8^3 / 16^3), default lambda
    for side in (8, 16):
        noisy, flags, _ = workloads.harmonics((side,) * 3, noise_seed=42, missing_seed=43)
        _record_solve(f"harm_{side}", (side,) * 3, flags, noisy[~flags], None)
    # empty mask (pure denoising) and a max_iters best-iterate case
    rng = np.random.default_rng(7004)
    b = rng.standard_normal(128)
    _record_solve("empty_128", (128,), np.zeros(128, bool), b, None)
    flags = np.zeros(64, bool)
    flags[rng.choice(64, 9, replace=False)] = True
    b = rng.standard_normal(64 - 9)
    _record_solve("maxit_64", (64,), flags, b, 0.4, max_iters=3)


def _sparse_1d(rng, n, n_missing, n_active, amplitude=(1.0, 2.0), noise=0.02):
    """Masked sparse 1D instance (the reference tests' conftest recipe)."""
    g = ref.GridShape((n,))
    mask = ref.Mask(np.sort(rng.choice(n, size=n_missing, replace=False)), g)
    beta = np.zeros(n)
    idx = rng.choice(n, size=n_active, replace=False)
    lo, hi = amplitude
    beta[idx] = (lo + (hi - lo) * rng.random(n_active)) * np.sign(rng.standard_normal(n_active))
    return ref.observe(beta, mask) + noise * rng.standard_normal(mask.n_observed), mask


def ista():
    """Reference diagnostics: soft_threshold and the ISTA oracle (diagnostics.py:325-360)."""
    from fftlasso import diagnostics as ref_diag

    x = np.concatenate([[0.0, -0.0, 0.3, -0.3, 0.30000000000000004, 1e300, -1e-300, np.inf, -np.inf],
                        np.random.default_rng(11).standard_normal(64)])
    arrays = dict(soft_x=x, soft_t=np.array(0.3), soft_out=ref_diag.soft_threshold(x, 0.3))
    cases = []
    rng = np.random.default_rng(3000)
    b, mask = _sparse_1d(rng, 64, 10, 3, amplitude=(1.0, 2.5), noise=0.05)
    cases.append(("c64", b, mask, 0.3))
    rng = np.random.default_rng(3001)
    b, mask = _sparse_1d(rng, 128, 19, 5, amplitude=(1.0, 2.5), noise=0.05)
    cases.append(("c128", b, mask, 0.3))
    rng = np.random.default_rng(3002)
    g = ref.GridShape((16, 16))
    flags = rng.random(256) < 0.12
    m2 = ref.Mask.from_bool(flags, g)
    bt = np.zeros(256)
    bt[rng.choice(256, 6, replace=False)] = rng.uniform(1.0, 2.0, 6)
    cases.append(("c16x16", ref.observe(bt, m2) + 0.03 * rng.standard_normal(m2.n_observed), m2, 0.25))
    noisy, flags, _ = workloads.harmonics((8, 8, 8), noise_seed=42, missing_seed=43)
    m3 = ref.Mask.from_bool(flags, ref.GridShape((8, 8, 8)))
    b3 = noisy[~flags]
    cases.append(("harm8", b3, m3, ref_ipm.default_penalty(b3, m3)))
    names = []
    for name, b, mask, lam in cases:
        beta, iters = ref_diag.ista_solve(b, mask, lam, tol=1e-10)
        om = orc.make_mask(mask.shape.dims, missing=mask.missing)
        obeta, oiters = orc.ista(b, om, lam, tol=1e-10)
        note("ista beta", beta, obeta)
        assert oiters == iters, (name, oiters, iters)
        arrays.update({f"{name}_dims": np.array(mask.shape.dims), f"{name}_missing": mask.missing,
                       f"{name}_b": b, f"{name}_lam": np.array(lam), f"{name}_beta": beta,
                       f"{name}_iters": np.array(iters),
                       f"{name}_objective": np.array(ref_ipm.lasso_objective(beta, b, mask, lam))})
        names.append(name)
        print(f"    {name}: {iters} ISTA iterations, lam {lam:.4g}")
    arrays["cases_json"] = np.array(json.dumps(names))
    save("ista", **arrays)


def spectrum():
    """Reference dense probes (diagnostics.py:94-224) on observer snapshots of a
    reference solve -> tests/golden/spectrum.npz (pins the oracle's restatement)."""
    from fftlasso import diagnostics as ref_diag

    rng = np.random.default_rng(7005)
    n = 24
    miss = np.sort(rng.choice(n, 3, replace=False))
    g = ref.GridShape((n,))
    mask = ref.Mask(miss, g)
    bt = np.zeros(n)
    bt[[2, 7]] = [1.5, -1.1]
    b = ref.observe(bt, mask) + 0.02 * rng.standard_normal(mask.n_observed)
    states = []
    fields = ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")
    ref.solve(b, mask, ref_ipm.IpmConfig(lam=0.35, tol=1e-8),
              observer=lambda s, r: states.append(ref_ipm.IpmState(mu=s.mu, **{f: getattr(s, f).copy() for f in fields})))
    arrays = dict(missing=miss)
    om = orc.make_mask((n,), missing=miss)
    for tag, st in (("first", states[0]), ("last", states[-1])):
        rep = ref_diag.preconditioned_spectrum(st, mask)
        k, p = ref_diag.dense_condensed_matrices(st, mask)
        for f in fields:
            arrays[f"{tag}__{f}"] = getattr(st, f)
        arrays[f"{tag}__eigs"] = rep.eigenvalues
        arrays[f"{tag}__K"] = k
        arrays[f"{tag}__P"] = p
        arrays[f"{tag}__scalars"] = np.array([rep.unit_cluster_size, rep.predicted_cluster_size, rep.kappa_observed,
                                              rep.kappa_predicted, rep.kappa_unpreconditioned, rep.n_active,
                                              rep.strict_complementarity, rep.duality_measure])
        note("spectrum", rep.eigenvalues, orc.preconditioned_spectrum(st, om)["eigenvalues"])
    save("spectrum", **arrays)


def _strip_wall(rows):
    return [{k: v for k, v in r.items() if k != "wall_time"} for r in rows]


def cli():
    """The reference CLI end to end (cli.py:37-144): files, reports, exit codes."""
    import tempfile

    from fftlasso import cli as ref_cli

    with tempfile.TemporaryDirectory() as tmp:
        sig, msk, byt = (os.path.join(tmp, f) for f in ("signal.f64", "mask.idx", "mask.byte"))
        beta, imp, rep = (os.path.join(tmp, f) for f in ("beta.f64", "imputed.f64", "report.jsonl"))
        assert ref_cli.main(["generate", "--dims", "8,8,8", "--noise-seed", "3", "--missing-seed", "4",
                             "--signal", sig, "--mask", msk]) == 0
        assert ref_cli.main(["generate", "--dims", "8,8,8", "--noise-seed", "3", "--missing-seed", "4",
                             "--signal", sig, "--mask", byt, "--mask-format", "bytemask"]) == 0
        code = ref_cli.main(["solve", "--input", sig, "--mask", msk, "--output", beta,
                             "--report", rep, "--impute", imp])
        with open(rep) as fh:
            records = [json.loads(line) for line in fh if line.strip()]
        code_max = ref_cli.main(["solve", "--input", sig, "--mask", msk, "--max-iters", "2",
                                 "--output", beta + ".2", "--report", rep + ".2"])
        with open(rep + ".2") as fh:
            records_max = [json.loads(line) for line in fh if line.strip()]
        bench = os.path.join(tmp, "bench.jsonl")
        code_bench = ref_cli.main(["bench", "--sizes", "4,8", "--seed", "7", "--report", bench])
        with open(bench) as fh:
            bench_rows = [json.loads(line) for line in fh if line.strip()]

        def raw(path):
            return np.frombuffer(open(path, "rb").read(), dtype=np.uint8)

        def side(path):
            return np.array(open(path + ".json").read())

        save("cli_8", signal=raw(sig), signal_json=side(sig), mask_idx=raw(msk), mask_idx_json=side(msk),
             mask_byte=raw(byt), mask_byte_json=side(byt), beta=raw(beta), imputed=raw(imp),
             code=np.array(code), code_max=np.array(code_max), code_bench=np.array(code_bench),
             records_json=np.array(json.dumps(_strip_wall(records))),
             records_max_json=np.array(json.dumps(_strip_wall(records_max))),
             bench_json=np.array(json.dumps(_strip_wall(bench_rows))))
        print(f"    cli: solve exit {code}, {records[-1]['status']} in {records[-1]['iterations']}; "
              f"max-iters exit {code_max}; bench exit {code_bench}")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    only = set(sys.argv[1:])
    for name, fn in (("transforms", transforms), ("masking", masking), ("newton", newton),
                     ("solves", solves), ("cli", cli), ("ista", ista), ("spectrum", spectrum)):
        if not only or name in only:
            print(name)
            fn()
    print("oracle vs reference worst relative deviation:")
    for k, v in WORST.items():
        print(f"  {k:16s} {v:.3e}")
