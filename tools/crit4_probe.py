"""Probe for reference acceptance criterion 4 (test_acceptance.py:160-170):
empty-mask solves must finish every condensed PCG in <= 2 steps.  Prints the
per-IPM-iteration PCG counts and final residuals of the GPU solve next to the
transform round-trip error of the GPU and scipy (oracle) transforms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2502_04217_b200 as fl  # noqa: E402
from oracle import fftlasso_oracle as O  # noqa: E402

for n, seed in [(64, 1), (256, 2), (1024, 3)]:
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(n)
    mask = fl.Mask(np.array([], dtype=np.int64), fl.GridShape((n,)))
    beta, rep = fl.solve(b, mask, fl.IpmConfig(tol=1e-8))
    recs = rep.records if hasattr(rep, "records") else []
    print(n, "krylov", rep.krylov_counts)
    print("   pcg_residual", [f"{r.pcg_residual:.2e}" for r in recs])
    x = rng.standard_normal(n)
    g = fl.analyze(fl.synthesize(x, fl.GridShape((n,))), fl.GridShape((n,)))
    o = O.analyze(O.synthesize(x, (n,)), (n,))
    print("   roundtrip rel err gpu %.3e  scipy %.3e" % (np.linalg.norm(g - x) / np.linalg.norm(x),
                                                       np.linalg.norm(o - x) / np.linalg.norm(x)))
    s_g = fl.synthesize(x, fl.GridShape((n,)))
    s_o = O.synthesize(x, (n,))
    print("   synth gpu vs scipy rel %.3e" % (np.linalg.norm(s_g - s_o) / np.linalg.norm(s_o)))

# per-IPM-iteration direction from the same (GPU-solve) states: GPU vs oracle PCG
print("--- same states, GPU newton_direction vs oracle (history) ---")
for n, seed in [(256, 2), (1024, 3)]:
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(n)
    mask = fl.Mask(np.array([], dtype=np.int64), fl.GridShape((n,)))
    states = []
    cfg = fl.IpmConfig(tol=1e-8)
    beta, rep = fl.solve(b, mask, cfg, observer=lambda s, rec: states.append(s))
    lam = fl.default_penalty(b, mask)
    om = O.make_mask((n,))
    ocfg = O.OConfig()
    from paper_2502_04217_b200 import ipm as gipm
    for k, s in enumerate(states[:-1]):
        d = gipm.newton_direction(s, b, mask, lam, cfg)
        ost = O.OState(**{f: np.asarray(getattr(s, f)) for f in ("beta", "z", "s1", "s2", "y1", "y2", "nu1", "nu2")}, mu=s.mu)
        diag = O.diagonals(ost.s1, ost.s2, ost.nu1, ost.nu2)
        rhs = O.newton_rhs(ost, b, om, lam)
        res = O.pcg(lambda v: np.concatenate(O.kkt_apply(v[:n], v[n:], diag, om)),
                    lambda v: np.concatenate(O.precond_apply(v[:n], v[n:], diag)),
                    np.concatenate([rhs["r_beta"], rhs["r_c"]]), abs_tol=1e-12, history=True)
        print(n, k + 1, "gpu", d.krylov_iters, f"{d.pcg_residual:.2e}", "oracle", res.iterations,
              [f"{h:.2e}" for h in (res.history or [])])
