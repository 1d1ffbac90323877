"""Convergence of the PCG solution: prints the least-squares energy error
||(d_t - Lap)(u - u_h)|| / ||f|| and the relative V_0, L^2 and H^1 errors (ls_error_norms) with
their observed rates, on the cube (u = prod sin(pi x_k) sin t, PAPER.md 1166) or, with
--annulus, on the 2D quarter annulus (u = -(x^2+y^2-1)(x^2+y^2-4) x y^2 sin(pi t),
PAPER.md 1128-1129, the setting of Fig. 2; P^G preconditioner).
    python tools/convergence.py [--d 3] [--p 2 3 4] [--nel 4 8 16 32] [--annulus]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1809_10026_b200 as ls
ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=3)
ap.add_argument("--p", type=int, nargs="+", default=[2, 3, 4])
ap.add_argument("--nel", type=int, nargs="+", default=[4, 8, 16, 32])
ap.add_argument("--annulus", action="store_true")
a = ap.parse_args()
if a.annulus:
    import synth
    a.d = 2
for p in a.p:
    errs = []
    for ne in a.nel:
        if a.annulus:
            ctx = ls.Context(2, p, [ne] * 3, geometry=synth.quarter_annulus(), precond=ls.LS_PRECOND_PG)
            kind = 2
        else:
            ctx = ls.Context(a.d, p, [ne] * (a.d + 1))
            kind = 1
        x, st = ctx.pcg(ctx.rhs(kind), tol=1e-12, max_iter=3000)
        e = ctx.energy_error(kind, x)
        n = ctx.error_norms(kind, x)
        errs.append([float(np.sqrt(max(e["J"], 0.0) / e["f2"])), n["rel_V0"], n["rel_L2"], n["rel_H1"]])
        ctx.close()
    E = np.array(errs)
    rates = np.log2(E[:-1] / E[1:]).T.tolist()
    print(json.dumps({"domain": "quarter annulus" if a.annulus else "cube", "d": a.d, "p": p, "n_el": a.nel,
                      "rel_energy_error": E[:, 0].tolist(), "rel_V0": E[:, 1].tolist(),
                      "rel_L2": E[:, 2].tolist(), "rel_H1": E[:, 3].tolist(),
                      "rates": {"energy": rates[0], "V0": rates[1], "L2": rates[2], "H1": rates[3]},
                      "expected": {"energy": p - 1, "V0": p - 1, "H1": p, "L2": p + 1 if p >= 3 else "suboptimal"}}),
          flush=True)
