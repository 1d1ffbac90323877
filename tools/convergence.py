"""Energy-norm convergence of the PCG solution: prints ||(d_t - Lap)(u - u_h)|| / ||f|| and
observed rates, on the cube (u = prod sin(pi x_k) sin t, PAPER.md 1166) or, with
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
        x, st = ctx.pcg(ctx.rhs(kind), tol=1e-12)
        e = ctx.energy_error(kind, x)
        errs.append(float(np.sqrt(max(e["J"], 0.0) / e["f2"])))
        ctx.close()
    rates = [float(np.log2(errs[i] / errs[i + 1])) for i in range(len(errs) - 1)]
    print(json.dumps({"domain": "quarter annulus" if a.annulus else "cube", "d": a.d, "p": p, "n_el": a.nel,
                      "rel_energy_error": errs, "rates": rates, "expected_rate": p - 1}))
