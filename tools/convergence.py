"""Energy-norm convergence of the PCG solution on the cube (u = prod sin(pi x_k) sin t,
PAPER.md 1166): prints ||(d_t - Lap)(u - u_h)|| / ||f|| and observed rates.
    python tools/convergence.py [--d 3] [--p 2 3 4] [--nel 4 8 16 32]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1809_10026_b200 as ls
ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=3)
ap.add_argument("--p", type=int, nargs="+", default=[2, 3, 4])
ap.add_argument("--nel", type=int, nargs="+", default=[4, 8, 16, 32])
a = ap.parse_args()
for p in a.p:
    errs = []
    for ne in a.nel:
        ctx = ls.Context(a.d, p, [ne] * (a.d + 1))
        x, st = ctx.pcg(ctx.rhs(1), tol=1e-12)
        e = ctx.energy_error(1, x)
        errs.append(float(np.sqrt(max(e["J"], 0.0) / e["f2"])))
        ctx.close()
    rates = [float(np.log2(errs[i] / errs[i + 1])) for i in range(len(errs) - 1)]
    print(json.dumps({"d": a.d, "p": p, "n_el": a.nel, "rel_energy_error": errs, "rates": rates,
                      "expected_rate": p - 1}))
