"""Write tests/golden/eig_mpmath.json (calls only oracle/ and the seeded input module).

High-precision references for the setup of Algorithm 1 (PAPER.md 939-962):
* eigenvalues lambda_1..lambda_5 and lambda_max of the space pencil (J-hat, M-hat) and the
  time pencil (K_t-hat, M_t-hat) (eq:eig_dec, PAPER.md 942-945), both for the EXACT rational
  pencil and for its entry-wise correctly rounded fp64 copy, by inertia bisection in
  mpmath (oracle/highprec.py) at 50 digits, stored with 40 significant digits;
* z = P^{-1} r (PAPER.md 733, 752-757; reading c2) by a banded Cholesky of the
  Kronecker-assembled P in mpmath (40 digits) on small anisotropic grids, r = synth.residual.

    python tools/make_golden_eig.py        (~2 min on one core)
"""
import json
import os
import sys
import time

import mpmath

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import highprec as hp  # noqa: E402
import synth  # noqa: E402

EIG_CASES = [(16, 2), (130, 2), (64, 3), (128, 6)]
# (n_el per direction (space 1..d, time), p, pencil entries exact or rounded to fp64, seed)
FD_CASES = [((6, 4, 5), 3, "exact", 11), ((3, 4, 2, 3), 2, "exact", 12),
            ((130, 4), 2, "fp64", 13), ((128, 3), 6, "fp64", 14)]


def s40(x):
    return mpmath.nstr(x, 40, strip_zeros=False)


def main():
    out = {"source": "tools/make_golden_eig.py (oracle/highprec.py: exact rational assembly, "
                     "mpmath inertia bisection, mpmath banded Cholesky of P)",
           "cite": "PAPER.md 939-945 (eq:eig_dec), 947-962 (Alg. 1), 733/752-757 (P)",
           "eig": [], "fd": []}
    for n_el, p in EIG_CASES:
        t0 = time.time()
        for name, (A, B) in (("space", hp.space_pencil(n_el, p)), ("time", hp.time_pencil(n_el, p))):
            n = len(A)
            ks = [1, 2, 3, 4, 5, n]
            ex = hp.eig_bisect(A, B, ks)
            rd = hp.eig_bisect(hp.round_fp64(A), hp.round_fp64(B), ks)
            out["eig"].append({"n_el": n_el, "p": p, "pencil": name, "n": n, "k": ks,
                               "exact": [s40(v) for v in ex], "fp64_pencil": [s40(v) for v in rd]})
        print(f"eig n_el={n_el} p={p}: {time.time() - t0:.1f} s", flush=True)
    for ne, p, kind, seed in FD_CASES:
        t0 = time.time()
        d = len(ne) - 1
        sp = [hp.space_pencil(n, p) for n in ne[:d]]
        tp = hp.time_pencil(ne[d], p)
        if kind == "fp64":
            sp = [(hp.round_fp64(J), hp.round_fp64(M)) for J, M in sp]
            tp = (hp.round_fp64(tp[0]), hp.round_fp64(tp[1]))
        shape = (len(tp[1]),) + tuple(len(M) for _, M in reversed(sp))
        r = synth.residual(shape, seed).ravel()
        z = hp.solve_P(sp, tp, r)
        out["fd"].append({"n_el": list(ne), "p": p, "pencil": kind, "seed": seed, "shape": list(shape),
                          "z": [mpmath.nstr(v, 25) for v in z]})
        print(f"fd {ne} p={p}: {time.time() - t0:.1f} s", flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "eig_mpmath.json"), "w") as f:
        json.dump(out, f, indent=0)


if __name__ == "__main__":
    main()
