"""Preconditioned conjugate gradient (oracle; test infrastructure).

PAPER.md 710-712 (A SPD, P SPD -> PCG) and 1109 ("tolerance of CG equal to
10^-8 and the initial guess equal to the null vector").  Textbook
Hestenes-Stiefel PCG.  Reading c7: stop when the recurrence residual satisfies
||r_k||_2 <= tol ||b||_2; the iteration count is the number of A-products.
Reading c8: max_iter = 1000, non-convergence is reported, not raised.
"""

import numpy as np


def pcg(apply_A, apply_Pinv, b, tol=1e-8, max_iter=1000, callback=None):
    """Returns (x, iters, converged, rel_res_history)."""
    b = np.asarray(b, dtype=np.float64)
    x = np.zeros_like(b)
    nb = np.sqrt(np.sum(b * b))
    if nb == 0.0:
        return x, 0, True, [0.0]
    r = b.copy()
    z = apply_Pinv(r)
    p = z.copy()
    rho = np.sum(r * z)
    hist = [1.0]
    for k in range(1, max_iter + 1):
        q = apply_A(p)
        alpha = rho / np.sum(p * q)
        x = x + alpha * p
        r = r - alpha * q
        rel = np.sqrt(np.sum(r * r)) / nb
        hist.append(rel)
        if callback is not None:
            callback(k, x, r)
        if rel <= tol:
            return x, k, True, hist
        z = apply_Pinv(r)
        rho_new = np.sum(r * z)
        beta = rho_new / rho
        rho = rho_new
        p = z + beta * p
    return x, max_iter, False, hist
