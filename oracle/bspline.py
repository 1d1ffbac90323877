"""Univariate B-splines by the Cox-de Boor recursion (oracle; test infrastructure).

PAPER.md lines 144-170 (Sec. 2.1): open knot vector
    Xi = {0 = xi_1 <= ... <= xi_{m+p+1} = 1},  xi_1 = ... = xi_{p+1} = 0,
    xi_m = ... = xi_{m+p+1} = 1,
degree 0:  b_{i,0}(eta) = 1 if xi_i <= eta < xi_{i+1}, else 0;
degree p:  b_{i,p} = (eta - xi_i)/(xi_{i+p} - xi_i) b_{i,p-1}
                     + (xi_{i+p+1} - eta)/(xi_{i+p+1} - xi_{i+1}) b_{i+1,p-1},
with the convention 0/0 = 0.

Indices here are 0-based: column i of every returned array is the paper's
b_{i+1,p}.

Reading (DESIGN.md R-endpoint): the degree-0 definition is half-open, which
would make every function vanish at eta = 1.  As is standard (and required for
W_t, PAPER.md 694, to be nonzero) the last non-empty knot span is taken closed,
i.e. values at eta = 1 are the left limits.
"""

import numpy as np


def open_uniform_knots(n_el, p, dtype=np.float64):
    """Open knot vector with n_el uniform elements on [0,1] (PAPER.md 144-147,
    1111-1112: h_s = h_t = h, n_el elements per parametric direction).
    No repeated interior knots, so the space is C^{p-1} (k-method, PAPER.md 60-61).
    The knots are i / n_el computed in ``dtype`` (np.longdouble for the
    extended-precision assembly of reading c17: fp64 knots are inexact when
    n_el is not a power of two and perturb the factor matrices by up to
    ~2.5e-14 relative at n_el = 130)."""
    interior = [dtype(i) / dtype(n_el) for i in range(1, n_el)]
    return np.array([dtype(0)] * (p + 1) + interior + [dtype(1)] * (p + 1), dtype=dtype)


def n_functions(knots, p):
    """m = (#knots) - p - 1 (the knot vector has m + p + 1 entries, PAPER.md 144)."""
    return len(knots) - p - 1


def _ratio(num, den):
    """num/den with the paper's 0/0 = 0 convention (den == 0 only occurs where the
    multiplied lower-degree function vanishes identically)."""
    if den == 0.0:
        return np.zeros_like(num)
    return num / den


def basis_values(knots, p, x, dtype=np.float64):
    """B[q, i] = b_{i,p}(x_q), i = 0..m-1, by the Cox-de Boor recursion
    (``dtype`` = np.longdouble for the extended-precision assembly, reading c17)."""
    knots = np.asarray(knots, dtype=dtype)
    x = np.atleast_1d(np.asarray(x, dtype=dtype))
    n0 = len(knots) - 1  # number of degree-0 functions
    B = np.zeros((len(x), n0), dtype=dtype)
    for i in range(n0):
        B[:, i] = ((x >= knots[i]) & (x < knots[i + 1])).astype(dtype)
    # right end point: left limit (last non-empty span closed), see module doc
    last = max(i for i in range(n0) if knots[i] < knots[i + 1])
    at_end = x == knots[-1]
    B[at_end, :] = 0.0
    B[at_end, last] = 1.0
    for q in range(1, p + 1):
        Bq = np.zeros((len(x), n0 - q), dtype=dtype)
        for i in range(n0 - q):
            Bq[:, i] = (_ratio(x - knots[i], knots[i + q] - knots[i]) * B[:, i]
                        + _ratio(knots[i + q + 1] - x, knots[i + q + 1] - knots[i + 1]) * B[:, i + 1])
        B = Bq
    return B


def basis_derivatives(knots, p, r, x, dtype=np.float64):
    """D[q, i] = d^r/deta^r b_{i,p}(x_q) by the derivative recursion of de Boor
    (the paper's reference for B-splines, PAPER.md 147 [DeBoor2001]):
        b'_{i,p} = p/(xi_{i+p} - xi_i) b_{i,p-1} - p/(xi_{i+p+1} - xi_{i+1}) b_{i+1,p-1},
    applied r times, with 0/0 = 0."""
    if r == 0:
        return basis_values(knots, p, x, dtype)
    knots = np.asarray(knots, dtype=dtype)
    D = basis_derivatives(knots, p - 1, r - 1, x, dtype)
    n = D.shape[1] - 1
    out = np.zeros((D.shape[0], n), dtype=dtype)
    for i in range(n):
        out[:, i] = p * (_ratio(D[:, i], knots[i + p] - knots[i])
                         - _ratio(D[:, i + 1], knots[i + p + 1] - knots[i + 1]))
    return out


def _leggauss(q, dtype):
    """Gauss-Legendre nodes/weights on [-1,1]; for extended precision the
    float64 nodes of numpy's leggauss are polished by Newton steps on the
    Legendre three-term recurrence in ``dtype``."""
    t, w = np.polynomial.legendre.leggauss(q)
    if dtype == np.float64:
        return t, w
    t = t.astype(dtype)

    def legendre(x):
        p0, p1 = np.ones_like(x), x.copy()
        for k in range(2, q + 1):
            p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
        if q == 1:
            p0 = np.ones_like(x)
        return p1, q * (x * p1 - p0) / (x * x - 1)

    for _ in range(3):
        pq, dp = legendre(t)
        t = t - pq / dp
    _, dp = legendre(t)
    return t, 2 / ((1 - t * t) * dp * dp)


def gauss_legendre_rule(knots, q, dtype=np.float64):
    """q-point Gauss-Legendre rule on every non-empty knot span (reading c6:
    the paper does not state its quadrature; with q = p+1 all integrands of the
    factor matrices -- piecewise polynomials of degree <= 2p -- are exact)."""
    t, w = _leggauss(q, dtype)
    breaks = np.unique(np.asarray(knots, dtype=dtype))
    xs, ws = [], []
    for a, b in zip(breaks[:-1], breaks[1:]):
        xs.append(0.5 * (a + b) + 0.5 * (b - a) * t)
        ws.append(0.5 * (b - a) * w)
    return np.concatenate(xs), np.concatenate(ws)
