"""Right-hand side b_i = F(B_i) (oracle; test infrastructure).

PAPER.md 409 (Sec. 3.1): F(w) = int_0^T int_Omega f (d_t w - Lap w).
For a separable forcing f(x,t) = g(t) prod_k s_k(x_k) on the identity map:
    b = (int g b_t') (x) [(x)_k int s_k b_k]
        - (int g b_t) (x) sum_k [ .. (x) int s_k b_k'' (x) .. ]      (slot k)
(direct expansion of d_t B_i - Lap B_i for a tensor-product B_i).

Reading c11 (forcings):  kind 0: f = e^t prod_k sin(pi x_k)  (BASELINE config 2);
kind 1: f = prod_k sin(pi x_k) (cos t + d pi^2 sin t), the forcing of the cube
benchmark's exact solution u = prod_k sin(pi x_k) sin t (PAPER.md 1166).
Reading c16: f is not polynomial, so the univariate integrals use q = p + 5
Gauss-Legendre points per element (the CUDA path's host setup uses the same rule).
"""

import numpy as np

from .bspline import basis_values, basis_derivatives, gauss_legendre_rule

Q_EXTRA = 5


def forcing(kind, d):
    """(g, s) with f(x, t) = g(t) prod_k s(x_k)."""
    s = lambda x: np.sin(np.pi * x)
    if kind == 0:
        return (lambda t: np.exp(t)), s
    if kind == 1:
        return (lambda t: np.cos(t) + d * np.pi ** 2 * np.sin(t)), s
    raise ValueError("unknown rhs kind")


def _integrals(knots, p, fn, sl, q):
    x, w = gauss_legendre_rule(knots, q)
    fx = fn(x) * w
    B0 = basis_values(knots, p, x)[:, sl]
    B1 = basis_derivatives(knots, p, 1, x)[:, sl]
    B2 = basis_derivatives(knots, p, 2, x)[:, sl] if p >= 2 else np.zeros_like(B0)
    return fx @ B0, fx @ B1, fx @ B2


def rhs(kind, space_knots, p_s, time_knots, p_t, T=1.0):
    """b as a tensor of shape (n_t, n_d, .., n_1) (separable evaluation)."""
    g, s = forcing(kind, len(space_knots))
    return rhs_separable([(g, [s] * len(space_knots))], space_knots, p_s, time_knots, p_t, T)


def rhs_separable(terms, space_knots, p_s, time_knots, p_t, T=1.0):
    """b for f = sum over terms (g, [s_1..s_d]) of g(t) prod_k s_k(x_k)."""
    out = 0.0
    for g, svec in terms:
        out = out + _rhs_one(g, svec, space_knots, p_s, time_knots, p_t, T)
    return out


def _rhs_one(g, svec, space_knots, p_s, time_knots, p_t, T):
    d = len(space_knots)
    S0, S2 = [], []
    for kn, s in zip(space_knots, svec):
        i0, _, i2 = _integrals(kn, p_s, s, slice(1, -1), p_s + Q_EXTRA)
        S0.append(i0)
        S2.append(i2)
    # time: t = T tau
    G0, G1, _ = _integrals(time_knots, p_t, lambda tau: g(T * tau), slice(1, None), p_t + Q_EXTRA)
    G0, G1 = G0 * T, G1  # int g b dt = T int g b dtau ; int g d_t b dt = int g b' dtau

    def outer(tvec, svecs):  # svecs[k-1] is direction k
        out = tvec
        for v in reversed(svecs):
            out = np.multiply.outer(out, v)
        return out

    b = outer(G1, S0)
    for k in range(d):
        sv = list(S0)
        sv[k] = S2[k]
        b = b - outer(G0, sv)
    return b


def rhs_dense_quadrature(kind, space_knots, p_s, time_knots, p_t, T=1.0):
    """Same b by direct space-time quadrature of f (d_t B_i - Lap B_i) over the
    full tensor grid (no separation); tiny grids only, used to pin ``rhs``."""
    d = len(space_knots)
    g, s = forcing(kind, d)
    tabs = []
    for kn in space_knots:
        x, w = gauss_legendre_rule(kn, p_s + Q_EXTRA)
        tabs.append((x, w, basis_values(kn, p_s, x)[:, 1:-1],
                     basis_derivatives(kn, p_s, 2, x)[:, 1:-1]))
    tau, wt = gauss_legendre_rule(time_knots, p_t + Q_EXTRA)
    T0 = basis_values(time_knots, p_t, tau)[:, 1:]
    T1 = basis_derivatives(time_knots, p_t, 1, tau)[:, 1:] / T
    t, wt = T * tau, wt * T
    # all points, slowest first (t, x_d, .., x_1)
    grids = np.meshgrid(t, *[tabs[k][0] for k in reversed(range(d))], indexing="ij")
    fval = g(grids[0])
    for j in range(1, d + 1):
        fval = fval * s(grids[j])
    wgt = wt
    for k in reversed(range(d)):
        wgt = np.multiply.outer(wgt, tabs[k][1])
    fw = (fval * wgt).ravel()

    def kr(mats):
        out = np.ones((1, 1))
        for A in mats:
            out = np.kron(out, A)
        return out

    order = list(reversed(range(d)))
    Dt = kr([T1] + [tabs[k][2] for k in order])
    Lap = np.zeros_like(Dt)
    for kk in range(d):
        Lap += kr([T0] + [tabs[k][3] if k == kk else tabs[k][2] for k in order])
    n_t = T0.shape[1]
    shape = (n_t,) + tuple(tabs[k][2].shape[1] for k in order)
    return (fw @ (Dt - Lap)).reshape(shape)
