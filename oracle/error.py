"""Discretisation error of a least-squares solution (oracle; test infrastructure).

The least-squares functional of the heat equation (PAPER.md 392-410, Sec. 3.1) at
u_h = sum_i c_i B_i is
    J(c) = int_0^T int_Omega (f - d_t u_h + Lap u_h)^2 = ||f||^2 - 2 F(u_h) + A(u_h, u_h)
(A(v, w) = int int (d_t v - Lap v)(d_t w - Lap w), F(w) = int int f (d_t w - Lap w),
eq:cont_problem).  When f = (d_t - Lap) u, J(c) = ||(d_t - Lap)(u - u_h)||^2, the
squared error in the least-squares energy norm, which is equivalent to the V_0 norm of
Thm teo:a-priori (PAPER.md 600-610): O(h^{p_s - 1} + h^{p_t}).

f_norm2: ||f||^2 in closed form for the built-in forcings (reading c11, T = 1).
ls_functional_quadrature: J(c) by direct space-time Gauss quadrature of the residual on
the full tensor grid (no use of A, b or the identity above); tiny grids only.
"""

import numpy as np

from .bspline import basis_values, basis_derivatives, gauss_legendre_rule
from .rhs import forcing, Q_EXTRA


def f_norm2(kind, d):
    """int_0^1 int_(0,1)^d f^2 for kind 0 (e^t prod sin) and kind 1 (prod sin (cos t + d pi^2 sin t))."""
    space = 0.5 ** d  # int_0^1 sin^2(pi x) dx = 1/2
    if kind == 0:
        return space * (np.exp(2.0) - 1.0) / 2.0
    if kind == 1:
        c = d * np.pi ** 2
        return space * ((0.5 + np.sin(2.0) / 4.0) + c * np.sin(1.0) ** 2 + c * c * (0.5 - np.sin(2.0) / 4.0))
    raise ValueError("unknown kind")


def ls_functional_quadrature(c, kind, space_knots, p_s, time_knots, p_t, T=1.0):
    """J(c) = int int (f - d_t u_h + Lap u_h)^2, c of shape (n_t, n_d, .., n_1)."""
    d = len(space_knots)
    g, s = forcing(kind, d)
    tabs = []
    for kn in space_knots:
        x, w = gauss_legendre_rule(kn, p_s + Q_EXTRA)
        tabs.append((x, w, basis_values(kn, p_s, x)[:, 1:-1], basis_derivatives(kn, p_s, 2, x)[:, 1:-1]))
    tau, wt = gauss_legendre_rule(time_knots, p_t + Q_EXTRA)
    T0 = basis_values(time_knots, p_t, tau)[:, 1:]
    T1 = basis_derivatives(time_knots, p_t, 1, tau)[:, 1:] / T
    t, wt = T * tau, wt * T
    grids = np.meshgrid(t, *[tabs[k][0] for k in reversed(range(d))], indexing="ij")
    fval = g(grids[0])
    for j in range(1, d + 1):
        fval = fval * s(grids[j])
    wgt = wt
    for k in reversed(range(d)):
        wgt = np.multiply.outer(wgt, tabs[k][1])

    def apply(mats, v):  # (mats[0] (x) mats[1] (x) ...) v, mats slowest first
        out = v
        for ax, A in enumerate(mats):
            out = np.moveaxis(np.tensordot(A, out, axes=([1], [ax])), 0, ax)
        return out

    order = list(reversed(range(d)))
    ut = apply([T1] + [tabs[k][2] for k in order], c)
    lap = 0.0
    for kk in range(d):
        lap = lap + apply([T0] + [tabs[k][3] if k == kk else tabs[k][2] for k in order], c)
    res = fval - ut + lap
    return float(np.sum(wgt * res * res))
