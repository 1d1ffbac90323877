"""Load vectors and least-squares energy error on mapped domains (oracle; test infrastructure).

Kind 3 (PAPER.md 1219-1221): the rotated quarter annulus with the forcing of the paper's
u = -(x^2+y^2-1)(x^2+y^2-4) x y^2 sin(z) and homogeneous data (reading c23).

The 2D benchmark of PAPER.md 1128-1129 (Sec. 5, Fig. 2): Omega = the quarter annulus
(radii 1, 2), T = 1, exact solution
    u = -(x^2 + y^2 - 1)(x^2 + y^2 - 4) x y^2 sin(pi t),
which vanishes on the whole boundary of Omega and at t = 0 (homogeneous data: no lifting),
so f = d_t u - Lap u.  Here f is obtained by SYMBOLIC differentiation of u (sympy), and
    b_i = F(B_i) = int int f (d_t B_i - Lap B_i)          (PAPER.md 409)
    ||f||^2 = int int f^2,
both by direct space-time Gauss quadrature of the mapped basis (p + 5 points per element
and direction: reading c16 extended to Omega), with no use of the separable structure of
f that the CUDA path exploits.  J(c) = ||f||^2 - 2 b.c + c.A c is then the squared
least-squares energy error ||(d_t - Lap)(u - u_h)||^2 (PAPER.md 392-410, 600-610).
"""

import numpy as np
import sympy as sp

from .bspline import basis_values, basis_derivatives, gauss_legendre_rule, open_uniform_knots
from .geometry import space_tables

Q_EXTRA = 5   # Gauss points per element = p + Q_EXTRA (reading c16)


def annulus_solution():
    """(u, f) as numpy callables u(x, y, t), f(x, y, t) from sympy (PAPER.md 1129)."""
    x, y, t = sp.symbols("x y t")
    u = -(x ** 2 + y ** 2 - 1) * (x ** 2 + y ** 2 - 4) * x * y ** 2 * sp.sin(sp.pi * t)
    f = sp.diff(u, t) - sp.diff(u, x, 2) - sp.diff(u, y, 2)
    return sp.lambdify((x, y, t), u, "numpy"), sp.lambdify((x, y, t), f, "numpy")


def revolved_solution():
    """(u, f) as numpy callables of (x, y, z, t) for the rotated quarter annulus
    (PAPER.md 1221): u = -(x^2 + y^2 - 1)(x^2 + y^2 - 4) x y^2 sin(z), time independent,
    f = d_t u - Lap u.  Reading c23: used with homogeneous data (the paper's lifting of
    u's non-zero boundary / initial values is out of scope)."""
    x, y, z, t = sp.symbols("x y z t")
    u = -(x ** 2 + y ** 2 - 1) * (x ** 2 + y ** 2 - 4) * x * y ** 2 * sp.sin(z)
    f = sp.diff(u, t) - sp.diff(u, x, 2) - sp.diff(u, y, 2) - sp.diff(u, z, 2)
    fl = sp.lambdify((x, y, z, t), f, "numpy")
    return sp.lambdify((x, y, z, t), u, "numpy"), lambda X, Y, Z, T: fl(X, Y, Z, T) + 0.0 * T


def _forcing(kind):
    if kind == 2:
        _, f = annulus_solution()
        return lambda X, t: f(X[None, :, 0], X[None, :, 1], t[:, None])
    if kind == 3:
        _, f = revolved_solution()
        return lambda X, t: f(X[None, :, 0], X[None, :, 1], X[None, :, 2], t[:, None])
    raise ValueError("unknown kind")


def _time_rule(n_el_t, p_t):
    kt = open_uniform_knots(n_el_t, p_t)
    xt, wt = gauss_legendre_rule(kt, p_t + Q_EXTRA)
    T0 = basis_values(kt, p_t, xt)[:, 1:]
    T1 = basis_derivatives(kt, p_t, 1, xt)[:, 1:]
    return xt, wt, T0, T1


def load_vector(geo, n_el_s, p_s, n_el_t, p_t, kind=2):
    """b of shape (n_t, n_d, .., n_1) for kind 2 (2D annulus) / 3 (rotated annulus),
    by direct quadrature."""
    f = _forcing(kind)
    st = space_tables(geo, n_el_s, p_s, q=p_s + Q_EXTRA)
    xt, wt, T0, T1 = _time_rule(n_el_t, p_t)
    X = st["X"]
    F = f(X, xt)                                               # [time pts][space pts]
    FW = (wt[:, None] * F) * st["W"][None, :]
    b = T1.T @ (st["Phi"].T @ FW.T).T - T0.T @ (st["Lap"].T @ FW.T).T
    return b.reshape((T0.shape[1],) + tuple(reversed(st["n_s"])))


def f_norm2(geo, n_el_s, p_s, n_el_t, p_t, kind=2):
    """||f||^2 = int int f^2 by the same quadrature."""
    f = _forcing(kind)
    st = space_tables(geo, n_el_s, p_s, q=p_s + Q_EXTRA)
    xt, wt, _, _ = _time_rule(n_el_t, p_t)
    X = st["X"]
    F = f(X, xt)
    return float(np.sum(wt[:, None] * st["W"][None, :] * F * F))
