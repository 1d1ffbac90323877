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


# ---------------------------------------------------------------------------------------
# V_0, L^2 and H^1 errors against the exact solution (Fig. 2)
# ---------------------------------------------------------------------------------------
Q_ERR = 3   # Gauss points per element and direction = p + Q_ERR (reading c24)


def exact_solution(kind, d):
    """The exact solution u(x_1..x_d, t) of a built-in benchmark and its derivatives
    (d_t u, grad_x u, Lap u) as numpy callables, by SYMBOLIC differentiation (sympy):
    kind 1: u = prod_k sin(pi x_k) sin t on the cube (PAPER.md 1166);
    kind 2: u = -(x^2 + y^2 - 1)(x^2 + y^2 - 4) x y^2 sin(pi t) (d = 2, PAPER.md 1129)."""
    import sympy as sp
    xs = sp.symbols("x1:%d" % (d + 1))
    t = sp.Symbol("t")
    if kind == 1:
        u = sp.sin(t)
        for x in xs:
            u = u * sp.sin(sp.pi * x)
    elif kind == 2 and d == 2:
        x, y = xs
        u = -(x ** 2 + y ** 2 - 1) * (x ** 2 + y ** 2 - 4) * x * y ** 2 * sp.sin(sp.pi * t)
    else:
        raise ValueError("no exact solution for this kind / d")
    args = tuple(xs) + (t,)
    lam = lambda e: sp.lambdify(args, e, "numpy")
    return {"u": lam(u), "ut": lam(sp.diff(u, t)), "grad": [lam(sp.diff(u, x)) for x in xs],
            "lap": lam(sum(sp.diff(u, x, 2) for x in xs)), "f": lam(sp.diff(u, t) - sum(sp.diff(u, x, 2) for x in xs))}


def error_norms(c, kind, geo, n_el_s, p_s, n_el_t, p_t):
    """The eight space-time integrals of ls_error_norms (err.cu header) by direct Gauss
    quadrature on the tensor grid (p_s + 3 points per element and space direction, p_t + 3 in
    time), e = u - u_h, u_h = sum_i c_i B_i on Omega = geo([0,1]^d) (the identity map for
    the cube: synth.affine_box([1]*d)):
        [0] int e^2, [1] int (d_t e)^2, [2] int |grad_x e|^2, [3] int (Lap e)^2, [4..7] same of u.
    The mapped basis' values / gradients / Laplacians come from oracle.geometry.space_tables
    (chain rule of PAPER.md 986-990); c has shape (n_t, n_d, .., n_1)."""
    from .geometry import space_tables
    from .bspline import open_uniform_knots
    d = geo["d"]
    tab = space_tables(geo, n_el_s, p_s, q=p_s + Q_ERR)
    kt = open_uniform_knots(n_el_t, p_t)
    tau, wt = gauss_legendre_rule(kt, p_t + Q_ERR)
    T0 = basis_values(kt, p_t, tau)[:, 1:]
    T1 = basis_derivatives(kt, p_t, 1, tau)[:, 1:]
    C = np.asarray(c, dtype=np.float64).reshape(T0.shape[1], -1)     # [n_t][N_s]
    uh = T0 @ (tab["Phi"] @ C.T).T                                    # [nq_t][nq_s]
    uth = T1 @ (tab["Phi"] @ C.T).T
    gh = [T0 @ (G @ C.T).T for G in tab["Grad"]]
    lh = T0 @ (tab["Lap"] @ C.T).T
    ex = exact_solution(kind, d)
    X = tab["X"]
    args = [X[None, :, k] for k in range(d)] + [tau[:, None]]
    u, ut, lu = ex["u"](*args), ex["ut"](*args), ex["lap"](*args)
    g = [np.broadcast_to(gk(*args), uh.shape) for gk in ex["grad"]]
    u, ut, lu = (np.broadcast_to(v, uh.shape) for v in (u, ut, lu))
    W = wt[:, None] * tab["W"][None, :]
    e_grad = sum((g[k] - gh[k]) ** 2 for k in range(d))
    u_grad = sum(g[k] ** 2 for k in range(d))
    return np.array([np.sum(W * (u - uh) ** 2), np.sum(W * (ut - uth) ** 2), np.sum(W * e_grad),
                     np.sum(W * (lu - lh) ** 2), np.sum(W * u ** 2), np.sum(W * ut ** 2), np.sum(W * u_grad),
                     np.sum(W * lu ** 2)])


def relative_errors(o):
    """(V_0, L^2, H^1) relative errors from the eight integrals (PAPER.md 318-323, 1131-1139)."""
    return (np.sqrt((o[1] + o[3]) / (o[5] + o[7])), np.sqrt(o[0] / o[4]),
            np.sqrt((o[0] + o[1] + o[2]) / (o[4] + o[5] + o[6])))


def grad_error_at_T(c, kind, geo, n_el_s, p_s, n_el_t, p_t):
    """int_Omega |grad_x e(x, T)|^2 (T = 1): the boundary term of eq:equivalent_A, by which
    ||(d_t - Lap) e||^2 = ||d_t e||^2 + ||Lap e||^2 + ||grad e(T)||^2 when e(0) = 0."""
    from .geometry import space_tables
    from .bspline import open_uniform_knots
    d = geo["d"]
    tab = space_tables(geo, n_el_s, p_s, q=p_s + Q_ERR)
    kt = open_uniform_knots(n_el_t, p_t)
    bT = basis_values(kt, p_t, [1.0])[0, 1:]
    C = np.asarray(c, dtype=np.float64).reshape(len(bT), -1)
    cT = bT @ C
    ex = exact_solution(kind, d)
    X = tab["X"]
    args = [X[:, k] for k in range(d)] + [np.ones(X.shape[0])]
    e2 = sum((ex["grad"][k](*args) - tab["Grad"][k] @ cT) ** 2 for k in range(d))
    return float(np.sum(tab["W"] * e2))
