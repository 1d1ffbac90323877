"""Mapped (non-identity) spatial domains (oracle; test infrastructure).

PAPER.md 226-250 (Sec. 2.2): Omega = F([0,1]^d), the discrete space is the
push-forward B_i = B^_i o F^{-1} of the constrained tensor B-spline basis
(eq:disc_space, PAPER.md 291-300).  eq:A_kron (PAPER.md 686-703) keeps its form
    A = K_t (x) M_s + M_t (x) J_s + W_t (x) L_s
but the spatial factors are the physical integrals
    [M_s]_ij = int_Omega B_i B_j,  [L_s]_ij = int_Omega grad B_i . grad B_j,
    [J_s]_ij = int_Omega Lap B_i Lap B_j,
no longer Kronecker products.  Reading c19: F is a tensor-product
NURBS (rational when ``weights`` is given) of its own degrees and knots.

Chain rule (PAPER.md 986-990, written for one x_i there; summed over i here):
with Jac[q][m][j] = dF_m/deta_j, Jinv = Jac^{-1} (Jinv[j][i] = d eta_j / d x_i),
    grad_x v = Jinv^T grad_eta v^,
    Lap v   = sum_{j,k} A_jk d_jk v^ - sum_m (sum_{j,k} A_jk d_jk F_m) (grad_x v)_m,
    A = Jinv Jinv^T.
(The Hessian of v o F^{-1} is Jinv^T (H^ v^ - sum_m (grad_x v)_m H^ F_m) Jinv,
whose trace is the line above; it equals the paper's formula with the derivative
of Jinv expanded by d(Jinv) = -Jinv (dJac) Jinv.)

Everything is evaluated at the tensor Gauss-Legendre points (p+1 per element,
reading c6) with quadrature weight times |det Jac|; the integrals of the rational
integrands are therefore not exact -- both sides of every comparison use the same
rule (reading c19).  Matrices are scipy.sparse, assembled as Phi^T W Phi from
evaluation matrices (points x DOFs): no element loop, no stencil format.
"""

import numpy as np
import scipy.sparse as sp

from .bspline import basis_values, basis_derivatives, gauss_legendre_rule, open_uniform_knots


def _ders(knots, p, r, x):
    """r-th derivative table of all B-splines of degree p (zero when r > p)."""
    if r > p:
        return np.zeros((len(x), len(knots) - p - 1))
    return basis_derivatives(knots, p, r, x)


def _kron_all(mats):
    """kron(mats[-1], ..., mats[0]): mats[k] belongs to direction k+1, so the
    result is in colex order (direction 1 fastest) for rows and columns."""
    out = sp.csr_matrix(np.ones((1, 1)))
    for A in reversed(mats):
        out = sp.kron(out, sp.csr_matrix(A), format="csr")
    return out


def _unit(d, j):
    e = [0] * d
    e[j] += 1
    return e


def _unit2(d, j, k):
    e = [0] * d
    e[j] += 1
    e[k] += 1
    return e


def _tensor_tables(tabs, order):
    """Tensor evaluation matrix for a derivative multi-index ``order`` (per direction),
    ``tabs[k][r]`` = univariate table of derivative r in direction k."""
    return _kron_all([tabs[k][order[k]] for k in range(len(tabs))])


def eval_map(geo, pts_per_dir):
    """F and its first and second parametric derivatives at the tensor grid of the
    univariate point lists ``pts_per_dir`` (colex order of points).

    Returns dict X [nq][d], Jac [nq][d][d] (Jac[q][m][j] = dF_m/deta_j),
    Hes [nq][d][d][d] (Hes[q][m][j][k] = d^2F_m/deta_j deta_k).
    Rational case by the quotient rule: F = N / W with N = sum w_c C_c R_c,
    W = sum w_c R_c."""
    d = geo["d"]
    tabs = [[_ders(geo["knots"][k], geo["degrees"][k], r, np.asarray(pts_per_dir[k], float))
             for r in range(3)] for k in range(d)]
    C = geo["ctrl"]
    w = geo["weights"] if geo["weights"] is not None else np.ones(C.shape[0])
    Cw = C * w[:, None]

    def ev(order):
        T = _tensor_tables(tabs, order)
        return T @ Cw, T @ w                       # (nq, d), (nq,)

    N0, W0 = ev([0] * d)
    N1 = [ev(_unit(d, j)) for j in range(d)]
    N2 = [[ev(_unit2(d, j, k)) for k in range(d)] for j in range(d)]
    X = N0 / W0[:, None]
    nq = X.shape[0]
    Jac = np.zeros((nq, d, d))
    for j in range(d):
        Nj, Wj = N1[j]
        Jac[:, :, j] = (Nj - X * Wj[:, None]) / W0[:, None]
    Hes = np.zeros((nq, d, d, d))
    for j in range(d):
        for k in range(d):
            Njk, Wjk = N2[j][k]
            Hes[:, :, j, k] = (Njk - Jac[:, :, j] * N1[k][1][:, None]
                               - Jac[:, :, k] * N1[j][1][:, None]
                               - X * Wjk[:, None]) / W0[:, None]
    return {"X": X, "Jac": Jac, "Hes": Hes}


def laplace_coefficients(Jac, Hes):
    """A[q] = Jinv Jinv^T (coefficient of d_jk v^) and b[q] with
    Lap v = sum_jk A_jk d_jk v^ + sum_j b_j d_j v^ (module docstring):
    b_j = -sum_m Jinv[j][m] c_m, c_m = sum_jk A_jk Hes[m][j][k]."""
    Jinv = np.linalg.inv(Jac)
    A = Jinv @ np.transpose(Jinv, (0, 2, 1))
    c = np.einsum("qjk,qmjk->qm", A, Hes)
    b = -np.einsum("qjm,qm->qj", Jinv, c)
    return Jinv, A, b


def physical_laplacian(v_grad, v_hess, Jac, Hes):
    """Lap_x (v^ o F^{-1}) at points from the parametric gradient [nq][d] and
    Hessian [nq][d][d] of v^ (the chain rule of the module docstring)."""
    _, A, b = laplace_coefficients(Jac, Hes)
    return np.einsum("qjk,qjk->q", A, v_hess) + np.einsum("qj,qj->q", b, v_grad)


def space_tables(geo, n_el, p, drop_boundary=True, q=None):
    """Physical evaluation matrices of the spatial basis at the tensor Gauss points
    (q per element and direction, default p + 1).

    ``n_el``: elements per direction (list of d).  Returns dict with W (quadrature
    weight x |det Jac|, [nq]), Phi (nq x N_s), Grad (list of d: d/dx_i, nq x N_s),
    Lap (nq x N_s), X (points), sizes.  The basis is the Dirichlet-constrained one
    (eq:basis_par: i_k = 2..m_k-1) unless drop_boundary is False (all m_k functions)."""
    d = geo["d"]
    knots = [open_uniform_knots(n_el[k], p) for k in range(d)]
    rules = [gauss_legendre_rule(kn, p + 1 if q is None else q) for kn in knots]
    sl = slice(1, -1) if drop_boundary else slice(None)
    tabs = [[_ders(knots[k], p, r, rules[k][0])[:, sl] for r in range(3)] for k in range(d)]
    g = eval_map(geo, [r[0] for r in rules])
    Jinv, A, b = laplace_coefficients(g["Jac"], g["Hes"])
    qw = _kron_all([r[1][:, None] for r in rules]).toarray().ravel()
    W = qw * np.abs(np.linalg.det(g["Jac"]))
    Phi = _tensor_tables(tabs, [0] * d)
    D1 = [_tensor_tables(tabs, _unit(d, j)) for j in range(d)]
    Grad = [sum(sp.diags(Jinv[:, j, i]) @ D1[j] for j in range(d)) for i in range(d)]
    Lap = sum(sp.diags(b[:, j]) @ D1[j] for j in range(d))
    for j in range(d):
        for k in range(d):
            Lap = Lap + sp.diags(A[:, j, k]) @ _tensor_tables(tabs, _unit2(d, j, k))
    return {"W": W, "Phi": Phi.tocsr(), "Grad": [G.tocsr() for G in Grad],
            "Lap": Lap.tocsr(), "X": g["X"], "knots": knots,
            "n_s": [t[0].shape[1] for t in tabs]}


def space_factors_physical(geo, n_el, p, drop_boundary=True):
    """The physical spatial factors of eq:A_kron (PAPER.md 697-703):
    M_s = Phi^T W Phi, L_s = sum_i Grad_i^T W Grad_i, J_s = Lap^T W Lap."""
    t = space_tables(geo, n_el, p, drop_boundary)
    Wd = sp.diags(t["W"])
    Ms = (t["Phi"].T @ Wd @ t["Phi"]).tocsr()
    Ls = sum(G.T @ Wd @ G for G in t["Grad"]).tocsr()
    Js = (t["Lap"].T @ Wd @ t["Lap"]).tocsr()
    return {"M": Ms, "L": Ls, "J": Js, "n_s": t["n_s"], "tables": t}


def apply_A_geo(x, sf, time):
    """y = A x with A = K_t (x) M_s + M_t (x) J_s + W_t (x) L_s (eq:A_kron) for the
    sparse physical spatial factors ``sf`` and the time dict of
    oracle.univariate.time_factors.  x has shape (n_t, n_d, .., n_1)."""
    shape = x.shape
    X = x.reshape(shape[0], -1)                       # [n_t][N_s], colex rows
    Y = (time["Kt"] @ (sf["M"] @ X.T).T + time["Mt"] @ (sf["J"] @ X.T).T
         + time["Wt"] @ (sf["L"] @ X.T).T)
    return Y.reshape(shape)


def dense_A_original_form_geo(geo, n_el_s, p_s, n_el_t, p_t, T=1.0):
    """Dense A from the ORIGINAL least-squares form (PAPER.md 406)
        A(v,w) = int int (d_t v - Lap v)(d_t w - Lap w)
    by space-time Gauss quadrature of the mapped basis (no eq:equivalent_A, no
    integration by parts, no Kronecker factorisation); tiny grids only."""
    t = space_tables(geo, n_el_s, p_s)
    kt = open_uniform_knots(n_el_t, p_t)
    xt, wt = gauss_legendre_rule(kt, p_t + 1)
    T0 = basis_values(kt, p_t, xt)[:, 1:]
    T1 = basis_derivatives(kt, p_t, 1, xt)[:, 1:] / T
    wt = wt * T
    Phi, Lap = t["Phi"].toarray(), t["Lap"].toarray()
    # space-time evaluation matrices, time slowest (colex)
    E = np.kron(T1, Phi) - np.kron(T0, Lap)
    W = np.kron(wt, t["W"])
    return E.T @ (E * W[:, None])
