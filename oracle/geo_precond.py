"""The geometry-aware preconditioner P^G (oracle; test infrastructure).

PAPER.md 969-1045 (Sec. 4.4).  With c_tau = |det J_F| T^{-1} and
c_k = (||row k of J_F^{-1}||_2)^4 |det J_F| T (reading c20: the coefficient of
(d^2 v^/d eta_k^2)^2 in (Lap v)^2 |det J_F|), sampled at one point per element
(the element midpoints), the rank-1 separable approximations
    c_k  ~ mu_1 .. omega_k .. mu_d mu_t,     c_tau ~ mu_1 .. mu_d omega_t
give the Kronecker matrix
    Pbar^G = K^G_t (x) M^G_s + M^G_t (x) J~^G_s
with weighted univariate factors [M^G_k]_ij = int mu_k b_i b_j,
[J^G_k]_ij = int omega_k b_i'' b_j'' (time: omega_t, mu_t), and finally
    P^G = D^{1/2} Pbar^G D^{1/2},   D_ii = A_ii / Pbar^G_ii.

Readings:
  c21  the separable approximation is the least-squares fit of the logarithms
       (the L2 form of the alternating Diliberto-Wachspress sweep; its products
       are unique, so P^G is well defined).  Here: one dense lstsq solve.
  c22  "extended by interpolation to all quadrature points": piecewise-linear
       interpolation of the factors between element midpoints, constant beyond
       the first / last midpoint, evaluated at the p+1 Gauss points per element
       of the standard rule (the weighted matrices use that rule).
  T = 1 only (reading c9): mu_t = omega_t = 1, so the time factors are K^_t, M^_t.
"""

import numpy as np

from . import fd
from .bspline import basis_values, basis_derivatives, gauss_legendre_rule, open_uniform_knots
from .geometry import eval_map


def midpoint_coefficients(geo, n_el, T=1.0):
    """c_tau and c_k (k = 1..d) at the tensor grid of element midpoints, each as an
    array of shape (n_el[d-1], .., n_el[0]) (direction 1 fastest)."""
    d = geo["d"]
    mids = [(np.arange(n) + 0.5) / n for n in n_el]
    g = eval_map(geo, mids)
    det = np.abs(np.linalg.det(g["Jac"]))
    Jinv = np.linalg.inv(g["Jac"])                      # Jinv[q][k][i] = d eta_k / d x_i
    shape = tuple(reversed(n_el))
    c_tau = (det / T).reshape(shape)
    c_k = [((np.sum(Jinv[:, k, :] ** 2, axis=1)) ** 2 * det * T).reshape(shape)
           for k in range(d)]
    return c_tau, c_k


def separable_fit(c_tau, c_k):
    """Least-squares fit of the logarithms (reading c21):
        log c_tau(e) ~ sum_j m_j(e_j),
        log c_k(e)   ~ o_k(e_k) + sum_{j != k} m_j(e_j),
    with mu_j = exp(m_j), omega_k = exp(o_k), omega_t = mu_t = 1.
    Returns (mu, omega): lists over directions of per-element values."""
    d = len(c_k)
    shape = c_tau.shape                                 # (n_d, .., n_1)
    n_el = list(reversed(shape))
    off_m = np.cumsum([0] + n_el)[:-1]
    off_o = off_m[-1] + n_el[-1] + np.cumsum([0] + n_el)[:-1]
    n_unk = 2 * sum(n_el)
    rows, rhs = [], []
    for idx in np.ndindex(*shape):
        e = idx[::-1]                                   # e[k] = element index in direction k+1
        for eq in range(d + 1):                         # eq = d: c_tau; eq = k: c_k
            a = np.zeros(n_unk)
            for j in range(d):
                if j == eq:
                    a[off_o[j] + e[j]] = 1.0
                else:
                    a[off_m[j] + e[j]] = 1.0
            rows.append(a)
            rhs.append(np.log(c_tau[idx] if eq == d else c_k[eq][idx]))
    sol = np.linalg.lstsq(np.array(rows), np.array(rhs), rcond=None)[0]
    mu = [np.exp(sol[off_m[j]:off_m[j] + n_el[j]]) for j in range(d)]
    om = [np.exp(sol[off_o[j]:off_o[j] + n_el[j]]) for j in range(d)]
    return mu, om


def interpolate_factor(values, x):
    """Reading c22: piecewise-linear through (element midpoint, value), constant
    beyond the outer midpoints."""
    n = len(values)
    mids = (np.arange(n) + 0.5) / n
    return np.interp(x, mids, values)


def weighted_space_factors(n_el, p, mu, omega):
    """Constrained (i = 2..m-1) [M^G]_ij = int mu b_i b_j, [J^G]_ij = int omega b_i'' b_j''
    with the p+1-point Gauss rule per element (reading c22)."""
    kn = open_uniform_knots(n_el, p)
    x, w = gauss_legendre_rule(kn, p + 1)
    B0 = basis_values(kn, p, x)[:, 1:-1]
    B2 = basis_derivatives(kn, p, 2, x)[:, 1:-1]
    wm = w * interpolate_factor(mu, x)
    wo = w * interpolate_factor(omega, x)
    return {"M": (B0.T * wm) @ B0, "J": (B2.T * wo) @ B2}


def setup(geo, n_el_s, p_s, time, A_diag):
    """P^G for the spatial grid n_el_s (list of d) and degree p_s; ``time`` the dict
    of oracle.univariate.time_factors (T = 1); ``A_diag`` the diagonal of A
    (shape (n_t, n_d, .., n_1)).  Returns the FD data of Pbar^G plus D^{-1/2}."""
    c_tau, c_k = midpoint_coefficients(geo, n_el_s)
    mu, om = separable_fit(c_tau, c_k)
    space = [weighted_space_factors(n_el_s[k], p_s, mu[k], om[k]) for k in range(len(n_el_s))]
    data = fd.setup(space, time)
    # diag(Pbar^G) from the Kronecker factor diagonals
    d = len(space)
    dM = [np.diag(f["M"]) for f in space]
    dJ = [np.diag(f["J"]) for f in space]

    def outer(vecs):                                   # vecs[k] for direction k+1
        out = vecs[-1]
        for v in reversed(vecs[:-1]):
            out = np.multiply.outer(out, v)
        return out

    Ms = outer(dM)
    Js = sum(outer([dJ[j] if j == k else dM[j] for j in range(d)]) for k in range(d))
    Pdiag = (np.multiply.outer(np.diag(time["Kt_hat"]), Ms)
             + np.multiply.outer(np.diag(time["Mt_hat"]), Js))
    data.update({"space": space, "Kt_hat_mat": time["Kt_hat"], "Mt_hat_mat": time["Mt_hat"], "mu": mu, "omega": om, "c_tau": c_tau, "c_k": c_k,
                 "Pbar_diag": Pdiag, "Dm12": np.sqrt(Pdiag / A_diag)})
    return data


def apply(r, data):
    """(P^G)^{-1} r = D^{-1/2} Pbar^{-1} D^{-1/2} r (Algorithm 1 for Pbar^G)."""
    return data["Dm12"] * fd.fd_apply(data["Dm12"] * r, data)


def A_diagonal(sf, time):
    """diag(A) = diag(K_t) (x) diag(M_s) + diag(M_t) (x) diag(J_s) + diag(W_t) (x) diag(L_s)
    for the sparse physical spatial factors of oracle.geometry.space_factors_physical."""
    shape = tuple(reversed(sf["n_s"]))
    dg = [np.asarray(sf[k].diagonal()).reshape(shape) for k in ("M", "J", "L")]
    return (np.multiply.outer(np.diag(time["Kt"]), dg[0])
            + np.multiply.outer(np.diag(time["Mt"]), dg[1])
            + np.multiply.outer(np.diag(time["Wt"]), dg[2]))


def dense_PG(data):
    """Dense P^G = D^{1/2} Pbar^G D^{1/2} by np.kron of the factors (tiny grids)."""
    space = data["space"]
    d = len(space)

    def kron(mats):                                    # mats[0] = time, then d, .., 1
        out = np.ones((1, 1))
        for A in mats:
            out = np.kron(out, A)
        return out

    Kt, Mt = data["Kt_hat_mat"], data["Mt_hat_mat"]
    Ms = kron([Kt] + [space[k]["M"] for k in reversed(range(d))])
    Js = sum(kron([Mt] + [space[k]["J"] if k == kk else space[k]["M"]
                          for k in reversed(range(d))]) for kk in range(d))
    D12 = 1.0 / data["Dm12"].ravel()
    return D12[:, None] * (Ms + Js) * D12[None, :]
