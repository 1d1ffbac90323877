"""Univariate factor matrices (oracle; test infrastructure).

Definitions (0-based indices; "full" = all m functions, before boundary conditions):
  M[i,j] = int_0^1 b_i b_j,      K[i,j] = int_0^1 b_i' b_j',
  J[i,j] = int_0^1 b_i'' b_j'',  G[i,j] = int_0^1 b_i'' b_j
(PAPER.md 738-757: K_t-hat, M_t-hat, J_k-hat, M_k-hat; G enters J_s through the
mixed terms of Delta B_i Delta B_j, PAPER.md 697-698).

Boundary / initial conditions, eq:basis_par (PAPER.md 266-267):
  space: i_k = 2..m_k-1  -> drop the first and the last function,
  time:  i_t = 2..m_t    -> drop the first function.
Reading c1: n_s = m - 2 (PAPER.md 285's "m_k - 1" is a typo).

W_t[i,j] = b_i(T) b_j(T) (PAPER.md 694).  Reading c9: physical time factors
K_t = K_t-hat / T, M_t = T M_t-hat, W_t unchanged (t = T tau, PAPER.md 246-249).
"""

import numpy as np

from .bspline import (open_uniform_knots, basis_values, basis_derivatives,
                      gauss_legendre_rule)


def full_matrices(knots, p, q=None):
    """Unconstrained (m x m) M, K, J, G by Gauss-Legendre with q points per element
    (default q = p + 1, exact for these degree-<=2p integrands; reading c6).

    Reading c17: evaluation, quadrature and summation run in 80-bit extended
    precision (np.longdouble) and the entries are rounded ONCE to fp64.  With
    plain fp64 assembly the last-ulp rounding of J perturbs the smallest
    eigenvalue of the pencil (J, M) -- the mode that dominates P^{-1} r -- by up
    to eps*lambda_max/lambda_min (measured 1e-8 relative at n_el=130, p=2),
    above the 1e-9 parity bar; correctly rounded entries remove that noise."""
    if q is None:
        q = p + 1
    ld = np.longdouble
    x, w = gauss_legendre_rule(knots, q, dtype=ld)
    B0 = basis_values(knots, p, x, dtype=ld)
    B1 = basis_derivatives(knots, p, 1, x, dtype=ld)
    B2 = basis_derivatives(knots, p, 2, x, dtype=ld) if p >= 2 else np.zeros_like(B0)
    M = (B0.T * w) @ B0
    K = (B1.T * w) @ B1
    J = (B2.T * w) @ B2
    G = (B2.T * w) @ B0
    return tuple(A.astype(np.float64) for A in (M, K, J, G))


def space_factors(n_el, p, knots=None):
    """Space pencil matrices on the Dirichlet-constrained basis i = 2..m-1.
    Returns dict with M, K, J, G, each (n_s x n_s), n_s = n_el + p - 2."""
    if knots is None:
        knots = open_uniform_knots(n_el, p, np.longdouble)
    M, K, J, G = full_matrices(knots, p)
    knots = np.asarray(knots, dtype=np.float64)
    s = slice(1, -1)
    return {"M": M[s, s], "K": K[s, s], "J": J[s, s], "G": G[s, s], "knots": knots}


def time_factors(n_el, p, T=1.0, knots=None):
    """Time matrices on the initial-condition-constrained basis i = 2..m.
    Returns dict with the parametric Kt_hat, Mt_hat (used by P) and the physical
    Kt, Mt, Wt (used by A), each (n_t x n_t), n_t = n_el + p - 1."""
    if knots is None:
        knots = open_uniform_knots(n_el, p, np.longdouble)
    M, K, _, _ = full_matrices(knots, p)
    knots = np.asarray(knots, dtype=np.float64)
    bT = basis_values(knots, p, [1.0])[0]
    s = slice(1, None)
    Mh, Kh = M[s, s], K[s, s]
    Wt = np.outer(bT, bT)[s, s]
    return {"Mt_hat": Mh, "Kt_hat": Kh, "Mt": T * Mh, "Kt": Kh / T, "Wt": Wt,
            "knots": knots}


def sizes(n_el, p):
    """(n_s, n_t) for uniform open knots (reading c1)."""
    return n_el + p - 2, n_el + p - 1
