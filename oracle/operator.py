"""The least-squares system matrix A (oracle; test infrastructure).

apply_A: y = A x with (eq:A_kron, PAPER.md 686-703)
    A = K_t (x) M_s + M_t (x) J_s + W_t (x) L_s,
    [M_s]_ij = int B_i B_j,  [L_s]_ij = int grad B_i . grad B_j,
    [J_s]_ij = int Lap B_i Lap B_j.
On the identity-mapped unit cube (the configs of BASELINE.json) B_i is a
product of univariate B-splines, so by direct expansion of the integrands
    M_s = M_d (x) ... (x) M_1,
    L_s = sum_k K_(k)                       (K in slot k, M elsewhere),
    J_s = sum_k J_(k) + sum_{k != l} G_(k) G^T_(l)
with G[i,j] = int b_i'' b_j (Lap B = sum_k d_kk B; the k != l cross terms are
int b''_{i_k} b_{j_k} * int b_{i_l} b''_{j_l}).  Each Kronecker term is applied
one axis at a time.  This is NOT the sum-factorisation the CUDA path uses.

dense_A_original_form: [A]_ij = A(B_i, B_j) with the ORIGINAL bilinear form
(PAPER.md 406, Sec. 3.1)
    A(v,w) = int int (d_t v d_t w + Lap v Lap w - d_t v Lap w - Lap v d_t w),
by direct space-time Gauss quadrature of the tensor basis.  It does not use
eq:equivalent_A, eq:A_kron or integration by parts; tiny grids only.
"""

import numpy as np

from .fd import mode_apply
from .bspline import basis_values, basis_derivatives, gauss_legendre_rule


def apply_kron(x, time_mat, space_mats):
    """(time_mat (x) space_mats[d-1] (x) ... (x) space_mats[0]) x, where
    space_mats[k-1] acts on direction k (axis d+1-k) and time_mat on axis 0.
    A ``None`` entry means identity."""
    d = len(space_mats)
    y = x
    for k in range(1, d + 1):
        if space_mats[k - 1] is not None:
            y = mode_apply(y, space_mats[k - 1], d + 1 - k)
    if time_mat is not None:
        y = mode_apply(y, time_mat, 0)
    return y


def apply_A(x, space, time):
    """y = A x, matrix-free from the univariate factors (eq:A_kron)."""
    d = len(space)
    M = [f["M"] for f in space]
    y = apply_kron(x, time["Kt"], M)                       # K_t (x) M_s
    for k in range(d):                                     # M_t (x) J_s
        mats = list(M)
        mats[k] = space[k]["J"]
        y = y + apply_kron(x, time["Mt"], mats)
        for l in range(d):
            if l == k:
                continue
            mats = list(M)
            mats[k] = space[k]["G"]
            mats[l] = space[l]["G"].T
            y = y + apply_kron(x, time["Mt"], mats)
    for k in range(d):                                     # W_t (x) L_s
        mats = list(M)
        mats[k] = space[k]["K"]
        y = y + apply_kron(x, time["Wt"], mats)
    return y


def _tables(knots, p, drop_first, drop_last, q):
    x, w = gauss_legendre_rule(knots, q)
    sl = slice(1 if drop_first else 0, -1 if drop_last else None)
    B0 = basis_values(knots, p, x)[:, sl]
    B1 = basis_derivatives(knots, p, 1, x)[:, sl]
    B2 = basis_derivatives(knots, p, 2, x)[:, sl] if p >= 2 else np.zeros_like(B0)
    return w, B0, B1, B2


def _kron_rows(mats):
    out = np.ones((1, 1))
    for A in mats:
        out = np.kron(out, A)
    return out


def dense_A_original_form(space_knots, p_s, time_knots, p_t, T=1.0):
    """Dense A from the original least-squares form (PAPER.md 406) by tensor
    Gauss quadrature (p+1 points per element per direction: exact).
    space_knots[k-1] is direction k.  Returns the (N x N) matrix in colex order."""
    d = len(space_knots)
    sp = [_tables(kn, p_s, True, True, p_s + 1) for kn in space_knots]
    wt, T0, T1, _ = _tables(time_knots, p_t, True, False, p_t + 1)
    # physical time t = T tau: d_t = (1/T) d_tau, dt = T dtau (PAPER.md 246-249)
    T1 = T1 / T
    wt = wt * T
    # evaluation matrices (points x DOFs); slowest factor first: time, d, ..., 1
    order = list(reversed(range(d)))
    W = _kron_rows([wt[None, :]] + [sp[k][0][None, :] for k in order]).ravel()
    Dt = _kron_rows([T1] + [sp[k][1] for k in order])
    Lap = np.zeros_like(Dt)
    for kk in range(d):
        Lap += _kron_rows([T0] + [sp[k][3] if k == kk else sp[k][1] for k in order])
    WD, WL = Dt * W[:, None], Lap * W[:, None]
    return Dt.T @ WD + Lap.T @ WL - Dt.T @ WL - Lap.T @ WD


def dense_A_from_factors(space, time):
    """Dense A by Kronecker assembly of the factors (eq:A_kron); used only to
    compare two independent constructions on tiny grids."""
    d = len(space)
    N_s = int(np.prod([f["M"].shape[0] for f in space]))
    n_t = time["Mt"].shape[0]
    I = np.eye(N_s * n_t)
    cols = [apply_A(I[:, j].reshape((n_t,) + tuple(f["M"].shape[0] for f in reversed(space))),
                    space, time).ravel() for j in range(N_s * n_t)]
    return np.array(cols).T
