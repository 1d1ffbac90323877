"""Pins for oracle/univariate.py: hand-integrated worked values, closed forms of
the unconstrained matrices, and structure fixed by PAPER.md 266-267, 694,
738-757."""

import numpy as np
import pytest

from oracle import univariate as uv, bspline as bs
from conftest import golden


def test_worked_p2_one_element():
    g = golden("univariate_one_element.json")["p2"]
    sf = uv.space_factors(1, 2)
    tf = uv.time_factors(1, 2)
    for key, mat in (("M_s", sf["M"]), ("J_s", sf["J"]), ("K_s", sf["K"]), ("G_s", sf["G"]),
                     ("Mt", tf["Mt"]), ("Kt", tf["Kt"]), ("Wt", tf["Wt"])):
        np.testing.assert_allclose(mat, np.array(g[key]), rtol=1e-14, atol=1e-14, err_msg=key)


def test_worked_p1_time_one_element():
    g = golden("univariate_one_element.json")["p1_time"]
    tf = uv.time_factors(1, 1)
    for key in ("Mt", "Kt", "Wt"):
        np.testing.assert_allclose(tf[key], np.array(g[key]), rtol=1e-14, atol=1e-15, err_msg=key)


@pytest.mark.parametrize("n_el,p", [(1, 2), (4, 2), (6, 3), (5, 5), (3, 8)])
def test_unconstrained_closed_forms(n_el, p):
    kn = bs.open_uniform_knots(n_el, p)
    M, K, J, G = uv.full_matrices(kn, p)
    m = n_el + p
    assert M.shape == (m, m)
    # sum_ij M_ij = int (sum_i b_i)^2 = 1 ; row sums = int b_i = (xi_{i+p+1}-xi_i)/(p+1)
    assert abs(M.sum() - 1.0) < 1e-13
    ints = (kn[p + 1:p + 1 + m] - kn[:m]) / (p + 1)
    np.testing.assert_allclose(M.sum(axis=1), ints, rtol=1e-13)
    # sum_j b_j == 1 => rows of K, J and columns of G (G_ij = int b_i'' b_j) vanish
    assert np.max(np.abs(K.sum(axis=1))) < 1e-10 * np.abs(K).max()
    assert np.max(np.abs(J.sum(axis=1))) < 1e-10 * np.abs(J).max()
    assert np.max(np.abs(G.sum(axis=0))) < 1e-10 * np.abs(G).max()  # sum_i b_i'' = 0
    # banded: support of b_i is p+1 spans
    i, j = np.nonzero(np.abs(M) > 0)
    assert np.max(np.abs(i - j)) <= p


@pytest.mark.parametrize("n_el,p", [(4, 2), (8, 3), (5, 6)])
def test_constrained_structure(n_el, p):
    sf = uv.space_factors(n_el, p)
    tf = uv.time_factors(n_el, p)
    n_s, n_t = uv.sizes(n_el, p)
    assert sf["M"].shape == (n_s, n_s) and tf["Mt"].shape == (n_t, n_t)
    for A in (sf["M"], sf["K"], sf["J"], tf["Mt"], tf["Kt"]):
        np.testing.assert_allclose(A, A.T, atol=1e-13 * np.abs(A).max())
        assert np.linalg.eigvalsh(A).min() > 0  # SPD on the constrained spaces
    # integration by parts with b_j(0) = b_j(1) = 0: int b_i'' b_j = -int b_i' b_j'
    np.testing.assert_allclose(sf["G"], -sf["K"], atol=1e-11 * np.abs(sf["K"]).max())
    # W_t = e_{n_t} e_{n_t}^T (only the last time function is nonzero at T)
    W = np.zeros((n_t, n_t))
    W[-1, -1] = 1.0
    np.testing.assert_array_equal(tf["Wt"], W)


def test_time_scaling():
    """t = T tau: K_t = K_hat/T, M_t = T M_hat, W_t unchanged (reading c9)."""
    a = uv.time_factors(4, 3, T=1.0)
    b = uv.time_factors(4, 3, T=2.0)
    np.testing.assert_allclose(b["Kt"], a["Kt"] / 2)
    np.testing.assert_allclose(b["Mt"], a["Mt"] * 2)
    np.testing.assert_array_equal(b["Wt"], a["Wt"])
