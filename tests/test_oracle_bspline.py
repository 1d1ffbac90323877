"""Pins for oracle/bspline.py against mathematics the paper fixes (Sec. 2.1,
PAPER.md 144-170) and an independent library implementation (scipy BSpline)."""

import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import bspline as bs

CASES = [(1, 1), (1, 2), (4, 2), (5, 3), (7, 4), (3, 6), (6, 8)]


@pytest.mark.parametrize("n_el,p", CASES)
def test_partition_of_unity(n_el, p):
    kn = bs.open_uniform_knots(n_el, p)
    x = np.random.default_rng(0).uniform(0, 1, 1000)
    x = np.concatenate([x, [0.0, 1.0], np.unique(kn)])
    B = bs.basis_values(kn, p, x)
    assert B.shape == (len(x), n_el + p)          # m = n_el + p functions
    assert np.all(B >= -1e-15)
    assert np.max(np.abs(B.sum(axis=1) - 1.0)) <= 1e-13


@pytest.mark.parametrize("n_el,p", CASES)
@pytest.mark.parametrize("r", [0, 1, 2])
def test_matches_scipy_bspline(n_el, p, r):
    """Independent evaluator (scipy's de Boor implementation), values and
    derivatives up to order 2, at random interior points."""
    if r > p:
        pytest.skip("derivative order above degree")
    kn = bs.open_uniform_knots(n_el, p)
    m = bs.n_functions(kn, p)
    x = np.random.default_rng(1).uniform(0, 1, 300)
    ours = bs.basis_derivatives(kn, p, r, x)
    for i in range(m):
        c = np.zeros(m)
        c[i] = 1.0
        ref = BSpline(kn, c, p, extrapolate=False)(x, nu=r)
        np.testing.assert_allclose(ours[:, i], ref, rtol=1e-12, atol=1e-10 * max(1, n_el) ** r)


@pytest.mark.parametrize("n_el,p", [(4, 2), (5, 3), (3, 5)])
def test_derivatives_finite_differences(n_el, p):
    kn = bs.open_uniform_knots(n_el, p)
    x = np.random.default_rng(2).uniform(0.01, 0.99, 50)
    h = 1e-5
    for r in (1, 2):
        lo = bs.basis_derivatives(kn, p, r - 1, x - h)
        hi = bs.basis_derivatives(kn, p, r - 1, x + h)
        fd = (hi - lo) / (2 * h)
        ex = bs.basis_derivatives(kn, p, r, x)
        # skip points within h of a knot (derivative jumps for r = p)
        near = np.min(np.abs(x[:, None] - np.unique(kn)[None, :]), axis=1) < 2 * h
        np.testing.assert_allclose(fd[~near], ex[~near], rtol=1e-5, atol=1e-5 * np.abs(ex).max())


@pytest.mark.parametrize("n_el,p", CASES)
def test_support_and_endpoints(n_el, p):
    kn = bs.open_uniform_knots(n_el, p)
    x = np.linspace(0, 1, 997)
    B = bs.basis_values(kn, p, x)
    for i in range(B.shape[1]):
        outside = (x < kn[i]) | (x > kn[i + p + 1])
        assert np.all(B[outside, i] == 0.0)
    # open knots interpolate the end points: only b_1(0) = 1 and b_m(1) = 1
    e0 = bs.basis_values(kn, p, [0.0])[0]
    e1 = bs.basis_values(kn, p, [1.0])[0]
    assert e0[0] == 1.0 and np.all(e0[1:] == 0.0)
    assert e1[-1] == 1.0 and np.all(e1[:-1] == 0.0)


@pytest.mark.parametrize("q", [1, 2, 3, 5])
def test_gauss_exactness(q):
    kn = bs.open_uniform_knots(3, 2)
    x, w = bs.gauss_legendre_rule(kn, q)
    assert np.all(w > 0)
    for deg in range(2 * q):
        assert abs(np.sum(w * x ** deg) - 1.0 / (deg + 1)) < 1e-14
