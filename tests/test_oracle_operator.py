"""Pins for oracle/operator.py and oracle/rhs.py: direct quadrature of the
original bilinear form (PAPER.md 406), SPD-ness (PAPER.md 710), Galerkin
exactness for a solution inside the discrete space, and the spectral
robustness of P^{-1}A (Thm spec_est, PAPER.md 905-911)."""

import numpy as np
import pytest
import scipy.linalg

from oracle import univariate as uv, operator as op, fd, rhs, bspline as bs


def _setup(n_els, p, n_el_t, p_t=None, T=1.0):
    p_t = p_t or p
    space = [uv.space_factors(n, p) for n in n_els]
    tf = uv.time_factors(n_el_t, p_t, T=T)
    kn_s = [bs.open_uniform_knots(n, p) for n in n_els]
    kn_t = bs.open_uniform_knots(n_el_t, p_t)
    return space, tf, kn_s, kn_t, p_t


@pytest.mark.parametrize("n_els,p,n_el_t,p_t,T", [
    ((4,), 2, 4, None, 1.0),
    ((3,), 3, 5, 2, 1.0),        # p_s = p_t + 1 (Fig. 2b configuration)
    ((3, 2), 2, 3, None, 1.0),
    ((2, 3), 3, 2, None, 2.5),   # T != 1 (reading c9)
    ((2, 1, 2), 2, 2, None, 1.0),
])
def test_matrix_free_A_equals_original_form(n_els, p, n_el_t, p_t, T):
    space, tf, kn_s, kn_t, p_t = _setup(n_els, p, n_el_t, p_t, T)
    A_orig = op.dense_A_original_form(kn_s, p, kn_t, p_t, T=T)
    A_mf = op.dense_A_from_factors(space, tf)
    assert np.max(np.abs(A_mf - A_orig)) <= 1e-12 * np.abs(A_orig).max()
    np.testing.assert_allclose(A_orig, A_orig.T, atol=1e-12 * np.abs(A_orig).max())
    scipy.linalg.cholesky(A_orig)  # SPD (Lemma coer, PAPER.md 435-454)


def test_galerkin_exactness():
    """u = x(1-x) y(1-y) t lies in V_h (p_s >= 2, u = 0 on the boundary and at
    t = 0), so the least-squares minimiser (PAPER.md 396) is u itself:
    A c_u = b(f) with f = d_t u - Lap u."""
    p, n_el = 3, 3
    space, tf, kn_s, kn_t, _ = _setup((n_el, n_el), p, n_el)
    q = lambda x: x * (1 - x)
    one = lambda x: np.ones_like(x)
    # f = x(1-x)y(1-y) + 2t y(1-y) + 2t x(1-x)   (slot order [s_1, s_2])
    terms = [(one, [q, q]),
             (lambda t: 2 * t, [q, one]),
             (lambda t: 2 * t, [one, q])]
    b = rhs.rhs_separable(terms, kn_s, p, kn_t, p)

    def coeffs(knots, p_, fn, sl):  # L2 projection (exact: fn in the span)
        x, w = bs.gauss_legendre_rule(knots, p_ + 3)
        B = bs.basis_values(knots, p_, x)[:, sl]
        return np.linalg.solve((B.T * w) @ B, (fn(x) * w) @ B)

    cs = coeffs(kn_s[0], p, q, slice(1, -1))
    ct = coeffs(kn_t, p, lambda t: t, slice(1, None))
    c = np.multiply.outer(np.multiply.outer(ct, cs), cs)
    Ac = op.apply_A(c, space, tf)
    assert np.linalg.norm(Ac - b) / np.linalg.norm(b) < 1e-12


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("n_els,p,n_el_t", [((3,), 2, 4), ((2, 3), 3, 2)])
def test_rhs_separable_vs_dense_quadrature(kind, n_els, p, n_el_t):
    _, _, kn_s, kn_t, _ = _setup(n_els, p, n_el_t)
    a = rhs.rhs(kind, kn_s, p, kn_t, p)
    b = rhs.rhs_dense_quadrature(kind, kn_s, p, kn_t, p)
    np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-13 * np.abs(b).max())


def test_spectral_robustness():
    """theta <= lambda(P^{-1} A) <= Theta independent of h and p (Thm spec_est,
    PAPER.md 905-911): over n_el in {2,4}, p in {2,3,4} (d = 2) the extremes
    vary by less than a factor 2 (SPEC.md 363)."""
    lo, hi = [], []
    for n_el in (2, 4):
        for p in (2, 3, 4):
            space, tf, _, _, _ = _setup((n_el, n_el), p, n_el)
            A = op.dense_A_from_factors(space, tf)
            P = fd.dense_P(space, tf)
            ev = scipy.linalg.eigh(A, P, eigvals_only=True)
            lo.append(ev.min())
            hi.append(ev.max())
    assert max(lo) / min(lo) < 2 and max(hi) / min(hi) < 2
    assert min(lo) > 0.1 and max(hi) < 10
