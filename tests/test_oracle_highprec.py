"""Pins for the extended-precision setup of reading c17 against
high-precision references that share nothing with the oracle's LAPACK + Ogita-Aishima path:

* oracle/highprec.py's EXACT rational univariate matrices (closed-form integration of the
  Cox-de Boor pieces, PAPER.md 148-152, 738-757) are themselves pinned to the hand-integrated
  worked example and to exact closed forms;
* the oracle's 80-bit quadrature assembly equals those exact matrices rounded once to fp64
  (within 2 ulp per entry; assembly noise <= 1e-16 of the row scale on exact zeros);
* tests/golden/eig_mpmath.json (tools/make_golden_eig.py: mpmath inertia bisection, 40 digits)
  pins the oracle's eigenvalues (eq:eig_dec, PAPER.md 942-945) to <= 1e-13 relative and
  z = P^{-1} r (Algorithm 1, PAPER.md 947-962) to <= 1e-12 against a banded Cholesky of the
  Kronecker-assembled P in mpmath.
"""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from conftest import golden
from oracle import highprec as hp, univariate as uv, fd
import synth

G = golden("eig_mpmath.json")


def _np(A):
    return np.array(hp.round_fp64(A))


# ----------------------------------------------------------- the exact reference itself

def test_exact_matrices_worked_example():
    """p = 2, one element: M_s = 2/15, J_s = 16, M_t = [[2/15, 1/10], [1/10, 1/5]],
    K_t = [[4/3, -2/3], [-2/3, 4/3]] (tests/golden/univariate_one_element.json derivation)."""
    J, M = hp.space_pencil(1, 2)
    assert J == [[Fraction(16)]] and M == [[Fraction(2, 15)]]
    Kt, Mt = hp.time_pencil(1, 2)
    assert Mt == [[Fraction(2, 15), Fraction(1, 10)], [Fraction(1, 10), Fraction(1, 5)]]
    assert Kt == [[Fraction(4, 3), Fraction(-2, 3)], [Fraction(-2, 3), Fraction(4, 3)]]


@pytest.mark.parametrize("n_el,p", [(1, 3), (5, 2), (7, 4), (4, 8)])
def test_exact_matrices_closed_forms(n_el, p):
    """Exactly: sum_ij M_ij = int 1 = 1; row sums of M = int b_i = (xi_{i+p+1} - xi_i)/(p+1);
    rows of K and J sum to 0 (partition of unity, PAPER.md 148-152); symmetry."""
    M, K, J = hp.exact_full_matrices(n_el, p)
    kn = hp.uniform_open_knots(n_el, p)
    m = n_el + p
    assert sum(sum(r) for r in M) == 1
    for i in range(m):
        assert sum(M[i]) == (kn[i + p + 1] - kn[i]) / (p + 1)
        assert sum(K[i]) == 0 and sum(J[i]) == 0
        for j in range(m):
            assert M[i][j] == M[j][i] and K[i][j] == K[j][i] and J[i][j] == J[j][i]
            if abs(i - j) > p:
                assert M[i][j] == K[i][j] == J[i][j] == 0


def test_bisection_matches_dense_mp_eigensolver():
    """The inertia bisection equals mpmath's dense symmetric eigensolver on the
    Cholesky-reduced pencil L^{-1} J L^{-T} (a different algorithm) on a small case."""
    J, M = hp.space_pencil(10, 3)
    n = len(J)
    ks = list(range(1, n + 1))
    with mpmath.workdps(40):
        Jm, Mm = mpmath.matrix([[mpmath.mpf(x.numerator) / x.denominator for x in r] for r in J]), \
            mpmath.matrix([[mpmath.mpf(x.numerator) / x.denominator for x in r] for r in M])
        L = mpmath.cholesky(Mm)
        Li = mpmath.inverse(L)
        C = Li * Jm * Li.T
        ev = sorted(mpmath.eigsy(C, eigvals_only=True))
        bi = hp.eig_bisect(J, M, ks, dps=40, rel=mpmath.mpf(10) ** -30)
        for a, b in zip(ev, bi):
            assert abs(a / b - 1) < mpmath.mpf(10) ** -25


# ----------------------------------------------------------- the oracle against it

@pytest.mark.parametrize("n_el,p", [(16, 2), (130, 2), (64, 3), (65, 3), (128, 6), (96, 8)])
def test_oracle_assembly_is_exact_rounded(n_el, p):
    """Reading c17: 80-bit assembly rounded once == the exact integrals rounded to fp64,
    up to 2 ulp (double rounding) and 1e-16 of the row scale (entries that are exactly 0)."""
    sf, tf = uv.space_factors(n_el, p), uv.time_factors(n_el, p)
    J, M = hp.space_pencil(n_el, p)
    Kt, Mt = hp.time_pencil(n_el, p)
    for ours, ex in ((sf["J"], J), (sf["M"], M), (tf["Kt_hat"], Kt), (tf["Mt_hat"], Mt)):
        R = _np(ex)
        tol = np.maximum(2 * np.spacing(np.abs(R)), 1e-16 * np.abs(R).max(axis=1, keepdims=True))
        assert np.all(np.abs(ours - R) <= tol)
        assert np.mean(ours == R) > 0.9


def _golden_eig():
    return [(e["n_el"], e["p"], e["pencil"]) for e in G["eig"]]


@pytest.mark.parametrize("n_el,p,pencil", _golden_eig())
def test_oracle_eigenvalues_vs_mpmath(n_el, p, pencil):
    """eq:eig_dec (PAPER.md 942-945): the oracle's generalized_eig on the correctly rounded
    pencil reproduces the 40-digit eigenvalues of that same pencil to 1e-13 relative
    (lambda_1..5 and lambda_max), and its eigenvalues of its own assembled pencil are
    within the fp64 rounding of the pencil (5e-10) of the EXACT pencil's."""
    e = next(e for e in G["eig"] if (e["n_el"], e["p"], e["pencil"]) == (n_el, p, pencil))
    A, B = hp.space_pencil(n_el, p) if pencil == "space" else hp.time_pencil(n_el, p)
    lam, U = fd.generalized_eig(_np(A), _np(B))
    idx = [k - 1 for k in e["k"]]
    ref = np.array([float(mpmath.mpf(v)) for v in e["fp64_pencil"]])
    np.testing.assert_allclose(lam[idx], ref, rtol=1e-13, atol=0)
    if pencil == "space":
        ours = uv.space_factors(n_el, p)
        lam2, _ = fd.generalized_eig(ours["J"], ours["M"])
    else:
        ours = uv.time_factors(n_el, p)
        lam2, _ = fd.generalized_eig(ours["Kt_hat"], ours["Mt_hat"])
    exact = np.array([float(mpmath.mpf(v)) for v in e["exact"]])
    np.testing.assert_allclose(lam2[idx], exact, rtol=5e-10, atol=0)


def test_plain_lapack_misses_the_bar():
    """Teeth of the pin above: fp64 LAPACK alone (refine=0) is > 1e-12 off the 40-digit
    smallest eigenvalue of the p = 6, n_el = 128 space pencil (reading c17)."""
    e = next(e for e in G["eig"] if (e["n_el"], e["p"], e["pencil"]) == (128, 6, "space"))
    A, B = hp.space_pencil(128, 6)
    lam0, _ = fd.generalized_eig(_np(A), _np(B), refine=0)
    ref = float(mpmath.mpf(e["fp64_pencil"][0]))
    assert abs(lam0[0] / ref - 1) > 1e-12


@pytest.mark.parametrize("i", range(len(G["fd"])))
def test_oracle_fd_apply_vs_mpmath_dense_solve(i):
    """Algorithm 1 (PAPER.md 947-962) == P^{-1} r by a 40-digit banded Cholesky of the
    Kronecker-assembled P (PAPER.md 733, 752-757) to 1e-12 relative: anisotropic d = 2, 3
    grids (exact pencils, the oracle's own assembly) and d = 1 grids with n_el = 130 / 128
    in space, where fp64 LAPACK alone is ~5e-9 off (correctly rounded pencils on both sides)."""
    c = G["fd"][i]
    ne, p = c["n_el"], c["p"]
    d = len(ne) - 1
    shape = tuple(c["shape"])
    r = synth.residual(shape, c["seed"])
    if c["pencil"] == "exact":
        fdd = fd.setup([uv.space_factors(n, p) for n in ne[:d]], uv.time_factors(ne[d], p))
    else:
        sp = [hp.space_pencil(n, p) for n in ne[:d]]
        Kt, Mt = hp.time_pencil(ne[d], p)
        fdd = fd.setup([{"J": _np(J), "M": _np(M)} for J, M in sp], {"Kt_hat": _np(Kt), "Mt_hat": _np(Mt)})
    z = fd.fd_apply(r, fdd)
    ref = np.array([float(v) for v in c["z"]]).reshape(shape)
    assert np.linalg.norm(z - ref) / np.linalg.norm(ref) <= 1e-12
