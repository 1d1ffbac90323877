"""Pins for oracle/pcg.py: the paper's Table 1 iteration counts (PAPER.md
1187-1191), exact-arithmetic properties of CG, robustness in p."""

import numpy as np
import pytest
import scipy.linalg

from oracle import univariate as uv, operator as op, fd, rhs, pcg, bspline as bs
from conftest import golden


def _cube_solve(n_el, p, d=3, kind=1, tol=1e-8):
    sf, tf = uv.space_factors(n_el, p), uv.time_factors(n_el, p)
    space = [sf] * d
    fdd = fd.setup(space, tf)
    kn = bs.open_uniform_knots(n_el, p)
    b = rhs.rhs(kind, [kn] * d, p, kn, p)
    x, it, conv, hist = pcg.pcg(lambda v: op.apply_A(v, space, tf),
                                lambda v: fd.fd_apply(v, fdd), b, tol=tol)
    true_rel = np.linalg.norm(b - op.apply_A(x, space, tf)) / np.linalg.norm(b)
    return it, conv, true_rel


@pytest.mark.parametrize("n_el", [8, 16])
@pytest.mark.parametrize("pi", [0, 1, 2, 3])
def test_table1_iterations(n_el, pi):
    g = golden("table1_iterations.json")
    p = g["p"][pi]
    it, conv, true_rel = _cube_solve(n_el, p)
    assert conv
    assert it == g["iterations"][str(n_el)][pi]
    assert true_rel <= 10 * 1e-8


def test_config2_iterations():
    """BASELINE config 2 (d=2, p=3, n_el=64, f = sin sin e^t): bounded
    iteration count in the Table 1 range (survey oracle run: 10)."""
    it, conv, true_rel = _cube_solve(64, 3, d=2, kind=0)
    assert conv and 9 <= it <= 13 and true_rel < 1e-7


def test_robust_in_p():
    """Thm spec_est: iterations bounded independently of p (d=3, n_el=8,
    p in {2,4,8}); spread <= 4 (SPEC.md 414)."""
    its = [_cube_solve(8, p)[0] for p in (2, 4, 8)]
    assert max(its) - min(its) <= 4 and max(its) <= 15


def _random_spd(n, seed):
    rng = np.random.default_rng(seed)
    Q = rng.standard_normal((n, n))
    return Q @ Q.T + n * np.eye(n)


def test_cg_solves_small_spd_exactly():
    A = _random_spd(16, 0)
    b = np.random.default_rng(1).standard_normal(16)
    x, it, conv, _ = pcg.pcg(lambda v: A @ v, lambda v: v, b, tol=1e-13, max_iter=100)
    assert conv and it <= 16 + 4
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-10)


def test_exact_preconditioner_one_iteration():
    A = _random_spd(20, 2)
    Ainv = np.linalg.inv(A)
    b = np.random.default_rng(3).standard_normal(20)
    x, it, conv, _ = pcg.pcg(lambda v: A @ v, lambda v: Ainv @ v, b)
    assert conv and it == 1


def test_cg_minimises_energy_over_krylov():
    """Iterate k of CG minimises the A-norm error over K_k(A, b): compare with
    a dense least-squares projection onto an explicit Krylov basis."""
    A = _random_spd(12, 4)
    b = np.random.default_rng(5).standard_normal(12)
    xs = {}
    pcg.pcg(lambda v: A @ v, lambda v: v, b, tol=0.0, max_iter=4,
            callback=lambda k, x, r: xs.__setitem__(k, x.copy()))
    L = np.linalg.cholesky(A)
    xstar = np.linalg.solve(A, b)
    for k in (1, 2, 3, 4):
        Kb = np.stack([np.linalg.matrix_power(A, j) @ b for j in range(k)], axis=1)
        Qk, _ = np.linalg.qr(Kb)
        c = np.linalg.lstsq(L.T @ Qk, L.T @ xstar, rcond=None)[0]
        np.testing.assert_allclose(xs[k], Qk @ c, rtol=1e-8, atol=1e-10)


def test_zero_rhs():
    x, it, conv, _ = pcg.pcg(lambda v: v, lambda v: v, np.zeros(5))
    assert it == 0 and conv and np.all(x == 0)
