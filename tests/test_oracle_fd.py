"""Pins for oracle/fd.py (Algorithm 1, PAPER.md 929-964): eigen invariants
(eq:eig_dec), Rayleigh-Ritz bounds against the continuous eigenproblems,
brute-force dense solves of P, special cases."""

import numpy as np
import pytest
import scipy.linalg

from oracle import univariate as uv, fd, bspline as bs


def _factors(n_els, p, n_el_t=None, p_t=None):
    space = [uv.space_factors(n, p) for n in n_els]
    tf = uv.time_factors(n_el_t if n_el_t is not None else n_els[0], p_t if p_t else p)
    return space, tf


@pytest.mark.parametrize("n_el,p", [(16, 2), (8, 3), (10, 6), (6, 8)])
def test_eig_invariants(n_el, p):
    """U^T M U = I, U^T J U = Lambda (PAPER.md 945)."""
    sf = uv.space_factors(n_el, p)
    tf = uv.time_factors(n_el, p)
    for K, M in ((sf["J"], sf["M"]), (tf["Kt_hat"], tf["Mt_hat"])):
        lam, U = fd.generalized_eig(K, M)
        n = len(lam)
        assert np.max(np.abs(U.T @ M @ U - np.eye(n))) < 1e-10
        assert np.max(np.abs(U.T @ K @ U - np.diag(lam))) < 1e-10 * lam.max()
        assert np.all(np.diff(lam) > 0) and lam[0] > 0


def test_rayleigh_ritz_limits():
    """Discrete eigenvalues of a conforming Galerkin pencil bound the continuous
    ones from above and converge to them: space pencil (J, M) -> (k pi)^4
    (int v'' w'' with v = 0 at both ends, eigenfunctions sin k pi x), time
    pencil (K_t, M_t) -> ((2k-1) pi / 2)^2 (v(0) = 0, natural at t = 1)."""
    ex_s = np.array([(k * np.pi) ** 4 for k in (1, 2, 3)])
    ex_t = np.array([((2 * k - 1) * np.pi / 2) ** 2 for k in (1, 2, 3)])
    errs = []
    for n_el in (8, 16, 32):
        sf, tf = uv.space_factors(n_el, 3), uv.time_factors(n_el, 3)
        ls, _ = fd.generalized_eig(sf["J"], sf["M"])
        lt, _ = fd.generalized_eig(tf["Kt_hat"], tf["Mt_hat"])
        assert np.all(ls[:3] >= ex_s * (1 - 1e-12))
        assert np.all(lt[:3] >= ex_t * (1 - 1e-10))
        errs.append((ls[0] - ex_s[0]) / ex_s[0])
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-6
    sf, tf = uv.space_factors(64, 3), uv.time_factors(64, 3)
    ls, _ = fd.generalized_eig(sf["J"], sf["M"])
    lt, _ = fd.generalized_eig(tf["Kt_hat"], tf["Mt_hat"])
    assert abs(ls[0] / np.pi ** 4 - 1) < 1e-7
    assert abs(lt[0] / (np.pi ** 2 / 4) - 1) < 1e-10


@pytest.mark.parametrize("n_els,p,n_el_t,seed", [
    ((16,), 2, 16, 0),          # BASELINE config 1 (272 DOFs)
    ((5, 3), 2, 4, 1),          # anisotropic d=2 (pins reading c3)
    ((3, 2, 4), 3, 2, 2),       # anisotropic d=3
    ((4, 4, 4), 2, 4, 3),
])
def test_fd_matches_dense_solve(n_els, p, n_el_t, seed):
    space, tf = _factors(n_els, p, n_el_t)
    P = fd.dense_P(space, tf)
    shape = (tf["Mt"].shape[0],) + tuple(f["M"].shape[0] for f in reversed(space))
    r = np.random.default_rng(seed).uniform(-1, 1, shape)
    z_dense = scipy.linalg.cho_solve(scipy.linalg.cho_factor(P), r.ravel())
    z = fd.fd_apply(r, fd.setup(space, tf))
    assert np.linalg.norm(z.ravel() - z_dense) / np.linalg.norm(z_dense) < 1e-9
    assert np.linalg.norm(P @ z.ravel() - r.ravel()) / np.linalg.norm(r) < 1e-9


def test_fd_dense_factorisation():
    """P = (U_t (x) U_s)^{-T} (Lambda_t (x) I + I (x) Lambda_s) (U_t (x) U_s)^{-1}
    (PAPER.md 950) assembled densely."""
    space, tf = _factors((4, 3), 2, 3)
    fdd = fd.setup(space, tf)
    U = fd.kron_list([fdd["U_t"]] + [fdd["U_s"][k] for k in reversed(range(2))])
    Ui = np.linalg.inv(U)
    D = np.diag(fd.divisor(fdd).ravel())
    np.testing.assert_allclose(Ui.T @ D @ Ui, fd.dense_P(space, tf), rtol=1e-9,
                               atol=1e-10 * np.abs(fd.dense_P(space, tf)).max())


def test_identity_special_case():
    """d=1, n_s = n_t = 2 with identity factor matrices: P = 2I, so z = r/2
    (SPEC.md 339)."""
    I = np.eye(2)
    space = [{"M": I, "J": I}]
    tf = {"Mt_hat": I, "Kt_hat": I}
    r = np.random.default_rng(5).uniform(-1, 1, (2, 2))
    np.testing.assert_allclose(fd.fd_apply(r, fd.setup(space, tf)), r / 2, rtol=1e-15)


def test_fd_symmetry_linearity():
    space, tf = _factors((6, 6, 6), 3, 6)
    fdd = fd.setup(space, tf)
    shape = (tf["Mt"].shape[0],) + (space[0]["M"].shape[0],) * 3
    rng = np.random.default_rng(7)
    r, s = rng.uniform(-1, 1, shape), rng.uniform(-1, 1, shape)
    Pr, Ps = fd.fd_apply(r, fdd), fd.fd_apply(s, fdd)
    assert abs(np.sum(r * Ps) - np.sum(s * Pr)) < 1e-12 * np.linalg.norm(r) * np.linalg.norm(Ps)
    np.testing.assert_allclose(fd.fd_apply(2 * r - 3 * s, fdd), 2 * Pr - 3 * Ps, rtol=1e-10,
                               atol=1e-13 * np.abs(Pr).max())
    assert np.all(fd.fd_apply(np.zeros(shape), fdd) == 0)


def test_mode_apply_kron_vec():
    """mode_apply along each axis equals the Kronecker matrix acting on the
    colex vector (eq:kron_vec, PAPER.md 646)."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((3, 4, 5))
    Cs = [rng.standard_normal((n, n)) for n in (3, 4, 5)]
    for axis in range(3):
        mats = [np.eye(n) for n in (3, 4, 5)]
        mats[axis] = Cs[axis]
        K = fd.kron_list(mats)
        np.testing.assert_allclose(fd.mode_apply(X, Cs[axis], axis).ravel(), K @ X.ravel(),
                                   rtol=1e-12, atol=1e-12)


def test_rank1_rows_match_full_fd():
    """The sampled rank-1 evaluator equals full Algorithm 1 on the same input."""
    space, tf = _factors((5, 4, 3), 3, 6)
    fdd = fd.setup(space, tf)
    shape = (tf["Mt"].shape[0],) + tuple(f["M"].shape[0] for f in reversed(space))
    rng = np.random.default_rng(11)
    facs = [rng.uniform(-1, 1, n) for n in shape]
    r = facs[0]
    for v in facs[1:]:
        r = np.multiply.outer(r, v)
    z = fd.fd_apply(r, fdd)
    rows = [(0, 0, 0), (shape[0] - 1, 2, 1), (3, shape[1] - 1, shape[2] - 1)]
    got = fd.fd_apply_rank1_rows(facs, fdd, rows)
    for j, idx in enumerate(rows):
        np.testing.assert_allclose(got[j], z[idx], rtol=1e-12, atol=1e-14 * np.abs(z).max())


@pytest.mark.parametrize("n_el,p", [(16, 2), (64, 3), (96, 2), (96, 4), (96, 8), (128, 6), (130, 2)])
def test_space_pencil_centrosymmetric(n_el, p):
    """Reading c25: on uniform open knots with Dirichlet conditions at both ends
    (PAPER.md 266-267, 1111-1112) the exact space matrices are centrosymmetric (b_i(1-x) =
    b_{n+1-i}(x)); the assembled fp64 ones are so to the last ulp, and the FD solution with the
    symmetrised pencil (J + RJR)/2, (M + RMR)/2 -- whose eigenbasis the library's split uses --
    differs from the oracle's by far less than the 1e-9 parity bar."""
    f = uv.space_factors(n_el, p)
    g = dict(f)
    for k in ("M", "K", "J"):
        A = f[k]
        R = A[::-1, ::-1]
        assert np.max(np.abs(A - R)) <= 4 * np.finfo(float).eps * np.abs(A).max()
        g[k] = 0.5 * (A + R)
    tf = uv.time_factors(6, p)
    r = np.random.default_rng(5).uniform(-1, 1, (tf["Mt_hat"].shape[0], f["M"].shape[0]))
    z = fd.fd_apply(r, fd.setup([f], tf))
    zs = fd.fd_apply(r, fd.setup([g], tf))
    assert np.linalg.norm(zs - z) / np.linalg.norm(z) <= 1e-12
