"""Pins of oracle/error.py: the closed-form ||f||^2 against quadrature, and the
least-squares identity J(c) = ||f||^2 - 2 b.c + c.A c (PAPER.md 392-410) against the
direct quadrature of the residual for random coefficient vectors."""

import numpy as np
import pytest

from oracle import bspline as bs, error as oerr, operator as op, rhs as orhs
from oracle.bspline import gauss_legendre_rule


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("d", [1, 2, 3])
def test_f_norm2_closed_form(kind, d):
    g, s = orhs.forcing(kind, d)
    x, w = gauss_legendre_rule(bs.open_uniform_knots(8, 2), 12)
    sx = float(np.sum(w * s(x) ** 2))
    gt = float(np.sum(w * g(x) ** 2))
    assert abs(oerr.f_norm2(kind, d) - sx ** d * gt) <= 1e-13 * oerr.f_norm2(kind, d)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("d,ps,pt,ne", [(1, 2, 2, [3, 4]), (1, 3, 2, [2, 3]), (2, 2, 3, [2, 3, 2])])
def test_ls_identity(kind, d, ps, pt, ne):
    sk = [bs.open_uniform_knots(n, ps) for n in ne[:d]]
    tk = bs.open_uniform_knots(ne[d], pt)
    A = op.dense_A_original_form(sk, ps, tk, pt)
    b = orhs.rhs(kind, sk, ps, tk, pt)
    c = np.random.default_rng(5).uniform(-1, 1, b.shape)
    J = oerr.ls_functional_quadrature(c, kind, sk, ps, tk, pt)
    ident = oerr.f_norm2(kind, d) - 2.0 * float(np.vdot(b, c)) + float(c.ravel() @ A @ c.ravel())
    assert abs(J - ident) <= 1e-9 * max(J, 1.0)
