"""Host logic of the P^G setup (ls_pg_factors, no GPU): the library's separable fit of the
midpoint coefficients (alternating sweeps, reading c21) against the oracle's dense least
squares, compared through gauge-invariant quantities, and its weighted factors through the
Kronecker sum Pbar^G (PAPER.md 1026-1045)."""

import warnings

import numpy as np
import pytest

import synth
from oracle import geo_precond as GP, univariate as uv

warnings.filterwarnings("ignore", category=DeprecationWarning)


def _outer(vs):
    out = vs[-1]
    for v in reversed(vs[:-1]):
        out = np.multiply.outer(out, v)
    return out


@pytest.mark.parametrize("name,ne,p", [("annulus2d", [6, 5], 3), ("annulus3d", [3, 4, 2], 2),
                                       ("affine", [3, 2, 4], 2)])
def test_pg_fit_and_factors_match_oracle(name, ne, p):
    import paper_1809_10026_b200 as ls
    geo = synth.GEOMETRIES[name]() if name != "affine" else synth.affine_box([2.0, 0.5, 1.5])
    d = geo["d"]
    mu, om, Mw, Jw, res = ls.pg_factors(geo, p, ne)
    c_tau, c_k = GP.midpoint_coefficients(geo, ne)
    mu_o, om_o = GP.separable_fit(c_tau, c_k)
    # gauge-invariant: the reconstructed c_tau and c_k
    assert np.allclose(_outer(mu), _outer(mu_o), rtol=1e-12)
    for k in range(d):
        rec = _outer([om[j] if j == k else mu[j] for j in range(d)])
        rec_o = _outer([om_o[j] if j == k else mu_o[j] for j in range(d)])
        assert np.allclose(rec, rec_o, rtol=1e-12)
    # the weighted factors: Pbar^G = K_t (x) (x)M^G + M_t (x) sum J^G (x) M^G is gauge invariant
    tf = uv.time_factors(2, p)
    sp_lib = [{"M": Mw[k], "J": Jw[k]} for k in range(d)]
    sp_ora = [GP.weighted_space_factors(ne[k], p, mu_o[k], om_o[k]) for k in range(d)]

    def pbar(space):
        def kron(mats):
            out = np.ones((1, 1))
            for A in mats:
                out = np.kron(out, A)
            return out
        P = kron([tf["Kt_hat"]] + [space[k]["M"] for k in reversed(range(d))])
        for kk in range(d):
            P = P + kron([tf["Mt_hat"]] + [space[k]["J"] if k == kk else space[k]["M"] for k in reversed(range(d))])
        return P

    P1, P2 = pbar(sp_lib), pbar(sp_ora)
    assert np.abs(P1 - P2).max() <= 1e-11 * np.abs(P2).max()
    if name == "affine":
        assert res < 1e-13


def test_pg_factors_rejects_folded_map():
    import paper_1809_10026_b200 as ls
    geo = dict(synth.quarter_annulus())
    c = geo["ctrl"].copy()
    c[0] = [3.0, 3.0]           # a corner dragged across the domain: det J_F changes sign
    geo["ctrl"] = c
    with pytest.raises(ls.LSError):
        ls.pg_factors(geo, 2, [4, 4])
