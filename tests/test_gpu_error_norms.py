"""GPU parity and convergence of ls_error_norms: the eight space-time
integrals of e = u - u_h and of u against oracle/error.py's direct quadrature (same rule,
reading c24), on the cube (kind 1, d = 1..3) and on the quarter annulus (kind 2, the Fig. 2
setting, PAPER.md 1128-1139); V_0 / H^1 / L^2 rates of the PCG solution."""
import numpy as np
import pytest

import synth
from oracle import error as oe

pytestmark = pytest.mark.gpu


def _ctx(d, p, ne, geo=None):
    import paper_1809_10026_b200 as ls
    if geo is None:
        return ls.Context(d, p, ne)
    return ls.Context(d, p, ne, geometry=geo, precond=ls.LS_PRECOND_PG)


def _cmp(got, ref):
    g = np.array([got[k] for k in ("e_L2", "e_dt", "e_grad", "e_lap", "u_L2", "u_dt", "u_grad", "u_lap")])
    scale = np.concatenate([ref[4:], ref[4:]])
    assert np.all(np.abs(g - ref) <= 1e-10 * scale + 1e-300), (g, ref)


@pytest.mark.parametrize("d,p,ne", [(1, 2, [5, 6]), (1, (3, 2), [4, 7]), (2, 3, [4, 5, 6]), (3, 2, [3, 4, 3, 5]),
                                    (3, 4, [2, 3, 2, 2])])
@pytest.mark.parametrize("which", ["random", "solution"])
def test_error_norms_cube_parity(d, p, ne, which):
    import torch
    ctx = _ctx(d, p, ne)
    if which == "random":
        x = torch.from_numpy(synth.residual(ctx.shape, 3)).cuda()
    else:
        x, st = ctx.pcg(ctx.rhs(1), tol=1e-10)
    got = ctx.error_norms(1, x)
    ps, pt = (p, p) if isinstance(p, int) else p
    ref = oe.error_norms(x.cpu().numpy(), 1, synth.affine_box([1.0] * d), ne[:d], ps, ne[d], pt)
    _cmp(got, ref)


@pytest.mark.parametrize("p,ne", [(2, [5, 4, 6]), (3, [6, 5, 4])])
def test_error_norms_annulus_parity(p, ne):
    import torch
    geo = synth.quarter_annulus()
    ctx = _ctx(2, p, ne, geo)
    x = torch.from_numpy(synth.residual(ctx.shape, 4)).cuda()
    _cmp(ctx.error_norms(2, x), oe.error_norms(x.cpu().numpy(), 2, geo, ne[:2], p, ne[2], p))
    x, st = ctx.pcg(ctx.rhs(2), tol=1e-10)
    _cmp(ctx.error_norms(2, x), oe.error_norms(x.cpu().numpy(), 2, geo, ne[:2], p, ne[2], p))


def _rates(errs):
    e = np.array(errs)
    return np.log2(e[:-1] / e[1:])


@pytest.mark.parametrize("p", [2, 3, 4])
def test_error_rates_cube_d3(p):
    """d = 3 (the 4D hypercube of configs 3-5), u of PAPER.md 1166: V_0 ~ h^(p-1)
    (Thm teo:a-priori), H^1 ~ h^p, L^2 ~ h^(p+1) for p >= 3 (PAPER.md 1136-1139)."""
    errs = []
    for n in (4, 8, 16):
        ctx = _ctx(3, p, [n] * 4)
        x, st = ctx.pcg(ctx.rhs(1), tol=1e-12)
        e = ctx.error_norms(1, x)
        errs.append((e["rel_V0"], e["rel_L2"], e["rel_H1"]))
    r = _rates(errs)[-1]
    assert abs(r[0] - (p - 1)) < 0.25 and abs(r[2] - p) < 0.3, (errs, r)
    if p >= 3:
        assert abs(r[1] - (p + 1)) < 0.35, (errs, r)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_error_rates_annulus(p):
    """Fig. 2 (PAPER.md 1128-1139): quarter annulus, p_s = p_t = p."""
    geo = synth.quarter_annulus()
    errs = []
    for n in (8, 16, 32):
        ctx = _ctx(2, p, [n] * 3, geo)
        x, st = ctx.pcg(ctx.rhs(2), tol=1e-12, max_iter=2000)
        e = ctx.error_norms(2, x)
        errs.append((e["rel_V0"], e["rel_L2"], e["rel_H1"]))
    r = _rates(errs)[-1]
    assert abs(r[0] - (p - 1)) < 0.25 and abs(r[2] - p) < 0.3, (errs, r)
    if p >= 3:
        assert abs(r[1] - (p + 1)) < 0.35, (errs, r)


def test_error_norms_unsupported_kinds():
    import torch
    import paper_1809_10026_b200 as ls
    ctx = _ctx(2, 2, [3, 3, 3])
    x = torch.zeros(ctx.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ls.LSError):
        ctx.error_norms(2, x)
    cg = _ctx(2, 2, [3, 3, 3], synth.quarter_annulus())
    with pytest.raises(ls.LSError):
        cg.error_norms(1, x)
