"""The graph-resident PCG loop (ls_tune LS_TUNE_PCG_GRAPH = 1, default on one GPU) against
the host-driven loop (= 0): the same kernels in the same order, so the iterates, the
iteration count and the status must agree bit for bit; plus the oracle PCG (reading c7)."""

import numpy as np
import pytest

import synth
from oracle import univariate as uv, fd, operator as op, pcg as opcg

pytestmark = pytest.mark.gpu

LS_TUNE_PCG_GRAPH = 5


def _solve(ctx, b, graph, **kw):
    ctx.tune(LS_TUNE_PCG_GRAPH, graph)
    x, st = ctx.pcg(b, **kw)
    return x.cpu().numpy(), st


@pytest.mark.parametrize("d,p,n_el,kind", [(2, 3, 16, 0), (3, 2, 8, 1), (3, 3, [5, 6, 7, 9], None),
                                           (3, 6, [8, 7, 9, 10], None), (2, 8, [20, 18, 22], 0)])
def test_graph_loop_equals_host_loop(d, p, n_el, kind):
    import torch
    import paper_1809_10026_b200 as ls
    ne = n_el if isinstance(n_el, list) else [n_el] * (d + 1)
    ctx = ls.Context(d, p, ne)
    b = ctx.rhs(kind) if kind is not None else torch.from_numpy(synth.residual(ctx.shape, 3)).cuda()
    xg, sg = _solve(ctx, b, 1)
    launches_g = ctx.launches
    xh, sh = _solve(ctx, b, 0)
    assert sg["status"] == sh["status"] == 0
    assert sg["iters"] == sh["iters"] and sg["iters"] > 1
    assert np.array_equal(xg, xh)
    assert sg["rel_res"] == sh["rel_res"]
    # the oracle PCG: same count, iterate within 1e-9
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    fdd = fd.setup(space, tf)
    x_ref, it, ok, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda r: fd.fd_apply(r, fdd),
                                b.cpu().numpy())
    assert ok and it == sg["iters"]
    assert np.linalg.norm(xg - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
    # a second solve reuses the instantiated graph
    xg2, sg2 = _solve(ctx, b, 1)
    assert np.array_equal(xg2, xg) and sg2["iters"] == sg["iters"]
    assert launches_g > 0


def test_graph_loop_noconv_and_max_iter():
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, 3, [6, 6, 6, 6])
    b = ctx.rhs(1)
    for mi in (1, 2, 5):
        xg, sg = _solve(ctx, b, 1, max_iter=mi)
        xh, sh = _solve(ctx, b, 0, max_iter=mi)
        assert sg["status"] == sh["status"] == ls.LS_ENOCONV
        assert sg["iters"] == sh["iters"] == mi
        assert np.array_equal(xg, xh)
    # tol change rebuilds the graph
    xg, sg = _solve(ctx, b, 1, tol=1e-4)
    xh, sh = _solve(ctx, b, 0, tol=1e-4)
    assert sg["iters"] == sh["iters"] and np.array_equal(xg, xh)


def test_graph_loop_mapped_domain_pg():
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(2, 3, [8, 8, 8], geometry=synth.quarter_annulus(), precond=ls.LS_PRECOND_PG)
    b = torch.from_numpy(synth.residual(ctx.shape, 4)).cuda()
    xg, sg = _solve(ctx, b, 1)
    xh, sh = _solve(ctx, b, 0)
    assert sg["status"] == 0 and sg["iters"] == sh["iters"] and np.array_equal(xg, xh)
