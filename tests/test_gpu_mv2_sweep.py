"""The register-sweep plane pass of the v2 matvec (p = 2, d = 3; ls_tune LS_TUNE_MV2_SWEEP = 16,
default 1; matvec2_kernels.cuh mv_sweep_kernel): directions 2 and 1 of eq:A_kron (PAPER.md
686-703) with one warp per (t, i3) plane and CW = ceil(n_1 / 32) columns per lane.  Same algebra
as the shared-memory plane pass (knob 16 = 0), so both must match the oracle's A x to 1e-12 and
each other to rounding.  Covered: CW = 2, 3, 4 (n_1 = 33 .. 128) at both ends, odd / even n_1,
n_2 shorter than the stencil ring and than 2p + 1, boundary rows and columns, per-rank slab rows
(ls_matvec_slab), the PCG solve through the graph."""

import numpy as np
import pytest

import synth
from oracle import univariate as uv, operator as op

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


CASES = [[31, 5, 4, 6], [32, 7, 5, 5], [62, 9, 3, 4], [64, 2, 6, 3], [94, 11, 4, 5], [96, 1, 3, 4],
         [100, 6, 5, 3], [126, 3, 2, 3], [40, 40, 3, 3], [70, 3, 40, 2]]


@pytest.mark.parametrize("ne", CASES)
def test_mv2_sweep_vs_oracle(ne):
    import torch
    import paper_1809_10026_b200 as ls
    d, p = 3, 2
    ctx = ls.Context(d, p, ne)
    ctx.tune(ls.LS_TUNE_MATVEC, 2)
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 19)
    xg = torch.from_numpy(x).cuda()
    ctx.tune(ls.LS_TUNE_MV2_SWEEP, 1)
    y = ctx.matvec(xg).cpu().numpy()
    ctx.tune(ls.LS_TUNE_MV2_SWEEP, 0)
    y0 = ctx.matvec(xg).cpu().numpy()
    y_ref = op.apply_A(x, space, tf)
    assert _rel(y, y_ref) <= 1e-12
    assert _rel(y, y0) <= 1e-14


@pytest.mark.parametrize("world", [2, 3])
def test_mv2_sweep_slab_rows(world):
    import torch
    import paper_1809_10026_b200 as ls
    d, p, ne = 3, 2, [96, 7, 5, 23]
    ctx = ls.Context(d, p, ne)
    ctx.tune(ls.LS_TUNE_MATVEC, 2)
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 21)
    y_ref = op.apply_A(x, space, tf)
    xg = torch.from_numpy(x).cuda()
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(ctx.shape[0], world, r, p)
        y = ctx.matvec_slab(xg[t0 - lo:t0 + ntl + hi].contiguous(), t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, (r, t0, ntl)


def test_mv2_sweep_pcg():
    """A PCG solve with the sweep (the automatic choice at p = 2) gives the oracle's count."""
    import paper_1809_10026_b200 as ls
    from oracle import fd, pcg as opcg
    d, p, ne = 3, 2, [40, 39, 5, 6]
    ctx = ls.Context(d, p, ne)
    b = ctx.rhs(1)
    x, st = ctx.pcg(b)
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    fdd = fd.setup(space, tf)
    x_ref, it, ok, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda r: fd.fd_apply(r, fdd), b.cpu().numpy())
    assert ok and it == st["iters"]
    assert np.linalg.norm(x.cpu().numpy() - x_ref) <= 1e-9 * np.linalg.norm(x_ref)
