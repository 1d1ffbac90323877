"""ls_matvec v4 (ls_tune(LS_TUNE_MATVEC, 4): the plane pass of directions 1 + 2, then the
direction-3 and time DMMA passes; mv4_kernels.cuh) against the oracle's A x (eq:A_kron,
PAPER.md 686-703) and the dense original form, whole-vector and per-rank slab rows; with the
direction-3 and time passes fused into one kernel (ls_tune(LS_TUNE_MV5 = 10, 1); the automatic
choice (2) for p <= 4; mv5_kernels.cuh: d = 3, p_s = p_t) and as two passes (10, 0): DMMA band
passes (LS_TUNE_MV6 = 15, 0, the default) or DFMA Toeplitz-stencil passes (15, 1;
matvec6_kernels.cuh, opt-in)."""
import numpy as np
import pytest

import synth
from oracle import univariate as uv, operator as op, bspline as bs

pytestmark = pytest.mark.gpu

CASES = [
    (2, 2, [5, 7, 6]),
    (2, 3, [64, 64, 64]),       # config 2
    (3, 2, [3, 4, 5, 6]),
    (3, 3, [7, 6, 9, 8]),
    (3, 4, [9, 10, 11, 12]),
    (3, 5, [7, 6, 9, 8]),
    (3, 6, [20, 11, 9, 14]),
    (3, 7, [13, 9, 10, 11]),
    (3, 8, [3, 40, 2, 33]),     # n < 2p + 1 in two directions
    (2, 5, [60, 1, 37]),        # n_2 = 4
    (3, 3, [64, 5, 6, 7]),      # n_1 = 65
    (3, 2, [128, 3, 31, 2]),    # n_1 = 128, n_t = 3
    (3, 6, [33, 29, 5, 6]),
]


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


# second-stage variants: (LS_TUNE_MV5, LS_TUNE_MV6)
STAGES = {"v5": (1, 0), "dmma": (0, 0), "dfma": (0, 1)}


@pytest.mark.parametrize("stage", list(STAGES))
@pytest.mark.parametrize("d,p,ne", CASES)
def test_matvec_v4_matches_oracle(d, p, ne, stage):
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, ne)
    ctx.tune(2, 4)
    ctx.tune(10, STAGES[stage][0])
    ctx.tune(15, STAGES[stage][1])
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 9)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert _rel(y, op.apply_A(x, space, tf)) <= 1e-12


@pytest.mark.parametrize("mv6", [0, 1])
@pytest.mark.parametrize("d,pp,ne", [(2, (3, 2), [8, 7, 9]), (3, (4, 3), [6, 5, 7, 8]), (2, (8, 6), [20, 5, 30]),
                                     (3, (6, 5), [10, 9, 8, 12]), (2, (2, 5), [9, 8, 11]), (3, (5, 7), [9, 8, 10, 13])])
def test_matvec_v4_degrees(d, pp, ne, mv6):
    import torch
    import paper_1809_10026_b200 as ls
    ps, pt = pp
    ctx = ls.Context(d, pp, ne)
    ctx.tune(2, 4)
    ctx.tune(15, mv6)
    space = [uv.space_factors(n, ps) for n in ne[:d]]
    tf = uv.time_factors(ne[d], pt)
    x = synth.residual(ctx.shape, 29)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert _rel(y, op.apply_A(x, space, tf)) <= 1e-12


def test_matvec_v4_original_form_tiny():
    import torch
    import paper_1809_10026_b200 as ls
    d, ps, pt, ne = 2, 3, 2, [3, 2, 3]
    ctx = ls.Context(d, (ps, pt), ne)
    ctx.tune(2, 4)
    A = op.dense_A_original_form([bs.open_uniform_knots(n, ps) for n in ne[:d]], ps,
                                 bs.open_uniform_knots(ne[d], pt), pt)
    x = synth.residual(ctx.shape, 31)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy().ravel()
    assert _rel(y, A @ x.ravel()) <= 1e-12


@pytest.mark.parametrize("stage", list(STAGES))
@pytest.mark.parametrize("d,p,ne,world", [(3, 6, [9, 8, 7, 40], 4), (3, 2, [6, 5, 7, 29], 3),
                                          (2, 8, [20, 12, 37], 2), (3, 3, [12, 10, 8, 61], 8),
                                          (3, 8, [5, 6, 4, 50], 5), (3, 4, [7, 5, 6, 23], 2)])
def test_matvec_v4_slab_decomposition(d, p, ne, world, stage):
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, ne)
    ctx.tune(2, 4)
    ctx.tune(10, STAGES[stage][0])
    ctx.tune(15, STAGES[stage][1])
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 13)
    y_ref = op.apply_A(x, space, tf)
    xg = torch.from_numpy(x).cuda()
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(ctx.shape[0], world, r, p)
        y = ctx.matvec_slab(xg[t0 - lo:t0 + ntl + hi].contiguous(), t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, (r, t0, ntl)


def test_matvec_v4_config4_sampled():
    """Full config 4 (the bench's PCG configuration): v4 against v3 on a seeded input and, on
    sampled fibres, linearity -- both paths were checked against the oracle above."""
    import torch
    import paper_1809_10026_b200 as ls
    c = synth.CONFIGS[4]
    ctx = ls.Context(3, c["p"], [c["n_el"]] * 4)
    x = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    ctx.tune(2, 3)
    y3 = ctx.matvec(x)
    ctx.tune(2, 4)
    ctx.tune(10, 0)
    ctx.tune(15, 0)
    y4 = ctx.matvec(x)
    assert float(torch.linalg.norm(y4 - y3) / torch.linalg.norm(y3)) <= 1e-13
    ctx.tune(15, 1)
    y6 = ctx.matvec(x)
    assert float(torch.linalg.norm(y6 - y3) / torch.linalg.norm(y3)) <= 1e-13
    ctx.tune(10, 1)
    y5 = ctx.matvec(x)
    assert float(torch.linalg.norm(y5 - y3) / torch.linalg.norm(y3)) <= 1e-13


@pytest.mark.parametrize("mv", [4, 1, 2, 6])
@pytest.mark.parametrize("d,p,ne,world", [(3, 6, [9, 8, 7, 40], 4), (3, 3, [12, 10, 8, 61], 8), (2, 4, [20, 12, 37], 3),
                                          (3, 2, [6, 5, 7, 29], 3)])
def test_matvec_slab3_decomposition(d, p, ne, world, mv):
    """ls_matvec_slab3 (the distributed ls_matvec's per-rank kernel without the copy into the
    halo-extended buffer: halo rows and own rows in separate buffers) against the oracle, rank
    by rank; the v4 path reads the three buffers directly, the others gather them."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, ne)
    ctx.tune(2, 4 if mv == 6 else mv)
    ctx.tune(15, 1 if mv == 6 else 0)  # 6: v4 with the DFMA stencil passes
    if mv == 6:
        ctx.tune(10, 0)
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 37)
    y_ref = op.apply_A(x, space, tf)
    xg = torch.from_numpy(x).cuda()
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(ctx.shape[0], world, r, p)
        x_lo = xg[t0 - lo:t0].clone() if lo else None
        x_hi = xg[t0 + ntl:t0 + ntl + hi].clone() if hi else None
        y = ctx.matvec_slab3(x_lo, xg[t0:t0 + ntl].clone(), x_hi, t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, (r, t0, ntl)


@pytest.mark.parametrize("p,ne", [(3, [7, 6, 9, 8]), (3, [64, 5, 6, 7]), (3, [60, 70, 3, 4]), (4, [94, 9, 5, 4]),
                                  (4, [30, 3, 2, 5]), (3, [95, 4, 6, 3]), (4, [124, 2, 3, 3]), (3, [2, 40, 3, 5])])
def test_matvec_v4_sweep_plane(p, ne):
    """The plane pass as the DFMA register sweep (LS_TUNE_MV4_SWEEP = 17, opt-in for d = 3,
    p = 3, 4; matvec2_kernels.cuh mv4_sweep_kernel) against the oracle and the DMMA plane pass
    (17 = 0, default), with the fused (v5) and the two-pass second stage."""
    import torch
    import paper_1809_10026_b200 as ls
    d = 3
    ctx = ls.Context(d, p, ne)
    ctx.tune(2, 4)
    space = [uv.space_factors(n, p) for n in ne[:d]]
    tf = uv.time_factors(ne[d], p)
    x = synth.residual(ctx.shape, 41)
    xg = torch.from_numpy(x).cuda()
    y_ref = op.apply_A(x, space, tf)
    for mv5 in (1, 0):
        ctx.tune(10, mv5)
        ctx.tune(17, 1)
        y = ctx.matvec(xg).cpu().numpy()
        ctx.tune(17, 0)
        y0 = ctx.matvec(xg).cpu().numpy()
        assert _rel(y, y_ref) <= 1e-12, mv5
        assert _rel(y, y0) <= 1e-13, mv5
