"""Spatial modes 1 + 2 of fd_apply fused per plane (ls_tune LS_TUNE_FD_PLANE = 14, opt-in;
csrc/fd_plane_kernel.cuh).

Algorithm 1 steps 2 and 4 (PAPER.md 959-962) for the two fastest spatial directions, both in
the centrosymmetric split (reading c25), as one kernel per (i_3, .., t) plane whose intermediate
stays in registers.  z = P^{-1} r is unique, so the fused path must match the
oracle at the parity bar and the per-direction path (knob 14 = 0) to rounding.  Covered: every
bucket (KS, NTH, MID) at both ends (odd and even n = 1 .. 136, the middle row / column of odd
extents, ragged last m-tiles and n-tiles), d = 2 and 3 (direction 3 and the time mode around
the plane pass), the 16-byte and 8-byte ring loads, fd_apply_stage's spatial stages on a few
time slices, and the fallbacks (n_1 != n_2; P^G, whose pencils are not centrosymmetric).
"""

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _oracle(d, p, n_elems, r):
    fdd = fd.setup([uv.space_factors(n, p) for n in n_elems[:d]], uv.time_factors(n_elems[d], p))
    return fd.fd_apply(r, fdd)


def _check(d, p, n_elems, seed=0):
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, n_elems)
    ctx.tune(ls.LS_TUNE_FD_PLANE, 1)
    r = synth.residual(ctx.shape, seed)
    rg = torch.from_numpy(r).cuda()
    z = ctx.fd_apply(rg).cpu().numpy()
    z_ref = _oracle(d, p, n_elems, r)
    assert _rel(z, z_ref) <= TOL
    assert np.max(np.abs(z - z_ref)) <= TOL * np.max(np.abs(z_ref))
    ctx.tune(ls.LS_TUNE_FD_PLANE, 0)
    z2 = ctx.fd_apply(rg).cpu().numpy()
    assert _rel(z, z2) <= 1e-12
    return ctx


# n_s = n_el + p - 2 (p = 2: n_s = n_el); d = 2 keeps the oracle cheap at n up to 136
N_2D = [1, 2, 3, 5, 16, 17, 30, 32, 33, 58, 63, 64, 65, 96, 97, 98, 99, 102, 103, 104, 105, 132]


@pytest.mark.parametrize("n", N_2D)
def test_plane_2d_vs_oracle(n):
    nt_el = 4 if n > 100 else 9
    _check(2, 2, [n, n, nt_el], seed=n)


@pytest.mark.parametrize("p,ne", [(3, [20, 20, 7, 6]), (3, [62, 62, 5, 4]), (2, [96, 96, 3, 3]), (6, [30, 30, 9, 5]),
                                  (4, [94, 94, 2, 3])])
def test_plane_3d_vs_oracle(p, ne):
    _check(3, p, ne, seed=1)


def test_plane_fallbacks():
    """n_1 != n_2 runs the per-direction kernels (one launch per direction)."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = _check(3, 2, [20, 21, 22, 5])
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    ctx.tune(ls.LS_TUNE_FD_PLANE, 1)
    ctx.fd_apply(r)
    torch.cuda.synchronize()
    n0 = ctx.launches
    ctx.fd_apply(r)
    torch.cuda.synchronize()
    assert ctx.launches - n0 == 2 * 3 + 1  # plane kernel not used: 6 spatial + 1 fused time launch
    ctx2 = ls.Context(3, 2, [20, 20, 22, 5])
    ctx2.tune(ls.LS_TUNE_FD_PLANE, 1)
    r2 = torch.from_numpy(synth.residual(ctx2.shape, 0)).cuda()
    ctx2.fd_apply(r2)
    torch.cuda.synchronize()
    n0 = ctx2.launches
    ctx2.fd_apply(r2)
    torch.cuda.synchronize()
    assert ctx2.launches - n0 == 2 * 2 + 1  # plane + direction 3, both ways, and the time mode


@pytest.mark.parametrize("rows", [1, 2, 3])
def test_plane_stage_slices(rows):
    """fd_apply_stage 0 / 2 (spatial modes on `rows` time slices) with the plane kernel equals
    the per-direction path."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, 3, [33, 33, 12, 8])
    Ns = int(np.prod(ctx.n_s))
    x = torch.from_numpy(synth.residual((rows, Ns), 4)).cuda()
    for stage in (0, 2):
        a = torch.empty_like(x)
        ctx.tune(ls.LS_TUNE_FD_PLANE, 1)
        ctx.fd_stage(stage, x, a, rows)
        b = torch.empty_like(x)
        ctx.tune(ls.LS_TUNE_FD_PLANE, 0)
        ctx.fd_stage(stage, x, b, rows)
        assert _rel(a.cpu().numpy(), b.cpu().numpy()) <= 1e-12


def test_plane_nonfinite_guard():
    """A NaN in one plane stays in that plane (planes never mix; padded ring rows are zero-filled)."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, 2, [24, 24, 6, 4])
    ctx.tune(ls.LS_TUNE_FD_PLANE, 1)
    Ns = int(np.prod(ctx.n_s))
    n = ctx.n_s[0]
    x = synth.residual((2, Ns), 3)
    x[1, 3 * n * n + 5] = np.nan  # time slice 1, plane i3 = 3
    out = torch.empty((2, Ns), dtype=torch.float64, device="cuda")
    ctx.fd_stage(0, torch.from_numpy(x).cuda(), out, 2)
    o = out.cpu().numpy().reshape(2, ctx.n_s[2], n * n)
    bad = ~np.isfinite(o)
    # direction 3 mixes the planes of one time slice, never two time slices
    assert bad[1].all()
    assert not bad[0].any()
