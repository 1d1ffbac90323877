"""Fused time mode of fd_apply (ls_tune LS_TUNE_FD_TIME = 13, default 1; csrc/fd_time_kernel.cuh).

Algorithm 1 steps 2-4 restricted to the time direction (PAPER.md 947-962): U_t^T along time,
the division by lambda_t[i_t] + Lambda_s[s] (reading c3), U_t along time -- one kernel whose
intermediate never leaves the registers (two fragment-ordered copies of U_t in shared memory up to
n_t = 104, one XOR-swizzled copy up to n_t = 136).  z = P^{-1} r is unique,
so the fused path must match the oracle at the parity bar and the two-launch path (knob 13 = 0)
to rounding.  Covered: every k-step bucket (3, 5, 9, 13, 17, 21, 25, 26) with n_t at both ends,
even row strides (16-byte vector path) and odd ones (scalar path), ragged last warp tiles,
n_t = 104 (largest fused) and 105 (falls back to two launches), separate degrees p_t != p_s,
d = 1, 2, 3, and the chunk entry point fd_apply_stage(1) at odd / even offsets and lengths.
"""

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _oracle(d, ps, pt, n_elems, r):
    fdd = fd.setup([uv.space_factors(n, ps) for n in n_elems[:d]], uv.time_factors(n_elems[d], pt))
    return fd.fd_apply(r, fdd)


# (d, p, n_elems): n_t = n_el_t + p_t - 1, N_s = prod(n_el + p_s - 2)
CASES = [
    (1, 2, [16, 8]),           # n_t = 9   (bucket 3),  N_s = 16 (one full warp tile)
    (2, 3, [13, 14, 10]),      # n_t = 12  (bucket 3),  N_s = 210 (even, ragged)
    (1, 2, [40, 16]),          # n_t = 17  (bucket 5),  N_s = 40
    (2, 3, [12, 14, 30]),      # n_t = 32  (bucket 9),  N_s = 195 (odd: scalar path)
    (2, 2, [40, 41, 49]),      # n_t = 50  (bucket 13), N_s = 1640
    (3, 3, [8, 9, 10, 64]),    # n_t = 66  (bucket 17), N_s = 990
    (3, 3, [10, 10, 10, 64]),  # n_t = 66  (bucket 17), N_s = 1331 (odd, config 3's parity)
    (2, 2, [30, 31, 66]),      # n_t = 67  (bucket 17)
    (2, 2, [30, 31, 80]),      # n_t = 81  (bucket 21)
    (2, 4, [20, 21, 96]),      # n_t = 99  (bucket 25), config 5 p = 4's n_t
    (2, 2, [24, 25, 96]),      # n_t = 97  (bucket 25), config 5 p = 2's n_t
    (2, 8, [10, 11, 96]),      # n_t = 103 (bucket 26), config 5 p = 8's n_t
    (1, 2, [50, 103]),         # n_t = 104 (largest two-copy bucket)
    (1, 2, [50, 104]),         # n_t = 105 (single swizzled copy, bucket 30)
    (2, 2, [30, 31, 119]),     # n_t = 120 (bucket 30, full)
    (2, 6, [9, 10, 124]),      # n_t = 129 (bucket 33)
    (3, 6, [4, 5, 6, 128]),    # n_t = 133 (bucket 34: config 4's n_t)
    (1, 2, [40, 135]),         # n_t = 136 (the cap)
]


@pytest.mark.parametrize("d,p,n_elems", CASES)
def test_time_fused_vs_oracle(d, p, n_elems):
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, n_elems)
    r = synth.residual(ctx.shape, 11)
    z_ref = _oracle(d, p, p, n_elems, r)
    rg = torch.from_numpy(r).cuda()
    z = ctx.fd_apply(rg).cpu().numpy()
    assert _rel(z, z_ref) <= TOL
    assert np.max(np.abs(z - z_ref)) <= TOL * np.max(np.abs(z_ref))
    # the two-launch path gives the same z up to rounding
    ctx.tune(ls.LS_TUNE_FD_TIME, 0)
    z2 = ctx.fd_apply(rg).cpu().numpy()
    assert _rel(z, z2) <= 1e-12


@pytest.mark.parametrize("ps,pt,n_elems", [(3, 1, [20, 21, 40]), (2, 5, [18, 19, 60]), (4, 2, [9, 10, 11, 70]),
                                          (2, 7, [12, 13, 120]), (5, 3, [6, 7, 8, 131])])
def test_time_fused_separate_degrees(ps, pt, n_elems):
    import torch
    import paper_1809_10026_b200 as ls
    d = len(n_elems) - 1
    ctx = ls.Context(d, (ps, pt), n_elems)
    r = synth.residual(ctx.shape, 5)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert _rel(z, _oracle(d, ps, pt, n_elems, r)) <= TOL


@pytest.mark.parametrize("a,b", [(0, 1), (0, 16), (3, 17), (16, 32), (5, 1000), (1, 1639)])
def test_time_fused_stage_chunks(a, b):
    """fd_apply_stage(1): the time mode of the spatial chunk [n_t][b] at offset a (the
    per-rank step of the distributed path) equals the two-launch path and the columns
    a .. a+b-1 of the whole time mode."""
    import torch
    import paper_1809_10026_b200 as ls
    d, p, ne = 2, 2, [40, 41, 49]
    ctx = ls.Context(d, p, ne)
    Ns = int(np.prod(ctx.n_s))
    x = torch.from_numpy(synth.residual((ctx.n_t, Ns), 3)).cuda()
    full = torch.empty_like(x)
    ctx.fd_stage(1, x, full, 0, Ns)
    chunk = x[:, a:a + b].contiguous()
    out = torch.empty_like(chunk)
    ctx.fd_stage(1, chunk, out, a, b)
    ref = full[:, a:a + b].cpu().numpy()
    assert _rel(out.cpu().numpy(), ref) <= 1e-12
    ctx.tune(ls.LS_TUNE_FD_TIME, 0)
    out2 = torch.empty_like(chunk)
    ctx.fd_stage(1, chunk, out2, a, b)
    assert _rel(out.cpu().numpy(), out2.cpu().numpy()) <= 1e-12


def test_time_fused_single_launch():
    """The fused path is one launch per time mode pair: 2d + 1 launches per fd_apply."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, 3, [8, 9, 10, 64])
    r = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
    ctx.fd_apply(r)
    torch.cuda.synchronize()
    n0 = ctx.launches
    ctx.fd_apply(r)
    torch.cuda.synchronize()
    assert ctx.launches - n0 == 2 * 3 + 1
    ctx.tune(ls.LS_TUNE_FD_TIME, 0)
    n1 = ctx.launches
    ctx.fd_apply(r)
    torch.cuda.synchronize()
    assert ctx.launches - n1 == 2 * 3 + 2


def test_time_fused_nonfinite_guard():
    """A NaN in one column of the time mode's input stays in that column (the fused tile
    never mixes columns; the padded rows / columns of a tile never reach a stored value)."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(2, 2, [40, 41, 49])
    Ns = int(np.prod(ctx.n_s))
    x = synth.residual((ctx.n_t, Ns), 2)
    x[:, 7] = np.nan
    out = torch.empty((ctx.n_t, Ns), dtype=torch.float64, device="cuda")
    ctx.fd_stage(1, torch.from_numpy(x).cuda(), out, 0, Ns)
    bad = ~np.isfinite(out.cpu().numpy())
    assert bad[:, 7].all()
    bad[:, 7] = False
    assert not bad.any()


def test_time_fused_mapped_pg_long_time():
    """The P^G preconditioner (PAPER.md 969-1045: D^{-1/2} scaling around the FD solve of the
    weighted pencils) with n_t = 133 (the single swizzled U_t copy) against the two-launch path."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(2, 3, [6, 6, 131], geometry=synth.quarter_annulus(), precond=ls.LS_PRECOND_PG)
    r = torch.from_numpy(synth.residual(ctx.shape, 9)).cuda()
    z = ctx.fd_apply(r).cpu().numpy()
    ctx.tune(ls.LS_TUNE_FD_TIME, 0)
    z0 = ctx.fd_apply(r).cpu().numpy()
    assert _rel(z, z0) <= 1e-12


@pytest.mark.parametrize("d,ps,pt,ne", [(1, 2, 1, [4, 1]), (2, 2, 1, [3, 4, 1]), (3, 2, 1, [2, 3, 2, 1]),
                                        (1, 3, 1, [40, 2]), (2, 2, 2, [1, 1, 1])])
def test_time_fused_edge_shapes(d, ps, pt, ne):
    """n_t = 1 and 2 (a single, mostly padded k-step), N_s = 1: the fused kernel against the oracle."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, (ps, pt), ne)
    r = synth.residual(ctx.shape, 1)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert _rel(z, _oracle(d, ps, pt, ne, r)) <= TOL
