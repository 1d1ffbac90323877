"""Centrosymmetric split of the spatial FD mode products (ls_tune LS_TUNE_FD_CS = 9, default 1;
fd_rd_kernel.cuh "CS", api.cu cs_eig, reading c25).

With uniform open knots and Dirichlet conditions at both ends (PAPER.md 266-267, 1111-1112)
the space pencil (J, M) commutes with the index reversal R, so its eigenvectors (eq:eig_dec,
PAPER.md 939-945) are even or odd and every spatial mode product splits into two half-size
products.  z = P^{-1} r is unique, so the split must reproduce the oracle's
fd_apply to the parity bar and the unsplit library path to rounding.  Covered here:
  * the eigenbasis: U^T M U = I, U^T J U = Lambda, the even / odd symmetry of the columns, the
    spectrum equal to the oracle's;
  * fd_apply against the oracle and against the unsplit kernels over even / odd extents
    n = 2 .. 136 (half extents in every k-step bucket 2 .. 17), d = 1, 2, 3, every mode
    position (contiguous / strided FAST / strided general);
  * the P^G preconditioner keeps the unsplit basis (its weighted pencils are not
    centrosymmetric): knob 9 has no effect there.
"""

import numpy as np
import pytest

from oracle import univariate as uv, fd
import synth

pytestmark = pytest.mark.gpu
TOL = 1e-9


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _fdd(d, p, n_elems):
    return fd.setup([uv.space_factors(n, p) for n in n_elems[:d]], uv.time_factors(n_elems[d], p))


# n_s = n_el + p - 2: even and odd extents, half extents ceil(n/2) across the buckets
EIG_CASES = [(2, 2), (3, 2), (3, 3), (16, 2), (64, 3), (63, 3), (96, 2), (96, 4), (96, 8), (128, 6), (131, 6)]


@pytest.mark.parametrize("n_el,p", EIG_CASES)
def test_cs_eigenbasis(n_el, p):
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(1, p, [n_el, 4])
    f = uv.space_factors(n_el, p)
    M, J = f["M"], f["J"]
    n = M.shape[0]
    he = (n + 1) // 2
    U = ctx.get_factor(7, 1)
    lam = ctx.get_factor(5, 1)
    assert np.max(np.abs(U.T @ M @ U - np.eye(n))) < 1e-10
    assert np.max(np.abs(U.T @ J @ U - np.diag(lam))) < 1e-10 * lam.max()
    # even columns first (u = R u), then odd ones (u = -R u), each half ascending
    assert np.array_equal(U[:, :he], U[::-1, :he])
    assert np.array_equal(U[:, he:], -U[::-1, he:])
    assert np.all(np.diff(lam[:he]) > 0) and np.all(np.diff(lam[he:]) > 0)
    lam_ref, _ = fd.generalized_eig(J, M)
    np.testing.assert_allclose(np.sort(lam), lam_ref, rtol=1e-10)


FD_CASES = [
    (1, 2, [2, 3]),             # n_s = 2 (he = ho = 1)
    (1, 3, [2, 5]),             # n_s = 3 (middle row only in the even half)
    (1, 2, [16, 16]),           # config 1
    (1, 4, [60, 9]),            # n_s = 62
    (1, 2, [130, 134]),         # n_s = 130 (he = 65, bucket 17)
    (1, 6, [130, 12]),          # n_s = 134 (he = 67)
    (1, 2, [136, 8]),           # n_s = 136, the largest extent (he = 68, bucket 17)
    (2, 3, [64, 64, 64]),       # config 2: n = 65 (he = 33, bucket 9); Q = 65 strided general
    (2, 2, [7, 9, 6]),          # n = 7 / 9, tiny
    (2, 6, [98, 20, 30]),       # n_1 = 102 (he = 51, bucket 13)
    (2, 5, [27, 40, 11]),       # n = 30 / 43
    (3, 2, [3, 4, 5, 6]),
    (3, 3, [6, 7, 8, 9]),       # odd and even extents in every direction
    (3, 4, [8, 9, 10, 11]),
    (3, 6, [10, 14, 12, 13]),   # Q = 14 (strided general), Q = 14*18 % 4 == 0 (FAST)
    (3, 2, [96, 3, 2, 5]),      # n_1 = 96 (he = 48, bucket 12): config 5 p = 2 extents
    (3, 4, [96, 2, 3, 4]),      # n_1 = 98 (he = 49, bucket 13): config 5 p = 4
    (3, 8, [96, 2, 2, 3]),      # n_1 = 102: config 5 p = 8
    (3, 6, [128, 2, 3, 5]),     # n_1 = 132 (he = 66, bucket 17): config 4 extents
]


@pytest.mark.parametrize("staged", [0, 1])
@pytest.mark.parametrize("d,p,n_elems", FD_CASES)
def test_cs_fd_apply(d, p, n_elems, staged):
    """staged = ls_tune LS_TUNE_FD_STAGED (11): the cp.async-staged split kernel for even
    extents (fd_rds_kernel.cuh), process-wide, restored to the default afterwards."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, n_elems)
    ctx.tune(11, staged)
    r = synth.residual(ctx.shape, 29)
    rg = torch.from_numpy(r).cuda()
    z_ref = fd.fd_apply(r, _fdd(d, p, n_elems))
    ctx.tune(9, 1)
    z1 = ctx.fd_apply(rg).cpu().numpy()
    assert _rel(z1, z_ref) <= TOL
    assert np.max(np.abs(z1 - z_ref)) <= TOL * np.abs(z_ref).max()
    ctx.tune(9, 0)
    z0 = ctx.fd_apply(rg).cpu().numpy()
    ctx.tune(11, 0)
    assert _rel(z0, z_ref) <= TOL
    assert _rel(z1, z0) <= 1e-12


def test_cs_in_place_and_linearity():
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, 3, [6, 7, 8, 9])
    r1 = torch.from_numpy(synth.residual(ctx.shape, 1)).cuda()
    r2 = torch.from_numpy(synth.residual(ctx.shape, 2)).cuda()
    z1, z2 = ctx.fd_apply(r1), ctx.fd_apply(r2)
    z12 = ctx.fd_apply(2.0 * r1 - 3.0 * r2)
    assert _rel((z12).cpu().numpy(), (2.0 * z1 - 3.0 * z2).cpu().numpy()) <= 1e-13
    x = r1.clone()
    ctx.fd_apply(x, x)
    assert _rel(x.cpu().numpy(), z1.cpu().numpy()) <= 1e-15


def test_cs_not_used_for_pg():
    """P^G's weighted pencils are not centrosymmetric: the basis stays ascending (no split)
    and knob 9 changes nothing bit for bit."""
    import torch
    import paper_1809_10026_b200 as ls
    geo = synth.quarter_annulus()
    ctx = ls.Context(2, 3, [6, 5, 7], geometry=geo, precond=ls.LS_PRECOND_PG)
    for k in (1, 2):
        assert np.all(np.diff(ctx.get_factor(5, k)) > 0)
    r = torch.from_numpy(synth.residual(ctx.shape, 3)).cuda()
    ctx.tune(9, 1)
    z1 = ctx.fd_apply(r).cpu().numpy()
    ctx.tune(9, 0)
    z0 = ctx.fd_apply(r).cpu().numpy()
    assert np.array_equal(z1, z0)


# DFMA tail rows of the split kernels (RDCfg::TR, fd_rd_kernel.cuh; ls_tune LS_TUNE_FD_TAIL = 7):
# half extents he = ceil(n/2) = 8 m + 1 or 8 m + 2 in an odd k-step bucket (5, 9, 13, 17), every
# mode position (contiguous / strided FAST / strided general), even and odd n
TAIL_CASES = [
    (1, 3, [64, 5]),            # n = 65 (he = 33, ho = 32), contiguous
    (2, 3, [64, 64, 6]),        # config 2 extents: contiguous + strided general (Q = 65)
    (2, 2, [66, 66, 3]),        # n = 66 (he = ho = 33): strided FAST, 1 n-tile per warp
    (2, 2, [33, 34, 4]),        # n = 33 / 34 (he = 17, bucket 5)
    (3, 4, [96, 2, 3, 4]),      # n_1 = 98 (he = 49, bucket 13): config 5 p = 4, contiguous
    (3, 4, [4, 96, 3, 3]),      # n_2 = 98 strided FAST (Q = 6)
    (3, 4, [3, 95, 3, 3]),      # n_2 = 97 (he = 49, ho = 48) strided general (Q = 5)
    (3, 6, [128, 2, 3, 5]),     # n_1 = 132 (he = 66, bucket 17): config 4, contiguous, 2 n-tiles
    (3, 6, [4, 128, 3, 3]),     # n_2 = 132 strided FAST (Q = 8)
    (3, 6, [3, 128, 3, 3]),     # n_2 = 132 strided general (Q = 7)
    (3, 6, [2, 2, 127, 4]),     # n_3 = 131 (he = 66, ho = 65), Q = 36
    (2, 6, [125, 5, 4]),        # n_1 = 129 (he = 65 = 8 * 8 + 1, ho = 64)
]


@pytest.mark.parametrize("d,p,n_elems", TAIL_CASES)
def test_cs_tail_rows(d, p, n_elems):
    """The last one or two rows of each half product on DFMAs (opt-in, knob value 2) against all-DMMA
    m-tiles and against the oracle (Algorithm 1, PAPER.md 955-964); two seeds so that a
    column tile's tail is non-trivial in every warp."""
    import torch
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(d, p, n_elems)
    fdd = _fdd(d, p, n_elems)
    try:
        for seed in (5, 6):
            r = synth.residual(ctx.shape, seed)
            rg = torch.from_numpy(r).cuda()
            z_ref = fd.fd_apply(r, fdd)
            ctx.tune(7, 2)
            z1 = ctx.fd_apply(rg).cpu().numpy()
            ctx.tune(7, 0)
            z0 = ctx.fd_apply(rg).cpu().numpy()
            assert _rel(z1, z_ref) <= TOL
            assert np.max(np.abs(z1 - z_ref)) <= TOL * np.abs(z_ref).max()
            assert _rel(z0, z_ref) <= TOL
            assert _rel(z1, z0) <= 1e-12
    finally:
        ctx.tune(7, 1)
