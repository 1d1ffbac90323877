"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on the
same seeded inputs.  Bar (BASELINE.json north_star): relative 2-norm error
<= 1e-9 in fp64; setup quantities to 1e-10."""

import numpy as np
import pytest

from oracle import univariate as uv, fd, operator as op, rhs as orhs, pcg as opcg, bspline as bs
import synth

pytestmark = pytest.mark.gpu

TOL = 1e-9


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _ctx(d, p, n_elems):
    import paper_1809_10026_b200 as ls
    return ls.Context(d, p, n_elems)


def _oracle(d, p, n_elems):
    space = [uv.space_factors(n, p) for n in n_elems[:d]]
    tf = uv.time_factors(n_elems[d], p)
    return space, tf, fd.setup(space, tf)


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


# (d, p, n_elems) -- BASELINE configs 1-2 plus shapes chosen to hit every kernel
# bucket (n up to 136), odd/even extents, several tiles and ragged tails.
FD_CASES = [
    (1, 2, [16, 16]),          # config 1
    (1, 5, [40, 31]),
    (1, 2, [130, 134]),        # n_s = 130, n_t = 135 (largest bucket)
    (2, 2, [5, 7, 6]),
    (2, 3, [64, 64, 64]),      # config 2
    (2, 6, [98, 20, 30]),      # n = 102 bucket
    (3, 2, [3, 4, 5, 6]),
    (3, 3, [6, 6, 6, 6]),
    (3, 4, [8, 9, 10, 11]),
    (3, 3, [20, 17, 9, 31]),
]


@pytest.mark.parametrize("d,p,n_elems", FD_CASES)
def test_setup_factors_match_oracle(torch_cuda, d, p, n_elems):
    ctx = _ctx(d, p, n_elems)
    space, tf, fdd = _oracle(d, p, n_elems)
    for k in range(1, d + 1):
        for which, key in ((0, "M"), (1, "K"), (2, "J")):
            A = space[k - 1][key]
            np.testing.assert_allclose(ctx.get_factor(which, k), A, rtol=0, atol=1e-12 * np.abs(A).max())
        lam = ctx.get_factor(5, k)  # eigen index order [even | odd] (LS_TUNE_FD_CS split)
        np.testing.assert_allclose(np.sort(lam), fdd["lam_s"][k - 1], rtol=1e-10)
        U = ctx.get_factor(7, k)
        M, J = space[k - 1]["M"], space[k - 1]["J"]
        n = M.shape[0]
        assert np.max(np.abs(U.T @ M @ U - np.eye(n))) < 1e-10
        assert np.max(np.abs(U.T @ J @ U - np.diag(lam))) < 1e-10 * lam.max()
    np.testing.assert_allclose(ctx.get_factor(3), tf["Mt_hat"], atol=1e-14)
    np.testing.assert_allclose(ctx.get_factor(4), tf["Kt_hat"], atol=1e-12 * np.abs(tf["Kt_hat"]).max())
    np.testing.assert_allclose(ctx.get_factor(6), fdd["lam_t"], rtol=1e-10)


@pytest.mark.parametrize("d,p,n_elems", FD_CASES)
@pytest.mark.parametrize("seed", [0, 1])
def test_fd_apply_matches_oracle(torch_cuda, d, p, n_elems, seed):
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, seed)
    z_ref = fd.fd_apply(r, fdd)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert _rel(z, z_ref) <= TOL
    # element-wise: every entry within 1e-9 of the largest
    assert np.max(np.abs(z - z_ref)) <= TOL * np.abs(z_ref).max()


VARIANT_CASES = FD_CASES + [
    (1, 2, [121, 125]),         # n = 121 / 126: k-step buckets wider than ceil(n/4) (33 vs 31, 32)
    (2, 3, [118, 5, 120]),      # n_1 = 119, n_t = 122
    (3, 6, [9, 7, 12, 10]),     # Q = 13 odd, n_t = 15
    (2, 2, [130, 7, 129]),      # n_1 = 130 (register-direct bucket), odd Q, n_t = 130
    (3, 2, [128, 3, 2, 131]),   # n_1 = 128, n_t = 132: FAST strided time mode (Q % 4 == 0)
    (1, 3, [130, 131]),         # d = 1, n = 131 / 133
]


@pytest.mark.parametrize("cs", [0, 1])
@pytest.mark.parametrize("variant", [1, 2])
@pytest.mark.parametrize("d,p,n_elems", VARIANT_CASES)
def test_fd_apply_kernel_variants(torch_cuda, variant, cs, d, p, n_elems):
    """Both FD mode-kernel families (ls_tune knob 1: 1 = smem-staged, 2 = register-
    direct) against the oracle, whatever the automatic dispatch picks; with and without the
    centrosymmetric split of the spatial modes (knob 9; with it the spatial modes always run
    the split register-direct kernel, the time modes the chosen family)."""
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    ctx.tune(1, variant)
    ctx.tune(9, cs)
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 11)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    z_ref = fd.fd_apply(r, fdd)
    assert _rel(z, z_ref) <= TOL
    assert np.max(np.abs(z - z_ref)) <= TOL * np.abs(z_ref).max()


def test_fd_apply_config1_dense_solve(torch_cuda):
    """BASELINE config 1: one fd_apply against a dense Kronecker solve of P."""
    import scipy.linalg
    torch = torch_cuda
    ctx = _ctx(1, 2, [16, 16])
    space, tf, _ = _oracle(1, 2, [16, 16])
    P = fd.dense_P(space, tf)
    r = synth.residual(ctx.shape, 0)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy().ravel()
    z_dense = scipy.linalg.cho_solve(scipy.linalg.cho_factor(P), r.ravel())
    assert _rel(z, z_dense) <= TOL
    assert np.linalg.norm(P @ z - r.ravel()) / np.linalg.norm(r) <= TOL


def test_fd_apply_in_place_and_zero(torch_cuda):
    torch = torch_cuda
    ctx = _ctx(3, 3, [6, 7, 8, 9])
    _, _, fdd = _oracle(3, 3, [6, 7, 8, 9])
    r = synth.residual(ctx.shape, 3)
    t = torch.from_numpy(r).cuda()
    ctx.fd_apply(t, t)
    assert _rel(t.cpu().numpy(), fd.fd_apply(r, fdd)) <= TOL
    zero = torch.zeros(ctx.shape, dtype=torch.float64, device="cuda")
    assert torch.count_nonzero(ctx.fd_apply(zero)).item() == 0


MV_CASES = [
    (1, 2, [16, 16]),
    (1, 4, [9, 13]),
    (2, 2, [5, 7, 6]),
    (2, 3, [64, 64, 64]),
    (3, 2, [3, 4, 5, 6]),
    (3, 5, [7, 6, 9, 8]),
]


MV_VARIANT_CASES = MV_CASES + [
    (3, 6, [20, 11, 9, 14]),     # interior Toeplitz zones in every direction, p = 6
    (3, 8, [3, 40, 2, 33]),      # n < 2p + 1 in two directions (no interior zone)
    (2, 5, [60, 1, 37]),         # n_2 = 4
    (3, 3, [64, 5, 6, 7]),       # n_1 = 65
    (3, 2, [128, 3, 31, 2]),     # n_1 = 128, n_t = 3 < 2p + 1
]


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
@pytest.mark.parametrize("d,p,n_elems", MV_VARIANT_CASES)
def test_matvec_variants_match_oracle(torch_cuda, variant, d, p, n_elems):
    """Every ls_matvec implementation (ls_tune knob 2: 1 = four banded passes,
    2 = three fused passes with Toeplitz stencils + boundary corrections, 3 = four DMMA band
    passes, 4 = DMMA plane pass + direction-3 / time passes, d >= 2)."""
    torch = torch_cuda
    if variant == 4 and d < 2:
        pytest.skip("v4 needs d >= 2 (LS_ENOTSUP)")
    ctx = _ctx(d, p, n_elems)
    ctx.tune(2, variant)
    space, tf, _ = _oracle(d, p, n_elems)
    x = synth.residual(ctx.shape, 9)
    y_ref = op.apply_A(x, space, tf)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert _rel(y, y_ref) <= 1e-12


@pytest.mark.parametrize("d,p,n_elems", MV_CASES)
def test_matvec_matches_oracle(torch_cuda, d, p, n_elems):
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    space, tf, _ = _oracle(d, p, n_elems)
    x = synth.residual(ctx.shape, 5)
    y_ref = op.apply_A(x, space, tf)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert _rel(y, y_ref) <= 1e-12


def test_matvec_original_form_tiny(torch_cuda):
    """Against the dense ORIGINAL least-squares form (PAPER.md 406)."""
    torch = torch_cuda
    d, p, ne = 2, 3, [3, 2, 3]
    ctx = _ctx(d, p, ne)
    A = op.dense_A_original_form([bs.open_uniform_knots(n, p) for n in ne[:d]], p,
                                 bs.open_uniform_knots(ne[d], p), p)
    x = synth.residual(ctx.shape, 6)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy().ravel()
    assert _rel(y, A @ x.ravel()) <= 1e-12


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("d,p,n_elems", [(1, 2, [16, 16]), (2, 3, [64, 64, 64]), (3, 4, [8, 9, 10, 11])])
def test_rhs_matches_oracle(torch_cuda, kind, d, p, n_elems):
    ctx = _ctx(d, p, n_elems)
    b_ref = orhs.rhs(kind, [bs.open_uniform_knots(n, p) for n in n_elems[:d]], p,
                     bs.open_uniform_knots(n_elems[d], p), p)
    b = ctx.rhs(kind).cpu().numpy()
    assert _rel(b, b_ref) <= 1e-12


@pytest.mark.parametrize("n_el", [8, 16])
@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_pcg_table1(torch_cuda, n_el, p):
    """Table 1 (PAPER.md 1187-1189) iteration counts on the GPU, and the
    solution against the oracle's PCG at the same iteration count."""
    from conftest import golden
    ctx = _ctx(3, p, [n_el] * 4)
    b = ctx.rhs(1)
    x, st = ctx.pcg(b, tol=1e-8)
    want = golden("table1_iterations.json")["iterations"][str(n_el)][p - 2]
    assert st["status"] == 0 and st["iters"] == want
    assert st["true_rel_res"] <= 1e-7
    space, tf, fdd = _oracle(3, p, [n_el] * 4)
    bo = b.cpu().numpy()
    xo, it, conv, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda v: fd.fd_apply(v, fdd), bo)
    assert it == st["iters"]
    assert _rel(x.cpu().numpy(), xo) <= TOL


def test_pcg_config2(torch_cuda):
    """BASELINE config 2: d=2, p=3, n_el=64, f = sin sin e^t (kind 0)."""
    ctx = _ctx(2, 3, [64, 64, 64])
    b = ctx.rhs(0)
    x, st = ctx.pcg(b, tol=1e-8)
    space, tf, fdd = _oracle(2, 3, [64, 64, 64])
    xo, it, conv, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda v: fd.fd_apply(v, fdd),
                               b.cpu().numpy())
    assert st["iters"] == it and st["status"] == 0
    assert _rel(x.cpu().numpy(), xo) <= TOL


def test_pcg_zero_rhs(torch_cuda):
    torch = torch_cuda
    ctx = _ctx(2, 2, [4, 4, 4])
    b = torch.zeros(ctx.shape, dtype=torch.float64, device="cuda")
    x, st = ctx.pcg(b)
    assert st["iters"] == 0 and torch.count_nonzero(x).item() == 0


@pytest.mark.parametrize("d,p,n_elems", [(2, 3, [12, 10, 9]),      # n_t = 11: pipelined copies
                                         (3, 2, [5, 6, 7, 4]),       # n_t = 5 < 8 chunks: plain path
                                         (1, 4, [30, 60])])
def test_fd_apply_host_roundtrip(torch_cuda, d, p, n_elems):
    """fd_apply_host (host buffers; chunked H2D / compute / D2H pipeline when n_t >= 8)."""
    ctx = _ctx(d, p, n_elems)
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 2)
    z = np.empty_like(r)
    ctx.fd_apply_host(r, z)
    assert _rel(z, fd.fd_apply(r, fdd)) <= TOL


def test_kernels_launched(torch_cuda):
    """The CUDA path is the one that runs: fd_apply launches 2d + 1 kernels (the two time modes
    fused), or 2(d+1) with the fused time mode off (LS_TUNE_FD_TIME = 0)."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx = _ctx(3, 3, [6, 6, 6, 6])
    r = torch.rand(ctx.shape, dtype=torch.float64, device="cuda")
    n0 = ctx.launches
    ctx.fd_apply(r)
    assert ctx.launches - n0 == 7
    ctx.tune(ls.LS_TUNE_FD_TIME, 0)
    n0 = ctx.launches
    ctx.fd_apply(r)
    assert ctx.launches - n0 == 8
    ctx2 = _ctx(1, 2, [10, 110])  # n_t = 111: the single-copy fused kernel
    r2 = torch.rand(ctx2.shape, dtype=torch.float64, device="cuda")
    n0 = ctx2.launches
    ctx2.fd_apply(r2)
    assert ctx2.launches - n0 == 3


EDGE_CASES = [
    (1, 2, [1, 1]),            # n_s = 1, n_t = 2 (smallest space-time grid)
    (2, 2, [1, 3, 1]),         # single-function directions
    (3, 2, [1, 1, 1, 1]),      # N = 2
    (3, 2, [2, 1, 40, 2]),     # extreme aspect ratio
    (1, 8, [128, 127]),        # n = 134 / n_t = 134 (near the 136 cap), p = 8
    (2, 4, [134, 1, 5]),       # n_1 = 136 (the cap)
]


@pytest.mark.parametrize("d,p,n_elems", EDGE_CASES)
def test_fd_apply_edge_shapes(torch_cuda, d, p, n_elems):
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 4)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    z_ref = fd.fd_apply(r, fdd)
    assert _rel(z, z_ref) <= TOL


@pytest.mark.parametrize("d,p,n_elems", EDGE_CASES[:4] + [(2, 8, [20, 3, 25])])
def test_matvec_edge_shapes(torch_cuda, d, p, n_elems):
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    space, tf, _ = _oracle(d, p, n_elems)
    x = synth.residual(ctx.shape, 8)
    y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert _rel(y, op.apply_A(x, space, tf)) <= 1e-12


def test_setup_rejects_too_large_extent(torch_cuda):
    import paper_1809_10026_b200 as ls
    with pytest.raises(ls.LSError) as e:
        ls.Context(1, 4, [10, 134])   # n_t = 137 > 136
    assert e.value.code == ls.LS_EINVAL


def test_matvec_rejects_aliasing(torch_cuda):
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    ctx = _ctx(2, 2, [4, 4, 4])
    x = torch.zeros(ctx.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ls.LSError):
        ctx.matvec(x, x)


def test_pcg_nonconvergence_status(torch_cuda):
    """max_iter too small -> LS_ENOCONV with stats filled (SPEC.md 405)."""
    import paper_1809_10026_b200 as ls
    ctx = _ctx(3, 3, [8, 8, 8, 8])
    x, st = ctx.pcg(ctx.rhs(1), tol=1e-12, max_iter=3)
    assert st["status"] == ls.LS_ENOCONV and st["iters"] == 3 and st["rel_res"] > 1e-12


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
@pytest.mark.parametrize("d,p,n_elems,world", [(3, 6, [9, 8, 7, 40], 4), (3, 2, [6, 5, 7, 29], 3),
                                                (2, 8, [20, 12, 37], 2), (1, 3, [30, 50], 5),
                                                (3, 3, [12, 10, 8, 61], 8)])
def test_matvec_slab_decomposition(torch_cuda, variant, d, p, n_elems, world):
    """The per-rank kernel of the distributed ls_matvec (ls_matvec_slab, time slab plus
    p halo slices each side, exactly what ls_matvec runs after its NCCL halo exchange),
    for every rank of a `world`-way split, against the oracle's full A x."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    if variant == 4 and d < 2:
        pytest.skip("v4 needs d >= 2 (LS_ENOTSUP)")
    ctx = _ctx(d, p, n_elems)
    ctx.tune(2, variant)
    space, tf, _ = _oracle(d, p, n_elems)
    x = synth.residual(ctx.shape, 13)
    y_ref = op.apply_A(x, space, tf)
    xg = torch.from_numpy(x).cuda()
    nt = ctx.shape[0]
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(nt, world, r, p)
        x_ext = xg[t0 - lo:t0 + ntl + hi].contiguous()
        y = ctx.matvec_slab(x_ext, t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, (r, t0, ntl)


@pytest.mark.parametrize("fdk", [1, 2])
@pytest.mark.parametrize("d,p,n_elems,world", [(3, 3, [8, 7, 6, 21], 4), (2, 6, [30, 25, 40], 3),
                                                (1, 2, [40, 17], 8), (3, 6, [30, 3, 2, 9], 2)])
def test_fd_apply_slab_chunk_decomposition(torch_cuda, fdk, d, p, n_elems, world):
    """The distributed fd_apply of ls_setup_dist emulated rank by rank on one GPU: forward
    spatial modes on every time slab (stage 0), the slab -> chunk all-to-all done here
    with the library's own plan (ls_a2a_plan), the fused time mode on every spatial chunk
    with its Lambda_s offset (stage 1), the transpose all-to-all, backward spatial modes
    (stage 2); against the oracle's fd_apply of the whole tensor."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    ctx.tune(1, fdk)
    ctx.tune(9, int(fdk == 2))  # the split with the register-direct family
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 17)
    nt = ctx.shape[0]
    Ns = int(np.prod(ctx.shape[1:]))
    rg = torch.from_numpy(r).cuda().reshape(nt, Ns)
    slabs = [ls.partition(nt, world, g) for g in range(world)]
    chunks = [ls.partition(Ns, world, h) for h in range(world)]
    fwd = []
    for (t0, ntl) in slabs:
        out = torch.empty(ntl, Ns, dtype=torch.float64, device="cuda")
        ctx.fd_stage(0, rg[t0:t0 + ntl].contiguous(), out, ntl)
        fwd.append(out)
    full = torch.cat(fwd)  # the all-to-all, by hand: chunk h = columns [c0, c0 + len) of every slab
    back = torch.empty_like(full)
    for (c0, ln) in chunks:
        if ln == 0:
            continue
        ch = full[:, c0:c0 + ln].contiguous()
        res = torch.empty_like(ch)
        ctx.fd_stage(1, ch, res, c0, ln)
        back[:, c0:c0 + ln] = res
    z = torch.empty_like(back)
    for (t0, ntl) in slabs:
        out = torch.empty(ntl, Ns, dtype=torch.float64, device="cuda")
        ctx.fd_stage(2, back[t0:t0 + ntl].contiguous(), out, ntl)
        z[t0:t0 + ntl] = out
    z_ref = fd.fd_apply(r, fdd)
    assert _rel(z.cpu().numpy().reshape(r.shape), z_ref) <= TOL


# the scattering epilogue is a FAST-path variant: n_1 ... n_{d-1} multiple of 4
@pytest.mark.parametrize("d,p,n_elems,world", [(3, 3, [5, 9, 6, 21], 4), (2, 2, [12, 25, 40], 3),
                                                (3, 6, [130, 2, 3, 9], 2), (2, 4, [6, 30, 17], 8)])
def test_fd_apply_fused_a2a_emulated(torch_cuda, d, p, n_elems, world):
    """The fused all-to-all path of the distributed fd_apply (LS_TUNE_A2A = 1), emulated rank
    by rank on one GPU: the scattering epilogues (fd_apply_scatter) write into per-rank
    receive buffers exactly as they write into peer memory in a multi-GPU run; the
    barriers are replaced by running the ranks one after the other.  Against the oracle."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    _, _, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 19)
    nt = ctx.shape[0]
    Ns = int(np.prod(ctx.shape[1:]))
    rg = torch.from_numpy(r).cuda().reshape(nt, Ns)
    slabs = [ls.partition(nt, world, g) for g in range(world)]
    chunks = [ls.partition(Ns, world, h) for h in range(world)]
    nan = float("nan")
    chunk_bufs = [torch.full((nt, 4 * ((ln + 3) // 4)), nan, dtype=torch.float64, device="cuda") for (_, ln) in chunks]
    for g, (t0, ntl) in enumerate(slabs):
        ctx.fd_scatter(0, rg[t0:t0 + ntl].contiguous(), ntl, 0, world, g, chunk_bufs)
    slab_bufs = [torch.full((ntl, Ns), nan, dtype=torch.float64, device="cuda") for (_, ntl) in slabs]
    for h, (c0, ln) in enumerate(chunks):
        ctx.fd_scatter(1, chunk_bufs[h], c0, ln, world, h, slab_bufs)
    z = torch.empty(nt, Ns, dtype=torch.float64, device="cuda")
    for g, (t0, ntl) in enumerate(slabs):
        out = torch.empty(ntl, Ns, dtype=torch.float64, device="cuda")
        ctx.fd_stage(2, slab_bufs[g], out, ntl)
        z[t0:t0 + ntl] = out
    z_ref = fd.fd_apply(r, fdd)
    assert _rel(z.cpu().numpy().reshape(r.shape), z_ref) <= TOL


GUARD_CASES = [(3, 3, [6, 7, 5, 9]), (2, 6, [29, 3, 11]), (1, 2, [121, 125]), (3, 2, [3, 4, 2, 6]),
               (2, 8, [130, 1, 14]), (3, 6, [128, 2, 3, 11]),
               (2, 3, [9, 9, 64]),        # n_t = 66: fused time mode with DFMA tail tiles; n_1 = n_2 (plane kernel)
               (3, 2, [5, 5, 6, 96])]     # n_t = 97 (tail, bucket 25), odd n_1 = n_2 = 5


def _guarded(torch, shape, fill, pad=4096):
    """A tensor of `shape` inside a larger allocation whose other entries are `fill`
    (compute-sanitizer is closed on this pool: NaN guards catch out-of-range reads that
    reach a result, canaries catch out-of-range writes)."""
    n = int(np.prod(shape))
    big = torch.full((n + 2 * pad,), fill, dtype=torch.float64, device="cuda")
    return big, big[pad:pad + n].view(shape), pad


@pytest.mark.parametrize("d,p,n_elems", GUARD_CASES)
def test_guarded_buffers_all_variants(torch_cuda, d, p, n_elems):
    """Inputs embedded in NaN-filled allocations, outputs inside canary-filled ones, for
    every FD kernel family and every matvec implementation: results match the oracle
    (no NaN leaked in from outside the input) and the canaries are untouched."""
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    space, tf, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 23)
    z_ref = fd.fd_apply(r, fdd)
    y_ref = op.apply_A(r, space, tf)
    canary = 1.2345e300
    # (FD kernel family, centrosymmetric split, fused time mode (knob 13), plane kernel (knob 14))
    for fdk, cs, ft, pl in ((1, 0, 1, 0), (2, 0, 1, 0), (1, 1, 1, 0), (2, 1, 1, 0), (2, 1, 0, 0), (2, 1, 1, 1)):
        ctx.tune(1, fdk)
        ctx.tune(9, cs)
        ctx.tune(13, ft)
        ctx.tune(14, pl)
        _, rin, _ = _guarded(torch, ctx.shape, float("nan"))
        rin.copy_(torch.from_numpy(r))
        obig, zout, pad = _guarded(torch, ctx.shape, canary)
        ctx.fd_apply(rin, zout)
        assert _rel(zout.cpu().numpy(), z_ref) <= TOL, (fdk, cs)
        assert bool((obig[:pad] == canary).all()) and bool((obig[pad + zout.numel():] == canary).all()), (fdk, cs)
    ctx.tune(1, 0)
    ctx.tune(13, 1)
    ctx.tune(14, 0)
    for mv in ((1, 2, 3, 4, 6) if d >= 2 else (1, 2, 3)):
        ctx.tune(2, 4 if mv == 6 else mv)  # 6: v4 with the DFMA stencil passes (knob 15)
        ctx.tune(15, 1 if mv == 6 else 0)
        _, xin, _ = _guarded(torch, ctx.shape, float("nan"))
        xin.copy_(torch.from_numpy(r))
        obig, yout, pad = _guarded(torch, ctx.shape, canary)
        ctx.matvec(xin, yout)
        assert _rel(yout.cpu().numpy(), y_ref) <= 1e-12, mv
        assert bool((obig[:pad] == canary).all()) and bool((obig[pad + yout.numel():] == canary).all()), mv


# separate degrees in space and time, p = (p_s, p_t) (PAPER.md 179-180;
# p_s = p_t + 1 as in Fig. 2b, PAPER.md 1132)
DEG_CASES = [(2, (3, 2), [8, 7, 9]), (3, (2, 1), [5, 6, 4, 7]), (3, (4, 3), [6, 5, 7, 8]),
             (1, (5, 4), [20, 17]), (2, (8, 6), [20, 5, 30]), (3, (6, 5), [10, 9, 8, 12]),
             (2, (2, 5), [9, 8, 11])]


def _oracle_deg(d, ps, pt, n_elems):
    space = [uv.space_factors(n, ps) for n in n_elems[:d]]
    tf = uv.time_factors(n_elems[d], pt)
    return space, tf, fd.setup(space, tf)


@pytest.mark.parametrize("d,pp,n_elems", DEG_CASES)
def test_degrees_fd_matvec_rhs_pcg(torch_cuda, d, pp, n_elems):
    """p_s != p_t: setup sizes, fd_apply, every ls_matvec implementation that supports the
    pair, ls_rhs and a PCG solve against the oracle."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    ps, pt = pp
    ctx = ls.Context(d, pp, n_elems)
    assert ctx.n_t == n_elems[d] + pt - 1 and ctx.n_s == [n + ps - 2 for n in n_elems[:d]]
    space, tf, fdd = _oracle_deg(d, ps, pt, n_elems)
    r = synth.residual(ctx.shape, 29)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert _rel(z, fd.fd_apply(r, fdd)) <= TOL
    y_ref = op.apply_A(r, space, tf)
    for mv in (1, 2, 3, 4):
        if (mv > 1 and pt < 2) or (mv == 4 and d < 2):
            continue
        ctx.tune(2, mv)
        y = ctx.matvec(torch.from_numpy(r).cuda()).cpu().numpy()
        assert _rel(y, y_ref) <= 1e-12, mv
    ctx.tune(2, 0)
    b_ref = orhs.rhs(1, [bs.open_uniform_knots(n, ps) for n in n_elems[:d]], ps,
                     bs.open_uniform_knots(n_elems[d], pt), pt)
    b = ctx.rhs(1)
    assert _rel(b.cpu().numpy(), b_ref) <= 1e-12
    x, st = ctx.pcg(b, tol=1e-8)
    xo, it, conv, _ = opcg.pcg(lambda v: op.apply_A(v, space, tf), lambda v: fd.fd_apply(v, fdd), b_ref)
    assert st["status"] == 0 and st["iters"] == it
    assert _rel(x.cpu().numpy(), xo) <= TOL


def test_degrees_matvec_original_form_tiny(torch_cuda):
    """p_s = 3, p_t = 2 against the dense ORIGINAL least-squares form (PAPER.md 406)."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    d, ps, pt, ne = 2, 3, 2, [3, 2, 3]
    ctx = ls.Context(d, (ps, pt), ne)
    A = op.dense_A_original_form([bs.open_uniform_knots(n, ps) for n in ne[:d]], ps,
                                 bs.open_uniform_knots(ne[d], pt), pt)
    x = synth.residual(ctx.shape, 31)
    for mv in (1, 2, 3, 4):
        ctx.tune(2, mv)
        y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy().ravel()
        assert _rel(y, A @ x.ravel()) <= 1e-12, mv


@pytest.mark.parametrize("variant", [1, 2, 3, 4])
def test_degrees_matvec_slab(torch_cuda, variant):
    """The halo of the distributed matvec is p_t slices wide."""
    import paper_1809_10026_b200 as ls
    torch = torch_cuda
    d, ps, pt, ne, world = 2, 3, 6, [6, 5, 40], 4
    ctx = ls.Context(d, (ps, pt), ne)
    ctx.tune(2, variant)
    space, tf, _ = _oracle_deg(d, ps, pt, ne)
    x = synth.residual(ctx.shape, 37)
    y_ref = op.apply_A(x, space, tf)
    xg = torch.from_numpy(x).cuda()
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(ctx.shape[0], world, r, pt)
        y = ctx.matvec_slab(xg[t0 - lo:t0 + ntl + hi].contiguous(), t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, r


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("d,pp,n_elems", [(1, (2, 2), [4, 5]), (2, (3, 2), [3, 2, 4]), (2, (2, 2), [3, 3, 3])])
def test_energy_error_matches_quadrature(torch_cuda, kind, d, pp, n_elems):
    """ls_energy_error at the PCG solution against the oracle's direct space-time
    quadrature of ||f - (d_t - Lap) u_h||^2 (PAPER.md 392-410)."""
    import paper_1809_10026_b200 as ls
    from oracle import error as oerr
    ps, pt = pp
    ctx = ls.Context(d, pp, n_elems)
    x, st = ctx.pcg(ctx.rhs(kind), tol=1e-12)
    e = ctx.energy_error(kind, x)
    J = oerr.ls_functional_quadrature(x.cpu().numpy(), kind, [bs.open_uniform_knots(n, ps) for n in n_elems[:d]],
                                      ps, bs.open_uniform_knots(n_elems[d], pt), pt)
    assert abs(e["J"] - J) <= 1e-10 * e["f2"]
    assert abs(e["f2"] - oerr.f_norm2(kind, d)) <= 1e-14 * e["f2"]


@pytest.mark.parametrize("p", [2, 3])
def test_energy_error_convergence_rate(torch_cuda, p):
    """The solve against the PDE: on the cube with u = prod sin(pi x_k) sin t (PAPER.md 1166),
    the least-squares energy error ||(d_t - Lap)(u - u_h)|| of the PCG solution decays as
    h^(p-1) for p_s = p_t = p (Thm teo:a-priori, PAPER.md 600-610; observed at PAPER.md 1131)."""
    import paper_1809_10026_b200 as ls
    errs = []
    for n_el in (4, 8, 16):
        ctx = ls.Context(2, p, [n_el] * 3)
        x, st = ctx.pcg(ctx.rhs(1), tol=1e-12)
        errs.append(np.sqrt(max(ctx.energy_error(1, x)["J"], 0.0)))
    rates = [np.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(abs(r - (p - 1)) <= 0.3 for r in rates), (errs, rates)


def test_pcg_rejects_aliasing(torch_cuda):
    import paper_1809_10026_b200 as ls
    ctx = _ctx(2, 2, [4, 4, 4])
    b = ctx.rhs(1)
    with pytest.raises(ls.LSError):
        ctx.pcg(b, x=b)


@pytest.mark.parametrize("d,p,n_elems", [(2, 3, [64, 63, 64]), (3, 2, [15, 16, 17, 17]), (1, 4, [95, 94]),
                                         (3, 3, [64, 8, 9, 63])])
def test_fd_tail_rows(torch_cuda, d, p, n_elems):
    """n = 8 m + 1 or 8 m + 2 in an odd k-step bucket (65, 66 in bucket 17; 17, 18 in bucket
    5; 97 in bucket 25): the last one or two output rows computed with DFMAs
    (LS_TUNE_FD_TAIL = 1, default) against the oracle and against all-DMMA tiles."""
    torch = torch_cuda
    ctx = _ctx(d, p, n_elems)
    space, tf, fdd = _oracle(d, p, n_elems)
    r = synth.residual(ctx.shape, 11)
    rg = torch.from_numpy(r).cuda()
    z_auto = ctx.fd_apply(rg).cpu().numpy()     # automatic dispatch (n = 97: register-direct)
    ctx.tune(1, 1)                               # the smem-staged family, which has the tail path
    ctx.tune(9, 0)                               # n x n spatial products (no split)
    z1 = ctx.fd_apply(rg).cpu().numpy()
    ctx.tune(7, 0)
    z0 = ctx.fd_apply(rg).cpu().numpy()
    ctx.tune(7, 1)
    z_ref = fd.fd_apply(r, fdd)
    assert _rel(z1, z_ref) <= TOL
    assert _rel(z1, z0) <= 1e-13
    assert _rel(z_auto, z_ref) <= TOL
