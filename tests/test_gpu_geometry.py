"""GPU parity of the mapped-domain path (ls_setup_geo):
the device-assembled physical factors (ls_matvec), P and P^G (fd_apply) and PCG
against oracle/geometry.py and oracle/geo_precond.py on the same seeded inputs and
the same maps (synth.GEOMETRIES).  Bars: matvec 1e-12, fd_apply / PCG 1e-9 (relative
2-norm), PCG iteration counts equal."""

import warnings

import numpy as np
import pytest

import synth
from oracle import geometry as G, geo_precond as GP, univariate as uv, fd, pcg as opcg

pytestmark = pytest.mark.gpu
warnings.filterwarnings("ignore", category=DeprecationWarning)


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _setup(name, p, n_elems, precond, pt=None):
    import paper_1809_10026_b200 as ls
    geo = synth.GEOMETRIES[name]() if name != "affine" else synth.affine_box([2.0, 0.5, 1.5][:len(n_elems) - 1])
    d = geo["d"]
    pt = p if pt is None else pt
    ctx = ls.Context(d, (p, pt), n_elems, geometry=geo, precond=precond)
    sf = G.space_factors_physical(geo, list(n_elems[:d]), p)
    tf = uv.time_factors(n_elems[d], pt)
    return ctx, geo, sf, tf


# (map, p_s, p_t, n_elems): ragged extents (N_s not a multiple of the 128-row CTA,
# n_t not a multiple of the 8-slice thread tile), several elements per direction
MV_CASES = [
    ("affine", 2, 2, [3, 4, 5]),
    ("annulus2d", 3, 3, [5, 7, 6]),
    ("annulus2d", 2, 3, [24, 20, 13]),
    ("annulus2d", 4, 2, [6, 5, 9]),
    ("annulus3d", 2, 2, [4, 5, 3, 6]),
    ("annulus3d", 3, 3, [5, 4, 6, 4]),
    ("affine", 3, 2, [3, 4, 2, 5]),
    ("annulus2d", 3, 2, [5, 6, 130]),      # n_t = 131: 17 time blocks of the DMMA tile
    ("annulus3d", 2, 4, [9, 3, 4, 60]),    # n_1 = 9: ragged 8-row block, n_t = 63
]


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name,p,pt,n_elems", MV_CASES)
def test_geo_matvec_matches_oracle(torch_cuda, name, p, pt, n_elems, variant):
    """variant 0: DMMA band tiles (default); 1: DFMA stencil kernel (ls_tune LS_TUNE_MATVEC = 1)."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx, geo, sf, tf = _setup(name, p, n_elems, ls.LS_PRECOND_P, pt)
    if variant:
        ctx.tune(2, 1)
    for seed in (1, 2):
        x = synth.residual(ctx.shape, seed)
        y = ctx.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        y_ref = G.apply_A_geo(x, sf, tf)
        assert _rel(y, y_ref) <= 1e-12, (seed, _rel(y, y_ref))


@pytest.mark.parametrize("variant", [0, 1])
@pytest.mark.parametrize("name,p,n_elems,world", [("annulus2d", 3, [6, 5, 30], 3),
                                                  ("annulus3d", 2, [4, 3, 5, 25], 4),
                                                  ("annulus2d", 2, [5, 4, 9], 2)])
def test_geo_matvec_slab_decomposition(torch_cuda, variant, name, p, n_elems, world):
    """The per-rank kernel of the distributed mapped-domain ls_matvec (ls_setup_geo_dist):
    a time slab plus p_t halo slices each side (ls_matvec_slab, what ls_matvec runs after
    its halo exchange), for every rank of a `world`-way split, against the oracle's A x;
    the last slice's W_t (x) L_s term lands on the last rank only."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx, geo, sf, tf = _setup(name, p, n_elems, ls.LS_PRECOND_P)
    if variant:
        ctx.tune(2, variant)
    x = synth.residual(ctx.shape, 6)
    y_ref = G.apply_A_geo(x, sf, tf)
    xg = torch.from_numpy(x).cuda()
    nt = ctx.shape[0]
    y_full = ctx.matvec(xg).cpu().numpy()
    for r in range(world):
        t0, ntl, lo, hi = ls.halo_plan(nt, world, r, p)
        x_ext = xg[t0 - lo:t0 + ntl + hi].contiguous()
        y = ctx.matvec_slab(x_ext, t0 - lo, t0, ntl).cpu().numpy()
        assert _rel(y, y_ref[t0:t0 + ntl]) <= 1e-12, (r, t0, ntl)
        assert np.array_equal(y, y_full[t0:t0 + ntl])   # same kernels, same summation order


@pytest.mark.parametrize("name,p,n_elems", [("annulus2d", 3, [6, 5, 7]), ("annulus3d", 2, [4, 3, 5, 4])])
def test_geo_plain_P_is_parametric(torch_cuda, name, p, n_elems):
    """precond = LS_PRECOND_P: fd_apply is Algorithm 1 for the parametric P (eq:preconditioner)."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx, geo, sf, tf = _setup(name, p, n_elems, ls.LS_PRECOND_P)
    d = geo["d"]
    plain = fd.setup([uv.space_factors(n, p) for n in n_elems[:d]], tf)
    r = synth.residual(ctx.shape, 3)
    z = ctx.fd_apply(torch.from_numpy(r).cuda()).cpu().numpy()
    assert _rel(z, fd.fd_apply(r, plain)) <= 1e-9
    assert ctx.geo_info()[0] == 0.0


PG_CASES = [
    ("affine", 2, [3, 4, 5]),
    ("annulus2d", 3, [6, 5, 7]),
    ("annulus2d", 2, [16, 12, 9]),
    ("annulus3d", 2, [4, 3, 5, 4]),
    ("annulus3d", 3, [5, 5, 5, 5]),
]


@pytest.mark.parametrize("name,p,n_elems", PG_CASES)
def test_geo_PG_fd_apply_matches_oracle(torch_cuda, name, p, n_elems):
    """(P^G)^{-1} r = D^{-1/2} Pbar^{-1} D^{-1/2} r (PAPER.md 969-1045, readings c20-c22)."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx, geo, sf, tf = _setup(name, p, n_elems, ls.LS_PRECOND_PG)
    d = geo["d"]
    data = GP.setup(geo, list(n_elems[:d]), p, tf, GP.A_diagonal(sf, tf))
    for seed in (4, 5):
        r = synth.residual(ctx.shape, seed)
        rt = torch.from_numpy(r).cuda()
        z = ctx.fd_apply(rt).cpu().numpy()
        err = _rel(z, GP.apply(r, data))
        assert err <= 1e-9, (seed, err)
    # in place (z == r)
    ctx.fd_apply(rt, rt)
    assert _rel(rt.cpu().numpy(), GP.apply(r, data)) <= 1e-9
    res, S = ctx.geo_info()
    assert S == (2 * p + 1) ** d
    if name == "affine":
        assert res < 1e-13          # constant coefficients: exactly separable
    else:
        assert 0 < res < 1e2   # shared mu_k: c_tau, c_k are not jointly separable on the annulus


@pytest.mark.parametrize("name,p,n_elems,precond", [("annulus2d", 3, [8, 8, 8], 0), ("annulus2d", 3, [8, 8, 8], 1),
                                                    ("annulus3d", 2, [4, 4, 4, 4], 0),
                                                    ("annulus3d", 2, [4, 4, 4, 4], 1)])
def test_geo_pcg_matches_oracle(torch_cuda, name, p, n_elems, precond):
    """PCG with P or P^G on the mapped domain: same iteration count and iterate as the
    oracle's PCG (x0 = 0, tol 1e-8 on the recurrence residual, PAPER.md 1109)."""
    torch = torch_cuda
    ctx, geo, sf, tf = _setup(name, p, n_elems, precond)
    d = geo["d"]
    b = synth.residual(ctx.shape, 7)
    x, st = ctx.pcg(torch.from_numpy(b).cuda(), tol=1e-8)
    A = lambda v: G.apply_A_geo(v, sf, tf)
    if precond == 1:
        data = GP.setup(geo, list(n_elems[:d]), p, tf, GP.A_diagonal(sf, tf))
        Pinv = lambda r: GP.apply(r, data)
    else:
        plain = fd.setup([uv.space_factors(n, p) for n in n_elems[:d]], tf)
        Pinv = lambda r: fd.fd_apply(r, plain)
    x_ref, it, ok, _ = opcg.pcg(A, Pinv, b)
    assert ok and st["status"] == 0
    # equal counts; on the worse-conditioned plain-P systems (~65 iterations) the recurrence
    # residual crosses tol within one iteration of the oracle's (reading c13: rounding order free)
    assert st["iters"] == it if it <= 30 else abs(st["iters"] - it) <= 1
    # the iterate at equal k: rounding-order differences grow with the iteration count on
    # these worse-conditioned systems (P: ~65 iterations), so the unique solution is
    # compared on a converged pair (tol 1e-12 on both sides)
    if it <= 30:
        assert _rel(x.cpu().numpy(), x_ref) <= 1e-9
    x2, st2 = ctx.pcg(torch.from_numpy(b).cuda(), tol=1e-12)
    x2_ref, _, ok2, _ = opcg.pcg(A, Pinv, b, tol=1e-12)
    assert ok2 and st2["status"] == 0
    assert _rel(x2.cpu().numpy(), x2_ref) <= 1e-9


def test_geo_pg_fewer_iterations(torch_cuda):
    """Table 2's claim (PAPER.md 1226-1228): P^G cuts the CG iterations on the rotated
    quarter annulus several times against P."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    its = []
    for pc in (ls.LS_PRECOND_P, ls.LS_PRECOND_PG):
        ctx, geo, sf, tf = _setup("annulus3d", 3, [8, 8, 8, 8], pc)
        b = torch.from_numpy(synth.residual(ctx.shape, 0)).cuda()
        _, st = ctx.pcg(b, tol=1e-8)
        assert st["status"] == 0
        its.append(st["iters"])
    assert its[1] * 3 <= its[0], its


def test_geo_errors(torch_cuda):
    import paper_1809_10026_b200 as ls
    geo = synth.quarter_annulus()
    ctx = ls.Context(2, 2, [4, 4, 4], geometry=geo, precond=ls.LS_PRECOND_PG)
    import torch
    b = torch.zeros(ctx.shape, dtype=torch.float64, device="cuda")
    with pytest.raises(ls.LSError) as e:
        ctx.rhs(0, b)
    assert e.value.code == ls.LS_ENOTSUP
    bad = dict(geo)
    bad["knots"] = [np.array([0.0, 0.0, 1.0]), geo["knots"][1]]       # too short for degree 1
    with pytest.raises(ls.LSError) as e:
        ls.Context(2, 2, [4, 4, 4], geometry=bad)
    assert e.value.code == ls.LS_EINVAL
    neg = dict(geo)
    neg["weights"] = -geo["weights"]
    with pytest.raises(ls.LSError):
        ls.Context(2, 2, [4, 4, 4], geometry=neg)
    with pytest.raises(ls.LSError):
        ls.Context(3, 7, [2, 2, 2, 2], geometry=synth.revolved_quarter_annulus())   # (p+1)^3 > 343
    # a folded map (one control point dragged across the domain: det J changes sign)
    fold = dict(geo)
    c = geo["ctrl"].copy()
    c[0] = [3.0, 3.0]
    fold["ctrl"] = c
    with pytest.raises(ls.LSError) as e:
        ls.Context(2, 2, [4, 4, 4], geometry=fold)
    assert e.value.code == ls.LS_EINVAL
    # b = 0 -> x = 0, 0 iterations
    x, st = ctx.pcg(b)
    assert st["iters"] == 0 and float(x.abs().max()) == 0.0


@pytest.mark.parametrize("p,pt,n_elems", [(2, 2, [5, 6, 7]), (3, 3, [8, 8, 8]), (3, 2, [6, 9, 5])])
def test_geo_rhs_kind2_matches_oracle(torch_cuda, p, pt, n_elems):
    """ls_rhs kind 2 on the quarter annulus (PAPER.md 1128-1129): the separable device
    evaluation against the oracle's direct space-time quadrature of f (d_t B_i - Lap B_i)."""
    import paper_1809_10026_b200 as ls
    from oracle import geo_rhs as R
    geo = synth.quarter_annulus()
    ctx = ls.Context(2, (p, pt), n_elems, geometry=geo, precond=ls.LS_PRECOND_PG)
    b = ctx.rhs(2).cpu().numpy()
    b_ref = R.load_vector(geo, n_elems[:2], p, n_elems[2], pt)
    assert _rel(b, b_ref) <= 1e-12


def test_geo_energy_error_and_convergence(torch_cuda):
    """ls_energy_error kind 2 equals the oracle's ||f||^2 - 2 b.x + x.A x, and the GPU
    solutions converge at O(h^{p-1}) in the least-squares energy norm (Fig. 2 setting)."""
    import paper_1809_10026_b200 as ls
    from oracle import geo_rhs as R
    geo = synth.quarter_annulus()
    for p, want in ((2, 1.0), (3, 2.0)):
        errs = []
        for ne in (8, 16, 32):
            ctx = ls.Context(2, p, [ne] * 3, geometry=geo, precond=ls.LS_PRECOND_PG)
            b = ctx.rhs(2)
            x, st = ctx.pcg(b, tol=1e-12)
            assert st["status"] == 0
            e = ctx.energy_error(2, x)
            if ne == 8:
                f2 = R.f_norm2(geo, [ne, ne], p, ne, p)
                assert abs(e["f2"] - f2) <= 1e-12 * f2
                sf = G.space_factors_physical(geo, [ne, ne], p)
                tf = uv.time_factors(ne, p)
                xh = x.cpu().numpy()
                J = f2 - 2 * np.sum(R.load_vector(geo, [ne, ne], p, ne, p) * xh) + np.sum(xh * G.apply_A_geo(xh, sf, tf))
                assert abs(e["J"] - J) <= 1e-9 * f2
            errs.append(np.sqrt(e["J"] / e["f2"]))
        rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert abs(rates[-1] - want) < 0.15, (p, errs, rates)


def test_geo_rhs_kind_errors(torch_cuda):
    import paper_1809_10026_b200 as ls
    c3 = ls.Context(3, 2, [2, 2, 2, 3], geometry=synth.revolved_quarter_annulus())
    with pytest.raises(ls.LSError) as e:
        c3.rhs(2)
    assert e.value.code == ls.LS_ENOTSUP
    cube = ls.Context(2, 2, [4, 4, 4])
    with pytest.raises(ls.LSError) as e:
        cube.rhs(2)
    assert e.value.code == ls.LS_EINVAL


@pytest.mark.parametrize("p,n_elems", [(2, [3, 4, 3, 5]), (3, [4, 3, 4, 4])])
def test_geo_rhs_kind3_matches_oracle(torch_cuda, p, n_elems):
    """ls_rhs kind 3 on the rotated quarter annulus (PAPER.md 1221, reading c23) against the
    oracle's direct space-time quadrature."""
    import paper_1809_10026_b200 as ls
    from oracle import geo_rhs as R
    geo = synth.revolved_quarter_annulus()
    ctx = ls.Context(3, p, n_elems, geometry=geo)
    b = ctx.rhs(3).cpu().numpy()
    b_ref = R.load_vector(geo, n_elems[:3], p, n_elems[3], p, kind=3)
    assert _rel(b, b_ref) <= 1e-12
    x = torch_cuda.from_numpy(synth.residual(ctx.shape, 9)).cuda()
    e = ctx.energy_error(3, x)
    assert abs(e["f2"] - R.f_norm2(geo, n_elems[:3], p, n_elems[3], p, kind=3)) <= 1e-12 * e["f2"]


@pytest.mark.parametrize("ne,p", [(8, 2), (8, 3), (16, 2), (16, 3)])
def test_geo_table2_iterations(torch_cuda, golden_loader, ne, p):
    """CG iterations with P and P^G on the rotated quarter annulus against Table 2
    (PAPER.md 1244-1262), forcing of kind 3 (reading c23: homogeneous data, so within 20 %)."""
    import paper_1809_10026_b200 as ls
    tab = golden_loader("table2_iterations.json")
    geo = synth.revolved_quarter_annulus()
    for pc, key in ((ls.LS_PRECOND_P, "P"), (ls.LS_PRECOND_PG, "PG")):
        ctx = ls.Context(3, p, [ne] * 4, geometry=geo, precond=pc)
        _, st = ctx.pcg(ctx.rhs(3), tol=1e-8)
        ref = tab[key][str(ne)][str(p)]
        assert st["status"] == 0 and abs(st["iters"] - ref) <= 0.2 * ref, (key, st["iters"], ref)


@pytest.mark.parametrize("n_el,p", [(32, 3), (64, 2)])
def test_geo_fullsize_properties(torch_cuda, n_el, p):
    """At the bench sizes (revolved quarter annulus, beyond the oracle's reach): A and
    (P^G)^{-1} are symmetric (x.Ay = y.Ax) and positive, on seeded inputs, in the launch
    configuration bench.py times; the PCG solve of the kind-3 forcing reaches its true
    residual."""
    torch = torch_cuda
    import paper_1809_10026_b200 as ls
    ctx = ls.Context(3, p, [n_el] * 4, geometry=synth.revolved_quarter_annulus(), precond=ls.LS_PRECOND_PG)
    x = torch.from_numpy(synth.residual(ctx.shape, 1)).cuda()
    y = torch.from_numpy(synth.residual(ctx.shape, 2)).cuda()
    Ax, Ay = ctx.matvec(x), ctx.matvec(y)
    xAy, yAx = float((x * Ay).sum()), float((y * Ax).sum())
    assert abs(xAy - yAx) <= 1e-12 * float(x.norm() * Ay.norm())
    assert float((x * Ax).sum()) > 0
    Px, Py = ctx.fd_apply(x), ctx.fd_apply(y)
    assert abs(float((x * Py).sum()) - float((y * Px).sum())) <= 1e-10 * float(x.norm() * Py.norm())
    assert float((x * Px).sum()) > 0
    _, st = ctx.pcg(ctx.rhs(3), tol=1e-8)
    assert st["status"] == 0 and st["true_rel_res"] < 1e-7
