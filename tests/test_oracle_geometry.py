"""Pins for oracle/geometry.py and oracle/geo_precond.py (SURVEY 8(f) NEXT-1/NEXT-2:
mapped domains, PAPER.md 226-300, 686-703, 969-1045).

Closed forms: the exact NURBS annulus radius, the quarter-annulus area 3 pi / 4 and
the Pappus volume of the revolved domain; the Laplacian of polynomials in x through
the chain rule; affine maps, whose physical factors and P^G are scaled parametric
ones; finite differences of the map; brute-force dense solves of P^G; the original
least-squares form (PAPER.md 406) against eq:A_kron with the physical factors."""

import warnings

import numpy as np
import pytest
import scipy.sparse as sp

import synth
from oracle import geometry as G, geo_precond as GP, univariate as uv, fd, pcg

warnings.filterwarnings("ignore", category=DeprecationWarning)


def test_annulus_exact_radius():
    """The rational quadratic arc is exact: |F(eta)| = 1 + eta_1 (PAPER.md 1219)."""
    e = np.linspace(0.0, 1.0, 11)
    g = G.eval_map(synth.quarter_annulus(), [e, e])
    eta1 = np.tile(e, 11)
    assert np.max(np.abs(np.linalg.norm(g["X"], axis=1) - (1 + eta1))) < 1e-14
    assert np.all(g["X"] >= -1e-15)
    # revolved: distance from the axis {y=-1, z=0} minus 1 is the planar y, so the
    # planar radius is recovered, and the revolution angle stays in [0, pi/2]
    g3 = G.eval_map(synth.revolved_quarter_annulus(), [e, e, e])
    x, yy, z = g3["X"].T
    y = np.hypot(yy + 1, z) - 1
    eta1 = np.tile(e, 121)
    assert np.max(np.abs(np.hypot(x, y) - (1 + eta1))) < 1e-14
    ang = np.arctan2(z, yy + 1)
    assert ang.min() > -1e-14 and ang.max() < np.pi / 2 + 1e-14


@pytest.mark.parametrize("name", ["annulus2d", "annulus3d"])
def test_map_derivatives_finite_differences(name):
    geo = synth.GEOMETRIES[name]()
    d = geo["d"]
    e = np.linspace(0.07, 0.93, 4)
    g = G.eval_map(geo, [e] * d)
    h = 1e-6
    for j in range(d):
        pp, pm = [e] * d, [e] * d
        pp[j], pm[j] = e + h, e - h
        a, b = G.eval_map(geo, pp), G.eval_map(geo, pm)
        assert np.max(np.abs((a["X"] - b["X"]) / (2 * h) - g["Jac"][:, :, j])) < 1e-7
        assert np.max(np.abs((a["Jac"] - b["Jac"]) / (2 * h) - g["Hes"][:, :, :, j])) < 1e-7


@pytest.mark.parametrize("name", ["annulus2d", "annulus3d"])
def test_laplacian_chain_rule_on_polynomials(name):
    """v(x) = |x|^2 + x_1^3: Lap v = 2d + 6 x_1, fed through v^ = v o F (forward chain
    rule from the map's own derivatives) and the inverse chain rule."""
    geo = synth.GEOMETRIES[name]()
    d = geo["d"]
    e = np.linspace(0.05, 0.95, 5)
    g = G.eval_map(geo, [e] * d)
    X = g["X"]
    gx = 2 * X.copy()
    gx[:, 0] += 3 * X[:, 0] ** 2
    H = np.zeros((len(X), d, d))
    H[:] = 2 * np.eye(d)
    H[:, 0, 0] += 6 * X[:, 0]
    vg = np.einsum("qm,qmj->qj", gx, g["Jac"])
    vh = (np.einsum("qmn,qmj,qnk->qjk", H, g["Jac"], g["Jac"])
          + np.einsum("qm,qmjk->qjk", gx, g["Hes"]))
    lap = G.physical_laplacian(vg, vh, g["Jac"], g["Hes"])
    assert np.max(np.abs(lap - (2 * d + 6 * X[:, 0]))) < 1e-12


def test_area_and_volume():
    """Sum of the unconstrained mass matrix = |Omega| (partition of unity):
    3 pi / 4 for the quarter annulus; Pappus for the revolved one:
    |Omega| * (pi / 2) * (distance of the centroid 28 / (9 pi) from the axis y = -1)."""
    sf = G.space_factors_physical(synth.quarter_annulus(), [8, 8], 3, drop_boundary=False)
    assert abs(sf["M"].sum() - 3 * np.pi / 4) < 1e-12
    vol = 3 * np.pi / 4 * np.pi / 2 * (28 / (9 * np.pi) + 1)
    errs = []
    for ne in (2, 4, 8):
        sf3 = G.space_factors_physical(synth.revolved_quarter_annulus(), [ne] * 3, 2,
                                       drop_boundary=False)
        errs.append(abs(sf3["M"].sum() - vol))
    assert errs[-1] < 5e-9 and errs[0] > errs[1] > errs[2]


def test_affine_map_closed_forms():
    """x = (a_1 eta_1, a_2 eta_2): M_s = a1 a2 M(x)M, L_s = (a2/a1) M(x)K + (a1/a2) K(x)M,
    J_s = (a2/a1^3) M(x)J + (a1/a2^3) J(x)M + (G^T(x)G + G(x)G^T)/(a1 a2)."""
    a = [2.0, 0.5]
    ne, p = [3, 4], 3
    sfa = G.space_factors_physical(synth.affine_box(a), ne, p)
    s = [uv.space_factors(ne[k], p) for k in range(2)]
    kr = lambda A, B: sp.kron(sp.csr_matrix(A), sp.csr_matrix(B))
    M = kr(s[1]["M"], s[0]["M"]) * a[0] * a[1]
    L = kr(s[1]["M"], s[0]["K"]) * a[1] / a[0] + kr(s[1]["K"], s[0]["M"]) * a[0] / a[1]
    J = (kr(s[1]["M"], s[0]["J"]) * a[1] / a[0] ** 3 + kr(s[1]["J"], s[0]["M"]) * a[0] / a[1] ** 3
         + (kr(s[1]["G"].T, s[0]["G"]) + kr(s[1]["G"], s[0]["G"].T)) / (a[0] * a[1]))
    for X, Y in ((sfa["M"], M), (sfa["L"], L), (sfa["J"], J)):
        assert abs(X - Y).max() <= 1e-13 * abs(Y).max()


@pytest.mark.parametrize("name,ne,p,net,pt", [("annulus2d", [3, 4], 3, 3, 2),
                                              ("annulus2d", [2, 3], 2, 2, 3),
                                              ("annulus3d", [2, 2, 3], 2, 2, 2)])
def test_original_form_equals_kron_form(name, ne, p, net, pt):
    """Direct space-time quadrature of A(v,w) = int int (d_t v - Lap v)(d_t w - Lap w)
    (PAPER.md 406) = K_t(x)M_s + M_t(x)J_s + W_t(x)L_s with the physical factors
    (eq:A_kron; the integration by parts of eq:equivalent_A holds on Omega).  A is SPD."""
    geo = synth.GEOMETRIES[name]()
    sf = G.space_factors_physical(geo, ne, p)
    tf = uv.time_factors(net, pt)
    Ad = G.dense_A_original_form_geo(geo, ne, p, net, pt)
    nt = tf["Mt"].shape[0]
    shape = (nt,) + tuple(reversed(sf["n_s"]))
    I = np.eye(Ad.shape[0])
    Ak = np.array([G.apply_A_geo(I[:, j].reshape(shape), sf, tf).ravel()
                   for j in range(Ad.shape[0])]).T
    assert np.abs(Ad - Ak).max() <= 1e-12 * np.abs(Ad).max()
    np.linalg.cholesky(Ad)


def test_separable_fit_exact_on_separable_data():
    """Products of univariate functions are recovered exactly (reading c21)."""
    rng = np.random.default_rng(3)
    n = [3, 4, 5]
    m = [rng.uniform(0.5, 2, k) for k in n]
    o = [rng.uniform(0.5, 2, k) for k in n]

    def outer(vs):
        out = vs[-1]
        for v in reversed(vs[:-1]):
            out = np.multiply.outer(out, v)
        return out

    c_tau = outer(m)
    c_k = [outer([o[j] if j == k else m[j] for j in range(3)]) for k in range(3)]
    mu, om = GP.separable_fit(c_tau, c_k)
    assert np.allclose(outer(mu), c_tau, rtol=1e-12)
    for k in range(3):
        assert np.allclose(outer([om[j] if j == k else mu[j] for j in range(3)]), c_k[k],
                           rtol=1e-12)


def test_PG_affine_closed_form():
    """Affine box: c_tau = a1 a2 a3, c_k = a1 a2 a3 / a_k^4 (constant, exactly separable),
    so Pbar^G = K_t (x) (prod a) M^ + M_t (x) sum_k (prod a / a_k^4) J_(k) and its
    diagonal scaling uses diag(A) of the physical factors."""
    a = [2.0, 0.5, 1.5]
    ne, p = [2, 3, 2], 2
    geo = synth.affine_box(a)
    c_tau, c_k = GP.midpoint_coefficients(geo, ne)
    pa = np.prod(a)
    assert np.allclose(c_tau, pa, rtol=1e-14)
    for k in range(3):
        assert np.allclose(c_k[k], pa / a[k] ** 4, rtol=1e-13)
    sf = G.space_factors_physical(geo, ne, p)
    tf = uv.time_factors(2, p)
    data = GP.setup(geo, ne, p, tf, GP.A_diagonal(sf, tf))
    Pd = GP.dense_PG(data)
    s = [uv.space_factors(ne[k], p) for k in range(3)]
    kron = lambda mats: np.kron(np.kron(np.kron(mats[0], mats[1]), mats[2]), mats[3])
    Pbar = kron([tf["Kt_hat"], s[2]["M"], s[1]["M"], s[0]["M"]]) * pa
    for k in range(3):
        mats = [tf["Mt_hat"]] + [s[j]["J"] if j == k else s[j]["M"] for j in (2, 1, 0)]
        Pbar = Pbar + kron(mats) * pa / a[k] ** 4
    D12 = np.sqrt(np.diag(G.dense_A_original_form_geo(geo, ne, p, 2, p)) / np.diag(Pbar))
    expect = D12[:, None] * Pbar * D12[None, :]
    assert np.abs(Pd - expect).max() <= 1e-12 * np.abs(expect).max()


@pytest.mark.parametrize("name,ne,p", [("annulus2d", [4, 3], 2), ("annulus3d", [2, 3, 2], 3)])
def test_PG_fd_equals_dense_solve(name, ne, p):
    """Algorithm 1 on Pbar^G with the D^{-1/2} scaling = brute-force dense solve of
    P^G = D^{1/2} Pbar^G D^{1/2} (PAPER.md 1040-1045)."""
    geo = synth.GEOMETRIES[name]()
    sf = G.space_factors_physical(geo, ne, p)
    tf = uv.time_factors(3, p)
    data = GP.setup(geo, ne, p, tf, GP.A_diagonal(sf, tf))
    assert all(np.all(m > 0) for m in data["mu"]) and all(np.all(o > 0) for o in data["omega"])
    nt = tf["Mt"].shape[0]
    shape = (nt,) + tuple(reversed(sf["n_s"]))
    r = synth.residual(shape, 5)
    z = GP.apply(r, data)
    z_ref = np.linalg.solve(GP.dense_PG(data), r.ravel()).reshape(shape)
    assert np.linalg.norm(z - z_ref) <= 1e-10 * np.linalg.norm(z_ref)
    # diag(P^G) = diag(A) by construction of D
    assert np.allclose(np.diag(GP.dense_PG(data)), GP.A_diagonal(sf, tf).ravel(), rtol=1e-12)


def test_interpolation_reading_c22():
    v = np.array([1.0, 3.0, 2.0, 5.0])
    x = np.array([0.0, 0.125, 0.25, 0.375, 0.5, 1.0])
    assert np.allclose(GP.interpolate_factor(v, x), [1.0, 1.0, 2.0, 3.0, 2.5, 5.0])


def test_PG_reduces_iterations_on_revolved_annulus():
    """Table 2 (PAPER.md 1244-1262): on the rotated quarter annulus P^G needs several
    times fewer CG iterations than P (107 -> 24 at n_sub = 8, p = 2 there, with the
    paper's manufactured data; seeded random right-hand side here)."""
    geo = synth.revolved_quarter_annulus()
    ne, p = 4, 2
    sf = G.space_factors_physical(geo, [ne] * 3, p)
    tf = uv.time_factors(ne, p)
    nt = tf["Mt"].shape[0]
    shape = (nt,) + tuple(reversed(sf["n_s"]))
    pg = GP.setup(geo, [ne] * 3, p, tf, GP.A_diagonal(sf, tf))
    plain = fd.setup([uv.space_factors(ne, p)] * 3, tf)
    b = synth.residual(shape, 0)
    A = lambda x: G.apply_A_geo(x, sf, tf)
    _, it_p, ok1, _ = pcg.pcg(A, lambda r: fd.fd_apply(r, plain), b)
    _, it_g, ok2, _ = pcg.pcg(A, lambda r: GP.apply(r, pg), b)
    assert ok1 and ok2
    assert it_g * 3 <= it_p, (it_p, it_g)


def test_annulus_benchmark_solution_has_homogeneous_data():
    """u = -(x^2+y^2-1)(x^2+y^2-4) x y^2 sin(pi t) (PAPER.md 1129) vanishes on the whole
    boundary of the quarter annulus and at t = 0, so no lifting is needed; the sympy f
    equals d_t u - Lap u by central differences."""
    from oracle import geo_rhs as R
    u, f = R.annulus_solution()
    geo = synth.quarter_annulus()
    e = np.linspace(0.0, 1.0, 9)
    for side in ([np.array([0.0]), e], [np.array([1.0]), e], [e, np.array([0.0])], [e, np.array([1.0])]):
        X = G.eval_map(geo, side)["X"]
        assert np.max(np.abs(u(X[:, 0], X[:, 1], 0.7))) < 1e-13
    X = G.eval_map(geo, [np.linspace(0.1, 0.9, 5)] * 2)["X"]
    assert np.max(np.abs(u(X[:, 0], X[:, 1], 0.0))) == 0.0
    h = 1e-4
    x, y, t = X[:, 0], X[:, 1], 0.37
    dt = (u(x, y, t + h) - u(x, y, t - h)) / (2 * h)
    lap = (u(x + h, y, t) + u(x - h, y, t) + u(x, y + h, t) + u(x, y - h, t) - 4 * u(x, y, t)) / h ** 2
    assert np.max(np.abs(f(x, y, t) - (dt - lap))) < 1e-5 * np.max(np.abs(f(x, y, t)))


def test_annulus_energy_error_converges_at_rate_p_minus_1():
    """Least-squares energy error ||(d_t - Lap)(u - u_h)|| on the quarter annulus (the
    setting of Fig. 2, PAPER.md 1128-1139) decreases as O(h^{p-1}) (Thm teo:a-priori)."""
    from oracle import geo_rhs as R
    geo = synth.quarter_annulus()
    for p, want in ((2, 1.0), (3, 2.0)):
        errs = []
        for ne in (4, 8, 16):
            sf = G.space_factors_physical(geo, [ne, ne], p)
            tf = uv.time_factors(ne, p)
            b = R.load_vector(geo, [ne, ne], p, ne, p)
            f2 = R.f_norm2(geo, [ne, ne], p, ne, p)
            A = lambda v: G.apply_A_geo(v, sf, tf)
            data = GP.setup(geo, [ne, ne], p, tf, GP.A_diagonal(sf, tf))
            x, _, ok, _ = pcg.pcg(A, lambda r: GP.apply(r, data), b, tol=1e-12)
            assert ok
            J = f2 - 2 * np.sum(b * x) + np.sum(x * A(x))
            assert J > 0 and np.sum(x * A(x)) <= f2     # J(c) >= 0, J(0) = ||f||^2
            errs.append(np.sqrt(J / f2))
        rates = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
        assert abs(rates[-1] - want) < 0.15, (p, errs, rates)


def test_revolved_forcing_and_table2_iterations(golden_loader):
    """Kind 3 (PAPER.md 1219-1221): f = -Lap u for the time-independent u of the rotated
    quarter annulus (central differences), and CG iteration counts with P and P^G on the
    n_sub = 8, p = 2 mesh against Table 2 (PAPER.md 1244-1262).  Reading c23: homogeneous
    data instead of the paper's lifting, so the counts agree within 20 %, not exactly."""
    from oracle import geo_rhs as R
    u, f = R.revolved_solution()
    geo = synth.revolved_quarter_annulus()
    X = G.eval_map(geo, [np.linspace(0.1, 0.9, 3)] * 3)["X"]
    x, y, z = X.T
    h = 1e-3
    lap = sum((u(*(X + h * np.eye(3)[k]).T, 0.0) + u(*(X - h * np.eye(3)[k]).T, 0.0) - 2 * u(x, y, z, 0.0)) / h ** 2
              for k in range(3))
    assert np.max(np.abs(f(x, y, z, 0.3) + lap)) < 1e-5 * np.max(np.abs(lap))
    tab = golden_loader("table2_iterations.json")
    ne, p = 8, 2
    sf = G.space_factors_physical(geo, [ne] * 3, p)
    tf = uv.time_factors(ne, p)
    b = R.load_vector(geo, [ne] * 3, p, ne, p, kind=3)
    A = lambda v: G.apply_A_geo(v, sf, tf)
    plain = fd.setup([uv.space_factors(ne, p)] * 3, tf)
    pg = GP.setup(geo, [ne] * 3, p, tf, GP.A_diagonal(sf, tf))
    _, it_p, _, _ = pcg.pcg(A, lambda r: fd.fd_apply(r, plain), b)
    _, it_g, _, _ = pcg.pcg(A, lambda r: GP.apply(r, pg), b)
    for it, ref in ((it_p, tab["P"]["8"]["2"]), (it_g, tab["PG"]["8"]["2"])):
        assert abs(it - ref) <= 0.2 * ref, (it, ref)
