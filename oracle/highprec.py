"""Exact / high-precision references for the setup of Algorithm 1 (oracle; test
infrastructure -- only tests/ and tools/make_golden_eig.py use it).

Used to pin the extended-precision setup of reading c17 against
something other than the oracle's own LAPACK + refinement:

* ``exact_full_matrices`` -- the univariate factor matrices M, K, J with EXACT
  rational entries (Python ``fractions.Fraction``).  The B-splines are built by
  the Cox-de Boor recursion (PAPER.md 148-152) as polynomial pieces on every
  knot span; the products of (derivatives of) two pieces are integrated in
  closed form (antiderivative at the span ends).  No quadrature, no rounding.
* ``space_pencil`` / ``time_pencil`` -- the constrained pencils (eq:basis_par,
  PAPER.md 266-267): (J-hat, M-hat) on i = 2..m-1 and (K_t-hat, M_t-hat) on
  i = 2..m (PAPER.md 738-757), exact.
* ``eig_bisect`` -- the k-th eigenvalue of a symmetric-definite banded pencil
  (A, B) (eq:eig_dec, PAPER.md 942-945) by bisection on Sylvester's law of
  inertia: #(lambda < sigma) = #negative pivots of the LDL^T factorisation of
  A - sigma B (B SPD).  mpmath at ``dps`` digits; a different algorithm from
  the oracle's (LAPACK + Ogita-Aishima refinement).
* ``solve_P`` -- z = P^{-1} r with P = K_t (x) M_s + M_t (x) J_s-tilde
  (PAPER.md 733, 752-757) assembled entry by entry in mpmath and solved by a
  banded Cholesky, unknowns ordered time-fastest so the half-bandwidth is
  small.  The brute-force definition of fd_apply (reading c2), in high
  precision.

Everything here is plain Python loops; sizes are the small / univariate ones of
tests/golden/eig_mpmath.json.
"""

from fractions import Fraction

import mpmath


# ---------------------------------------------------------------- polynomials
# A polynomial is a list of Fraction coefficients, c[k] multiplies u^k (local coordinate).

def _padd(a, b):
    n = max(len(a), len(b))
    return [(a[k] if k < len(a) else 0) + (b[k] if k < len(b) else 0) for k in range(n)]


def _pmul(a, b):
    out = [Fraction(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        if x == 0:
            continue
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def _pder(a):
    return [k * a[k] for k in range(1, len(a))] or [Fraction(0)]


def _pint01(a):
    """int_0^1 a(u) du, exactly."""
    return sum((c / (k + 1) for k, c in enumerate(a)), Fraction(0))


def uniform_open_knots(n_el, p):
    """Open knot vector with n_el uniform elements (PAPER.md 144-147, 1111-1112),
    exact rationals."""
    return [Fraction(0)] * (p + 1) + [Fraction(i, n_el) for i in range(1, n_el)] + [Fraction(1)] * (p + 1)


def bspline_pieces(knots, p):
    """pieces[s][i] = polynomial in the local coordinate u in [0, 1]
    (eta = xi_s + h_s u) of b_{i,p} on the knot span [xi_s, xi_{s+1}) (0-based i),
    for every non-empty span s.  Cox-de Boor (PAPER.md 148-152):
    b_{i,0} = 1 on [xi_i, xi_{i+1}); b_{i,q} = (eta - xi_i)/(xi_{i+q} - xi_i) b_{i,q-1}
    + (xi_{i+q+1} - eta)/(xi_{i+q+1} - xi_{i+1}) b_{i+1,q-1}, 0/0 = 0."""
    n0 = len(knots) - 1
    out = {}
    for s in range(n0):
        lo, h = knots[s], knots[s + 1] - knots[s]
        if h == 0:
            continue
        B = [[Fraction(1)] if i == s else [Fraction(0)] for i in range(n0)]
        for q in range(1, p + 1):
            Bq = []
            for i in range(n0 - q):
                term = [Fraction(0)]
                den = knots[i + q] - knots[i]
                if den != 0 and any(B[i]):
                    term = _padd(term, _pmul([(lo - knots[i]) / den, h / den], B[i]))
                den = knots[i + q + 1] - knots[i + 1]
                if den != 0 and any(B[i + 1]):
                    term = _padd(term, _pmul([(knots[i + q + 1] - lo) / den, -h / den], B[i + 1]))
                Bq.append(term)
            B = Bq
        out[s] = (h, B)
    return out


def exact_full_matrices(n_el, p):
    """Unconstrained m x m M = int b_i b_j, K = int b_i' b_j', J = int b_i'' b_j''
    (PAPER.md 738-757) as exact Fractions, by closed-form integration of the
    polynomial pieces (d/d eta = h^{-1} d/du, d eta = h du).  Returns (M, K, J)
    as lists of lists."""
    knots = uniform_open_knots(n_el, p)
    m = len(knots) - p - 1
    M = [[Fraction(0)] * m for _ in range(m)]
    K = [[Fraction(0)] * m for _ in range(m)]
    J = [[Fraction(0)] * m for _ in range(m)]
    for s, (h, B) in bspline_pieces(knots, p).items():
        live = [i for i in range(m) if any(B[i])]
        d0 = {i: B[i] for i in live}
        d1 = {i: _pder(B[i]) for i in live}
        d2 = {i: _pder(d1[i]) for i in live}
        for i in live:
            for j in live:
                if j < i:
                    continue
                vm = h * _pint01(_pmul(d0[i], d0[j]))
                vk = _pint01(_pmul(d1[i], d1[j])) / h
                vj = _pint01(_pmul(d2[i], d2[j])) / h ** 3
                for A, v in ((M, vm), (K, vk), (J, vj)):
                    A[i][j] += v
                    if j != i:
                        A[j][i] += v
    return M, K, J


def space_pencil(n_el, p):
    """(J-hat, M-hat) on the Dirichlet-constrained functions i = 2..m-1 (PAPER.md 266)."""
    M, _, J = exact_full_matrices(n_el, p)
    sl = lambda A: [row[1:-1] for row in A[1:-1]]
    return sl(J), sl(M)


def time_pencil(n_el, p):
    """(K_t-hat, M_t-hat) on the initial-condition-constrained functions i = 2..m (PAPER.md 267)."""
    M, K, _ = exact_full_matrices(n_el, p)
    sl = lambda A: [row[1:] for row in A[1:]]
    return sl(K), sl(M)


def round_fp64(A):
    """Entry-wise correctly rounded fp64 (float(Fraction) rounds to nearest)."""
    return [[float(x) for x in row] for row in A]


# ---------------------------------------------------------------- eigenvalues

def _to_mp(A):
    return [[mpmath.mpf(x.numerator) / x.denominator if isinstance(x, Fraction) else mpmath.mpf(x)
             for x in row] for row in A]


def _bandwidth(A):
    n = len(A)
    return max((j - i for i in range(n) for j in range(i, n) if A[i][j] != 0), default=0)


def inertia_count(A, B, sigma, w):
    """#eigenvalues of (A, B) below sigma = #negative pivots of LDL^T(A - sigma B)
    (Sylvester; B SPD).  A, B mpmath lists, half-bandwidth w."""
    n = len(A)
    L = [dict() for _ in range(n)]   # L[j][k] for k in [j-w, j)
    D = [None] * n
    neg = 0
    for j in range(n):
        lo = max(0, j - w)
        # column j of L below the diagonal is computed when rows are reached;
        # row-oriented: l_jk = (c_jk - sum_{m<k} l_jm l_km d_m) / d_k
        for k in range(lo, j):
            s = A[j][k] - sigma * B[j][k]
            for mm in range(max(lo, k - w), k):
                s -= L[j].get(mm, 0) * L[k].get(mm, 0) * D[mm]
            L[j][k] = s / D[k]
        s = A[j][j] - sigma * B[j][j]
        for k in range(lo, j):
            s -= L[j][k] * L[j][k] * D[k]
        if s == 0:   # sigma is an eigenvalue of a leading block: perturb (standard Sturm rule)
            s = -mpmath.eps * (abs(A[j][j]) + abs(sigma * B[j][j]))
        D[j] = s
        if s < 0:
            neg += 1
    return neg


def eig_bisect(A, B, ks, dps=50, rel=mpmath.mpf(10) ** -40):
    """Eigenvalues number ks (1-based, ascending) of the SPD pencil (A, B) to
    relative accuracy ``rel`` by inertia bisection (mpmath, ``dps`` digits)."""
    with mpmath.workdps(dps):
        Am, Bm = _to_mp(A), _to_mp(B)
        w = max(_bandwidth(A), _bandwidth(B))
        out = []
        for k in ks:
            lo, hi = mpmath.mpf(0), 1 + mpmath.sqrt(2) / 1000   # not a dyadic rational
            while inertia_count(Am, Bm, hi, w) < k:
                lo, hi = hi, hi * 2
            while hi - lo > rel * hi:
                mid = (lo + hi) / 2
                if inertia_count(Am, Bm, mid, w) >= k:
                    hi = mid
                else:
                    lo = mid
            out.append((lo + hi) / 2)
        return out


# ---------------------------------------------------------------- P^{-1} r

def solve_P(space, time, r, dps=40):
    """z = P^{-1} r, P = K_t (x) M_s + M_t (x) J_s-tilde (PAPER.md 733, 752-757),
    M_s = M_d (x) .. (x) M_1, J_s-tilde = sum_k M_d (x) .. J_k .. (x) M_1.

    ``space`` = [(J_k, M_k) for k = 1..d], ``time`` = (K_t, M_t): matrices as
    lists (Fraction or float).  ``r`` is a flat sequence in the paper's colex
    order (direction 1 fastest, time slowest, PAPER.md 271-285).  Every entry of
    P is formed from its Kronecker definition (a sum over the d + 1 terms of
    products of univariate entries); the system is solved by a banded Cholesky
    with the unknowns reordered so that the longest axis is the slowest (small
    half-bandwidth).  Returns z as a list of mpf in colex order."""
    d = len(space)
    with mpmath.workdps(dps):
        # axes: 0 = time, k = direction k; per axis the matrices of each Kronecker term
        Kt, Mt = _to_mp(time[0]), _to_mp(time[1])
        Sp = [(_to_mp(Jk), _to_mp(Mk)) for Jk, Mk in space]
        terms = [[Kt] + [Sp[k][1] for k in range(d)]]
        for j in range(d):
            terms.append([Mt] + [Sp[k][0] if k == j else Sp[k][1] for k in range(d)])
        ext = [len(Kt)] + [len(Sp[k][1]) for k in range(d)]
        band = [max(j - i for T in terms for i in range(ext[a]) for j in range(ext[a]) if T[a][i][j] != 0)
                for a in range(d + 1)]
        order = sorted(range(d + 1), key=lambda a: -ext[a])      # slowest first
        stride, s_ = [0] * (d + 1), 1
        for a in reversed(order):
            stride[a] = s_
            s_ *= ext[a]
        N = s_
        w = sum(band[a] * stride[a] for a in range(d + 1))
        colex_stride, s_ = [0] * (d + 1), 1
        for a in list(range(1, d + 1)) + [0]:                  # direction 1 fastest, time slowest
            colex_stride[a] = s_
            s_ *= ext[a]

        def midx(i):
            return [(i // stride[a]) % ext[a] for a in range(d + 1)]
        multi = [midx(i) for i in range(N)]

        def entry(x, y):
            ix, iy = multi[x], multi[y]
            tot = mpmath.mpf(0)
            for T in terms:
                v = mpmath.mpf(1)
                for a in range(d + 1):
                    v *= T[a][ix[a]][iy[a]]
                    if v == 0:
                        break
                tot += v
            return tot

        L = [dict() for _ in range(N)]
        for j in range(N):
            lo = max(0, j - w)
            for k in range(lo, j + 1):
                s = entry(j, k)
                Lj, Lk = L[j], L[k]
                for mm, lk in Lk.items():
                    if mm < k:
                        lj = Lj.get(mm)
                        if lj is not None:
                            s -= lj * lk
                if k == j:
                    if s <= 0:
                        raise ValueError("P not SPD")
                    Lj[j] = mpmath.sqrt(s)
                elif s != 0:
                    Lj[k] = s / Lk[k]
        perm = [sum(multi[i][a] * colex_stride[a] for a in range(d + 1)) for i in range(N)]
        y = [None] * N
        for j in range(N):
            s = mpmath.mpf(r[perm[j]])
            for k, v in L[j].items():
                if k < j:
                    s -= v * y[k]
            y[j] = s / L[j][j]
        x = [None] * N
        Lt = [dict() for _ in range(N)]
        for j in range(N):
            for k, v in L[j].items():
                if k < j:
                    Lt[k][j] = v
        for j in reversed(range(N)):
            s = y[j]
            for k, v in Lt[j].items():
                s -= v * x[k]
            x[j] = s / L[j][j]
        z = [None] * N
        for i in range(N):
            z[perm[i]] = x[i]
        return z
