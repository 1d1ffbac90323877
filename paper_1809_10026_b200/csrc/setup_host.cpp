// Host-side univariate setup.  See setup_host.hpp.
#include "setup_host.hpp"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>

namespace ls {

std::vector<double> open_uniform_knots(int n_el, int p) {
  std::vector<double> kn;
  kn.reserve(n_el + 2 * p + 1);
  for (int i = 0; i <= p; ++i) kn.push_back(0.0);
  for (int i = 1; i < n_el; ++i) kn.push_back(double(i) / double(n_el));
  for (int i = 0; i <= p; ++i) kn.push_back(1.0);
  return kn;
}

// The same knots i / n_el in 80-bit (reading c17): fp64 knots are inexact unless n_el is a
// power of two and would perturb the assembled matrices by up to ~2.5e-14 relative
// (n_el = 130; tests/test_oracle_highprec.py pins the assembly to the exact rationals).
std::vector<long double> open_uniform_knots_ld(int n_el, int p) {
  std::vector<long double> kn;
  kn.reserve(n_el + 2 * p + 1);
  for (int i = 0; i <= p; ++i) kn.push_back(0.0L);
  for (int i = 1; i < n_el; ++i) kn.push_back((long double)i / (long double)n_el);
  for (int i = 0; i <= p; ++i) kn.push_back(1.0L);
  return kn;
}

void gauss_legendre(int q, std::vector<long double>& x, std::vector<long double>& w) {
  typedef long double R;
  x.assign(q, 0.0L);
  w.assign(q, 0.0L);
  const R pi = 3.141592653589793238462643383279502884L;
  auto legendre = [q](R z, R& pq, R& dpq) {  // P_q(z) and P_q'(z)
    R p0 = 1.0L, p1 = z;
    for (int k = 2; k <= q; ++k) {
      R p2 = ((2.0L * k - 1.0L) * z * p1 - (k - 1.0L) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (q == 1) p0 = 1.0L;
    pq = p1;
    dpq = q * (z * p1 - p0) / (z * z - 1.0L);
  };
  for (int i = 0; i < (q + 1) / 2; ++i) {
    R z = cosl(pi * (i + 0.75L) / (q + 0.5L)), pq, dp;
    for (int it = 0; it < 100; ++it) {
      legendre(z, pq, dp);
      const R dz = pq / dp;
      z -= dz;
      if (fabsl(dz) < 1e-19L) break;
    }
    legendre(z, pq, dp);
    x[i] = -z;
    x[q - 1 - i] = z;
    w[i] = w[q - 1 - i] = 2.0L / ((1.0L - z * z) * dp * dp);
  }
  if (q % 2 == 1) x[q / 2] = 0.0L;
}

static inline long double ratio(long double num, long double den) { return den == 0.0L ? 0.0L : num / den; }

void bspline_eval(const std::vector<double>& kd, int p, long double x, long double* v0,
                  long double* v1, long double* v2) {
  bspline_eval(std::vector<long double>(kd.begin(), kd.end()), p, x, v0, v1, v2);
}

void bspline_eval(const std::vector<long double>& kn, int p, long double x, long double* v0,
                  long double* v1, long double* v2) {
  typedef long double R;
  const int n0 = int(kn.size()) - 1;
  // N[q][i] for degrees 0..p (Cox-de Boor, PAPER.md 148-166)
  std::vector<std::vector<R>> N(p + 1);
  N[0].assign(n0, 0.0L);
  int last = 0;
  for (int i = 0; i < n0; ++i)
    if (kn[i] < kn[i + 1]) last = i;
  if (x >= kn.back()) {
    N[0][last] = 1.0L;  // right end: left limit (reading R-endpoint)
  } else {
    for (int i = 0; i < n0; ++i) N[0][i] = (kn[i] <= x && x < kn[i + 1]) ? 1.0L : 0.0L;
  }
  for (int q = 1; q <= p; ++q) {
    N[q].assign(n0 - q, 0.0L);
    for (int i = 0; i < n0 - q; ++i)
      N[q][i] = ratio(x - kn[i], kn[i + q] - kn[i]) * N[q - 1][i] +
                ratio(kn[i + q + 1] - x, kn[i + q + 1] - kn[i + 1]) * N[q - 1][i + 1];
  }
  const int m = n0 - p;
  // first derivative of degree-q functions from degree q-1 values (de Boor)
  auto d1 = [&](int q, int i) {
    return q * (ratio(N[q - 1][i], kn[i + q] - kn[i]) - ratio(N[q - 1][i + 1], kn[i + q + 1] - kn[i + 1]));
  };
  for (int i = 0; i < m; ++i) {
    v0[i] = N[p][i];
    v1[i] = p >= 1 ? d1(p, i) : 0.0L;
    if (p >= 2) {
      R a = d1(p - 1, i), b = d1(p - 1, i + 1);
      v2[i] = p * (ratio(a, kn[i + p] - kn[i]) - ratio(b, kn[i + p + 1] - kn[i + 1]));
    } else {
      v2[i] = 0.0L;
    }
  }
}

// Dense unconstrained m x m matrices M = int b b, K = int b' b', J = int b'' b''
// with q = p + 1 Gauss points per element (exact, reading c6), evaluated and summed
// in 80-bit extended precision and rounded once to fp64 (reading c17).
static void assemble_full(const std::vector<long double>& kn, int p, std::vector<double>& Mo,
                          std::vector<double>& Ko, std::vector<double>& Jo) {
  typedef long double R;
  const int m = int(kn.size()) - p - 1;
  std::vector<R> M(size_t(m) * m, 0.0L), K(size_t(m) * m, 0.0L), J(size_t(m) * m, 0.0L);
  std::vector<R> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  std::vector<R> v0(m), v1(m), v2(m);
  for (size_t e = 0; e + 1 < kn.size(); ++e) {
    const R a = kn[e], b = kn[e + 1];
    if (!(a < b)) continue;
    for (size_t g = 0; g < gx.size(); ++g) {
      const R x = 0.5L * (a + b) + 0.5L * (b - a) * gx[g];
      const R w = 0.5L * (b - a) * gw[g];
      bspline_eval(kn, p, x, v0.data(), v1.data(), v2.data());
      int lo = std::max(0, int(e) - p), hi = std::min(m - 1, int(e));
      for (int i = lo; i <= hi; ++i)
        for (int j = lo; j <= hi; ++j) {
          M[size_t(i) * m + j] += w * v0[i] * v0[j];
          K[size_t(i) * m + j] += w * v1[i] * v1[j];
          J[size_t(i) * m + j] += w * v2[i] * v2[j];
        }
    }
  }
  Mo.assign(M.begin(), M.end());
  Ko.assign(K.begin(), K.end());
  Jo.assign(J.begin(), J.end());
}

static std::vector<double> slice(const std::vector<double>& A, int m, int lo, int n) {
  std::vector<double> out(size_t(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[size_t(i) * n + j] = A[size_t(i + lo) * m + (j + lo)];
  return out;
}

Factors space_factors(int n_el, int p) {
  auto kn = open_uniform_knots_ld(n_el, p);
  const int m = n_el + p;
  std::vector<double> M, K, J;
  assemble_full(kn, p, M, K, J);
  Factors f;
  f.n = m - 2;  // i = 2..m-1 (eq:basis_par, reading c1)
  f.M = slice(M, m, 1, f.n);
  f.K = slice(K, m, 1, f.n);
  f.J = slice(J, m, 1, f.n);
  return f;
}

Factors time_factors(int n_el, int p) {
  auto kn = open_uniform_knots_ld(n_el, p);
  const int m = n_el + p;
  std::vector<double> M, K, J;
  assemble_full(kn, p, M, K, J);
  Factors f;
  f.n = m - 1;  // i = 2..m
  f.M = slice(M, m, 1, f.n);
  f.K = slice(K, m, 1, f.n);
  return f;
}

void load_integrals(int n_el, int p, bool space, int fn, double c, std::vector<double>& i0,
                    std::vector<double>& i1, std::vector<double>& i2) {
  typedef long double R;
  auto kn = open_uniform_knots_ld(n_el, p);
  const int m = n_el + p;
  const int lo = 1, n = space ? m - 2 : m - 1;
  std::vector<R> a0(n, 0.0L), a1(n, 0.0L), a2(n, 0.0L);
  std::vector<R> gx, gw;
  gauss_legendre(p + 5, gx, gw);
  std::vector<R> v0(m), v1(m), v2(m);
  const R pi = 3.141592653589793238462643383279502884L;
  for (size_t e = 0; e + 1 < kn.size(); ++e) {
    const R a = kn[e], b = kn[e + 1];
    if (!(a < b)) continue;
    for (size_t g = 0; g < gx.size(); ++g) {
      const R x = 0.5L * (a + b) + 0.5L * (b - a) * gx[g];
      const R w = 0.5L * (b - a) * gw[g];
      const R f = fn == 0 ? sinl(pi * x) : fn == 1 ? expl(x) : fn == 3 ? cosl(pi * x) : fn == 4 ? 1.0L
                                                                                  : cosl(x) + R(c) * sinl(x);
      bspline_eval(kn, p, x, v0.data(), v1.data(), v2.data());
      for (int i = 0; i < n; ++i) {
        a0[i] += w * f * v0[i + lo];
        a1[i] += w * f * v1[i + lo];
        a2[i] += w * f * v2[i + lo];
      }
    }
  }
  i0.assign(a0.begin(), a0.end());
  i1.assign(a1.begin(), a1.end());
  i2.assign(a2.begin(), a2.end());
}

} // namespace ls

// ------------------------------------------------------------------------------------------
// Generalized symmetric-definite eigenproblem K U = M U Lambda, U^T M U = I
// (eq:eig_dec, PAPER.md 939-945) in 80-bit extended precision on the host:
// Cholesky M = L L^T, C = L^{-1} K L^{-T}, cyclic Jacobi on C with the relative
// (Demmel-Veselic) stopping rule, U = L^{-T} Q.  The smallest eigenvalues of
// (J, M) dominate P^{-1} r and sit ~1e10 below the largest; double-precision
// solvers lose ~eps*lambda_max/lambda_min of their relative accuracy (cuSOLVER
// Dsygvd: ~5e-9, measured), extended precision keeps them exact
// to double rounding.  O(n^3) per sweep, n <= 136: ~0.1 s per pencil.
// ------------------------------------------------------------------------------------------
namespace ls {

template <class T>
static int generalized_eig_t(const std::vector<T>& Kd, const std::vector<T>& Md, int n,
                             std::vector<double>& lam, std::vector<double>& Uout) {
  typedef long double R;
  std::vector<R> L(size_t(n) * n, 0.0L), C(size_t(n) * n), Q(size_t(n) * n, 0.0L);
  // Cholesky M = L L^T
  for (int j = 0; j < n; ++j) {
    R s = Md[size_t(j) * n + j];
    for (int k = 0; k < j; ++k) s -= L[size_t(j) * n + k] * L[size_t(j) * n + k];
    if (!(s > 0)) return 1;
    const R ljj = sqrtl(s);
    L[size_t(j) * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      R t = Md[size_t(i) * n + j];
      for (int k = 0; k < j; ++k) t -= L[size_t(i) * n + k] * L[size_t(j) * n + k];
      L[size_t(i) * n + j] = t / ljj;
    }
  }
  // Y = L^{-1} K (forward substitution, column by column)
  std::vector<R> Y(size_t(n) * n);
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      R t = Kd[size_t(i) * n + c];
      for (int k = 0; k < i; ++k) t -= L[size_t(i) * n + k] * Y[size_t(k) * n + c];
      Y[size_t(i) * n + c] = t / L[size_t(i) * n + i];
    }
  // C = L^{-1} Y^T  (= L^{-1} K L^{-T} since K is symmetric), then symmetrise
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      R t = Y[size_t(c) * n + i];
      for (int k = 0; k < i; ++k) t -= L[size_t(i) * n + k] * C[size_t(k) * n + c];
      C[size_t(i) * n + c] = t / L[size_t(i) * n + i];
    }
  for (int i = 0; i < n; ++i)
    for (int j = i + 1; j < n; ++j) {
      R a = 0.5L * (C[size_t(i) * n + j] + C[size_t(j) * n + i]);
      C[size_t(i) * n + j] = C[size_t(j) * n + i] = a;
    }
  // cyclic Jacobi: Q^T C Q = diag
  for (int i = 0; i < n; ++i) Q[size_t(i) * n + i] = 1.0L;
  const R eps = LDBL_EPSILON;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        const R apq = C[size_t(p) * n + q];
        const R app = C[size_t(p) * n + p], aqq = C[size_t(q) * n + q];
        if (fabsl(apq) <= eps * sqrtl(fabsl(app * aqq))) {
          C[size_t(p) * n + q] = C[size_t(q) * n + p] = 0.0L;
          continue;
        }
        rotated = true;
        const R theta = (aqq - app) / (2.0L * apq);
        const R t = (theta >= 0 ? 1.0L : -1.0L) / (fabsl(theta) + sqrtl(1.0L + theta * theta));
        const R c = 1.0L / sqrtl(1.0L + t * t), s = t * c;
        for (int k = 0; k < n; ++k) {  // columns p, q
          const R akp = C[size_t(k) * n + p], akq = C[size_t(k) * n + q];
          C[size_t(k) * n + p] = c * akp - s * akq;
          C[size_t(k) * n + q] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rows p, q
          const R apk = C[size_t(p) * n + k], aqk = C[size_t(q) * n + k];
          C[size_t(p) * n + k] = c * apk - s * aqk;
          C[size_t(q) * n + k] = s * apk + c * aqk;
        }
        C[size_t(p) * n + q] = C[size_t(q) * n + p] = 0.0L;
        for (int k = 0; k < n; ++k) {
          const R vkp = Q[size_t(k) * n + p], vkq = Q[size_t(k) * n + q];
          Q[size_t(k) * n + p] = c * vkp - s * vkq;
          Q[size_t(k) * n + q] = s * vkp + c * vkq;
        }
      }
    if (!rotated) break;
  }
  // U = L^{-T} Q (back substitution)
  std::vector<R> U(size_t(n) * n);
  for (int c = 0; c < n; ++c)
    for (int i = n - 1; i >= 0; --i) {
      R t = Q[size_t(i) * n + c];
      for (int k = i + 1; k < n; ++k) t -= L[size_t(k) * n + i] * U[size_t(k) * n + c];
      U[size_t(i) * n + c] = t / L[size_t(i) * n + i];
    }
  // sort ascending; fix signs (largest |component| positive) for determinism
  std::vector<int> ord(n);
  for (int i = 0; i < n; ++i) ord[i] = i;
  std::sort(ord.begin(), ord.end(),
            [&](int a, int b) { return C[size_t(a) * n + a] < C[size_t(b) * n + b]; });
  lam.assign(n, 0.0);
  Uout.assign(size_t(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    const int o = ord[j];
    lam[j] = double(C[size_t(o) * n + o]);
    int imax = 0;
    for (int i = 1; i < n; ++i)
      if (fabsl(U[size_t(i) * n + o]) > fabsl(U[size_t(imax) * n + o])) imax = i;
    const R sg = U[size_t(imax) * n + o] < 0 ? -1.0L : 1.0L;
    for (int i = 0; i < n; ++i) Uout[size_t(i) * n + j] = double(sg * U[size_t(i) * n + o]);
  }
  return 0;
}

int generalized_eig(const std::vector<double>& K, const std::vector<double>& M, int n,
                    std::vector<double>& lam, std::vector<double>& U) {
  return generalized_eig_t(K, M, n, lam, U);
}

int generalized_eig(const std::vector<long double>& K, const std::vector<long double>& M, int n,
                    std::vector<double>& lam, std::vector<double>& U) {
  return generalized_eig_t(K, M, n, lam, U);
}

} // namespace ls
