// Host-side univariate setup.  See setup_host.hpp.
#include "setup_host.hpp"

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

void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  const double pi = 3.14159265358979323846;
  for (int i = 0; i < (q + 1) / 2; ++i) {
    double z = std::cos(pi * (i + 0.75) / (q + 0.5));
    double dp = 1.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;  // P_0, P_1
      for (int k = 2; k <= q; ++k) {
        double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) { p1 = z; p0 = 1.0; }
      dp = q * (z * p1 - p0) / (z * z - 1.0);  // P_q'
      double dz = p1 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    // recompute derivative at the converged node
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= q; ++k) {
      double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    if (q == 1) { p1 = z; p0 = 1.0; }
    dp = q * (z * p1 - p0) / (z * z - 1.0);
    x[i] = -z;
    x[q - 1 - i] = z;
    w[i] = w[q - 1 - i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
  if (q % 2 == 1) x[q / 2] = 0.0;
}

static inline double ratio(double num, double den) { return den == 0.0 ? 0.0 : num / den; }

void bspline_eval(const std::vector<double>& kn, int p, double x, double* v0, double* v1,
                  double* v2) {
  const int n0 = int(kn.size()) - 1;
  // N[q][i] for degrees 0..p (Cox-de Boor); only degrees p-2..p are needed below
  std::vector<std::vector<double>> N(p + 1);
  N[0].assign(n0, 0.0);
  int last = 0;
  for (int i = 0; i < n0; ++i)
    if (kn[i] < kn[i + 1]) last = i;
  if (x >= kn.back()) {
    N[0][last] = 1.0;  // right end: left limit (reading R-endpoint)
  } else {
    for (int i = 0; i < n0; ++i) N[0][i] = (kn[i] <= x && x < kn[i + 1]) ? 1.0 : 0.0;
  }
  for (int q = 1; q <= p; ++q) {
    N[q].assign(n0 - q, 0.0);
    for (int i = 0; i < n0 - q; ++i)
      N[q][i] = ratio(x - kn[i], kn[i + q] - kn[i]) * N[q - 1][i] +
                ratio(kn[i + q + 1] - x, kn[i + q + 1] - kn[i + 1]) * N[q - 1][i + 1];
  }
  const int m = n0 - p;
  // first derivatives of degree q from degree q-1 values
  auto d1 = [&](int q, int i) {
    return q * (ratio(N[q - 1][i], kn[i + q] - kn[i]) - ratio(N[q - 1][i + 1], kn[i + q + 1] - kn[i + 1]));
  };
  for (int i = 0; i < m; ++i) {
    v0[i] = N[p][i];
    v1[i] = p >= 1 ? d1(p, i) : 0.0;
    if (p >= 2) {
      double a = d1(p - 1, i), b = d1(p - 1, i + 1);
      v2[i] = p * (ratio(a, kn[i + p] - kn[i]) - ratio(b, kn[i + p + 1] - kn[i + 1]));
    } else {
      v2[i] = 0.0;
    }
  }
}

// Dense unconstrained m x m matrices M = int b b, K = int b' b', J = int b'' b''
// with q = p + 1 Gauss points per element (exact, reading c6).
static void assemble_full(const std::vector<double>& kn, int p, std::vector<double>& M,
                          std::vector<double>& K, std::vector<double>& J) {
  const int m = int(kn.size()) - p - 1;
  M.assign(size_t(m) * m, 0.0);
  K.assign(size_t(m) * m, 0.0);
  J.assign(size_t(m) * m, 0.0);
  std::vector<double> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  std::vector<double> v0(m), v1(m), v2(m);
  for (size_t e = 0; e + 1 < kn.size(); ++e) {
    double a = kn[e], b = kn[e + 1];
    if (!(a < b)) continue;
    for (size_t g = 0; g < gx.size(); ++g) {
      double x = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      double w = 0.5 * (b - a) * gw[g];
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
}

static std::vector<double> slice(const std::vector<double>& A, int m, int lo, int n) {
  std::vector<double> out(size_t(n) * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[size_t(i) * n + j] = A[size_t(i + lo) * m + (j + lo)];
  return out;
}

Factors space_factors(int n_el, int p) {
  auto kn = open_uniform_knots(n_el, p);
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
  auto kn = open_uniform_knots(n_el, p);
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
  auto kn = open_uniform_knots(n_el, p);
  const int m = n_el + p;
  const int lo = 1, n = space ? m - 2 : m - 1;
  i0.assign(n, 0.0);
  i1.assign(n, 0.0);
  i2.assign(n, 0.0);
  std::vector<double> gx, gw;
  gauss_legendre(p + 5, gx, gw);
  std::vector<double> v0(m), v1(m), v2(m);
  const double pi = 3.14159265358979323846;
  for (size_t e = 0; e + 1 < kn.size(); ++e) {
    double a = kn[e], b = kn[e + 1];
    if (!(a < b)) continue;
    for (size_t g = 0; g < gx.size(); ++g) {
      double x = 0.5 * (a + b) + 0.5 * (b - a) * gx[g];
      double w = 0.5 * (b - a) * gw[g];
      double f = fn == 0 ? std::sin(pi * x) : fn == 1 ? std::exp(x) : std::cos(x) + c * std::sin(x);
      bspline_eval(kn, p, x, v0.data(), v1.data(), v2.data());
      for (int i = 0; i < n; ++i) {
        i0[i] += w * f * v0[i + lo];
        i1[i] += w * f * v1[i + lo];
        i2[i] += w * f * v2[i + lo];
      }
    }
  }
}

} // namespace ls
