// Host side of the mapped-domain path (geo.hpp): map validation / evaluation and the
// P^G setup of PAPER.md 969-1045 (readings c19-c22 in DESIGN.md).  O(#elements) work,
// once per ls_setup_geo.
#include <algorithm>
#include <cmath>
#include <vector>

#include "geo.hpp"
#include "setup_host.hpp"

namespace ls {

int geo_copy(const ls_geometry* g, int d, GeoMap& out) {
  if (!g || !g->ctrl) return LS_EINVAL;
  out = GeoMap();
  out.d = d;
  int64_t total = 1;
  for (int k = 0; k < d; ++k) {
    const int q = g->degree[k];
    const int64_t nk = g->n_knots[k];
    if (q < 1 || q > 8 || !g->knots[k] || nk < 2 * (q + 1) || nk > 4096) return LS_EINVAL;
    out.q[k] = q;
    out.knots[k].assign(g->knots[k], g->knots[k] + nk);
    const auto& kn = out.knots[k];
    for (int64_t i = 0; i + 1 < nk; ++i)
      if (!(kn[i] <= kn[i + 1])) return LS_EINVAL;
    // open knot vector on [0, 1] (Ass. 1: F defined on the parametric unit cube)
    for (int i = 0; i <= q; ++i)
      if (kn[i] != 0.0 || kn[nk - 1 - i] != 1.0) return LS_EINVAL;
    out.m[k] = int(nk - q - 1);
    total *= out.m[k];
  }
  out.ctrl.assign(g->ctrl, g->ctrl + total * d);
  out.w.assign(total, 1.0);
  if (g->weights)
    for (int64_t i = 0; i < total; ++i) {
      if (!(g->weights[i] > 0.0) || !std::isfinite(g->weights[i])) return LS_EINVAL;
      out.w[i] = g->weights[i];
    }
  for (double c : out.ctrl)
    if (!std::isfinite(c)) return LS_EINVAL;
  return LS_OK;
}

typedef long double R;

// values / first derivatives of all geometry functions of direction k at eta
static void dir_eval(const GeoMap& g, int k, R eta, std::vector<R>& v0, std::vector<R>& v1) {
  const int m = g.m[k];
  std::vector<R> v2(m);
  v0.assign(m, 0);
  v1.assign(m, 0);
  bspline_eval(g.knots[k], g.q[k], eta, v0.data(), v1.data(), v2.data());
}

// F and Jac at one point from per-direction tables (quotient rule, PAPER.md 226-250)
static void tensor_eval(const GeoMap& g, const R* const* v0, const R* const* v1, R* x, R* jac) {
  const int d = g.d;
  R N[3] = {0, 0, 0}, W = 0, dN[3][3] = {{0}}, dW[3] = {0, 0, 0};
  const int m1 = g.m[0], m2 = d >= 2 ? g.m[1] : 1, m3 = d >= 3 ? g.m[2] : 1;
  for (int c3 = 0; c3 < m3; ++c3)
    for (int c2 = 0; c2 < m2; ++c2)
      for (int c1 = 0; c1 < m1; ++c1) {
        const int c[3] = {c1, c2, c3};
        const int64_t idx = c1 + int64_t(m1) * (c2 + int64_t(m2) * c3);
        R val = 1, der[3] = {1, 1, 1};
        for (int k = 0; k < d; ++k) val *= v0[k][c[k]];
        for (int j = 0; j < d; ++j)
          for (int k = 0; k < d; ++k) der[j] *= (k == j) ? v1[k][c[k]] : v0[k][c[k]];
        const R w = g.w[idx];
        W += w * val;
        for (int j = 0; j < d; ++j) dW[j] += w * der[j];
        for (int i = 0; i < d; ++i) {
          const R cw = w * R(g.ctrl[idx * d + i]);
          N[i] += cw * val;
          for (int j = 0; j < d; ++j) dN[i][j] += cw * der[j];
        }
      }
  for (int i = 0; i < d; ++i) {
    x[i] = N[i] / W;
    for (int j = 0; j < d; ++j) jac[i * d + j] = (dN[i][j] - x[i] * dW[j]) / W;
  }
}

void geo_eval(const GeoMap& g, const double* eta, double* x, double* jac) {
  std::vector<R> v0[3], v1[3];
  for (int k = 0; k < g.d; ++k) dir_eval(g, k, eta[k], v0[k], v1[k]);
  const R* p0[3] = {v0[0].data(), v0[1].data(), v0[2].data()};
  const R* p1[3] = {v1[0].data(), v1[1].data(), v1[2].data()};
  R xr[3], jr[9];
  tensor_eval(g, p0, p1, xr, jr);
  for (int i = 0; i < g.d; ++i) x[i] = double(xr[i]);
  for (int i = 0; i < g.d * g.d; ++i) jac[i] = double(jr[i]);
}

// inverse and determinant of a d x d matrix (d <= 3)
static R inv_det(int d, const R* a, R* inv) {
  if (d == 1) {
    inv[0] = 1 / a[0];
    return a[0];
  }
  if (d == 2) {
    const R det = a[0] * a[3] - a[1] * a[2];
    inv[0] = a[3] / det;
    inv[1] = -a[1] / det;
    inv[2] = -a[2] / det;
    inv[3] = a[0] / det;
    return det;
  }
  const R c00 = a[4] * a[8] - a[5] * a[7], c01 = a[5] * a[6] - a[3] * a[8], c02 = a[3] * a[7] - a[4] * a[6];
  const R det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  inv[0] = c00 / det;
  inv[3] = c01 / det;
  inv[6] = c02 / det;
  inv[1] = (a[2] * a[7] - a[1] * a[8]) / det;
  inv[4] = (a[0] * a[8] - a[2] * a[6]) / det;
  inv[7] = (a[1] * a[6] - a[0] * a[7]) / det;
  inv[2] = (a[1] * a[5] - a[2] * a[4]) / det;
  inv[5] = (a[2] * a[3] - a[0] * a[5]) / det;
  inv[8] = (a[0] * a[4] - a[1] * a[3]) / det;
  return det;
}

int pg_weights(const GeoMap& g, const int64_t* n_el, std::vector<double> mu[3], std::vector<double> om[3],
               double* fit_rel_res) {
  const int d = g.d;
  int ne[3] = {1, 1, 1};
  for (int k = 0; k < d; ++k) ne[k] = int(n_el[k]);
  // per-direction geometry tables at the element midpoints (one point per element)
  std::vector<std::vector<R>> t0[3], t1[3];
  for (int k = 0; k < d; ++k) {
    t0[k].resize(ne[k]);
    t1[k].resize(ne[k]);
    for (int e = 0; e < ne[k]; ++e) dir_eval(g, k, (R(e) + 0.5L) / R(ne[k]), t0[k][e], t1[k][e]);
  }
  const int64_t NE = int64_t(ne[0]) * ne[1] * ne[2];
  // logarithms of c_tau and c_k (T = 1; reading c20 for c_k)
  std::vector<R> L(size_t(NE) * (d + 1));
  int signs = 0;
  for (int64_t e = 0; e < NE; ++e) {
    const int ei[3] = {int(e % ne[0]), int((e / ne[0]) % ne[1]), int(e / (int64_t(ne[0]) * ne[1]))};
    const R* v0[3] = {nullptr, nullptr, nullptr};
    const R* v1[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < d; ++k) {
      v0[k] = t0[k][ei[k]].data();
      v1[k] = t1[k][ei[k]].data();
    }
    R x[3], jac[9], inv[9];
    tensor_eval(g, v0, v1, x, jac);
    const R sdet = inv_det(d, jac, inv);
    const R det = std::fabs(sdet);
    if (!(det > 0) || !std::isfinite(double(det))) return LS_EINVAL;  // singular map
    signs |= sdet > 0 ? 1 : 2;
    if (signs == 3) return LS_EINVAL;  // det J_F changes sign: a folded map (Assumption 4)
    L[size_t(e) * (d + 1) + d] = std::log(det);
    for (int k = 0; k < d; ++k) {
      R s = 0;
      for (int i = 0; i < d; ++i) s += inv[k * d + i] * inv[k * d + i];  // row k of J^{-1}
      L[size_t(e) * (d + 1) + k] = std::log(s * s * det);
    }
  }
  // alternating least-squares sweeps on the logarithms (reading c21):
  //   log c_tau(e) ~ sum_j m_j(e_j);  log c_k(e) ~ o_k(e_k) + sum_{j != k} m_j(e_j)
  // Every update is an average over the elements with e_j = v of separable terms, so it
  // needs only the marginals A_q[j][v] = sum_{e: e_j = v} L_q(e) (one pass over the
  // elements) and the sums S(m_l), S(o_k): O(d^2 n_el) per sweep.
  std::vector<R> m[3], o[3], Am[4][3];
  for (int k = 0; k < 3; ++k) {
    m[k].assign(ne[k], 0);
    o[k].assign(ne[k], 0);
  }
  for (int q = 0; q <= d; ++q)
    for (int j = 0; j < d; ++j) Am[q][j].assign(ne[j], 0);
  for (int64_t e = 0; e < NE; ++e) {
    const int ei[3] = {int(e % ne[0]), int((e / ne[0]) % ne[1]), int(e / (int64_t(ne[0]) * ne[1]))};
    for (int q = 0; q <= d; ++q)
      for (int j = 0; j < d; ++j) Am[q][j][ei[j]] += L[size_t(e) * (d + 1) + q];
  }
  auto sum = [](const std::vector<R>& v) {
    R s = 0;
    for (R x : v) s += x;
    return s;
  };
  for (int sweep = 0; sweep < 5000; ++sweep) {
    R change = 0;
    for (int j = 0; j < d; ++j) {  // m_j: the c_tau equation and the c_k equations, k != j
      const R cnt = R(NE / ne[j]);
      for (int v = 0; v < ne[j]; ++v) {
        R t = Am[d][j][v];  // c_tau: L_tau - sum_{l != j} m_l
        for (int l = 0; l < d; ++l)
          if (l != j) t -= cnt / ne[l] * sum(m[l]);
        for (int k = 0; k < d; ++k) {  // c_k: L_k - o_k - sum_{l != j, k} m_l
          if (k == j) continue;
          t += Am[k][j][v] - cnt / ne[k] * sum(o[k]);
          for (int l = 0; l < d; ++l)
            if (l != j && l != k) t -= cnt / ne[l] * sum(m[l]);
        }
        const R nv = t / (cnt * R(d));
        change = std::max(change, std::fabs(nv - m[j][v]));
        m[j][v] = nv;
      }
    }
    for (int k = 0; k < d; ++k) {  // o_k: only the c_k equation
      const R cnt = R(NE / ne[k]);
      for (int v = 0; v < ne[k]; ++v) {
        R t = Am[k][k][v];
        for (int l = 0; l < d; ++l)
          if (l != k) t -= cnt / ne[l] * sum(m[l]);
        const R nv = t / cnt;
        change = std::max(change, std::fabs(nv - o[k][v]));
        o[k][v] = nv;
      }
    }
    if (change < 1e-16L) break;
  }
  // relative residual of the fit (max over equations of |c - approx| / c), reported
  R res = 0;
  for (int64_t e = 0; e < NE; ++e) {
    const int ei[3] = {int(e % ne[0]), int((e / ne[0]) % ne[1]), int(e / (int64_t(ne[0]) * ne[1]))};
    R sm = 0;
    for (int l = 0; l < d; ++l) sm += m[l][ei[l]];
    res = std::max(res, std::fabs(std::expm1(sm - L[size_t(e) * (d + 1) + d])));
    for (int k = 0; k < d; ++k)
      res = std::max(res, std::fabs(std::expm1(sm - m[k][ei[k]] + o[k][ei[k]] - L[size_t(e) * (d + 1) + k])));
  }
  if (fit_rel_res) *fit_rel_res = double(res);
  for (int k = 0; k < d; ++k) {
    mu[k].resize(ne[k]);
    om[k].resize(ne[k]);
    for (int v = 0; v < ne[k]; ++v) {
      mu[k][v] = double(std::exp(m[k][v]));
      om[k][v] = double(std::exp(o[k][v]));
    }
  }
  return LS_OK;
}

// reading c22: piecewise linear through (midpoint, value), constant beyond the outer midpoints
static R interp(const std::vector<double>& v, R x) {
  const int n = int(v.size());
  const R t = x * n - 0.5L;  // midpoint coordinate
  if (t <= 0) return v[0];
  if (t >= n - 1) return v[n - 1];
  const int i = int(t);
  const R f = t - i;
  return (1 - f) * R(v[i]) + f * R(v[i + 1]);
}

void weighted_space_factors(int n_el, int p, const std::vector<double>& mu, const std::vector<double>& om,
                            std::vector<double>& Mo, std::vector<double>& Jo) {
  auto kn = open_uniform_knots(n_el, p);
  const int m = n_el + p;
  std::vector<R> M(size_t(m) * m, 0), J(size_t(m) * m, 0);
  std::vector<R> gx, gw;
  gauss_legendre(p + 1, gx, gw);
  std::vector<R> v0(m), v1(m), v2(m);
  for (int e = 0; e < n_el; ++e) {
    const R a = kn[p + e], b = kn[p + e + 1];
    for (size_t g = 0; g < gx.size(); ++g) {
      const R x = 0.5L * (a + b) + 0.5L * (b - a) * gx[g];
      const R w = 0.5L * (b - a) * gw[g];
      const R wm = w * interp(mu, x), wo = w * interp(om, x);
      bspline_eval(kn, p, x, v0.data(), v1.data(), v2.data());
      for (int i = e; i <= e + p; ++i)
        for (int j = e; j <= e + p; ++j) {
          M[size_t(i) * m + j] += wm * v0[i] * v0[j];
          J[size_t(i) * m + j] += wo * v2[i] * v2[j];
        }
    }
  }
  const int n = m - 2;  // i = 2..m-1
  Mo.assign(size_t(n) * n, 0.0);
  Jo.assign(size_t(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      Mo[size_t(i) * n + j] = double(M[size_t(i + 1) * m + (j + 1)]);
      Jo[size_t(i) * n + j] = double(J[size_t(i + 1) * m + (j + 1)]);
    }
}

}  // namespace ls
