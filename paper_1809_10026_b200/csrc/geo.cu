// Device side of the mapped-domain path (geo.hpp).
//
// Layout of the physical spatial factors (PAPER.md 697-703) on the device: for each of
// M_s, J_s, L_s a stencil array st[mat][o][i], i = the constrained spatial row (colex),
// o = (o_1 + (2p+1)(o_2 + (2p+1) o_3)) with o_k = j_k - i_k + p the offset of the column
// in direction k (tensor B-splines of degree p couple |j_k - i_k| <= p).  Entries whose
// column falls outside the constrained grid stay 0.  Row-contiguous in i for every
// offset, so consecutive threads (consecutive rows) read coalesced coefficients.
//
// Kernels:
//   geo_qpoint_kernel   map derivatives at every tensor Gauss point -> |det J| w_q, J^{-1},
//                       the first-order Laplacian coefficients b (chain rule, PAPER.md 986-990)
//   geo_assemble_kernel one CTA per element: physical values / gradients / Laplacians of the
//                       (p+1)^d local functions at a chunk of points in shared memory, pair
//                       sums in registers, added into the stencil rows (one launch per
//                       element colour class: deterministic, no atomics)
//   geo_time_kernel     t1 = K_t x, t2 = M_t x (banded, half-bandwidth p_t)
//   geo_dmma_kernel     y = M_s t1 + J_s t2 (+ L_s x on the last slice: W_t = e e^T) as DMMA
//                       band tiles (default)
//   geo_stencil_kernel  the same with DFMAs, one thread per row and 8 time slices (ls_tune)
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <vector>

#include "geo.hpp"
#include "setup_host.hpp"

namespace ls {

#define GEO_CUDA(x)                                                                  \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::fprintf(stderr, "[libls] CUDA error %s at %s:%d\n", cudaGetErrorString(e_), \
                   __FILE__, __LINE__);                                              \
      return LS_ECUDA;                                                               \
    }                                                                                \
  } while (0)

GeoDev::~GeoDev() {
  for (void* a : allocs) cudaFree(a);
}

static int dalloc(std::vector<void*>& allocs, double** p, size_t n) {
  void* v = nullptr;
  if (cudaMalloc(&v, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) return LS_ENOMEM;
  allocs.push_back(v);
  *p = static_cast<double*>(v);
  return LS_OK;
}

#define LS_CHECK_RC(x)     \
  do {                     \
    int rc_ = (x);         \
    if (rc_ != LS_OK) return rc_; \
  } while (0)

static int dupload(std::vector<void*>& allocs, const std::vector<double>& h, double** p) {
  int rc = dalloc(allocs, p, h.size());
  if (rc != LS_OK) return rc;
  GEO_CUDA(cudaMemcpy(*p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// geometry at the quadrature points
// ------------------------------------------------------------------------------------------
struct GeoQArgs {
  int d;
  int nq[3];                 // Gauss points per direction (n_el (p+1))
  int q[3];                  // geometry degrees
  int m[3];                  // geometry functions per direction
  const int* span[3];        // first non-zero geometry function at each point
  const double* gt[3];       // [nq_k][q_k+1][3] values, 1st, 2nd derivatives
  const double* wq[3];       // [nq_k] Gauss weights (element length included)
  const double* ctrl;        // [prod m][d]
  const double* w;           // [prod m]
  double* out;               // [16][NQ]: wdet, Jinv[3][3] (row j = grad eta_j), b[3], x[3]
  int64_t NQ;
  int* flags;                // bit 0: det J <= 0 seen, bit 1: det J >= 0 seen, bit 2: det J = 0 / non-finite
};

__global__ void geo_qpoint_kernel(GeoQArgs a) {
  for (int64_t qi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; qi < a.NQ;
       qi += int64_t(gridDim.x) * blockDim.x) {
    const int d = a.d;
    int iq[3] = {0, 0, 0};
    int64_t r = qi;
    for (int k = 0; k < d; ++k) {
      iq[k] = int(r % a.nq[k]);
      r /= a.nq[k];
    }
    double N[3] = {0, 0, 0}, W = 0, dN[3][3] = {}, dW[3] = {}, hN[3][3][3] = {}, hW[3][3] = {};
    const int c1n = a.q[0] + 1, c2n = d >= 2 ? a.q[1] + 1 : 1, c3n = d >= 3 ? a.q[2] + 1 : 1;
    for (int c3 = 0; c3 < c3n; ++c3)
      for (int c2 = 0; c2 < c2n; ++c2)
        for (int c1 = 0; c1 < c1n; ++c1) {
          const int cl[3] = {c1, c2, c3};
          double v[3][3];  // [dir][deriv]
          int64_t idx = 0, stride = 1;
          for (int k = 0; k < 3; ++k) {
            if (k < d) {
              const double* t = a.gt[k] + (size_t(iq[k]) * (a.q[k] + 1) + cl[k]) * 3;
              v[k][0] = t[0];
              v[k][1] = t[1];
              v[k][2] = t[2];
              idx += stride * (a.span[k][iq[k]] + cl[k]);
              stride *= a.m[k];
            } else {
              v[k][0] = 1;
              v[k][1] = 0;
              v[k][2] = 0;
            }
          }
          const double wc = a.w[idx];
          double val = v[0][0] * v[1][0] * v[2][0];
          double der[3], hes[3][3];
          for (int j = 0; j < 3; ++j) {
            der[j] = 1;
            for (int k = 0; k < 3; ++k) der[j] *= v[k][k == j ? 1 : 0];
          }
          for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) {
              double h = 1;
              for (int k = 0; k < 3; ++k) h *= v[k][(k == j) + (k == l)];
              hes[j][l] = h;
            }
          W += wc * val;
          for (int j = 0; j < d; ++j) {
            dW[j] += wc * der[j];
            for (int l = 0; l < d; ++l) hW[j][l] += wc * hes[j][l];
          }
          for (int i = 0; i < d; ++i) {
            const double cw = wc * a.ctrl[idx * d + i];
            N[i] += cw * val;
            for (int j = 0; j < d; ++j) {
              dN[i][j] += cw * der[j];
              for (int l = 0; l < d; ++l) hN[i][j][l] += cw * hes[j][l];
            }
          }
        }
    // quotient rule: F = N / W
    double F[3], J[3][3] = {}, H[3][3][3] = {};
    for (int i = 0; i < d; ++i) F[i] = N[i] / W;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) J[i][j] = (dN[i][j] - F[i] * dW[j]) / W;
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j)
        for (int l = 0; l < d; ++l)
          H[i][j][l] = (hN[i][j][l] - J[i][j] * dW[l] - J[i][l] * dW[j] - F[i] * hW[j][l]) / W;
    // inverse (Jinv[j][i] = d eta_j / d x_i) and determinant
    double inv[3][3] = {}, det;
    if (d == 1) {
      det = J[0][0];
      inv[0][0] = 1.0 / det;
    } else if (d == 2) {
      det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
      inv[0][0] = J[1][1] / det;
      inv[0][1] = -J[0][1] / det;
      inv[1][0] = -J[1][0] / det;
      inv[1][1] = J[0][0] / det;
    } else {
      const double c00 = J[1][1] * J[2][2] - J[1][2] * J[2][1];
      const double c01 = J[1][2] * J[2][0] - J[1][0] * J[2][2];
      const double c02 = J[1][0] * J[2][1] - J[1][1] * J[2][0];
      det = J[0][0] * c00 + J[0][1] * c01 + J[0][2] * c02;
      inv[0][0] = c00 / det;
      inv[1][0] = c01 / det;
      inv[2][0] = c02 / det;
      inv[0][1] = (J[0][2] * J[2][1] - J[0][1] * J[2][2]) / det;
      inv[1][1] = (J[0][0] * J[2][2] - J[0][2] * J[2][0]) / det;
      inv[2][1] = (J[0][1] * J[2][0] - J[0][0] * J[2][1]) / det;
      inv[0][2] = (J[0][1] * J[1][2] - J[0][2] * J[1][1]) / det;
      inv[1][2] = (J[0][2] * J[1][0] - J[0][0] * J[1][2]) / det;
      inv[2][2] = (J[0][0] * J[1][1] - J[0][1] * J[1][0]) / det;
    }
    // A = Jinv Jinv^T; c_m = sum_jl A_jl H[m][j][l]; b_j = -sum_m Jinv[j][m] c_m
    double A[3][3] = {}, c[3] = {}, b[3] = {};
    for (int j = 0; j < d; ++j)
      for (int l = 0; l < d; ++l)
        for (int i = 0; i < d; ++i) A[j][l] += inv[j][i] * inv[l][i];
    for (int m_ = 0; m_ < d; ++m_)
      for (int j = 0; j < d; ++j)
        for (int l = 0; l < d; ++l) c[m_] += A[j][l] * H[m_][j][l];
    for (int j = 0; j < d; ++j)
      for (int m_ = 0; m_ < d; ++m_) b[j] -= inv[j][m_] * c[m_];
    // Ass. 4: F^{-1} with bounded derivatives -> det J of one sign, bounded away from 0
    if (!(fabs(det) > 1e-300) || !isfinite(det) || !isfinite(b[0] + b[1] + b[2])) atomicOr(a.flags, 4);
    else atomicOr(a.flags, det < 0 ? 1 : 2);
    double wq = 1;
    for (int k = 0; k < d; ++k) wq *= a.wq[k][iq[k]];
    a.out[qi] = wq * fabs(det);
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 3; ++i) a.out[(1 + j * 3 + i) * a.NQ + qi] = inv[j][i];
    for (int j = 0; j < 3; ++j) a.out[(10 + j) * a.NQ + qi] = b[j];
    for (int j = 0; j < 3; ++j) a.out[(13 + j) * a.NQ + qi] = j < d ? F[j] : 0.0;
  }
}

// ------------------------------------------------------------------------------------------
// element assembly
// ------------------------------------------------------------------------------------------
struct GeoAsmArgs {
  int d, p, nloc;
  int nel[3], m[3], n[3];     // elements, full functions (n_el + p), constrained sizes
  int nq[3];
  const double* bt[3];        // [n_el][p+1 points][p+1 functions][3]
  const double* qd;           // [13][NQ]
  int64_t NQ, Ns;
  int qc;                     // points per shared-memory chunk
  int color[3];               // element colour class of this launch
  double* st;                 // [3][S][Ns]
  int S;
};

constexpr int ASM_THREADS = 256;
constexpr int ASM_PP = 4;     // pairs per thread per round

__global__ void __launch_bounds__(ASM_THREADS) geo_assemble_kernel(GeoAsmArgs a) {
  extern __shared__ double sm[];
  const int d = a.d, p = a.p, P1 = p + 1, nloc = a.nloc;
  double* tab = sm;                               // [qc][nloc][5]: phi, grad_x (3), Lap
  double* wts = sm + size_t(a.qc) * nloc * 5;     // [qc]
  // colour class (c_1..c_d): elements e_k = c_k + (p+1) m_k.  Two elements of one class are
  // >= p+1 apart in some direction, so they share no basis function and the stencil updates
  // below never collide: plain read-modify-write, deterministic summation order.
  int e[3] = {0, 0, 0};
  {
    int64_t r = blockIdx.x;
    for (int k = 0; k < d; ++k) {
      const int cnt = (a.nel[k] - a.color[k] + p) / (p + 1);
      e[k] = a.color[k] + (p + 1) * int(r % cnt);
      r /= cnt;
    }
  }
  const int Q = nloc;  // (p+1)^d points per element
  const int npairs = nloc * nloc;
  for (int base = 0; base < npairs; base += ASM_THREADS * ASM_PP) {
    double acc[ASM_PP][3];
#pragma unroll
    for (int j = 0; j < ASM_PP; ++j) acc[j][0] = acc[j][1] = acc[j][2] = 0;
    for (int q0 = 0; q0 < Q; q0 += a.qc) {
      const int qn = min(a.qc, Q - q0);
      __syncthreads();
      for (int idx = threadIdx.x; idx < qn * nloc; idx += ASM_THREADS) {
        const int ql = q0 + idx / nloc, f = idx % nloc;
        int g[3] = {0, 0, 0}, fa[3] = {0, 0, 0};
        int64_t qi = 0, stride = 1;
        {
          int rq = ql, rf = f;
          for (int k = 0; k < d; ++k) {
            g[k] = rq % P1;
            rq /= P1;
            fa[k] = rf % P1;
            rf /= P1;
            qi += stride * (int64_t(e[k]) * P1 + g[k]);
            stride *= a.nq[k];
          }
        }
        double v[3][3];
        for (int k = 0; k < 3; ++k) {
          if (k < d) {
            const double* t = a.bt[k] + ((size_t(e[k]) * P1 + g[k]) * P1 + fa[k]) * 3;
            v[k][0] = t[0];
            v[k][1] = t[1];
            v[k][2] = t[2];
          } else {
            v[k][0] = 1;
            v[k][1] = 0;
            v[k][2] = 0;
          }
        }
        const double phi = v[0][0] * v[1][0] * v[2][0];
        double gr[3], hs[3][3];
        for (int j = 0; j < 3; ++j) {
          gr[j] = 1;
          for (int k = 0; k < 3; ++k) gr[j] *= v[k][k == j ? 1 : 0];
        }
        for (int j = 0; j < 3; ++j)
          for (int l = 0; l < 3; ++l) {
            double h = 1;
            for (int k = 0; k < 3; ++k) h *= v[k][(k == j) + (k == l)];
            hs[j][l] = h;
          }
        double inv[3][3], b[3];
        for (int j = 0; j < 3; ++j)
          for (int i = 0; i < 3; ++i) inv[j][i] = a.qd[(1 + j * 3 + i) * a.NQ + qi];
        for (int j = 0; j < 3; ++j) b[j] = a.qd[(10 + j) * a.NQ + qi];
        // grad_x = Jinv^T grad_eta ; Lap = sum_jl (Jinv Jinv^T)_jl d_jl + b . grad_eta
        double gx[3];
        for (int i = 0; i < 3; ++i) gx[i] = inv[0][i] * gr[0] + inv[1][i] * gr[1] + inv[2][i] * gr[2];
        double lap = b[0] * gr[0] + b[1] * gr[1] + b[2] * gr[2];
        for (int j = 0; j < d; ++j)
          for (int l = 0; l < d; ++l) {
            const double Ajl = inv[j][0] * inv[l][0] + inv[j][1] * inv[l][1] + inv[j][2] * inv[l][2];
            lap += Ajl * hs[j][l];
          }
        double* o = tab + (size_t(idx / nloc) * nloc + f) * 5;
        o[0] = phi;
        o[1] = gx[0];
        o[2] = gx[1];
        o[3] = gx[2];
        o[4] = lap;
        if (f == 0) wts[idx / nloc] = a.qd[qi];
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < ASM_PP; ++j) {
        const int pid = base + j * ASM_THREADS + threadIdx.x;
        if (pid >= npairs) continue;
        const int fa = pid / nloc, fb = pid % nloc;
        double s0 = 0, s1 = 0, s2 = 0;
        for (int q = 0; q < qn; ++q) {
          const double* ta = tab + (size_t(q) * nloc + fa) * 5;
          const double* tb = tab + (size_t(q) * nloc + fb) * 5;
          const double w = wts[q];
          s0 += w * ta[0] * tb[0];
          s1 += w * ta[4] * tb[4];
          s2 += w * (ta[1] * tb[1] + ta[2] * tb[2] + ta[3] * tb[3]);
        }
        acc[j][0] += s0;
        acc[j][1] += s1;
        acc[j][2] += s2;
      }
    }
    // scatter into the stencil rows of the constrained functions
#pragma unroll
    for (int j = 0; j < ASM_PP; ++j) {
      const int pid = base + j * ASM_THREADS + threadIdx.x;
      if (pid >= npairs) continue;
      int fa = pid / nloc, fb = pid % nloc;
      int64_t row = 0, rs = 1;
      int o = 0, os = 1;
      bool ok = true;
      for (int k = 0; k < d; ++k) {
        const int ga = e[k] + fa % P1, gb = e[k] + fb % P1;  // full indices
        fa /= P1;
        fb /= P1;
        ok = ok && ga >= 1 && ga <= a.m[k] - 2 && gb >= 1 && gb <= a.m[k] - 2;
        row += rs * (ga - 1);
        rs *= a.n[k];
        o += os * (gb - ga + p);
        os *= 2 * p + 1;
      }
      if (!ok) continue;
      a.st[(size_t(0) * a.S + o) * a.Ns + row] += acc[j][0];
      a.st[(size_t(1) * a.S + o) * a.Ns + row] += acc[j][1];
      a.st[(size_t(2) * a.S + o) * a.Ns + row] += acc[j][2];
    }
  }
}

// host tables of one direction: Gauss points / weights, discretisation basis per element
// host tables of one direction for qpe Gauss points per element: points / weights and the
// p+1 local basis functions' values, 1st and 2nd derivatives [n_el][qpe][p+1][3]
void dir_tables(int n_el, int p, int qpe, std::vector<double>& xq, std::vector<double>& wq,
                       std::vector<double>& bt) {
  auto kn = open_uniform_knots(n_el, p);
  const int m = n_el + p, P1 = p + 1, QP = qpe;
  std::vector<long double> gx, gw;
  gauss_legendre(QP, gx, gw);
  std::vector<long double> v0(m), v1(m), v2(m);
  xq.assign(size_t(n_el) * QP, 0);
  wq.assign(size_t(n_el) * QP, 0);
  bt.assign(size_t(n_el) * QP * P1 * 3, 0);
  for (int e = 0; e < n_el; ++e) {
    const long double a = kn[p + e], b = kn[p + e + 1];
    for (int g = 0; g < QP; ++g) {
      const long double x = 0.5L * (a + b) + 0.5L * (b - a) * gx[g];
      xq[size_t(e) * QP + g] = double(x);
      wq[size_t(e) * QP + g] = double(0.5L * (b - a) * gw[g]);
      bspline_eval(kn, p, x, v0.data(), v1.data(), v2.data());
      for (int f = 0; f < P1; ++f) {
        double* t = &bt[((size_t(e) * QP + g) * P1 + f) * 3];
        t[0] = double(v0[e + f]);
        t[1] = double(v1[e + f]);
        t[2] = double(v2[e + f]);
      }
    }
  }
}

// Point data of the mapped domain at qpe Gauss points per element and direction: the
// discretisation tables (bt) and, from geo_qpoint_kernel, |det J| w, J^{-1}, the Laplacian's
// first-order coefficients and x (qd, [16][NQ]).  LS_EINVAL for a singular / folded map.
struct GeoPts {
  double* qd = nullptr;
  const double* bt[3] = {nullptr, nullptr, nullptr};
  int nq[3] = {1, 1, 1};
  int64_t NQ = 1;
  int qpe = 0;
};

static int geo_points(const GeoMap& g, int d, int p, const int64_t* n_el, int qpe, std::vector<void*>& allocs,
                      cudaStream_t s, GeoPts& out, int64_t* launches) {
  GeoQArgs qa{};
  qa.d = d;
  out.qpe = qpe;
  out.NQ = 1;
  for (int k = 0; k < d; ++k) {
    out.nq[k] = int(n_el[k]) * qpe;
    out.NQ *= out.nq[k];
  }
  qa.NQ = out.NQ;
  for (int k = 0; k < d; ++k) {
    std::vector<double> xq, wq, bt;
    dir_tables(int(n_el[k]), p, qpe, xq, wq, bt);
    // geometry basis at the points: span (first non-zero function) and q+1 values
    const int q = g.q[k], mg = g.m[k];
    std::vector<double> gt(xq.size() * (q + 1) * 3);
    std::vector<int> span(xq.size());
    std::vector<long double> v0(mg), v1(mg), v2(mg);
    const auto& kn = g.knots[k];
    for (size_t i = 0; i < xq.size(); ++i) {
      const double x = xq[i];
      int sp = q;  // knot span: kn[sp] <= x < kn[sp+1], sp in [q, mg-1]
      while (sp < mg - 1 && kn[sp + 1] <= x) ++sp;
      span[i] = sp - q;
      bspline_eval(kn, q, x, v0.data(), v1.data(), v2.data());
      for (int c = 0; c <= q; ++c) {
        gt[(i * (q + 1) + c) * 3 + 0] = double(v0[sp - q + c]);
        gt[(i * (q + 1) + c) * 3 + 1] = double(v1[sp - q + c]);
        gt[(i * (q + 1) + c) * 3 + 2] = double(v2[sp - q + c]);
      }
    }
    double *dgt, *dwq, *dbt;
    int rc = dupload(allocs, gt, &dgt);
    if (rc == LS_OK) rc = dupload(allocs, wq, &dwq);
    if (rc == LS_OK) rc = dupload(allocs, bt, &dbt);
    if (rc != LS_OK) return rc;
    int* dspan = nullptr;
    GEO_CUDA(cudaMalloc(&dspan, span.size() * sizeof(int)));
    allocs.push_back(dspan);
    GEO_CUDA(cudaMemcpy(dspan, span.data(), span.size() * sizeof(int), cudaMemcpyHostToDevice));
    qa.nq[k] = out.nq[k];
    qa.q[k] = q;
    qa.m[k] = mg;
    qa.span[k] = dspan;
    qa.gt[k] = dgt;
    qa.wq[k] = dwq;
    out.bt[k] = dbt;
  }
  double *dctrl, *dw;
  int rc = dupload(allocs, g.ctrl, &dctrl);
  if (rc == LS_OK) rc = dupload(allocs, g.w, &dw);
  if (rc == LS_OK) rc = dalloc(allocs, &out.qd, size_t(16) * out.NQ);
  if (rc != LS_OK) return rc;
  qa.ctrl = dctrl;
  qa.w = dw;
  qa.out = out.qd;
  GEO_CUDA(cudaMemsetAsync(out.qd, 0, size_t(16) * out.NQ * sizeof(double), s));
  int* dflags = nullptr;
  GEO_CUDA(cudaMalloc(&dflags, sizeof(int)));
  allocs.push_back(dflags);
  GEO_CUDA(cudaMemsetAsync(dflags, 0, sizeof(int), s));
  qa.flags = dflags;
  geo_qpoint_kernel<<<unsigned(std::min<int64_t>((out.NQ + 255) / 256, 148 * 16)), 256, 0, s>>>(qa);
  GEO_CUDA(cudaGetLastError());
  if (launches) *launches += 1;
  int hflags = 0;
  GEO_CUDA(cudaMemcpyAsync(&hflags, dflags, sizeof(int), cudaMemcpyDeviceToHost, s));
  GEO_CUDA(cudaStreamSynchronize(s));
  if ((hflags & 4) || (hflags & 3) == 3) return LS_EINVAL;  // singular or folded map
  return LS_OK;
}

int geo_point_data(const GeoMap& g, int d, int p, const int64_t* n_el, int qpe, std::vector<void*>& allocs,
                   cudaStream_t s, double** qd, int64_t* NQ, int64_t* launches) {
  GeoPts pts;
  const int rc = geo_points(g, d, p, n_el, qpe, allocs, s, pts, launches);
  *qd = pts.qd;
  *NQ = pts.NQ;
  return rc;
}

int geo_assemble(GeoDev& gd, const GeoMap& g, int d, int p, const int64_t* n_el, cudaStream_t s,
                 int64_t* launches) {
  gd.d = d;
  gd.p = p;
  gd.Ns = 1;
  gd.S = 1;
  int nq[3] = {1, 1, 1}, m[3] = {1, 1, 1};
  for (int k = 0; k < d; ++k) {
    gd.nel[k] = int(n_el[k]);
    gd.n[k] = int(n_el[k]) + p - 2;
    m[k] = int(n_el[k]) + p;
    nq[k] = int(n_el[k]) * (p + 1);
    gd.Ns *= gd.n[k];
    gd.S *= 2 * p + 1;
  }
  int64_t NQ = 1, NE = 1;
  for (int k = 0; k < d; ++k) {
    NQ *= nq[k];
    NE *= n_el[k];
  }
  GeoAsmArgs aa{};
  GeoPts pts;
  LS_CHECK_RC(geo_points(g, d, p, n_el, p + 1, gd.allocs, s, pts, launches));
  for (int k = 0; k < d; ++k) aa.bt[k] = pts.bt[k];
  double* qd = pts.qd;
  LS_CHECK_RC(dalloc(gd.allocs, &gd.st, size_t(3) * gd.S * gd.Ns));
  GEO_CUDA(cudaMemsetAsync(gd.st, 0, size_t(3) * gd.S * gd.Ns * sizeof(double), s));
  // assembly
  aa.d = d;
  aa.p = p;
  aa.nloc = 1;
  for (int k = 0; k < d; ++k) aa.nloc *= p + 1;
  for (int k = 0; k < 3; ++k) {
    aa.nel[k] = k < d ? int(n_el[k]) : 1;
    aa.m[k] = m[k];
    aa.n[k] = gd.n[k];
    aa.nq[k] = nq[k];
  }
  aa.qd = qd;
  aa.NQ = NQ;
  aa.Ns = gd.Ns;
  aa.st = gd.st;
  aa.S = gd.S;
  const size_t smem_budget = 96 * 1024;
  aa.qc = int(std::max<size_t>(1, smem_budget / (size_t(aa.nloc) * 5 * 8 + 8)));
  aa.qc = std::min(aa.qc, aa.nloc);
  const size_t smem = (size_t(aa.qc) * aa.nloc * 5 + aa.qc) * sizeof(double);
  GEO_CUDA(cudaFuncSetAttribute(geo_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  int ncol = 1;
  for (int k = 0; k < d; ++k) ncol *= p + 1;
  int nlaunch = 0;
  for (int c = 0; c < ncol; ++c) {
    int64_t cnt = 1;
    int r = c;
    for (int k = 0; k < 3; ++k) {
      aa.color[k] = 0;
      if (k < d) {
        aa.color[k] = r % (p + 1);
        r /= p + 1;
        cnt *= (n_el[k] - aa.color[k] + p) / (p + 1);
      }
    }
    if (cnt == 0) continue;  // fewer than p+1 elements in some direction
    geo_assemble_kernel<<<unsigned(cnt), ASM_THREADS, smem, s>>>(aa);
    GEO_CUDA(cudaGetLastError());
    ++nlaunch;
  }
  GEO_CUDA(cudaStreamSynchronize(s));
  if (launches) *launches += nlaunch;
  int centre = 0, cs = 1;
  for (int k = 0; k < d; ++k) {
    centre += cs * p;
    cs *= 2 * p + 1;
  }
  for (int mat = 0; mat < 3; ++mat) gd.diag[mat] = gd.st + (size_t(mat) * gd.S + centre) * gd.Ns;
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// load vectors of the mapped-domain benchmarks (ls_rhs kinds 2, 3)
// ------------------------------------------------------------------------------------------
// P(x, y) = -(x^2 + y^2 - 1)(x^2 + y^2 - 4) x y^2,
// Lap P   = -2x (x^4 + 22 x^2 y^2 - 5 x^2 + 21 y^4 - 45 y^2 + 4)   (2D Laplacian).
// kind 2 (2D quarter annulus, PAPER.md 1128-1129): u = P sin(pi t),
//   f = pi cos(pi t) P - sin(pi t) Lap P: two terms (s_1 = P, g_1 = pi cos(pi t)),
//   (s_2 = -Lap P, g_2 = sin(pi t)).
// kind 3 (rotated quarter annulus, PAPER.md 1219-1221): u = P sin(z) (time independent),
//   f = -Lap_3D u = (P - Lap P) sin(z): one term (s_1 = f, g_1 = 1) -- the paper's forcing
//   for homogeneous data (reading c23: Table 2's lifting is out of scope).
__device__ __forceinline__ double annulus_P(double x, double y) {
  const double r2 = x * x + y * y;
  return -(r2 - 1.0) * (r2 - 4.0) * x * y * y;
}
__device__ __forceinline__ double annulus_lapP(double x, double y) {
  const double x2 = x * x, y2 = y * y;
  return -2.0 * x * (x2 * x2 + 22.0 * x2 * y2 - 5.0 * x2 + 21.0 * y2 * y2 - 45.0 * y2 + 4.0);
}
// the spatial factors s_1, s_2 of the kind at a physical point
__device__ __forceinline__ void load_terms(int kind, double x, double y, double z, double& s1, double& s2) {
  if (kind == 2) {
    s1 = annulus_P(x, y);
    s2 = -annulus_lapP(x, y);
  } else {
    s1 = (annulus_P(x, y) - annulus_lapP(x, y)) * sin(z);
    s2 = 0.0;
  }
}

struct GeoLoadArgs {
  int d, p, qpe, kind;
  int nel[3], m[3], n[3], nq[3];
  int color[3];
  const double* bt[3];   // [n_el][qpe][p+1][3]
  const double* qd;      // [16][NQ]
  int64_t NQ, Ns;
  double* lv;            // [4][Ns]: int s_1 phi, int s_2 phi, int s_1 Lap phi, int s_2 Lap phi
};

// one CTA per element of a colour class (e_k mod (p+1) fixed: no two CTAs share a row),
// threads over the local functions
__global__ void geo_load_kernel(GeoLoadArgs a) {
  const int d = a.d, P1 = a.p + 1, QP = a.qpe;
  int nloc = 1, nqe = 1;
  for (int k = 0; k < d; ++k) {
    nloc *= P1;
    nqe *= QP;
  }
  int e[3] = {0, 0, 0};
  {
    int64_t r = blockIdx.x;
    for (int k = 0; k < d; ++k) {
      const int cnt = (a.nel[k] - a.color[k] + a.p) / P1;
      e[k] = a.color[k] + P1 * int(r % cnt);
      r /= cnt;
    }
  }
  for (int f = threadIdx.x; f < nloc; f += blockDim.x) {
    int fl[3] = {0, 0, 0};
    int64_t row = 0, rs = 1;
    bool ok = true;
    {
      int r = f;
      for (int k = 0; k < d; ++k) {
        fl[k] = r % P1;
        r /= P1;
        const int gk = e[k] + fl[k];  // full index
        ok = ok && gk >= 1 && gk <= a.m[k] - 2;
        row += rs * (gk - 1);
        rs *= a.n[k];
      }
    }
    if (!ok) continue;  // Dirichlet
    double s0a = 0, s0b = 0, s2a = 0, s2b = 0;
    for (int ql = 0; ql < nqe; ++ql) {
      double v[3][3];
      int64_t qi = 0, qs = 1;
      int r = ql;
      for (int k = 0; k < 3; ++k) {
        if (k < d) {
          const int g = r % QP;
          r /= QP;
          const double* t = a.bt[k] + ((size_t(e[k]) * QP + g) * P1 + fl[k]) * 3;
          v[k][0] = t[0];
          v[k][1] = t[1];
          v[k][2] = t[2];
          qi += qs * (int64_t(e[k]) * QP + g);
          qs *= a.nq[k];
        } else {
          v[k][0] = 1;
          v[k][1] = 0;
          v[k][2] = 0;
        }
      }
      const double phi = v[0][0] * v[1][0] * v[2][0];
      double gr[3], hs[3][3];
      for (int j = 0; j < 3; ++j) {
        gr[j] = 1;
        for (int k = 0; k < 3; ++k) gr[j] *= v[k][k == j ? 1 : 0];
      }
      for (int j = 0; j < 3; ++j)
        for (int l = 0; l < 3; ++l) {
          double h = 1;
          for (int k = 0; k < 3; ++k) h *= v[k][(k == j) + (k == l)];
          hs[j][l] = h;
        }
      double inv[3][3], b[3];
      for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) inv[j][i] = a.qd[(1 + j * 3 + i) * a.NQ + qi];
      for (int j = 0; j < 3; ++j) b[j] = a.qd[(10 + j) * a.NQ + qi];
      double lap = b[0] * gr[0] + b[1] * gr[1] + b[2] * gr[2];
      for (int j = 0; j < d; ++j)
        for (int l = 0; l < d; ++l)
          lap += (inv[j][0] * inv[l][0] + inv[j][1] * inv[l][1] + inv[j][2] * inv[l][2]) * hs[j][l];
      const double w = a.qd[qi];
      double s1, s2;
      load_terms(a.kind, a.qd[13 * a.NQ + qi], a.qd[14 * a.NQ + qi], a.qd[15 * a.NQ + qi], s1, s2);
      s0a += w * s1 * phi;
      s0b += w * s2 * phi;
      s2a += w * s1 * lap;
      s2b += w * s2 * lap;
    }
    a.lv[row] += s0a;
    a.lv[a.Ns + row] += s0b;
    a.lv[2 * a.Ns + row] += s2a;
    a.lv[3 * a.Ns + row] += s2b;
  }
}

// int_Omega s_1^2 and int_Omega s_2^2 (||f||^2 of ls_energy_error)
__global__ void geo_fnorm_kernel(const double* __restrict__ qd, int64_t NQ, int kind, double* out2) {
  double a0 = 0, a1 = 0;
  for (int64_t qi = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; qi < NQ; qi += int64_t(gridDim.x) * blockDim.x) {
    double s1, s2;
    load_terms(kind, qd[13 * NQ + qi], qd[14 * NQ + qi], qd[15 * NQ + qi], s1, s2);
    const double w = qd[qi];
    a0 += w * s1 * s1;
    a1 += w * s2 * s2;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_down_sync(0xffffffffu, a0, o);
    a1 += __shfl_down_sync(0xffffffffu, a1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out2, a0);
    atomicAdd(out2 + 1, a1);
  }
}

int geo_load(GeoDev& gd, const GeoMap& g, const int64_t* n_el, int kind, cudaStream_t s, int64_t* launches) {
  if (!((kind == 2 && gd.d == 2) || (kind == 3 && gd.d == 3))) return LS_ENOTSUP;
  if (gd.lv && gd.lv_kind == kind) return LS_OK;  // cached
  const int d = gd.d, p = gd.p, qpe = p + 5;  // reading c16 on Omega
  std::vector<void*> tmp;  // point data of this computation only
  GeoPts pts;
  int rc = geo_points(g, d, p, n_el, qpe, tmp, s, pts, launches);
  if (rc == LS_OK && !gd.lv) rc = dalloc(gd.allocs, &gd.lv, size_t(4) * gd.Ns);
  double* dn = nullptr;
  if (rc == LS_OK) rc = dalloc(tmp, &dn, 2);
  if (rc == LS_OK) {
    GEO_CUDA(cudaMemsetAsync(gd.lv, 0, size_t(4) * gd.Ns * sizeof(double), s));
    GEO_CUDA(cudaMemsetAsync(dn, 0, 2 * sizeof(double), s));
    GeoLoadArgs la{};
    la.d = d;
    la.p = p;
    la.qpe = qpe;
    la.kind = kind;
    for (int k = 0; k < 3; ++k) {
      la.nel[k] = k < d ? int(n_el[k]) : 1;
      la.m[k] = k < d ? int(n_el[k]) + p : 1;
      la.n[k] = gd.n[k];
      la.nq[k] = pts.nq[k];
      la.bt[k] = pts.bt[k];
    }
    la.qd = pts.qd;
    la.NQ = pts.NQ;
    la.Ns = gd.Ns;
    la.lv = gd.lv;
    const int P1 = p + 1;
    int ncol = 1;
    for (int k = 0; k < d; ++k) ncol *= P1;
    for (int c = 0; c < ncol; ++c) {
      int64_t cnt = 1;
      int r = c;
      for (int k = 0; k < 3; ++k) {
        la.color[k] = 0;
        if (k < d) {
          la.color[k] = r % P1;
          r /= P1;
          cnt *= (n_el[k] - la.color[k] + p) / P1;
        }
      }
      if (cnt == 0) continue;
      geo_load_kernel<<<unsigned(cnt), 64, 0, s>>>(la);
      GEO_CUDA(cudaGetLastError());
      if (launches) *launches += 1;
    }
    geo_fnorm_kernel<<<unsigned(std::min<int64_t>((pts.NQ + 255) / 256, 148 * 8)), 256, 0, s>>>(pts.qd, pts.NQ, kind,
                                                                                                dn);
    GEO_CUDA(cudaGetLastError());
    if (launches) *launches += 1;
    GEO_CUDA(cudaMemcpyAsync(gd.fint, dn, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    GEO_CUDA(cudaStreamSynchronize(s));
    gd.lv_kind = kind;
  }
  for (void* v : tmp) cudaFree(v);
  return rc;
}

// b[t][i] = G1_1[t] S0_1[i] - G0_1[t] S2_1[i] + G1_2[t] S0_2[i] - G0_2[t] S2_2[i] with
// G0_m = int g_m b_t, G1_m = int g_m b_t' (host, 80-bit), G = [G0_1 | G1_1 | G0_2 | G1_2]
__global__ void geo_rhs_kernel(const double* __restrict__ lv, const double* __restrict__ G, double* __restrict__ b,
                               int t0, int nrows, int nt, int64_t Ns) {
  const int64_t total = int64_t(nrows) * Ns;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int t = t0 + int(idx / Ns);
    const int64_t i = idx % Ns;
    b[idx] = G[nt + t] * lv[i] - G[t] * lv[2 * Ns + i] + G[3 * nt + t] * lv[Ns + i] - G[2 * nt + t] * lv[3 * Ns + i];
  }
}

int geo_rhs(const GeoDev& gd, const double* G, double* b, int t0, int nrows, int nt, cudaStream_t s,
            int64_t* launches) {
  const int64_t total = int64_t(nrows) * gd.Ns;
  geo_rhs_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(gd.lv, G, b, t0, nrows,
                                                                                           nt, gd.Ns);
  GEO_CUDA(cudaGetLastError());
  if (launches) *launches += 1;
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// matvec
// ------------------------------------------------------------------------------------------
// rows [t_first, t_first + nout) of t1 = K_t x, t2 = M_t x (global time indices; the band is
// clipped to [0, n_t)); x_ext holds the global rows [s_first, s_first + ...) that the band of
// every output row needs (the time halo of a slab)
__global__ void geo_time_kernel(const double* __restrict__ x, double* __restrict__ t1, double* __restrict__ t2,
                                const double* __restrict__ bK, const double* __restrict__ bM, int nt, int pt,
                                int64_t Ns, int s_first, int t_first, int nout) {
  const int W = 2 * pt + 1;
  const int64_t total = int64_t(nout) * Ns;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int tl = int(idx / Ns);
    const int64_t i = idx - int64_t(tl) * Ns;
    const int t = t_first + tl;
    double a = 0, b = 0;
    const int lo = max(0, t - pt), hi = min(nt - 1, t + pt);
    for (int s = lo; s <= hi; ++s) {
      const double v = __ldg(x + int64_t(s - s_first) * Ns + i);
      a += __ldg(bK + t * W + (s - t + pt)) * v;
      b += __ldg(bM + t * W + (s - t + pt)) * v;
    }
    t1[idx] = a;
    t2[idx] = b;
  }
}

constexpr int ST_TC = 8;      // time slices per thread
constexpr int ST_THREADS = 128;

__global__ void __launch_bounds__(ST_THREADS) geo_stencil_kernel(
    const double* __restrict__ st, const double* __restrict__ t1, const double* __restrict__ t2,
    const double* __restrict__ xl, double* __restrict__ y, int d, int p, int n1, int n2, int n3, int64_t Ns,
    int S, int nt, int lastl) {
  // nt: output rows (local); lastl: local row of the global last slice, -1 if not here;
  // xl: that slice of x (W_t (x) L_s, W_t = e_{n_t} e_{n_t}^T)
  const int64_t i = blockIdx.x * int64_t(ST_THREADS) + threadIdx.x;
  if (i >= Ns) return;
  const int t0 = blockIdx.y * ST_TC;
  const int tn = min(ST_TC, nt - t0);
  const bool last = lastl >= t0 && lastl < t0 + tn;
  const int i1 = int(i % n1), i2 = int((i / n1) % n2), i3 = int(i / (int64_t(n1) * n2));
  const int W = 2 * p + 1;
  const int r2 = d >= 2 ? p : 0, r3 = d >= 3 ? p : 0;
  double acc[ST_TC];
#pragma unroll
  for (int k = 0; k < ST_TC; ++k) acc[k] = 0;
  double accL = 0;
  const double* Ms = st;
  const double* Js = st + size_t(S) * Ns;
  const double* Ls = st + size_t(2) * S * Ns;
  for (int o3 = -r3; o3 <= r3; ++o3) {
    const int j3 = i3 + o3;
    if (j3 < 0 || j3 >= n3) continue;
    for (int o2 = -r2; o2 <= r2; ++o2) {
      const int j2 = i2 + o2;
      if (j2 < 0 || j2 >= n2) continue;
      const int ob = ((o3 + r3) * (d >= 2 ? W : 1) + (o2 + r2)) * W;
      const int64_t jb = (int64_t(j3) * n2 + j2) * n1;
      for (int o1 = -p; o1 <= p; ++o1) {
        const int j1 = i1 + o1;
        if (j1 < 0 || j1 >= n1) continue;
        const int o = ob + o1 + p;
        const int64_t j = jb + j1;
        const double cm = __ldg(Ms + size_t(o) * Ns + i);
        const double cj = __ldg(Js + size_t(o) * Ns + i);
#pragma unroll
        for (int k = 0; k < ST_TC; ++k)
          if (k < tn) {
            const int64_t off = int64_t(t0 + k) * Ns + j;
            acc[k] += cm * __ldg(t1 + off) + cj * __ldg(t2 + off);
          }
        if (last) accL += __ldg(Ls + size_t(o) * Ns + i) * __ldg(xl + j);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < ST_TC; ++k)
    if (k < tn) y[int64_t(t0 + k) * Ns + i] = acc[k] + ((last && t0 + k == lastl) ? accL : 0.0);
}

// ---- tensor-core variant (default): the stencil pass as DMMA.8x8x4 tiles -------------------
// For a line L = (i_2, i_3) and a block of 8 consecutive rows i_1 in [8 rb, 8 rb + 8), the
// coupling to the source line (i_2 + o_2, i_3 + o_3) is an 8 x (8 + 2p) band block B.  With
// time as the M dimension: D[t][i] += sum_j T[t][j] B^T[j][i], i.e. m8n8k4 with A = 8 time
// slices x 4 source columns (loaded straight from t1 / t2, 32 B per time row) and B = the
// band block gathered from the compact stencil rows into registers once per source line
// and reused for every time block.  M_s on t1 and J_s on t2 accumulate into the same tile;
// L_s on x enters the tile of the last time block with only the row t = n_t - 1 non-zero.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

struct FragGeom {
  int d, p, n1, n2, n3, RB, KS, Q, W2;
  int64_t NL, Ns;
};

// CTAs per SM (register cap): 4 (128 registers) for up to 3 time blocks per warp, where
// that fits without spills, else 3
#ifndef GEO_DMMA_CTAS
#define GEO_DMMA_CTAS 3
#endif
#ifndef GEO_DMMA_CTAS_SMALL
#define GEO_DMMA_CTAS_SMALL 4
#endif
#ifndef GEO_TBM_MAX
#define GEO_TBM_MAX 5
#endif
template <int TBM, int KS>
__global__ void __launch_bounds__(128, (TBM <= 3 ? GEO_DMMA_CTAS_SMALL : GEO_DMMA_CTAS)) geo_dmma_kernel(const double* __restrict__ st,
                                                         const double* __restrict__ t1,
                                                         const double* __restrict__ t2,
                                                         const double* __restrict__ xl, double* __restrict__ y,
                                                         FragGeom g, int nt, int S, int lastl) {
  const int lane = threadIdx.x & 31;
  // work item = (time chunk of TBM blocks, line, 8-row block), the time chunk slowest: the
  // warps resident at one time share it, so the t1 / t2 rows they read stay in L2
  const int nchunk = (nt + 8 * TBM - 1) / (8 * TBM);
  const int64_t nwarps = g.NL * g.RB * nchunk;
  const int r2 = g.d >= 2 ? g.p : 0, r3 = g.d >= 3 ? g.p : 0;
  const int W = 2 * g.p + 1;
  const int trow = lane >> 2, kc = lane & 3;
  const double* Ms = st;
  const double* Js = st + size_t(S) * g.Ns;
  const double* Ls = st + size_t(2) * S * g.Ns;
  for (int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5; w < nwarps;
       w += (int64_t(gridDim.x) * blockDim.x) >> 5) {
    const int chunk = int(w / (g.NL * g.RB));
    const int64_t wl = w - int64_t(chunk) * g.NL * g.RB;
    const int64_t L = wl / g.RB;
    const int rb = int(wl - L * g.RB);
    const int i2 = int(L % g.n2), i3 = int(L / g.n2);
    const int tb0 = chunk * TBM;
    const int ntb = min(TBM, (nt + 7) / 8 - tb0);  // blocks of this chunk
    // local block of the global last slice (W_t = e e^T), -1 / out of range if not in this chunk
    const int tbl = lastl >= 0 ? lastl / 8 - tb0 : -1;
    const bool chunk_last = tbl >= 0 && tbl < ntb;                // warp-uniform
    const bool row_last = chunk_last && (tb0 + tbl) * 8 + trow == lastl;  // A row of this lane
    const int i1 = rb * 8 + trow;                  // B-fragment row of this lane (n = lane >> 2)
    const bool iok = i1 < g.n1;
    const int64_t brow = L * g.n1 + i1;
    int64_t toff[TBM];
    bool tok[TBM];
#pragma unroll
    for (int tb = 0; tb < TBM; ++tb) {
      const int t = (tb0 + tb) * 8 + trow;
      tok[tb] = tb < ntb && t < nt;
      toff[tb] = int64_t(t) * g.Ns;
    }
    double acc[TBM][2];
#pragma unroll
    for (int tb = 0; tb < TBM; ++tb) acc[tb][0] = acc[tb][1] = 0.0;
    for (int q = 0; q < g.Q; ++q) {
      const int j2 = i2 + q % g.W2 - r2, j3 = i3 + q / g.W2 - r3;
      if (j2 < 0 || j2 >= g.n2 || j3 < 0 || j3 >= g.n3) continue;  // warp-uniform
      const int64_t src = (int64_t(j3) * g.n2 + j2) * g.n1;
      // every load of this source line first (B: band entries (i_1, o_1 = 4 ks + k - n) gathered
      // from the compact stencil rows; A: t1 / t2 rows), then the DMMAs: one exposed latency
      // per source line, overlapped by the other resident warps' tensor work
      double bM[KS], bJ[KS], bL[KS], aM[KS][TBM], aJ[KS][TBM], aL[KS];
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int o1 = ks * 4 + kc - trow;
        const bool ok = iok && o1 >= 0 && o1 < W;
        const size_t off = size_t(o1 + W * q) * g.Ns + brow;
        bM[ks] = ok ? __ldg(Ms + off) : 0.0;
        bJ[ks] = ok ? __ldg(Js + off) : 0.0;
        bL[ks] = (ok && chunk_last) ? __ldg(Ls + off) : 0.0;
        const int j1 = rb * 8 - g.p + ks * 4 + kc;   // A-fragment column (k = lane & 3)
        const bool jok = j1 >= 0 && j1 < g.n1;
#pragma unroll
        for (int tb = 0; tb < TBM; ++tb) {
          const bool okt = jok && tok[tb];
          aM[ks][tb] = okt ? __ldg(t1 + toff[tb] + src + j1) : 0.0;
          aJ[ks][tb] = okt ? __ldg(t2 + toff[tb] + src + j1) : 0.0;
        }
        aL[ks] = (jok && row_last) ? __ldg(xl + src + j1) : 0.0;
      }
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int tb = 0; tb < TBM; ++tb) {
          if (tb < ntb) {
            dmma(acc[tb], aM[ks][tb], bM[ks]);
            dmma(acc[tb], aJ[ks][tb], bJ[ks]);
          }
          if (tb == tbl) dmma(acc[tb], aL[ks], bL[ks]);
        }
      }
    }
#pragma unroll
    for (int tb = 0; tb < TBM; ++tb) {
      const int t = (tb0 + tb) * 8 + trow;
      const int o1 = rb * 8 + 2 * kc;
      if (tb < ntb && t < nt) {
        double* yr = y + int64_t(t) * g.Ns + L * g.n1;
        if (o1 < g.n1) yr[o1] = acc[tb][0];
        if (o1 + 1 < g.n1) yr[o1 + 1] = acc[tb][1];
      }
    }
  }
}

static FragGeom frag_geom(const GeoDev& gd) {
  FragGeom g;
  g.d = gd.d;
  g.p = gd.p;
  g.n1 = gd.n[0];
  g.n2 = gd.d >= 2 ? gd.n[1] : 1;
  g.n3 = gd.d >= 3 ? gd.n[2] : 1;
  g.RB = (g.n1 + 7) / 8;
  g.KS = (8 + 2 * gd.p + 3) / 4;
  g.W2 = gd.d >= 2 ? 2 * gd.p + 1 : 1;
  g.Q = g.W2 * (gd.d >= 3 ? 2 * gd.p + 1 : 1);
  g.NL = int64_t(g.n2) * g.n3;
  g.Ns = gd.Ns;
  return g;
}

int geo_matvec(const GeoDev& gd, const double* bKt, const double* bMt, int nt_global, const double* x,
               int s_first, int t_first, int nout, double* y, double* t1, double* t2, cudaStream_t s,
               int64_t* launches) {
  if (nout <= 0) return LS_OK;
  const int64_t total = int64_t(nout) * gd.Ns;
  geo_time_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(
      x, t1, t2, bKt, bMt, nt_global, gd.pt, gd.Ns, s_first, t_first, nout);
  GEO_CUDA(cudaGetLastError());
  const int nt = nout;  // rows of t1, t2, y below
  const int lastl = (nt_global - 1 >= t_first && nt_global - 1 < t_first + nout) ? nt_global - 1 - t_first : -1;
  const double* xl = x + int64_t(nt_global - 1 - s_first) * gd.Ns;  // dereferenced only if lastl >= 0
  if (gd.variant != 1) {
    const FragGeom g = frag_geom(gd);
    const int ntb = (nt + 7) / 8;
    // time blocks per warp: the largest of 5..2 with the fewest idle blocks in the last chunk
    int tbm = GEO_TBM_MAX, waste = 1 << 30;
    for (int c = GEO_TBM_MAX; c >= 2; --c) {
      const int wst = (ntb + c - 1) / c * c - ntb;
      if (wst < waste) {
        waste = wst;
        tbm = c;
      }
    }
    if (ntb == 1) tbm = 2;
    const int64_t warps = g.NL * g.RB * ((ntb + tbm - 1) / tbm);
    const unsigned grid = unsigned(std::min<int64_t>((warps + 3) / 4, int64_t(1) << 30));
    // k-steps per 8-row band block: ceil((8 + 2p) / 4) = 3 (p = 2), 4 (p = 3, 4), 5 (p = 5, 6)
#define GEO_DMMA(TB)                                                                                      \
  do {                                                                                                    \
    if (g.KS == 3)                                                                                        \
      geo_dmma_kernel<TB, 3><<<grid, 128, 0, s>>>(gd.st, t1, t2, xl, y, g, nt, gd.S, lastl);              \
    else if (g.KS == 4)                                                                                   \
      geo_dmma_kernel<TB, 4><<<grid, 128, 0, s>>>(gd.st, t1, t2, xl, y, g, nt, gd.S, lastl);              \
    else                                                                                                  \
      geo_dmma_kernel<TB, 5><<<grid, 128, 0, s>>>(gd.st, t1, t2, xl, y, g, nt, gd.S, lastl);              \
  } while (0)
    switch (tbm) {
      case 2: GEO_DMMA(2); break;
      case 3: GEO_DMMA(3); break;
      case 4: GEO_DMMA(4); break;
      default: GEO_DMMA(5); break;
    }
#undef GEO_DMMA
    GEO_CUDA(cudaGetLastError());
    if (launches) *launches += 2;
    return LS_OK;
  }
  dim3 grid(unsigned((gd.Ns + ST_THREADS - 1) / ST_THREADS), unsigned((nt + ST_TC - 1) / ST_TC));
  geo_stencil_kernel<<<grid, ST_THREADS, 0, s>>>(gd.st, t1, t2, xl, y, gd.d, gd.p, gd.n[0], gd.n[1], gd.n[2],
                                                 gd.Ns, gd.S, nt, lastl);
  GEO_CUDA(cudaGetLastError());
  if (launches) *launches += 2;
  return LS_OK;
}

// ------------------------------------------------------------------------------------------
// P^G diagonal scaling
// ------------------------------------------------------------------------------------------
__global__ void pg_scaling_kernel(const double* __restrict__ Md, const double* __restrict__ Jd,
                                  const double* __restrict__ Ld, const double* __restrict__ bK,
                                  const double* __restrict__ bM, int pt, const double* __restrict__ pdt,
                                  const double* __restrict__ pds, double* __restrict__ out, int nt, int64_t Ns,
                                  int t0, int nrows) {
  const int W = 2 * pt + 1;
  const int64_t total = int64_t(nrows) * Ns;
  for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
       idx += int64_t(gridDim.x) * blockDim.x) {
    const int t = t0 + int(idx / Ns);  // global time index of this slab row
    const int64_t i = idx % Ns;
    double a = bK[t * W + pt] * Md[i] + bM[t * W + pt] * Jd[i];
    if (t == nt - 1) a += Ld[i];  // W_t = e_{n_t} e_{n_t}^T
    const double pb = pdt[t] * pds[i] + pdt[nt + t] * pds[Ns + i];
    out[idx] = sqrt(pb / a);
  }
}

int pg_scaling(const GeoDev& gd, const double* bKt, const double* bMt, int nt, const double* pdiag_t,
               const double* pdiag_s, double* dm12, int t0, int nrows, cudaStream_t s, int64_t* launches) {
  const int64_t total = int64_t(nrows) * gd.Ns;
  pg_scaling_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 16)), 256, 0, s>>>(
      gd.diag[0], gd.diag[1], gd.diag[2], bKt, bMt, gd.pt, pdiag_t, pdiag_s, dm12, nt, gd.Ns, t0, nrows);
  GEO_CUDA(cudaGetLastError());
  if (launches) *launches += 1;
  return LS_OK;
}

__global__ void scale_vec_kernel(const double* __restrict__ sc, const double* __restrict__ x,
                                 double* __restrict__ y, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = sc[i] * x[i];
}

int scale_vec(const double* sc, const double* x, double* y, int64_t n, cudaStream_t s, int64_t* launches) {
  scale_vec_kernel<<<unsigned(std::min<int64_t>((n + 255) / 256, 148 * 8)), 256, 0, s>>>(sc, x, y, n);
  GEO_CUDA(cudaGetLastError());
  if (launches) *launches += 1;
  return LS_OK;
}

}  // namespace ls
