// Discretisation-error norms of a least-squares solution.
//
// For u_h = sum_i x_i B_i and the exact solution u of a built-in benchmark, by direct
// space-time Gauss quadrature (Q = p_s + 3 points per element and space direction,
// QT = p_t + 3 in time; reading c24):
//     out[0] = int int (u - u_h)^2                out[4] = int int u^2
//     out[1] = int int (d_t (u - u_h))^2          out[5] = int int (d_t u)^2
//     out[2] = int int |grad_x (u - u_h)|^2       out[6] = int int |grad_x u|^2
//     out[3] = int int (Lap (u - u_h))^2          out[7] = int int (Lap u)^2
// so ||e||_V0^2 = out[1] + out[3] (PAPER.md 318-323), ||e||_L2^2 = out[0] and the space-time
// ||e||_H1^2 = out[0] + out[1] + out[2] (Fig. 2, PAPER.md 1131-1139).
//
// Kernel: one CTA per space-time element at a time (grid-stride over elements, fixed per
// CTA: deterministic).  The element's (p_t+1)(p_s+1)^d coefficients are staged in shared
// memory; for each time Gauss point the time contraction (values and d/dt) and then, per
// spatial derivative multi-index, d successive sum-factorised contractions with the local
// univariate tables give u_h's parametric derivatives at the Q^d spatial points.  Physical
// gradient / Laplacian by the chain rule of PAPER.md 986-990 with the map data of
// geo_point_data (mapped domains) or the identity (cube).  Per-CTA partial sums, then one
// single-block reduction in a fixed order.
#include <cmath>
#include <vector>

#include "err.hpp"
#include "geo.hpp"

namespace ls {

namespace {

constexpr int ERR_THREADS = 128;
constexpr double kPi = 3.14159265358979323846;

struct ErrArgs {
  int d, ps, pt, kind;
  int nel[3], nelt;
  int n[3], nt;          // constrained sizes
  int Q, QT;             // Gauss points per element: space, time
  const double* bt[3];   // [nel][Q][ps+1][3] local basis values / 1st / 2nd derivatives
  const double* xq[3];   // [nel * Q] parametric points
  const double* wq[3];   // [nel * Q] weights
  const double* btt;     // [nelt][QT][pt+1][3]
  const double* xqt;     // [nelt * QT]
  const double* wqt;
  const double* qd;      // mapped: [16][NQ] (geo_point_data), nullptr on the cube
  int64_t NQ;
  int nq[3];
  const double* x;       // [nt][N_s]
  int64_t Ns, nelem;
  double* partials;      // [gridDim][8]
};

// spatial derivative multi-indices per field (direction 1 first); the last field is d/dt
template <int D>
struct Fields;
template <>
struct Fields<1> {
  static constexpr int NF = 4;
  __device__ static int alpha(int f, int k) { return f == 3 ? 0 : f; }
};
template <>
struct Fields<2> {
  static constexpr int NF = 7;  // (0,0) (1,0) (0,1) (2,0) (0,2) (1,1) | t
  __device__ static int alpha(int f, int k) {
    const int a[7][2] = {{0, 0}, {1, 0}, {0, 1}, {2, 0}, {0, 2}, {1, 1}, {0, 0}};
    return a[f][k];
  }
};
template <>
struct Fields<3> {
  static constexpr int NF = 11;  // 0, d1, d2, d3, d11, d22, d33, d12, d13, d23 | t
  __device__ static int alpha(int f, int k) {
    const int a[11][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {2, 0, 0}, {0, 2, 0},
                          {0, 0, 2}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}, {0, 0, 0}};
    return a[f][k];
  }
};

// exact solutions (value, d/dt, grad_x, Lap) of the built-in benchmarks
__device__ void exact_u(int kind, int D, const double* X, double t, double& u, double& ut, double* g,
                        double& lap) {
  if (kind == 1) {  // cube, u = prod_k sin(pi x_k) sin t (PAPER.md 1166)
    double s[3], c[3], S = 1.0;
    for (int k = 0; k < D; ++k) {
      sincospi(X[k], &s[k], &c[k]);
      S *= s[k];
    }
    const double st = sin(t), ct = cos(t);
    u = S * st;
    ut = S * ct;
    for (int k = 0; k < D; ++k) {
      double o = kPi * c[k];
      for (int j = 0; j < D; ++j)
        if (j != k) o *= s[j];
      g[k] = o * st;
    }
    lap = -D * kPi * kPi * u;
  } else {  // kind 2, quarter annulus (PAPER.md 1129): u = P(x, y) sin(pi t)
    const double x = X[0], y = X[1], x2 = x * x, y2 = y * y, r2 = x2 + y2;
    const double gg = (r2 - 1.0) * (r2 - 4.0), g1 = 2.0 * r2 - 5.0;  // g(r^2), dg/d(r^2)
    const double P = -gg * x * y2;
    const double Px = -y2 * (2.0 * x2 * g1 + gg);
    const double Py = -2.0 * x * y * (y2 * g1 + gg);
    const double LP = -2.0 * x * (x2 * x2 + 22.0 * x2 * y2 - 5.0 * x2 + 21.0 * y2 * y2 - 45.0 * y2 + 4.0);
    double sp, cp;
    sincospi(t, &sp, &cp);
    u = P * sp;
    ut = kPi * cp * P;
    g[0] = Px * sp;
    g[1] = Py * sp;
    lap = LP * sp;
  }
}

template <int D>
__global__ void __launch_bounds__(ERR_THREADS) err_norm_kernel(const ErrArgs a) {
  using Fd = Fields<D>;
  constexpr int NF = Fd::NF;
  extern __shared__ double sm[];
  const int P1 = a.ps + 1, PT = a.pt + 1, Q = a.Q;
  int P1d = 1, Qd = 1;
  for (int k = 0; k < D; ++k) {
    P1d *= P1;
    Qd *= Q;
  }
  double* xl = sm;                // [PT][P1^D]
  double* X0 = xl + PT * P1d;     // [P1^D]
  double* X1 = X0 + P1d;
  double* bufA = X1 + P1d;        // ping-pong of the contractions: <= max(P1, Q)^D each
  int mx = 1;
  for (int k = 0; k < D; ++k) mx *= (P1 > Q ? P1 : Q);
  double* bufB = bufA + mx;
  double* F = bufB + mx;          // [NF][Q^D]
  double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int tid = threadIdx.x;
  int64_t nels = 1;
  for (int k = 0; k < D; ++k) nels *= a.nel[k];

  for (int64_t el = blockIdx.x; el < a.nelem; el += gridDim.x) {
    int e[3] = {0, 0, 0};
    int64_t r = el;
    for (int k = 0; k < D; ++k) {
      e[k] = int(r % a.nel[k]);
      r /= a.nel[k];
    }
    const int et = int(r);
    // element coefficients: full local function e + a_k -> constrained index e + a_k - 1
    __syncthreads();
    for (int i = tid; i < PT * P1d; i += ERR_THREADS) {
      int rr = i % P1d;
      const int at = i / P1d;
      int64_t off = 0, st = 1;
      bool ok = true;
      for (int k = 0; k < D; ++k) {
        const int g = e[k] + rr % P1 - 1;
        rr /= P1;
        ok = ok && g >= 0 && g < a.n[k];
        off += st * g;
        st *= a.n[k];
      }
      const int gt = et + at - 1;
      ok = ok && gt >= 0 && gt < a.nt;
      xl[i] = ok ? a.x[int64_t(gt) * a.Ns + off] : 0.0;
    }
    for (int qt = 0; qt < a.QT; ++qt) {
      const double* tt = a.btt + (size_t(et) * a.QT + qt) * PT * 3;
      __syncthreads();
      for (int i = tid; i < P1d; i += ERR_THREADS) {
        double v0 = 0.0, v1 = 0.0;
        for (int at = 0; at < PT; ++at) {
          const double c = xl[at * P1d + i];
          v0 += tt[at * 3 + 0] * c;
          v1 += tt[at * 3 + 1] * c;
        }
        X0[i] = v0;
        X1[i] = v1;
      }
      for (int f = 0; f < NF; ++f) {
        const double* in = (f == NF - 1) ? X1 : X0;
        // stage k: [P1^(D-k)][P1][Q^(k-1)] -> [P1^(D-k)][Q][Q^(k-1)]
        int S = P1d / P1, Fst = 1;
        for (int k = 0; k < D; ++k) {
          double* out = (k == D - 1) ? F + f * Qd : ((k & 1) ? bufB : bufA);
          const int al = Fd::alpha(f, k);
          const double* T = a.bt[k] + size_t(e[k]) * Q * P1 * 3 + al;
          __syncthreads();
          const int tot = S * Q * Fst;
          for (int i = tid; i < tot; i += ERR_THREADS) {
            const int s = i / (Q * Fst), rem = i % (Q * Fst), q = rem / Fst, fi = rem % Fst;
            double v = 0.0;
            for (int aa = 0; aa < P1; ++aa) v += T[(q * P1 + aa) * 3] * in[(s * P1 + aa) * Fst + fi];
            out[i] = v;
          }
          in = out;
          S /= P1;
          Fst *= Q;
        }
      }
      __syncthreads();
      const double t = a.xqt[size_t(et) * a.QT + qt];
      const double wt = a.wqt[size_t(et) * a.QT + qt];
      for (int i = tid; i < Qd; i += ERR_THREADS) {
        int q[3] = {0, 0, 0}, rr = i;
        for (int k = 0; k < D; ++k) {
          q[k] = rr % Q;
          rr /= Q;
        }
        double X[3] = {0, 0, 0}, Ji[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}}, b[3] = {0, 0, 0}, w;
        if (a.qd) {
          int64_t qi = 0, st = 1;
          for (int k = 0; k < D; ++k) {
            qi += st * (int64_t(e[k]) * Q + q[k]);
            st *= a.nq[k];
          }
          w = a.qd[qi];
          for (int j = 0; j < 3; ++j)
            for (int l = 0; l < 3; ++l) Ji[j][l] = a.qd[(1 + 3 * j + l) * a.NQ + qi];
          for (int j = 0; j < 3; ++j) b[j] = a.qd[(10 + j) * a.NQ + qi];
          for (int j = 0; j < 3; ++j) X[j] = a.qd[(13 + j) * a.NQ + qi];
        } else {
          w = 1.0;
          for (int k = 0; k < D; ++k) {
            X[k] = a.xq[k][size_t(e[k]) * Q + q[k]];
            w *= a.wq[k][size_t(e[k]) * Q + q[k]];
          }
        }
        w *= wt;
        // parametric derivatives of u_h
        double gh[3] = {0, 0, 0}, H[3][3] = {};
        const double uh = F[i];
        for (int j = 0; j < D; ++j) gh[j] = F[(1 + j) * Qd + i];
        for (int j = 0; j < D; ++j) H[j][j] = F[(1 + D + j) * Qd + i];
        if (D == 2) H[0][1] = H[1][0] = F[5 * Qd + i];
        if (D == 3) {
          H[0][1] = H[1][0] = F[7 * Qd + i];
          H[0][2] = H[2][0] = F[8 * Qd + i];
          H[1][2] = H[2][1] = F[9 * Qd + i];
        }
        const double uth = F[(NF - 1) * Qd + i];
        // chain rule: grad_x = Jinv^T grad_eta, Lap = sum_jl A_jl H_jl + b . grad_eta
        double gx[3] = {0, 0, 0}, lap = 0.0;
        for (int ii = 0; ii < D; ++ii)
          for (int j = 0; j < D; ++j) gx[ii] += Ji[j][ii] * gh[j];
        for (int j = 0; j < D; ++j) {
          lap += b[j] * gh[j];
          for (int l = 0; l < D; ++l) {
            double A = 0.0;
            for (int ii = 0; ii < D; ++ii) A += Ji[j][ii] * Ji[l][ii];
            lap += A * H[j][l];
          }
        }
        double u, ut, g[3] = {0, 0, 0}, lu;
        exact_u(a.kind, D, X, t, u, ut, g, lu);
        const double e0 = u - uh, e1 = ut - uth, e3 = lu - lap;
        double e2 = 0.0, g2 = 0.0;
        for (int k = 0; k < D; ++k) {
          e2 += (g[k] - gx[k]) * (g[k] - gx[k]);
          g2 += g[k] * g[k];
        }
        acc[0] += w * e0 * e0;
        acc[1] += w * e1 * e1;
        acc[2] += w * e2;
        acc[3] += w * e3 * e3;
        acc[4] += w * u * u;
        acc[5] += w * ut * ut;
        acc[6] += w * g2;
        acc[7] += w * lu * lu;
      }
    }
  }
  // CTA reduction (fixed order): warp shuffles, then warp 0
  __shared__ double red[ERR_THREADS / 32][8];
  for (int j = 0; j < 8; ++j) {
    double v = acc[j];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5][j] = v;
  }
  __syncthreads();
  if (tid < 8) {
    double v = 0.0;
    for (int w = 0; w < ERR_THREADS / 32; ++w) v += red[w][tid];
    a.partials[size_t(blockIdx.x) * 8 + tid] = v;
  }
}

// out[j] = sum_b partials[b][j], one block, fixed order
__global__ void err_reduce_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double s[256];
  for (int j = 0; j < 8; ++j) {
    double v = 0.0;
    for (int b = threadIdx.x; b < nb; b += 256) v += part[size_t(b) * 8 + j];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (int(threadIdx.x) < o) s[threadIdx.x] += s[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[j] = s[0];
    __syncthreads();
  }
}

struct Buf {
  std::vector<void*> v;
  ~Buf() {
    for (void* p : v) cudaFree(p);
  }
  double* up(const std::vector<double>& h) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(h.size(), 1) * sizeof(double)) != cudaSuccess) return nullptr;
    v.push_back(p);
    if (cudaMemcpy(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return static_cast<double*>(p);
  }
  double* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) return nullptr;
    v.push_back(p);
    return static_cast<double*>(p);
  }
};

}  // namespace

int error_norms(const ErrSetup& es, const double* x, cudaStream_t s, int64_t* launches, double* out8) {
  const int d = es.d;
  if (d < 1 || d > 3 || !(es.kind == 1 || (es.kind == 2 && d == 2 && es.gmap))) return LS_ENOTSUP;
  if ((es.kind == 1) == bool(es.gmap)) return LS_ENOTSUP;
  ErrArgs a{};
  a.d = d;
  a.ps = es.ps;
  a.pt = es.pt;
  a.kind = es.kind;
  a.Q = es.ps + 3;
  a.QT = es.pt + 3;
  a.nt = es.nt;
  a.nelt = int(es.n_el[d]);
  a.x = x;
  a.Ns = 1;
  Buf buf;
  for (int k = 0; k < 3; ++k) {
    a.nel[k] = 1;
    a.n[k] = 1;
  }
  a.nelem = es.n_el[d];
  for (int k = 0; k < d; ++k) {
    a.nel[k] = int(es.n_el[k]);
    a.n[k] = int(es.n_el[k]) + es.ps - 2;
    a.Ns *= a.n[k];
    a.nelem *= es.n_el[k];
    std::vector<double> xq, wq, bt;
    dir_tables(int(es.n_el[k]), es.ps, a.Q, xq, wq, bt);
    a.xq[k] = buf.up(xq);
    a.wq[k] = buf.up(wq);
    a.bt[k] = buf.up(bt);
    a.nq[k] = int(es.n_el[k]) * a.Q;
    if (!a.xq[k] || !a.wq[k] || !a.bt[k]) return LS_ENOMEM;
  }
  {
    std::vector<double> xq, wq, bt;
    dir_tables(a.nelt, es.pt, a.QT, xq, wq, bt);
    a.xqt = buf.up(xq);
    a.wqt = buf.up(wq);
    a.btt = buf.up(bt);
    if (!a.xqt || !a.wqt || !a.btt) return LS_ENOMEM;
  }
  if (es.gmap) {
    double* qd = nullptr;
    const int rc = geo_point_data(*es.gmap, d, es.ps, es.n_el, a.Q, buf.v, s, &qd, &a.NQ, launches);
    if (rc != LS_OK) return rc;
    a.qd = qd;
  }
  const int P1 = es.ps + 1, PT = es.pt + 1;
  int P1d = 1, Qd = 1, mx = 1;
  for (int k = 0; k < d; ++k) {
    P1d *= P1;
    Qd *= a.Q;
    mx *= std::max(P1, a.Q);
  }
  const int NF = d == 1 ? 4 : d == 2 ? 7 : 11;
  const size_t smem = sizeof(double) * (size_t(PT) * P1d + 2 * P1d + 2 * mx + size_t(NF) * Qd);
  if (smem > 200 * 1024) return LS_ENOTSUP;
  const int grid = int(std::min<int64_t>(a.nelem, 148 * 8));
  double* part = buf.alloc(size_t(grid) * 8);
  double* dout = buf.alloc(8);
  if (!part || !dout) return LS_ENOMEM;
  a.partials = part;
  cudaError_t e = cudaSuccess;
  if (d == 1) {
    cudaFuncSetAttribute(err_norm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    err_norm_kernel<1><<<grid, ERR_THREADS, smem, s>>>(a);
  } else if (d == 2) {
    cudaFuncSetAttribute(err_norm_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    err_norm_kernel<2><<<grid, ERR_THREADS, smem, s>>>(a);
  } else {
    cudaFuncSetAttribute(err_norm_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    err_norm_kernel<3><<<grid, ERR_THREADS, smem, s>>>(a);
  }
  err_reduce_kernel<<<1, 256, 0, s>>>(part, grid, dout);
  e = cudaGetLastError();
  if (e != cudaSuccess) return LS_ECUDA;
  if (launches) *launches += 2;
  if (cudaMemcpyAsync(out8, dout, 8 * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess) return LS_ECUDA;
  if (cudaStreamSynchronize(s) != cudaSuccess) return LS_ECUDA;
  return LS_OK;
}

}  // namespace ls
