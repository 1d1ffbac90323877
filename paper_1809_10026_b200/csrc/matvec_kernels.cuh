// Matrix-free y = A x on the identity map (eq:A_kron, PAPER.md 686-703),
// sum-factorised over the banded univariate factors (half-bandwidth p).
//
// With M_s = (x)_k M_k, L_s = sum_k K_(k), J_s = sum_k J_(k) + sum_{k!=l} K_(k) K_(l)
// (the last by integration by parts, int b_i'' b_j = -int b_i' b_j' on the
// Dirichlet basis), three running spatial tensors are carried
// direction by direction:
//     after direction 1:   S_M = M_1 x,   S_K = K_1 x,   S_J = J_1 x
//     direction k >= 2:    S_M <- M_k S_M
//                          S_K <- K_k S_M + M_k S_K
//                          S_J <- J_k S_M + M_k S_J + 2 K_k S_K
// so that after direction d: S_M = M_s x, S_K = L_s x, S_J = J_s x (per time
// slice), and finally, along time,
//     y = K_t S_M + M_t S_J + W_t S_K,   W_t = e_{n_t} e_{n_t}^T (PAPER.md 694).
// One kernel per direction reads the (up to) three inputs and writes the three
// outputs: d + 1 launches, HBM-bound.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ls {

struct BandArgs {
  const double* SM;  // inputs (SK, SJ null for the first direction)
  const double* SK;
  const double* SJ;
  double* oM;
  double* oK;
  double* oJ;
  const double* bM;  // bands [n][2hb+1], entry (a, i) at a*(2hb+1) + (i - a + hb)
  const double* bK;
  const double* bJ;
  int n, hb;
  uint32_t Q;         // product of faster extents
  uint64_t total;     // number of output elements
};

// FIRST: direction 1 (inputs: SM = x only).
template <bool FIRST>
__global__ void __launch_bounds__(256) band_triple_kernel(BandArgs a) {
  const int W = 2 * a.hb + 1;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < a.total;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t pq = e / (uint64_t(a.n) * a.Q);
    const uint32_t rem = uint32_t(e - pq * uint64_t(a.n) * a.Q);
    const int row = rem / a.Q;
    const uint32_t q = rem - row * a.Q;
    const uint64_t base = pq * uint64_t(a.n) * a.Q + q;
    const int lo = max(0, row - a.hb), hi = min(a.n - 1, row + a.hb);
    const double* bm = a.bM + size_t(row) * W - row + a.hb;
    const double* bk = a.bK + size_t(row) * W - row + a.hb;
    const double* bj = a.bJ + size_t(row) * W - row + a.hb;
    double m = 0, k = 0, j = 0;
    for (int i = lo; i <= hi; ++i) {
      const uint64_t off = base + uint64_t(i) * a.Q;
      const double xm = __ldg(a.SM + off);
      const double cm = __ldg(bm + i), ck = __ldg(bk + i), cj = __ldg(bj + i);
      if (FIRST) {
        m = fma(cm, xm, m);
        k = fma(ck, xm, k);
        j = fma(cj, xm, j);
      } else {
        const double xk = __ldg(a.SK + off), xj = __ldg(a.SJ + off);
        m = fma(cm, xm, m);
        k = fma(ck, xm, fma(cm, xk, k));
        j = fma(cj, xm, fma(cm, xj, fma(2.0 * ck, xk, j)));
      }
    }
    a.oM[e] = m;
    a.oK[e] = k;
    a.oJ[e] = j;
  }
}

struct TimeArgs {
  const double* SM;
  const double* SK;
  const double* SJ;
  double* y;
  const double* bKt;  // bands of K_t, M_t
  const double* bMt;
  int nt, hb;
  int t_first;   // global time index of output row 0
  int s_first;   // global time index of S row 0 (extended slab incl. halo)
  uint32_t Ns;
  uint64_t total;  // output rows * Ns
};

// y[t][s] = sum_i K_t[t][i] S_M[i][s] + M_t[t][i] S_J[i][s] + [t == n_t-1] S_K[t][s]
// (t, i global time indices; S rows are stored from global row s_first)
__global__ void __launch_bounds__(256) band_time_kernel(TimeArgs a) {
  const int W = 2 * a.hb + 1;
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < a.total;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const int tl = int(e / a.Ns);
    const uint32_t s = uint32_t(e - uint64_t(tl) * a.Ns);
    const int t = a.t_first + tl;
    const int lo = max(0, t - a.hb), hi = min(a.nt - 1, t + a.hb);
    const double* bk = a.bKt + size_t(t) * W - t + a.hb;
    const double* bm = a.bMt + size_t(t) * W - t + a.hb;
    double y = 0;
    for (int i = lo; i <= hi; ++i) {
      const uint64_t off = uint64_t(i - a.s_first) * a.Ns + s;
      y = fma(__ldg(bk + i), __ldg(a.SM + off), fma(__ldg(bm + i), __ldg(a.SJ + off), y));
    }
    if (t == a.nt - 1) y += __ldg(a.SK + uint64_t(t - a.s_first) * a.Ns + s);
    a.y[e] = y;
  }
}

} // namespace ls
