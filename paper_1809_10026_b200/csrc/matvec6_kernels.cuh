// ls_matvec v6 (LS_TUNE_MV6): the direction-3 and time passes of v4 (mv4_kernels.cuh plane
// pass: P_M = M2 M1 x, P_K = (K2 M1 + M2 K1) x, P_J = (J2 M1 + M2 J1 + 2 K2 K1) x) as
// streaming DFMA stencil passes instead of DMMA band tiles (eq:A_kron, PAPER.md 686-703):
//   direction 3:  S_M = M3 P_M,  S_J = M3 P_J + J3 P_M + 2 K3 P_K,
//                 on the last time slice also L = M3 P_K + K3 P_M (the L_s x of W_t (x) L_s)
//   time:         y = K_t S_M + M_t S_J  (+ L on the global row n_t - 1: W_t = e_{n_t} e_{n_t}^T)
// Why: a banded product on 8 x 4 DMMA tiles executes (8 + 2p) / (2p + 1) ... 1.54x its
// multiply-adds at p = 6 (the parallelogram of the band in whole tiles), which made the v4
// direction-3 pass FP64-pipe bound (66 % DMMA pipe, 3.28 ms at config 4) although its HBM
// traffic (40 B/DOF) needs 1.9 ms.  A Toeplitz stencil in DFMAs executes exactly 2p + 1
// multiply-adds per output (52 per DOF here, 0.9 ms of FP64 pipe at config 4), so both
// passes become HBM-bound.
// Banded products: the v2 split B = T + E (matvec2_kernels.cuh, reading c18): one stencil
// (constant-bank DFMA operands) on every row plus exact per-row corrections of the boundary
// rows.  Work item = one warp: 32 consecutive columns of one time slice (lane = column,
// coalesced 256-byte rows) x R consecutive rows of the banded direction; the window of
// R + 2p input rows sits in registers.  Warps are persistent over the items; the items of a
// column block are consecutive, so the 2p halo rows of neighbouring chunks hit L1 / L2.
// Time pass: fused PCG p.q (dotp != nullptr): every stored y element times p at the same
// offset, warp sums -> CTA sum in a fixed order -> dot_part[blockIdx.x] (fixed grid).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "matvec2_kernels.cuh"  // MVArgs, mv_stencil, mv_correct, mv_ld

namespace ls {

constexpr int MV6_WARPS = 8;
constexpr int MV6_THREADS = 32 * MV6_WARPS;
constexpr unsigned MV6_MAX_DOT_GRID = 1184;  // = RED_BLOCKS (pcg_kernels.cuh): entries of ctx->partials

struct MV6Args {
  MVArgs m;           // stencils: d3 pass 0 M3, 1 J3, 2 K3, 3 2K3; time pass 0 K_t, 1 M_t
  const double* dotp;  // time pass: fused p.q (nullptr: none)
  double* dot_part;
  uint32_t Q;          // d3 pass: n1 n2 (columns per time slice); time pass: N_s
  int rows;            // d3 pass: time slices of the inputs; time pass: see MVArgs s_first / s_rows
  int tT;              // d3 pass: local time slice that also produces L (or -1)
  double* L;           // d3 pass: L output [n3][Q] (the last slice)
};

// direction-3 pass: in[0] = P_M, in[1] = P_K, in[2] = P_J ([rows][n3][Q]); out[0] = S_M, out[1] = S_J
template <int P, int R>
__global__ void __launch_bounds__(MV6_THREADS) mv6_d3_kernel(const __grid_constant__ MV6Args A) {
  pdl_wait();
  const MVArgs& a = A.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = a.n;
  const uint32_t Q = A.Q;
  const uint32_t nqb = (Q + 31) / 32;
  const uint32_t nch = (n + R - 1) / R;
  const uint64_t items = uint64_t(A.rows) * nqb * nch;
  for (uint64_t it = uint64_t(blockIdx.x) * MV6_WARPS + warp; it < items; it += uint64_t(gridDim.x) * MV6_WARPS) {
    const uint32_t ch = uint32_t(it % nch);
    const uint64_t cb = it / nch;
    const uint32_t qb = uint32_t(cb % nqb), pt = uint32_t(cb / nqb);
    const uint32_t q = qb * 32 + lane;
    const bool qv = q < Q;
    const int r0 = int(ch) * R;
    const size_t base = size_t(pt) * n * Q + (qv ? q : 0);
    const bool corr = r0 < a.r_lo || r0 + R > a.r_hi;
    const bool last = int(pt) == A.tT;
    double w[R + 2 * P];
    auto window = [&](const double* src) {
#pragma unroll
      for (int j = 0; j < R + 2 * P; ++j) {
        const int r = r0 - P + j;
        w[j] = (qv && r >= 0 && r < n) ? mv_ld(src + base + size_t(r) * Q) : 0.0;
      }
    };
    auto apply = [&](double (&acc)[R], int m) {
      mv_stencil<P, R>(acc, w, a.st[m]);
      if (corr) mv_correct<P, R>(acc, w, a.E[m], r0, n, a.r_lo, a.r_hi);
    };
    auto put = [&](const double (&acc)[R], double* dst) {
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (qv && r0 + i < n) dst[size_t(r0 + i) * Q] = acc[i];
    };
    double sj[R], sl[R];
#pragma unroll
    for (int i = 0; i < R; ++i) sj[i] = sl[i] = 0.0;
    {  // P_M: S_M = M3 P_M (stored), S_J += J3 P_M, L += K3 P_M
      window(a.in[0]);
      double sm[R];
#pragma unroll
      for (int i = 0; i < R; ++i) sm[i] = 0.0;
      apply(sm, 0);
      put(sm, a.out[0] + base);
      apply(sj, 1);
      if (last) apply(sl, 2);
    }
    window(a.in[1]);  // P_K: S_J += 2 K3 P_K, L += M3 P_K
    apply(sj, 3);
    if (last) {
      apply(sl, 0);
      put(sl, A.L + (qv ? q : 0));
    }
    window(a.in[2]);  // P_J: S_J += M3 P_J
    apply(sj, 0);
    put(sj, a.out[1] + base);
  }
}

// time pass: in[0] = S_M, in[1] = S_J (stored global rows [s_first, s_first + s_rows) of
// [.][Q]); xT = L (one slice, or nullptr if this rank does not own row n_t - 1);
// out[0] = y on the output rows [t_first, t_first + nout)
template <int P, int R>
__global__ void __launch_bounds__(MV6_THREADS) mv6_time_kernel(const __grid_constant__ MV6Args A) {
  pdl_wait();
  const MVArgs& a = A.m;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = a.n;
  const uint32_t Q = A.Q;
  const uint32_t nqb = (Q + 31) / 32;
  const uint32_t nch = (a.nout + R - 1) / R;
  const uint64_t items = uint64_t(nqb) * nch;
  double dacc = 0.0;
  for (uint64_t it = uint64_t(blockIdx.x) * MV6_WARPS + warp; it < items; it += uint64_t(gridDim.x) * MV6_WARPS) {
    const uint32_t ch = uint32_t(it % nch), qb = uint32_t(it / nch);
    const uint32_t q = qb * 32 + lane;
    const bool qv = q < Q;
    const int r0 = int(ch) * R;      // local output row of acc[0]
    const int g0 = a.t_first + r0;   // its global row
    const bool corr = g0 < a.r_lo || g0 + R > a.r_hi;
    double w[R + 2 * P], acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0.0;
#pragma unroll
    for (int m = 0; m < 2; ++m) {  // m = 0: K_t S_M, m = 1: M_t S_J
      const double* src = a.in[m] + (qv ? q : 0);
#pragma unroll
      for (int j = 0; j < R + 2 * P; ++j) {
        const int g = g0 - P + j;
        const bool ok = qv && g >= 0 && g < n && g >= a.s_first && g < a.s_first + a.s_rows;
        w[j] = ok ? mv_ld(src + size_t(g - a.s_first) * Q) : 0.0;
      }
      mv_stencil<P, R>(acc, w, a.st[m]);
      if (corr) mv_correct<P, R>(acc, w, a.E[m], g0, n, a.r_lo, a.r_hi);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int lr = r0 + i;
      if (!qv || lr >= a.nout) continue;
      double v = acc[i];
      if (a.xT && g0 + i == n - 1) v += mv_ld(a.xT + q);  // W_t L on the last global row
      a.out[0][size_t(lr) * Q + q] = v;
      if (A.dotp) dacc = fma(v, A.dotp[size_t(lr) * Q + q], dacc);
    }
  }
  if (A.dotp) {  // CTA sum in a fixed order
    __shared__ double red[MV6_WARPS];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) red[warp] = dacc;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < MV6_WARPS; ++w) t += red[w];
      A.dot_part[blockIdx.x] = t;
    }
  }
}

// host side (mv6.cu): grid = min(items / 8, num_sms * 4) CTAs (<= RED_BLOCKS for the dot)
cudaError_t mv6_run_d3(const MV6Args& a, int p, int num_sms, cudaStream_t s);
cudaError_t mv6_run_time(const MV6Args& a, int pt, int num_sms, cudaStream_t s, unsigned* grid);

}  // namespace ls
