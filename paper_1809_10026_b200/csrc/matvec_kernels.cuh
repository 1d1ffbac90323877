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
//
// One launch per direction (d + 1), each HBM-bound.  Both kernels are
// persistent, cp.async-pipelined tile kernels in the style of fd_mode_kernel:
//   * band_tile_kernel (directions >= 2 and time): a tile = BN = 32 columns of
//     the mode-k unfolding (columns c = (p, q) of the [P][n][Q] view) x all band
//     rows, staged in shared memory with P zero rows above and below (no bounds
//     checks in the stencil); the inputs of a direction stream one after the
//     other through an NSTAGE ring; lane = column (coalesced loads/stores),
//     warp = a block of RB consecutive output rows whose RB + 2P window is read
//     from shared memory once and reused by all RB outputs; the coefficients of
//     the warp's rows are warp-uniform shared-memory broadcasts.
//   * band_first_kernel (direction 1, contiguous axis): the tile is a contiguous
//     chunk [BN][n] staged [BN][n + 2P + 1]; thread = output row a, its 3(2P+1)
//     coefficients in registers, sweeping the tile's columns.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"  // cp.async helpers

namespace ls {

struct BandArgs {
  const double* in[3];   // KIND 1: S_M, S_K, S_J ; first: x ; KIND 2: S_M, S_J, S_K (last row only)
  double* out[3];        // first/KIND 1: M-, K-, J-outputs ; KIND 2: y
  const double* band[3]; // [n][2p+1] row-major: first/KIND 1: M, K, J ; KIND 2: M_t, K_t, -
  int n;                 // extent of the mode (size of the band matrices)
  uint32_t Q;            // product of the faster extents (KIND 2: N_s)
  uint32_t ncols;        // columns of the unfolding
  uint32_t ntiles;
  // time (KIND 2): output rows are global [t_first, t_first + nout); input rows are
  // stored from global s_first, s_rows of them (extended slab incl. halo)
  int t_first, s_first, s_rows, nout;
};

template <int P, int RB, int KIND, int NSTAGE, int NW_ = 8>
struct BandCfg {
  static constexpr int W = 2 * P + 1;
  static constexpr int NWARPS = NW_, THREADS = 32 * NW_, BN = 32;
  static constexpr int ROWS = NWARPS * RB;                   // output rows covered
  static constexpr int NR = ROWS + 2 * P;                    // staged rows: band rows -P .. ROWS+P-1
  static constexpr int NIN = (KIND == 1) ? 3 : 2;            // streamed inputs per tile
  static constexpr int LD = BN + 1;                          // odd stride
  static constexpr int TILE = NR * LD;
  static constexpr int WP = W + 1;                           // padded row (even: LDS.128 pairs)
  static constexpr int NCOEF = 3 * ROWS * WP;                // coefficient table, rows 0..ROWS-1
  static constexpr size_t SMEM = size_t(NCOEF + TILE * NSTAGE) * sizeof(double);
};

// KIND 1 (directions >= 2) and KIND 2 (time).
template <int P, int RB, int KIND, int NSTAGE, int NWARPS>
// two CTAs per SM for RB <= 9 (<= 128 registers: config 3 matvec 0.81 -> 0.75 ms, n_el = 48
// 0.31 -> 0.28 ms); larger row blocks keep one (they would spill)
__global__ void __launch_bounds__(32 * NWARPS, (RB <= 9 ? 2 : 1)) band_tile_kernel(BandArgs a) {
  pdl_wait();
  using C = BandCfg<P, RB, KIND, NSTAGE, NWARPS>;
  constexpr int W = C::W;
  constexpr int NIN = C::NIN;
  extern __shared__ __align__(16) double smem[];
  constexpr int WP = C::WP;
  double* coef = smem;  // [3][ROWS][WP]
  double* tiles = smem + C::NCOEF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrows = (KIND == 2) ? a.nout : a.n;   // output rows
  const int g_off = (KIND == 2) ? a.t_first : 0;  // band row of output row 0
  for (int e = tid; e < C::NCOEF; e += C::THREADS) {
    const int m = e / (C::ROWS * WP), r = (e / WP) % C::ROWS, k = e % WP;
    const int g = g_off + r, i = g - P + k;
    coef[e] = (k < W && r < nrows && i >= 0 && i < a.n && a.band[m] != nullptr)
                  ? __ldg(a.band[m] + size_t(g) * W + k) : 0.0;
  }
  // staged row s <-> band index i = g_off - P + s
  auto row_valid = [&](int s) {
    const int i = g_off - P + s;
    if (KIND == 1) return i >= 0 && i < a.n;
    return i >= 0 && i < a.n && i >= a.s_first && i < a.s_first + a.s_rows;
  };
  for (int st = 0; st < NSTAGE; ++st)  // zero invalid staged rows once (never loaded)
    for (int e = tid; e < C::TILE; e += C::THREADS)
      if (!row_valid(e / C::LD)) tiles[st * C::TILE + e] = 0.0;

  const uint32_t Q = a.Q;
  auto load = [&](uint32_t tile, int which, int stage) {
    double* t = tiles + stage * C::TILE;
    const double* src = a.in[which];
    const int cc = tid & 31;
    const uint32_t c = tile * C::BN + cc;
    if (c >= a.ncols) return;
    size_t base;
    if (KIND == 1) {
      const uint32_t p = c / Q, q = c - p * Q;
      base = size_t(p) * a.n * Q + q;
    } else {
      base = c;
    }
    for (int s = tid >> 5; s < C::NR; s += C::NWARPS) {
      if (!row_valid(s)) continue;
      const int i = g_off - P + s;
      const int ri = (KIND == 1) ? i : i - a.s_first;
      cp_async8(t + s * C::LD + cc, src + base + size_t(ri) * Q);
    }
  };

  const uint32_t stride = gridDim.x;
  const uint32_t my_tiles = (a.ntiles > blockIdx.x) ? (a.ntiles - blockIdx.x + stride - 1) / stride : 0;
  const uint32_t units = my_tiles * NIN;
  auto unit_tile = [&](uint32_t u) { return blockIdx.x + (u / NIN) * stride; };
  __syncthreads();
#pragma unroll 1
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (uint32_t(s) < units) load(unit_tile(s), s % NIN, s);
    cp_async_commit();
  }

  const int r0 = warp * RB;  // first output row of this warp
  const double2* cM = reinterpret_cast<const double2*>(coef + (0 * C::ROWS + r0) * WP);
  const double2* cK = reinterpret_cast<const double2*>(coef + (1 * C::ROWS + r0) * WP);
  const double2* cJ = reinterpret_cast<const double2*>(coef + (2 * C::ROWS + r0) * WP);
  constexpr int HP = WP / 2;  // coefficient pairs per row
  double acc[3][RB];
#pragma unroll 1
  for (uint32_t u = 0; u < units; ++u) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    {
      const uint32_t un = u + NSTAGE - 1;
      if (un < units) load(unit_tile(un), un % NIN, un % NSTAGE);
      cp_async_commit();
    }
    const int which = u % NIN;
    if (which == 0) {
#pragma unroll
      for (int m = 0; m < 3; ++m)
#pragma unroll
        for (int r = 0; r < RB; ++r) acc[m][r] = 0.0;
    }
    const double* t = tiles + (u % NSTAGE) * C::TILE + lane;
    double win[RB + 2 * P];  // staged rows r0 .. r0 + RB + 2P - 1 (band rows r0-P ..)
#pragma unroll
    for (int w = 0; w < RB + 2 * P; ++w) win[w] = t[(r0 + w) * C::LD];
    if (KIND == 1) {
      if (which == 0) {         // S_M -> M, K, J
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int h = 0; h < HP; ++h) {
            const double2 m2 = cM[r * HP + h], k2 = cK[r * HP + h], j2 = cJ[r * HP + h];
            const double v0 = win[r + 2 * h], v1 = (2 * h + 1 < W) ? win[r + 2 * h + 1] : 0.0;
            acc[0][r] = fma(m2.x, v0, acc[0][r]);
            acc[1][r] = fma(k2.x, v0, acc[1][r]);
            acc[2][r] = fma(j2.x, v0, acc[2][r]);
            if (2 * h + 1 < W) {
              acc[0][r] = fma(m2.y, v1, acc[0][r]);
              acc[1][r] = fma(k2.y, v1, acc[1][r]);
              acc[2][r] = fma(j2.y, v1, acc[2][r]);
            }
          }
      } else if (which == 1) {  // S_K -> M into K, 2K into J
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int h = 0; h < HP; ++h) {
            const double2 m2 = cM[r * HP + h], k2 = cK[r * HP + h];
            const double v0 = win[r + 2 * h], v1 = (2 * h + 1 < W) ? win[r + 2 * h + 1] : 0.0;
            acc[1][r] = fma(m2.x, v0, acc[1][r]);
            acc[2][r] = fma(k2.x, 2.0 * v0, acc[2][r]);
            if (2 * h + 1 < W) {
              acc[1][r] = fma(m2.y, v1, acc[1][r]);
              acc[2][r] = fma(k2.y, 2.0 * v1, acc[2][r]);
            }
          }
      } else {                  // S_J -> M into J
#pragma unroll
        for (int r = 0; r < RB; ++r)
#pragma unroll
          for (int h = 0; h < HP; ++h) {
            const double2 m2 = cM[r * HP + h];
            acc[2][r] = fma(m2.x, win[r + 2 * h], acc[2][r]);
            if (2 * h + 1 < W) acc[2][r] = fma(m2.y, win[r + 2 * h + 1], acc[2][r]);
          }
      }
    } else {
      // time: band[0] = M_t, band[1] = K_t; input 0 = S_M (K_t), input 1 = S_J (M_t)
      const double2* cc = (which == 0) ? cK : cM;
#pragma unroll
      for (int r = 0; r < RB; ++r)
#pragma unroll
        for (int h = 0; h < HP; ++h) {
          const double2 c2 = cc[r * HP + h];
          acc[0][r] = fma(c2.x, win[r + 2 * h], acc[0][r]);
          if (2 * h + 1 < W) acc[0][r] = fma(c2.y, win[r + 2 * h + 1], acc[0][r]);
        }
    }
    if (which == NIN - 1) {  // epilogue: this warp's RB rows of column `lane`
      const uint32_t c = unit_tile(u) * C::BN + lane;
      if (c < a.ncols) {
        if (KIND == 1) {
          const uint32_t p = c / Q, q = c - p * Q;
          const size_t base = size_t(p) * a.n * Q + q;
#pragma unroll
          for (int r = 0; r < RB; ++r)
            if (r0 + r < a.n) {
              const size_t o = base + size_t(r0 + r) * Q;
              a.out[0][o] = acc[0][r];
              a.out[1][o] = acc[1][r];
              a.out[2][o] = acc[2][r];
            }
        } else {
#pragma unroll
          for (int r = 0; r < RB; ++r)
            if (r0 + r < a.nout) {
              const int tg = a.t_first + r0 + r;
              double v = acc[0][r];
              if (tg == a.n - 1) v += __ldg(a.in[2] + size_t(tg - a.s_first) * Q + c);  // W_t S_K
              a.out[0][size_t(r0 + r) * Q + c] = v;
            }
        }
      }
    }
  }
  cp_async_wait<0>();
}

template <int P, int NMAX, int NSTAGE>
struct FirstCfg {
  static constexpr int BN = 32;
  static constexpr int LD = NMAX + 2 * P + 1;  // per-column stride (odd when NMAX even)
  static constexpr int TILE = BN * LD;
  static constexpr size_t SMEM = size_t(TILE) * NSTAGE * sizeof(double);
};

// Direction 1 (contiguous axis): x viewed as [ncols][n].
template <int P, int NMAX, int NSTAGE>
__global__ void __launch_bounds__(256, 2) band_first_kernel(BandArgs a) {
  pdl_wait();
  using C = FirstCfg<P, NMAX, NSTAGE>;
  constexpr int W = 2 * P + 1;
  constexpr int BN = C::BN, LD = C::LD, TILE = C::TILE;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int n = a.n;
  const int groups = 256 / n;  // column groups (>= 1 for n <= 256)
  const int row = tid % n, g = tid / n;
  const bool active = g < groups;
  double cm[W], ck[W], cj[W];
#pragma unroll
  for (int k = 0; k < W; ++k) {
    const int i = row - P + k;
    const bool in = active && i >= 0 && i < n;
    cm[k] = in ? __ldg(a.band[0] + size_t(row) * W + k) : 0.0;
    ck[k] = in ? __ldg(a.band[1] + size_t(row) * W + k) : 0.0;
    cj[k] = in ? __ldg(a.band[2] + size_t(row) * W + k) : 0.0;
  }
  for (int st = 0; st < NSTAGE; ++st)  // zero the P-entry borders of every column once
    for (int e = tid; e < BN * 2 * P; e += 256) {
      const int c = e / (2 * P), s = e % (2 * P);
      smem[st * TILE + c * LD + (s < P ? s : n + s)] = 0.0;
    }
  auto load = [&](uint32_t tile, int stage) {
    double* t = smem + stage * TILE;
    const uint32_t c0 = tile * BN;
    const uint32_t cend = min(c0 + (uint32_t)BN, a.ncols);
    const uint32_t total = (cend - c0) * (uint32_t)n;
    const double* src = a.in[0] + size_t(c0) * n;
    uint32_t c = tid / n, i = tid % n;
    const uint32_t dq = 256 / n, dr = 256 % n;
    for (uint32_t e = tid; e < total; e += 256) {
      cp_async8(t + c * LD + P + i, src + e);
      c += dq;
      i += dr;
      if (i >= (uint32_t)n) { i -= n; ++c; }
    }
  };
  const uint32_t stride = gridDim.x;
  uint32_t tile = blockIdx.x;
  __syncthreads();
#pragma unroll 1
  for (int s = 0; s < NSTAGE - 1; ++s) {
    if (tile + s * stride < a.ntiles) load(tile + s * stride, s);
    cp_async_commit();
  }
#pragma unroll 1
  for (int j = 0; tile < a.ntiles; ++j, tile += stride) {
    cp_async_wait<NSTAGE - 2>();
    __syncthreads();
    {
      const uint32_t tn = tile + (NSTAGE - 1) * stride;
      if (tn < a.ntiles) load(tn, (j + NSTAGE - 1) % NSTAGE);
      cp_async_commit();
    }
    if (!active) continue;
    const double* t = smem + (j % NSTAGE) * TILE;
    const uint32_t c0 = tile * BN;
#pragma unroll 2
    for (int c = g; c < BN; c += groups) {
      if (c0 + c >= a.ncols) break;
      const double* col = t + c * LD + row;  // col[k] = staged entry of band index row - P + k
      double m = 0, kk = 0, jj = 0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        const double v = col[k];
        m = fma(cm[k], v, m);
        kk = fma(ck[k], v, kk);
        jj = fma(cj[k], v, jj);
      }
      const size_t o = size_t(c0 + c) * n + row;
      a.out[0][o] = m;
      a.out[1][o] = kk;
      a.out[2][o] = jj;
    }
  }
  cp_async_wait<0>();
}

} // namespace ls
