// Matrix-free y = A x on the identity map (eq:A_kron, PAPER.md 686-703), v2:
// three fused banded passes, 96 B/DOF of HBM traffic (v1, matvec_kernels.cuh:
// four passes, 152 B/DOF).
//
// Algebra.  With M_s = (x)_k M_k, L_s = sum_k K_(k) and
// J_s = sum_k J_(k) + sum_{k != l} K_(k) K_(l) (integration by parts on the
// Dirichlet basis), expand A direction by direction starting from
// time with a triple (A, B, C):
//     A0 = K_t x,   B0 = M_t x,   C0 = W_t x        (W_t = e_{n_t} e_{n_t}^T)
//     direction k:  A <- M_k A + J_k B + K_k C
//                   B <- M_k B
//                   C <- 2 K_k B + M_k C
// and after the last direction y = A.  (Induction: after directions d..k the
// triple holds the time/space terms whose remaining factors are M, J and K
// respectively; every ordered pair k != l of the K K cross terms appears once in
// each order, hence the 2.)  Passes:
//   mv_time_kernel  (time):          x -> Kx = K_t x, Mx = M_t x            8 + 16 B/DOF
//   mv_dir_kernel   (direction d):   Kx, Mx (+ x at t = n_t - 1) -> A, B, C  16 + 24 B/DOF
//   mv_plane_kernel (directions d-1 .. 1, i.e. 2 and 1 fused per plane for
//                    d = 3, 1 for d = 2):  A, B, C -> y                      24 + 8 B/DOF
// (d = 1: mv_dir_kernel in A-only mode writes y.)
//
// Banded products.  The univariate matrices of uniform open knots are Toeplitz
// away from the boundary (translation invariance of the interior B-splines).
// Each band matrix B (half-bandwidth P) is split as B = T + E: T applies ONE
// stencil s[0..2P] on every row (inputs outside [0, n) are zero), and E holds the
// per-row corrections of the boundary rows [0, r_lo) and [r_hi, n) (interior
// rows agree with s to rounding, reading c18).  The stencils are
// kernel parameters (__grid_constant__): the DFMAs take them as constant-bank
// operands, so the hot loops issue only data loads and DFMAs.
// Thread mapping: lane = column of the banded direction (coalesced rows), each
// thread sweeps its column in chunks of R rows with a window of R + 2P values;
// the boundary chunks add the E rows (warp-uniform broadcast loads).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pdl.cuh"

namespace ls {

constexpr int MV_MAXW = 17;  // 2P + 1 for P <= 8
constexpr int MV_NST = 7;    // stencils per pass (plane pass: M2 J2 K2 2K2 M1 J1 K1)

struct MVArgs {
  double st[MV_NST][MV_MAXW];  // Toeplitz stencils (constant-bank operands)
  const double* E[MV_NST];     // boundary corrections [nb][2P+1]: rows [0, r_lo) then [r_hi, n)
  int r_lo, r_hi;              // interior zone of the pass direction (plane: direction 2)
  int r_lo1, r_hi1;            // plane pass: interior zone of direction 1
  const double* in[3];
  double* out[3];
  const double* xT;   // mv_dir: x rows of the last time slice [n][Q] (nullptr if not owned)
  int n;              // extent of the banded direction (time: n_t; dir: n_d; plane: n_2)
  int n1;             // plane pass: extent of direction 1
  uint32_t Q;         // dir pass: product of the faster extents
  uint32_t ncols;     // dir / time: columns; plane: number of planes (or rows when d = 2)
  int t_first, s_first, s_rows, nout;  // time pass: global output rows / stored input rows
  int tT;             // dir pass: local time index of global t = n_t - 1 (or -1)
};

__device__ __forceinline__ double mv_ld(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// acc[i] += sum_j s[j] w[i + j] (Toeplitz part; s is a compile-time-indexed parameter)
template <int P, int R>
__device__ __forceinline__ void mv_stencil(double (&acc)[R], const double (&w)[R + 2 * P], const double* s) {
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < 2 * P + 1; ++j) acc[i] = fma(s[j], w[i + j], acc[i]);
}

// boundary corrections for rows r0 .. r0+R-1 of a band direction with zone [lo, hi)
template <int P, int R>
__device__ __forceinline__ void mv_correct(double (&acc)[R], const double (&w)[R + 2 * P], const double* E,
                                           int r0, int n, int lo, int hi) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int r = r0 + i;
    if (r < n && (r < lo || r >= hi)) {
      const double* e = E + (r < lo ? r : lo + (r - hi)) * (2 * P + 1);
#pragma unroll
      for (int j = 0; j < 2 * P + 1; ++j) acc[i] = fma(__ldg(e + j), w[i + j], acc[i]);
    }
  }
}

// --------------------------------------------------------------------------------------
// time pass: Kx = K_t x, Mx = M_t x on every spatial column (Q = N_s columns)
// --------------------------------------------------------------------------------------
// block (32, MV_CY): x = column, y = chunk of R output rows; one chunk per thread, the
// halo rows of neighbouring chunks hit L1
constexpr int MV_CY = 8;

template <int P, int R>
__global__ void __launch_bounds__(32 * MV_CY) mv_time_kernel(const __grid_constant__ MVArgs a) {
  pdl_wait();
  const uint32_t c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = (blockIdx.y * MV_CY + threadIdx.y) * R;  // local output row of acc[0]
  if (c >= a.ncols || r0 >= a.nout) return;
  const size_t Q = a.ncols;
  const int n = a.n;
  const double* x = a.in[0];
  const int g0 = a.t_first + r0;  // global output row of acc[0]
  double w[R + 2 * P];
#pragma unroll
  for (int j = 0; j < R + 2 * P; ++j) {
    const int g = g0 - P + j;
    const bool ok = g >= 0 && g < n && g >= a.s_first && g < a.s_first + a.s_rows;
    w[j] = ok ? mv_ld(x + size_t(g - a.s_first) * Q + c) : 0.0;
  }
  const bool corr = g0 < a.r_lo || g0 + R > a.r_hi;
#pragma unroll
  for (int m = 0; m < 2; ++m) {  // m = 0: Kx (stencil 0), m = 1: Mx (stencil 1)
    double acc[R];
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0.0;
    mv_stencil<P, R>(acc, w, a.st[m]);
    if (corr) mv_correct<P, R>(acc, w, a.E[m], g0, n, a.r_lo, a.r_hi);
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (r0 + i < a.nout) a.out[m][size_t(r0 + i) * Q + c] = acc[i];
  }
}

// --------------------------------------------------------------------------------------
// direction-d pass on [P_t][n][Q] (P_t = local time slices): stencils 0 M, 1 J, 2 K, 3 2K
//   A = M Kx + J Mx (+ K xT),  B = M Mx,  C = 2K Mx (+ M xT)     (xT only at t = tT)
// AONLY (d = 1): only A, written to out[0] (= y).
// --------------------------------------------------------------------------------------
template <int P, int R, bool AONLY>
__global__ void __launch_bounds__(32 * MV_CY) mv_dir_kernel(const __grid_constant__ MVArgs a) {
  pdl_wait();
  const uint32_t c = blockIdx.x * 32 + threadIdx.x;
  const int r0 = (blockIdx.y * MV_CY + threadIdx.y) * R;
  const int n = a.n;
  if (c >= a.ncols || r0 >= n) return;
  const uint32_t Q = a.Q;
  const uint32_t pt = c / Q, q = c - pt * Q;
  const size_t base = size_t(pt) * n * Q + q;
  const bool last = int(pt) == a.tT;
  const bool corr = r0 < a.r_lo || r0 + R > a.r_hi;
  double acc[R], w[R + 2 * P];
  auto window = [&](const double* src) {
#pragma unroll
    for (int j = 0; j < R + 2 * P; ++j) {
      const int r = r0 - P + j;
      w[j] = (r >= 0 && r < n) ? mv_ld(src + size_t(r) * Q) : 0.0;
    }
  };
  auto zero = [&]() {
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] = 0.0;
  };
  auto apply = [&](int m) {
    mv_stencil<P, R>(acc, w, a.st[m]);
    if (corr) mv_correct<P, R>(acc, w, a.E[m], r0, n, a.r_lo, a.r_hi);
  };
  auto put = [&](int o) {
#pragma unroll
    for (int i = 0; i < R; ++i)
      if (r0 + i < n) a.out[o][base + size_t(r0 + i) * Q] = acc[i];
  };
  // A = M Kx + J Mx (+ K xT)
  zero();
  window(a.in[0] + base);
  apply(0);
  window(a.in[1] + base);
  apply(1);
  if (last) {
    window(a.xT + q);
    apply(2);
  }
  put(0);
  if (AONLY) return;
  // C = (M xT) + 2K Mx
  zero();
  if (last) apply(0);  // w holds the xT window
  window(a.in[1] + base);
  apply(3);
  put(2);
  // B = M Mx (w holds the Mx window)
  zero();
  apply(0);
  put(1);
}

// --------------------------------------------------------------------------------------
// plane pass.  PHASE1 (d = 3): a work item = up to 32 consecutive rows i2 of one
// (t, i3) plane [n2][n1]; phase 1 applies direction 2 (stencils 0 M2, 1 J2, 2 K2,
// 3 2K2) from global memory into shared rows
//     A2 = M2 A + J2 B + K2 C,  B2 = M2 B,  C2 = 2K2 B + M2 C,
// phase 2 applies direction 1 (stencils 4 M1, 5 J1, 6 K1) along the shared rows
//     y = M1 A2 + J1 B2 + K1 C2
// with lane = row and warp = segment of direction-1 outputs (warp-uniform output
// positions, so boundary corrections are broadcasts), and the outputs are staged
// back through shared memory for coalesced stores.  !PHASE1 (d = 2): the work item
// is 32 consecutive rows of [rows][n1], phase 1 only copies A, B, C into shared.
// --------------------------------------------------------------------------------------
// geometry (tools/mv2_ab.sh, config 5 p = 2): 8-row work items, 3 warps, 8 CTAs per SM
// (80 registers; spills grow with P, so P > 3 keeps 4 CTAs)
#ifndef MV_PLANE_WARPS
#define MV_PLANE_WARPS 3
#endif
#ifndef MV_PLANE_CTAS
#define MV_PLANE_CTAS 8
#endif
#ifndef MV_PLANE_CTAS_HI
#define MV_PLANE_CTAS_HI 4
#endif
#ifndef MV_PLANE_ROWS_
#define MV_PLANE_ROWS_ 8
#endif
constexpr int MV_PLANE_THREADS = 32 * MV_PLANE_WARPS;
constexpr int MV_PLANE_ROWS = MV_PLANE_ROWS_;  // rows per work item
__host__ __device__ constexpr int mv_plane_ctas(int P) { return P <= 3 ? MV_PLANE_CTAS : MV_PLANE_CTAS_HI; }

__host__ __device__ inline int mv_plane_pitch(int n1, int P) {
  const int w = n1 + 2 * P;
  return (w & 1) ? w : w + 1;  // odd pitch: lane = row reads are conflict-free
}

template <int P, int R, bool PHASE1>
__global__ void __launch_bounds__(MV_PLANE_THREADS, mv_plane_ctas(P)) mv_plane_kernel(const __grid_constant__ MVArgs a) {
  pdl_wait();
  extern __shared__ __align__(16) double sm[];
  const int n1 = a.n1, n2 = a.n;
  const int pitch = mv_plane_pitch(n1, P);
  const int slab = MV_PLANE_ROWS * pitch;
  double* S0 = sm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // zero the P-column borders once (never written afterwards)
  for (int e = tid; e < 3 * MV_PLANE_ROWS * 2 * P; e += MV_PLANE_THREADS) {
    const int m = e / (MV_PLANE_ROWS * 2 * P), rem = e % (MV_PLANE_ROWS * 2 * P);
    const int r = rem / (2 * P), j = rem % (2 * P);
    S0[m * slab + r * pitch + (j < P ? j : P + n1 + (j - P))] = 0.0;
  }
  const int bpp = PHASE1 ? (n2 + MV_PLANE_ROWS - 1) / MV_PLANE_ROWS : 1;  // blocks per plane
  const uint32_t nitems = PHASE1 ? a.ncols * uint32_t(bpp) : (a.ncols + MV_PLANE_ROWS - 1) / MV_PLANE_ROWS;
  // phase 2: thread = (row, segment of R direction-1 outputs)
  static_assert(32 % MV_PLANE_ROWS == 0, "a warp covers whole row groups");
  constexpr int SEGW = 32 / MV_PLANE_ROWS;  // segments per warp and phase-2 step
  const int prow = lane % MV_PLANE_ROWS;
  const int nseg = (n1 + R - 1) / R;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    size_t row0;  // global row (of the [rows][n1] view) of local row 0
    int nr, i2_0 = 0;
    uint32_t plane = 0;
    if (PHASE1) {
      plane = it / bpp;
      const int b = it - plane * bpp;
      i2_0 = (b * n2) / bpp;
      nr = ((b + 1) * n2) / bpp - i2_0;  // balanced blocks (<= 16 rows)
      row0 = size_t(plane) * n2 + i2_0;
    } else {
      row0 = size_t(it) * MV_PLANE_ROWS;
      nr = int(min(size_t(MV_PLANE_ROWS), size_t(a.ncols) - row0));
    }
    __syncthreads();  // previous item's shared rows fully consumed
    if (PHASE1) {
      // ---- phase 1: direction 2, thread = (column i1, chunk of R rows)
      const int nch = (nr + R - 1) / R;
      for (int job = tid; job < nch * n1; job += MV_PLANE_THREADS) {
        const int i1 = job % n1, lr = (job / n1) * R;
        const size_t cbase = size_t(plane) * n2 * n1 + i1;
        const int r0 = i2_0 + lr;  // row of the direction-2 band
        const bool corr = r0 < a.r_lo || r0 + R > a.r_hi;
        double acc[R], w[R + 2 * P];
        auto window = [&](const double* src) {
#pragma unroll
          for (int j = 0; j < R + 2 * P; ++j) {
            const int r = r0 - P + j;
            w[j] = (r >= 0 && r < n2) ? mv_ld(src + cbase + size_t(r) * n1) : 0.0;
          }
        };
        auto zero = [&]() {
#pragma unroll
          for (int i = 0; i < R; ++i) acc[i] = 0.0;
        };
        auto apply = [&](int m) {
          mv_stencil<P, R>(acc, w, a.st[m]);
          if (corr) mv_correct<P, R>(acc, w, a.E[m], r0, n2, a.r_lo, a.r_hi);
        };
        auto put = [&](int m) {
#pragma unroll
          for (int i = 0; i < R; ++i)
            if (lr + i < nr) S0[m * slab + (lr + i) * pitch + P + i1] = acc[i];
        };
        // A2 = M2 A + J2 B + K2 C
        zero();
        window(a.in[0]);
        apply(0);
        window(a.in[1]);
        apply(1);
        window(a.in[2]);
        apply(2);
        put(0);
        // C2 = M2 C + 2K2 B  (w holds the C window)
        zero();
        apply(0);
        window(a.in[1]);
        apply(3);
        put(2);
        // B2 = M2 B  (w holds the B window)
        zero();
        apply(0);
        put(1);
      }
    } else {
      for (int e = tid; e < nr * n1; e += MV_PLANE_THREADS) {
        const int r = e / n1, i1 = e - r * n1;
        const size_t g = (row0 + r) * n1 + i1;
        const int o = r * pitch + P + i1;
        S0[o] = mv_ld(a.in[0] + g);
        S0[slab + o] = mv_ld(a.in[1] + g);
        S0[2 * slab + o] = mv_ld(a.in[2] + g);
      }
    }
    __syncthreads();
    // ---- phase 2: direction 1 along the shared rows; thread = (row, segment); outputs go
    //      straight to global memory (a thread's R outputs are contiguous)
    for (int seg = warp * SEGW + lane / MV_PLANE_ROWS; seg < nseg; seg += SEGW * (MV_PLANE_THREADS / 32)) {
      if (prow >= nr) continue;
      const int c0 = seg * R;
      const bool corr = c0 < a.r_lo1 || c0 + R > a.r_hi1;
      double acc[R], w[R + 2 * P];
#pragma unroll
      for (int i = 0; i < R; ++i) acc[i] = 0.0;
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const double* row = S0 + m * slab + prow * pitch + c0;  // staged column c0 - P
#pragma unroll
        for (int j = 0; j < R + 2 * P; ++j) w[j] = (c0 - P + j < n1 + P) ? row[j] : 0.0;
        mv_stencil<P, R>(acc, w, a.st[4 + m]);
        if (corr) mv_correct<P, R>(acc, w, a.E[4 + m], c0, n1, a.r_lo1, a.r_hi1);
      }
      double* yrow = a.out[0] + (row0 + prow) * n1;
#pragma unroll
      for (int i = 0; i < R; ++i)
        if (c0 + i < n1) yrow[c0 + i] = acc[i];
    }
  }
}

// --------------------------------------------------------------------------------------
// sweep variant of the d = 3 plane pass (r02, LS_TUNE_MV2_SWEEP): the same algebra as
// mv_plane_kernel (A2 = M2 A + J2 B + K2 C, B2 = M2 B, C2 = 2K2 B + M2 C along direction 2,
// then y = M1 A2 + J1 B2 + K1 C2 along direction 1, stencils + boundary corrections), but
// without shared memory or barriers: one warp owns a whole (t, i3) plane, lane l holds the CW
// direction-1 columns CW l .. CW l + CW - 1 (32 CW >= n1), and the warp sweeps direction 2
// row by row with a register ring of the 2P + 1 + D input rows of A, B, C (rows are loaded D
// steps ahead).  Direction 1's P neighbours of a lane's columns come from the adjacent lanes
// (shuffles).  Each input is read once, y written once: 32 B/DOF, streamed.
// Why (ncu of mv_plane_kernel, config 5 p = 2): 2.6 TB/s, barrier and long-scoreboard stalls —
// its two phases do not overlap inside a CTA.
// --------------------------------------------------------------------------------------
#ifndef LS_MV2_SWEEP_SPLIT
#define LS_MV2_SWEEP_SPLIT 0
#endif
template <int P, int CW, int D>
__global__ void __launch_bounds__(256, 1) mv_sweep_kernel(const __grid_constant__ MVArgs a) {
  static_assert(CW >= P, "direction-1 neighbours come from the adjacent lanes only");
  constexpr int W = 2 * P + 1, R = W + D;  // stencil width, ring rows
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n1 = a.n1, n2 = a.n;
  const int c0 = lane * CW;  // the lane's first column
  const uint32_t planes = a.ncols;
  for (uint32_t pl = blockIdx.x * 8u + warp; pl < planes; pl += gridDim.x * 8u) {
    const size_t base = size_t(pl) * n2 * n1 + c0;
    double w[3][R][CW];  // ring slot (r + P) % R holds input row r
    auto load = [&](int slot, int row) {
      const bool rv = row >= 0 && row < n2;
#pragma unroll
      for (int f = 0; f < 3; ++f)
#pragma unroll
        for (int m = 0; m < CW; ++m)
          w[f][slot][m] = (rv && c0 + m < n1) ? mv_ld(a.in[f] + base + size_t(row) * n1 + m) : 0.0;
    };
#pragma unroll
    for (int j = 0; j < R - 1; ++j) load(j, j - P);
#pragma unroll 1
    for (int i2b = 0; i2b < n2; i2b += R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int i2 = i2b + u;
        if (i2 >= n2) break;
        load((u + R - 1) % R, i2 + P + D);  // D rows ahead: the slot of row i2 - P - 1
        // ---- direction 2 at row i2 (ring slots (u + j) % R hold rows i2 - P + j)
        double A2[CW], B2[CW], C2[CW];
#pragma unroll
        for (int m = 0; m < CW; ++m) A2[m] = B2[m] = C2[m] = 0.0;
#if LS_MV2_SWEEP_SPLIT
        // one accumulator chain per input field (W links each instead of 3W / 2W), summed at the end
        double A2b[CW], A2c[CW], C2b[CW];
#pragma unroll
        for (int m = 0; m < CW; ++m) A2b[m] = A2c[m] = C2b[m] = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int sl = (u + j) % R;
#pragma unroll
          for (int m = 0; m < CW; ++m) {
            A2[m] = fma(a.st[0][j], w[0][sl][m], A2[m]);
            A2b[m] = fma(a.st[1][j], w[1][sl][m], A2b[m]);
            A2c[m] = fma(a.st[2][j], w[2][sl][m], A2c[m]);
            B2[m] = fma(a.st[0][j], w[1][sl][m], B2[m]);
            C2[m] = fma(a.st[0][j], w[2][sl][m], C2[m]);
            C2b[m] = fma(a.st[3][j], w[1][sl][m], C2b[m]);
          }
        }
#pragma unroll
        for (int m = 0; m < CW; ++m) {
          A2[m] = (A2[m] + A2b[m]) + A2c[m];
          C2[m] += C2b[m];
        }
#else
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int sl = (u + j) % R;
#pragma unroll
          for (int m = 0; m < CW; ++m) {
            A2[m] = fma(a.st[0][j], w[0][sl][m], fma(a.st[1][j], w[1][sl][m], fma(a.st[2][j], w[2][sl][m], A2[m])));
            B2[m] = fma(a.st[0][j], w[1][sl][m], B2[m]);
            C2[m] = fma(a.st[3][j], w[1][sl][m], fma(a.st[0][j], w[2][sl][m], C2[m]));
          }
        }
#endif
        if (i2 < a.r_lo || i2 >= a.r_hi) {  // boundary row of direction 2 (warp-uniform)
          const int er = (i2 < a.r_lo ? i2 : a.r_lo + (i2 - a.r_hi)) * W;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            const int sl = (u + j) % R;
            const double eM = __ldg(a.E[0] + er + j), eJ = __ldg(a.E[1] + er + j), eK = __ldg(a.E[2] + er + j),
                         e2K = __ldg(a.E[3] + er + j);
#pragma unroll
            for (int m = 0; m < CW; ++m) {
              A2[m] = fma(eM, w[0][sl][m], fma(eJ, w[1][sl][m], fma(eK, w[2][sl][m], A2[m])));
              B2[m] = fma(eM, w[1][sl][m], B2[m]);
              C2[m] = fma(e2K, w[1][sl][m], fma(eM, w[2][sl][m], C2[m]));
            }
          }
        }
        // ---- direction 1: columns c0 - P .. c0 + CW - 1 + P (neighbours from lanes l -+ 1;
        //      columns outside [0, n1) are zero: invalid columns hold 0 from the zero inputs)
        double x[3][CW + 2 * P];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          const double* v = f == 0 ? A2 : (f == 1 ? B2 : C2);
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const double lft = __shfl_up_sync(0xffffffffu, v[CW - P + k], 1);
            const double rgt = __shfl_down_sync(0xffffffffu, v[k], 1);
            x[f][k] = lane == 0 ? 0.0 : lft;
            x[f][P + CW + k] = lane == 31 ? 0.0 : rgt;
          }
#pragma unroll
          for (int m = 0; m < CW; ++m) x[f][P + m] = v[m];
        }
        double* yrow = a.out[0] + base + size_t(i2) * n1;
#pragma unroll
        for (int m = 0; m < CW; ++m) {
          const int c = c0 + m;
          double y = 0.0;
#if LS_MV2_SWEEP_SPLIT
          double yb = 0.0, yc = 0.0;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            y = fma(a.st[4][j], x[0][m + j], y);
            yb = fma(a.st[5][j], x[1][m + j], yb);
            yc = fma(a.st[6][j], x[2][m + j], yc);
          }
          y = (y + yb) + yc;
#else
#pragma unroll
          for (int j = 0; j < W; ++j)
            y = fma(a.st[4][j], x[0][m + j], fma(a.st[5][j], x[1][m + j], fma(a.st[6][j], x[2][m + j], y)));
#endif
          if (c < n1 && (c < a.r_lo1 || c >= a.r_hi1)) {  // boundary column of direction 1
            const int er = (c < a.r_lo1 ? c : a.r_lo1 + (c - a.r_hi1)) * W;
#pragma unroll
            for (int j = 0; j < W; ++j)
              y = fma(__ldg(a.E[4] + er + j), x[0][m + j],
                      fma(__ldg(a.E[5] + er + j), x[1][m + j], fma(__ldg(a.E[6] + er + j), x[2][m + j], y)));
          }
          if (c < n1) yrow[m] = y;
        }
      }
    }
  }
}

// --------------------------------------------------------------------------------------
// the v4 plane pass (mv4_kernels.cuh: P_M = M2 M1 x, P_K = (K2 M1 + M2 K1) x,
// P_J = (J2 M1 + M2 J1 + 2 K2 K1) x) as the same register sweep (r02, LS_TUNE_MV4_SWEEP; p <= 4):
// direction 2 first on the single input x (ring of the 2P + 1 + D rows of x),
//     v_M = M2 x, v_K = K2 x, v_J = J2 x,
// then direction 1 across the lanes,
//     P_M = M1 v_M,  P_K = M1 v_K + K1 v_M,  P_J = M1 v_J + J1 v_M + 2 K1 v_K
// (the Kronecker factors of different directions commute).  Exactly 2P + 1 DFMAs per banded
// output (9 products: 81 DFMA / DOF at p = 4) instead of the DMMA band tiles' parallelogram
// (8-row tiles over 8 + 2P columns: 56 % useful at p = 4); x read once, P_* written once.
// Stencil slots: 0 M2, 1 J2, 2 K2, 4 M1, 5 J1, 6 K1 (+ boundary corrections E[.]).
// --------------------------------------------------------------------------------------
template <int P, int CW, int D>
__global__ void __launch_bounds__(256, 1) mv4_sweep_kernel(const __grid_constant__ MVArgs a) {
  static_assert(CW >= P, "direction-1 neighbours come from the adjacent lanes only");
  constexpr int W = 2 * P + 1, R = W + D;
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n1 = a.n1, n2 = a.n;
  const int c0 = lane * CW;
  const uint32_t planes = a.ncols;
  for (uint32_t pl = blockIdx.x * 8u + warp; pl < planes; pl += gridDim.x * 8u) {
    const size_t base = size_t(pl) * n2 * n1 + c0;
    double w[R][CW];  // ring slot (r + P) % R holds row r of x
    auto load = [&](int slot, int row) {
      const bool rv = row >= 0 && row < n2;
#pragma unroll
      for (int m = 0; m < CW; ++m) w[slot][m] = (rv && c0 + m < n1) ? mv_ld(a.in[0] + base + size_t(row) * n1 + m) : 0.0;
    };
#pragma unroll
    for (int j = 0; j < R - 1; ++j) load(j, j - P);
#pragma unroll 1
    for (int i2b = 0; i2b < n2; i2b += R) {
#pragma unroll
      for (int u = 0; u < R; ++u) {
        const int i2 = i2b + u;
        if (i2 >= n2) break;
        load((u + R - 1) % R, i2 + P + D);
        // ---- direction 2 at row i2: v_M, v_J, v_K
        double v[3][CW];  // 0 M, 1 J, 2 K
#pragma unroll
        for (int m = 0; m < CW; ++m) v[0][m] = v[1][m] = v[2][m] = 0.0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const int sl = (u + j) % R;
#pragma unroll
          for (int m = 0; m < CW; ++m) {
            v[0][m] = fma(a.st[0][j], w[sl][m], v[0][m]);
            v[1][m] = fma(a.st[1][j], w[sl][m], v[1][m]);
            v[2][m] = fma(a.st[2][j], w[sl][m], v[2][m]);
          }
        }
        if (i2 < a.r_lo || i2 >= a.r_hi) {  // boundary row of direction 2 (warp-uniform)
          const int er = (i2 < a.r_lo ? i2 : a.r_lo + (i2 - a.r_hi)) * W;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            const int sl = (u + j) % R;
            const double eM = __ldg(a.E[0] + er + j), eJ = __ldg(a.E[1] + er + j), eK = __ldg(a.E[2] + er + j);
#pragma unroll
            for (int m = 0; m < CW; ++m) {
              v[0][m] = fma(eM, w[sl][m], v[0][m]);
              v[1][m] = fma(eJ, w[sl][m], v[1][m]);
              v[2][m] = fma(eK, w[sl][m], v[2][m]);
            }
          }
        }
        // ---- direction 1: columns c0 - P .. c0 + CW - 1 + P of v_M, v_J, v_K
        double x[3][CW + 2 * P];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
#pragma unroll
          for (int k = 0; k < P; ++k) {
            const double lft = __shfl_up_sync(0xffffffffu, v[f][CW - P + k], 1);
            const double rgt = __shfl_down_sync(0xffffffffu, v[f][k], 1);
            x[f][k] = lane == 0 ? 0.0 : lft;
            x[f][P + CW + k] = lane == 31 ? 0.0 : rgt;
          }
#pragma unroll
          for (int m = 0; m < CW; ++m) x[f][P + m] = v[f][m];
        }
        const size_t ro = base + size_t(i2) * n1;
#pragma unroll
        for (int m = 0; m < CW; ++m) {
          const int c = c0 + m;
          double pm = 0.0, pk = 0.0, pj = 0.0;
#pragma unroll
          for (int j = 0; j < W; ++j) {
            const double xm = x[0][m + j], xj = x[1][m + j], xk = x[2][m + j];
            pm = fma(a.st[4][j], xm, pm);
            pk = fma(a.st[4][j], xk, fma(a.st[6][j], xm, pk));
            pj = fma(a.st[4][j], xj, fma(a.st[5][j], xm, fma(2.0 * a.st[6][j], xk, pj)));
          }
          if (c < n1 && (c < a.r_lo1 || c >= a.r_hi1)) {  // boundary column of direction 1
            const int er = (c < a.r_lo1 ? c : a.r_lo1 + (c - a.r_hi1)) * W;
#pragma unroll
            for (int j = 0; j < W; ++j) {
              const double eM = __ldg(a.E[4] + er + j), eJ = __ldg(a.E[5] + er + j), eK = __ldg(a.E[6] + er + j);
              const double xm = x[0][m + j], xj = x[1][m + j], xk = x[2][m + j];
              pm = fma(eM, xm, pm);
              pk = fma(eM, xk, fma(eK, xm, pk));
              pj = fma(eM, xj, fma(eJ, xm, fma(2.0 * eK, xk, pj)));
            }
          }
          if (c < n1) {
            a.out[0][ro + m] = pm;
            a.out[1][ro + m] = pk;
            a.out[2][ro + m] = pj;
          }
        }
      }
    }
  }
}
cudaError_t mv4_sweep_run(const MVArgs& a, int p, int cw, int num_sms, cudaStream_t s);

// launch plan built by the host (api.cu) and executed by mv2.cu (own translation unit)
struct MV2Plan {
  MVArgs time, dir, plane;
  int d;
  unsigned grid_time, grid_dir, grid_plane;
  size_t smem_plane;
  int sweep_cw;  // > 0: the d = 3 plane pass runs mv_sweep_kernel with CW columns per lane
  cudaStream_t stream;
  int num_sms;
};
// returns the CUDA error of the launches; *launches += number of kernels launched
// p: space degree (direction passes), pt: time degree (time pass)
cudaError_t mv2_run(int p, int pt, const MV2Plan& plan, int64_t* launches);

}  // namespace ls
