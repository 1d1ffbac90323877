// FD mode-k product kernels (Algorithm 1 steps 2-4, PAPER.md 959-962) for sm_100a.
//
// A d+1-mode tensor in colex layout is viewed, for the mode being applied, as
// X[P][n][Q] (row-major; n = the mode's extent, Q = product of the faster
// extents, P = product of the slower ones).  The mode-k product with a dense
// n x n matrix W is, for every column c = (p, q) of the (n x P*Q) unfolding,
//     Y[p][a][q] = sum_i W[a][i] X[p][i][q],
// i.e. a GEMM  Y_(k) = W X_(k)  with M = n, K = n, N = P*Q (the mode-k
// unfolding of Kolda-Bader; eq:kron_vec, PAPER.md 646).
//
// FP64 on B200 has no tcgen05 kind, so the contraction runs on
// the FP64 tensor path: mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4, 37.0 TF/s
// measured (profiles/peaks_fp64_r01.json).  Design:
//   * W (U^T or U, <= 136 x 136) is WEIGHT-STATIONARY IN REGISTERS: warp-row
//     wm owns m-tiles [wm*MT, wm*MT+MT) for all K, loaded once per CTA.
//   * The streamed operand X is staged in shared memory tile by tile
//     (BN columns x Kp rows) with cp.async, NSTAGE-deep ring, persistent CTAs.
//   * Shared-memory row strides are = 4 (mod 16) doubles so the m8n8k4
//     B-fragment reads (lane -> row lane%4, col lane/4) are bank-conflict free.
//   * Ragged extents: K padded to Kp = 4*ceil(n/4) (zero rows in smem, zero
//     columns in W), M to 8*ceil(n/8) (zero W rows; never stored), N tail
//     columns skipped at the store.
//   * Optional epilogue (the time mode, the last forward mode): Algorithm 1
//     step 3, Y[a][c] /= (lambda_t[a] + Lambda_s[c]) (reading c3), with the
//     reciprocal from rcp.approx + 2 Newton steps (rel. err ~1e-16).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ls {

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double fast_rcp(double d) {
  double x;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(d));
  double e = fma(-d, x, 1.0);
  x = fma(x, e, x);
  e = fma(-d, x, 1.0);
  return fma(x, e, x);
}

constexpr int pad4mod16(int v) {  // smallest s >= v with s % 16 == 4
  return v + ((4 - v % 16) + 16) % 16;
}

template <int MT_, int NT_, int WM_, int WN_, int KS_, bool MODE1_, bool SCALE_, int NSTAGE_>
struct ModeCfg {
  static constexpr int MT = MT_, NT = NT_, WM = WM_, WN = WN_, KS = KS_, NSTAGE = NSTAGE_;
  static constexpr bool MODE1 = MODE1_, SCALE = SCALE_;
  static constexpr int THREADS = 32 * WM * WN;
  static constexpr int BN = 8 * NT * WN;  // columns per tile
  static constexpr int KP = 4 * KS;       // padded K
  // non-MODE1 tile: [KP][SN]; MODE1 tile: [BN][SK]
  static constexpr int SN = pad4mod16(BN);
  static constexpr int SK = pad4mod16(KP);
  static constexpr int TILE = MODE1 ? BN * SK : KP * SN;  // doubles
  static constexpr size_t SMEM = size_t(TILE) * NSTAGE * sizeof(double);
  static_assert(THREADS % BN == 0 || MODE1, "loader needs THREADS % BN == 0");
};

struct ModeArgs {
  const double* X;
  double* Y;
  const double* W;      // n x n row-major, Y = W X along the mode
  const double* lam_a;  // SCALE: lambda per output mode index (lambda_t)
  const double* lam_c;  // SCALE: Lambda_s per column (P == 1)
  int n;
  uint32_t P, Q;
  uint32_t ncols;   // P * Q
  uint32_t ntiles;  // ceil(ncols / BN)
};

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) fd_mode_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int wm = warp % C::WM;  // warp-row: output rows
  const int wn = warp / C::WM;  // warp-col: columns
  const int n = args.n;
  const uint32_t Q = args.Q;
  const uint32_t ncols = args.ncols;
  const int mtiles = (n + 7) >> 3;

  // ---- weights: W fragments for this warp's m-tiles, all k-steps (registers)
  double wreg[C::MT][C::KS];
#pragma unroll
  for (int mt = 0; mt < C::MT; ++mt) {
    const int a = (wm * C::MT + mt) * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      const int i = ks * 4 + (lane & 3);
      wreg[mt][ks] = (a < n && i < n) ? __ldg(args.W + size_t(a) * n + i) : 0.0;
    }
  }

  // ---- zero the K padding of every stage once (never written by the loader)
  for (int s = 0; s < C::NSTAGE; ++s) {
    double* t = smem + s * C::TILE;
    if (C::MODE1) {
      for (int e = tid; e < C::BN * (C::SK - n); e += C::THREADS) {
        int r = e / (C::SK - n), cidx = n + e % (C::SK - n);
        t[r * C::SK + cidx] = 0.0;
      }
    } else {
      for (int e = tid; e < (C::KP - n) * C::SN; e += C::THREADS) t[n * C::SN + e] = 0.0;
    }
  }

  // ---- loader: tile -> stage
  auto load_tile = [&](uint32_t tile, int stage) {
    double* t = smem + stage * C::TILE;
    const uint32_t c0 = tile * C::BN;
    if (C::MODE1) {
      // columns are rows of length n, contiguous: chunk X[c0*n, (c0+BN)*n)
      const uint32_t cend = min(c0 + (uint32_t)C::BN, ncols);
      const uint32_t total = (cend - c0) * (uint32_t)n;
      const double* src = args.X + size_t(c0) * n;
      uint32_t cc = tid / n, i = tid % n;
      const uint32_t dq = C::THREADS / n, dr = C::THREADS % n;
      for (uint32_t e = tid; e < total; e += C::THREADS) {
        cp_async8(t + cc * C::SK + i, src + e);
        cc += dq;
        i += dr;
        if (i >= (uint32_t)n) { i -= n; ++cc; }
      }
    } else {
      const int cc = tid % C::BN;
      const uint32_t c = c0 + cc;
      if (c < ncols) {
        const uint32_t p = c / Q, q = c - p * Q;
        const double* src = args.X + (size_t(p) * n) * Q + q;
        for (int i = tid / C::BN; i < n; i += C::THREADS / C::BN)
          cp_async8(t + i * C::SN + cc, src + size_t(i) * Q);
      }
    }
  };

  const uint32_t stride = gridDim.x;
  uint32_t tile = blockIdx.x;
#pragma unroll 1
  for (int s = 0; s < C::NSTAGE - 1; ++s) {
    uint32_t tt = tile + s * stride;
    if (tt < args.ntiles) load_tile(tt, s);
    cp_async_commit();
  }

#pragma unroll 1
  for (int j = 0; tile < args.ntiles; ++j, tile += stride) {
    cp_async_wait<C::NSTAGE - 2>();
    __syncthreads();
    {
      uint32_t tn = tile + (C::NSTAGE - 1) * stride;
      if (tn < args.ntiles) load_tile(tn, (j + C::NSTAGE - 1) % C::NSTAGE);
      cp_async_commit();
    }
    const double* t = smem + (j % C::NSTAGE) * C::TILE;

    double acc[C::MT][C::NT][2];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;

    const int colbase = wn * C::NT * 8 + (lane >> 2);
#pragma unroll
    for (int ks = 0; ks < C::KS; ++ks) {
      double xf[C::NT];
      const int krow = ks * 4 + (lane & 3);
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        const int col = colbase + nt * 8;
        xf[nt] = C::MODE1 ? t[col * C::SK + krow] : t[krow * C::SN + col];
      }
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        if (wm * C::MT + mt < mtiles) {
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt) dmma_8x8x4(acc[mt][nt], wreg[mt][ks], xf[nt]);
        }
      }
    }

    // ---- epilogue: registers -> global (optionally scaled, Alg. 1 step 3)
    const uint32_t c0 = tile * C::BN;
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        const uint32_t c = c0 + wn * C::NT * 8 + nt * 8 + 2 * (lane & 3) + jj;
        if (c >= ncols) continue;
        size_t base;
        if (C::MODE1) {
          base = size_t(c) * n;
        } else {
          const uint32_t p = c / Q, q = c - p * Q;
          base = size_t(p) * n * Q + q;
        }
        double lc = 0.0;
        if (C::SCALE) lc = __ldg(args.lam_c + c);
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const int a = (wm * C::MT + mt) * 8 + (lane >> 2);
          if (a < n) {
            double v = acc[mt][nt][jj];
            if (C::SCALE) v *= fast_rcp(__ldg(args.lam_a + a) + lc);
            args.Y[base + (C::MODE1 ? size_t(a) : size_t(a) * Q)] = v;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

} // namespace ls
