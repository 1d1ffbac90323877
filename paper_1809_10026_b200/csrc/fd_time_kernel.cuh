// Fused time mode of fd_apply (Algorithm 1 steps 2-4 for the time direction, PAPER.md
// 959-962; SURVEY.md 3 "k_time_fused"): for every spatial column s of X[t][s]
//     Y[j][s] = sum_t U_t[t][j] X[t][s]                       (U_t^T, forward time mode)
//     Y[j][s] /= (lambda_t[j] + Lambda_s[s])                    (step 3, reading c3)
//     Z[t'][s] = sum_j U_t[t'][j] Y[j][s]                      (U_t, backward time mode)
// in ONE kernel: Y never leaves the registers (one HBM round trip, 16 B/DOF, instead of two).
//
// Operand roles (m8n8k4, FP64 DMMA; fd_kernels.cuh): the streamed X is the A operand of
// the first product, A[m = s][k = t] (Y^T = X^T U_t), so its accumulators (C fragments:
// lane (r = l/4, c = l%4) holds rows m = r, columns n = 2c, 2c+1 of every n-tile) are,
// register for register, the A fragments of the second product Z^T = Y^T U_t^T
// (A[m = r][k = c] of k-step (jt, h) is column 2c + h of n-tile jt).  The k order of a
// contraction is free, so the eigen index j of column n = 2c + h of n-tile jt is chosen as
// j = 8 jt + 4 h + c: k-step (jt, h) of the second product then covers j = 8jt+4h .. +3,
// and the k-steps past 4 KS (all-zero columns) are skipped.
// M mapping: a warp owns 16 consecutive columns s0 .. s0+15; row r of m-tile ms is column
// s = s0 + 2 r + ms, so a lane's two m-tile elements are one 16-byte pair (LDG.128 / STG.128
// when the row stride is even: VEC).
// Both U_t operands sit in shared memory in B-fragment order, two k-steps per LDS.128:
//   B1 (first product):  b1[((jt*KSP + ks/2)*32 + l)*2 + ks%2] = U_t[4ks + l%4][8jt + 4((l/4)%2) + l/8]
//   B2 (second product): b2[((tt*NJ + jt)*32 + l)*2 + h]      = U_t[8tt + l/4][8jt + 4h + l%4]
// (zero outside n_t x n_t).  Each LDS.128 feeds 4 DMMAs (2 k-steps x 2 m-tiles).
// X loads stream through a rolling register window D k-steps ahead that crosses into the
// warp's next tile, so the second product of one tile overlaps the first loads of the next.
// Sizes: n_t <= 4 KS, KS <= 26 (n_t <= 104: both fragment sets fit in shared memory).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_rd_kernel.cuh"  // ldg_stream, dmma_8x8x4, fast_rcp

namespace ls {

struct FTArgs {
  const double* X;       // [n_t][ld] (columns 0 .. ncols-1 used)
  double* Z;             // [n_t][ld]; may equal X (a warp reads its columns before writing them)
  const double* U;       // U_t, n_t x n_t row-major (row = time index t, column = eigen index j)
  const double* lam_t;   // lambda_t [n_t]
  const double* lam_s;   // Lambda_s per column [ncols]
  int nt;
  uint32_t ncols;
  uint64_t ld;           // row stride (elements)
};

template <int KS_, bool VEC_, int D_, int MINB_, int TV_ = 0, bool SC_ = false>
struct FTCfg {
  static constexpr int KS = KS_, D = D_, MINB = MINB_;
  static constexpr bool VEC = VEC_;
  static constexpr int NJ = (KS + 1) / 2;      // 8-wide n-tiles of j (and of t' in the output)
  // TAIL (n_t = 8 (NJ - 1) + 1 .. + TV, TV = 2 or 4): the last n-tile of j and the last output
  // tile of t' hold at most TV valid indices; they are computed with DFMAs instead of mostly
  // padded DMMA tiles (the eigen columns j0 + v and output rows j0 + w, j0 = 8 (NJ - 1), v, w < TV)
  static constexpr int TV = TV_;
  static constexpr bool TAIL = TV > 0;
  static constexpr int NJD = TAIL ? NJ - 1 : NJ;  // DMMA n-tiles / output tiles
  static constexpr int UTN = TV * 8 * NJ;  // ut[t][v] = U_t[t][j0 + v]
  static constexpr int UON = TV * 8 * NJ;  // uo[j][w] = U_t[j0 + w][j]
  static_assert(TV == 0 || TV == 2 || TV == 4, "tail width");
  static constexpr int KSP = NJ;               // k-step pairs of the first product
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  static constexpr int TW = 16;                // columns per warp tile (2 m-tiles)
  // SC (single copy, n_t up to 136): ONE copy of U_t in 8 x 8 blocks, element (a, b) of block
  // (T, J) at 8a + (b ^ m(a)), m(a) = 6 if a & 2 else 0 -- an XOR swizzle under which both
  // fragment patterns (first product: 4 rows x 8 columns of a block, second: 8 rows x 4 columns)
  // are bank-conflict free (one LDS.64 per fragment instead of one LDS.128 per two); 148 KB at
  // n_t = 133 where the two fragment-ordered copies would need 296 KB
  static constexpr bool SC = SC_;
  static constexpr int B1N = SC ? 0 : NJ * KSP * 64;    // doubles
  static constexpr int B2N = SC ? 0 : NJ * NJ * 64;
  static constexpr int UBN = SC ? NJ * NJ * 64 : 0;
  static constexpr int LAMN = 8 * NJ;
  static constexpr int KSE = ((KS + D - 1) / D) * D;  // k-steps rounded up to the window
  static constexpr size_t SMEM = size_t(B1N + B2N + UBN + LAMN + UTN + UON) * sizeof(double);
  static_assert(SC ? KS <= 34 : KS <= 26, "n_t <= 104 (two fragment copies) / 136 (single copy)");
  static_assert(SMEM <= 232448, "shared memory budget");
};

template <class C>
__global__ void __launch_bounds__(256, C::MINB) fd_time_fused_kernel(FTArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* b1 = smem;
  double* b2 = smem + C::B1N;
  double* ub = b2 + C::B2N;  // SC: the swizzled single copy
  double* lam = ub + C::UBN;
  double* ut = lam + C::LAMN;  // TAIL tables (16-byte aligned: all offsets are multiples of 8 doubles)
  double* uo = ut + C::UTN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c = lane & 3, r = lane >> 2;
  const int nt = a.nt;

  // U_t -> B-fragment order (see the header); lambda_t padded with 1 (the padded
  // accumulator columns are 0, a finite divisor keeps them 0)
  for (int e = tid; e < C::B1N; e += C::THREADS) {
    const int h = e & 1, l = (e >> 1) & 31, ksp = (e >> 6) % C::KSP, jt = (e >> 6) / C::KSP;
    const int t = 4 * (2 * ksp + h) + (l & 3);
    const int j = 8 * jt + 4 * ((l >> 2) & 1) + (l >> 3);
    b1[e] = (t < nt && j < nt) ? __ldg(a.U + size_t(t) * nt + j) : 0.0;
  }
  for (int e = tid; e < C::B2N; e += C::THREADS) {
    const int h = e & 1, l = (e >> 1) & 31, jt = (e >> 6) % C::NJ, tt = (e >> 6) / C::NJ;
    const int t = 8 * tt + (l >> 2);
    const int j = 8 * jt + 4 * h + (l & 3);
    b2[e] = (t < nt && j < nt) ? __ldg(a.U + size_t(t) * nt + j) : 0.0;
  }
  for (int e = tid; e < C::UBN; e += C::THREADS) {
    const int blk = e >> 6, pos = e & 63, ra = pos >> 3;
    const int t = 8 * (blk / C::NJ) + ra;
    const int j = 8 * (blk % C::NJ) + ((pos & 7) ^ ((ra & 2) ? 6 : 0));
    ub[e] = (t < nt && j < nt) ? __ldg(a.U + size_t(t) * nt + j) : 0.0;
  }
  for (int e = tid; e < C::LAMN; e += C::THREADS) lam[e] = e < nt ? __ldg(a.lam_t + e) : 1.0;
  constexpr int J0 = 8 * (C::NJ - 1);
  if constexpr (C::TAIL) {
    for (int e = tid; e < C::UTN; e += C::THREADS) {
      const int t = e / C::TV, v = e % C::TV;
      ut[e] = (t < nt && J0 + v < nt) ? __ldg(a.U + size_t(t) * nt + J0 + v) : 0.0;
      uo[e] = (t < nt && J0 + v < nt) ? __ldg(a.U + size_t(J0 + v) * nt + t) : 0.0;  // uo[j][w], j = t
    }
  }
  __syncthreads();

  const uint32_t ncols = a.ncols;
  const uint32_t ntw = (ncols + C::TW - 1) / C::TW;
  const uint32_t wstride = gridDim.x * C::WARPS;
  uint32_t tile = blockIdx.x * C::WARPS + warp;
  if (tile >= ntw) return;
  const size_t ld = a.ld;
  const size_t kstep = 4 * ld;

  pdl_wait();  // X is the previous kernel's output

  // lane's A elements of k-step ks: X[4ks + c][s0 + 2r + {0, 1}]
  const double* lp;
  uint32_t cnt = 0;  // valid columns of the lane's pair (0, 1, 2)
  auto set_ptr = [&](uint32_t tl) {
    const uint32_t s = tl * C::TW + 2 * r;
    lp = a.X + size_t(c) * ld + s;
    cnt = s >= ncols ? 0u : (s + 1 >= ncols ? 1u : 2u);
  };
  auto load = [&](double2& dst, int ks) {
    const bool ok = 4 * ks + c < nt;
    if (C::VEC) {
      dst = (ok && cnt == 2) ? ldg_stream2(lp) : make_double2(0.0, 0.0);
    } else {
      dst.x = (ok && cnt >= 1) ? ldg_stream(lp) : 0.0;
      dst.y = (ok && cnt == 2) ? ldg_stream(lp + 1) : 0.0;
    }
    lp += kstep;
  };
  double2 win[C::D];
  set_ptr(tile);
#pragma unroll
  for (int s = 0; s < C::D; ++s)
    if (s < C::KS) load(win[s], s);

  const double* b1l = b1 + 2 * lane;
  const double* b2l = b2 + 2 * lane;
  // SC lane offsets inside a block: first product (row 4 (ks & 1) + c, column pi(r)),
  // second product (row r, column 4h + c)
  const int l1 = 8 * c + ((4 * (r & 1) + (r >> 1)) ^ ((c & 2) ? 6 : 0));
  const int l20 = 8 * r + (c ^ ((r & 2) ? 6 : 0));
  const int l21 = 8 * r + ((4 + c) ^ ((r & 2) ? 6 : 0));

#pragma unroll 1
  for (; tile < ntw; tile += wstride) {
    const uint32_t nxt = tile + wstride;
    const uint32_t s0 = tile * C::TW + 2 * r;  // the lane's column pair
    double ls0 = 1.0, ls1 = 1.0;                // Lambda_s of the pair (loaded ahead of use)
    if (s0 < ncols) ls0 = __ldg(a.lam_s + s0);
    if (s0 + 1 < ncols) ls1 = __ldg(a.lam_s + s0 + 1);

    // ---- first product: acc[ms][jt] = (X^T U_t) rows s0 + ms, columns of n-tile jt
    double acc[2][C::NJ][2];
#pragma unroll
    for (int ms = 0; ms < 2; ++ms)
#pragma unroll
      for (int jt = 0; jt < C::NJ; ++jt) acc[ms][jt][0] = acc[ms][jt][1] = 0.0;
    double py[2][C::TV > 0 ? C::TV : 1];  // TAIL: lane-partial Y^T[s0 + ms][J0 + v] (t = c mod 4)
#pragma unroll
    for (int v = 0; v < C::TV; ++v) py[0][v] = py[1][v] = 0.0;
#pragma unroll
    for (int ksp = 0; ksp < C::KSE / 2 + (C::KSE & 1); ++ksp) {
      const int k0 = 2 * ksp, k1 = 2 * ksp + 1;
      if (k0 < C::KS) {
        const double2 x0 = win[k0 % C::D];
        const double2 x1 = (k1 < C::KS) ? win[k1 % C::D] : make_double2(0.0, 0.0);
        if (C::TAIL) {
#pragma unroll
          for (int v = 0; v < C::TV; v += 2) {
            const double2 u0 = *reinterpret_cast<const double2*>(ut + C::TV * (4 * k0 + c) + v);
            py[0][v] = fma(x0.x, u0.x, py[0][v]);
            py[0][v + 1] = fma(x0.x, u0.y, py[0][v + 1]);
            py[1][v] = fma(x0.y, u0.x, py[1][v]);
            py[1][v + 1] = fma(x0.y, u0.y, py[1][v + 1]);
            if (k1 < C::KS) {
              const double2 u1 = *reinterpret_cast<const double2*>(ut + C::TV * (4 * k1 + c) + v);
              py[0][v] = fma(x1.x, u1.x, py[0][v]);
              py[0][v + 1] = fma(x1.x, u1.y, py[0][v + 1]);
              py[1][v] = fma(x1.y, u1.x, py[1][v]);
              py[1][v + 1] = fma(x1.y, u1.y, py[1][v + 1]);
            }
          }
        }
#pragma unroll
        for (int jt = 0; jt < C::NJD; ++jt) {
          double2 bf;
          if constexpr (C::SC) {
            const double* blk = ub + (ksp * C::NJ + jt) * 64;
            bf.x = blk[l1];
            bf.y = blk[l1 + 32];
          } else {
            bf = *reinterpret_cast<const double2*>(b1l + (jt * C::KSP + ksp) * 64);
          }
          dmma_8x8x4(acc[0][jt], x0.x, bf.x);
          dmma_8x8x4(acc[1][jt], x0.y, bf.x);
          if (k1 < C::KS) {
            dmma_8x8x4(acc[0][jt], x1.x, bf.y);
            dmma_8x8x4(acc[1][jt], x1.y, bf.y);
          }
        }
      }
      // refill the consumed slots: k + D of this tile, or the next tile's first k-steps
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = k0 + h;
        if (k >= C::KSE) continue;
        const int kk = k + C::D;
        if (kk < C::KS) {
          load(win[k % C::D], kk);
        } else if (kk >= C::KSE) {
          const int s = kk - C::KSE;  // the next tile's k-step s, same slot (KSE % D == 0)
          if (s == 0) set_ptr(nxt);
          if (s < C::KS) load(win[k % C::D], s);
        }
      }
    }

    // ---- step 3: acc[ms][jt][h] is Y^T[s0 + ms][j = 8jt + 4h + c]
    if (C::TAIL) {  // quad sum of the tail partials (t = c mod 4), then the same division
#pragma unroll
      for (int ms = 0; ms < 2; ++ms)
#pragma unroll
        for (int v = 0; v < C::TV; ++v) {
          double y = py[ms][v];
          y += __shfl_xor_sync(0xffffffffu, y, 1);
          y += __shfl_xor_sync(0xffffffffu, y, 2);
          py[ms][v] = y * fast_rcp(lam[J0 + v] + (ms ? ls1 : ls0));
        }
    }
#pragma unroll
    for (int jt = 0; jt < C::NJD; ++jt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double lt = lam[8 * jt + 4 * h + c];
        acc[0][jt][h] *= fast_rcp(lt + ls0);
        acc[1][jt][h] *= fast_rcp(lt + ls1);
      }

    // ---- second product, two output n-tiles (t' = 8tt + 2c + {0,1}) at a time
    double* zp = a.Z + s0;
#pragma unroll 1
    for (int tt = 0; tt < C::NJD; tt += 2) {
      const bool two = tt + 1 < C::NJD;
      double o[2][2][2];  // [tile of the pair][ms][column half]
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int ms = 0; ms < 2; ++ms) o[u][ms][0] = o[u][ms][1] = 0.0;
      if (C::TAIL) {  // the tail columns' rank-TV update: o += Y^T[., J0 + v] U_t[t'][J0 + v]
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int v = 0; v < C::TV; v += 2) {
              const double2 w = *reinterpret_cast<const double2*>(ut + C::TV * (8 * (tt + u) + 2 * c + h) + v);
#pragma unroll
              for (int ms = 0; ms < 2; ++ms)
                o[u][ms][h] = fma(py[ms][v + 1], w.y, fma(py[ms][v], w.x, o[u][ms][h]));
            }
      }
#pragma unroll
      for (int jt = 0; jt < C::NJD; ++jt) {
        const bool h1 = 2 * jt + 1 < C::KS;  // k-step (jt, 1) has valid columns
        double2 f0;
        if constexpr (C::SC) {
          const double* blk = ub + (tt * C::NJ + jt) * 64;
          f0 = make_double2(blk[l20], blk[l21]);
        } else {
          f0 = *reinterpret_cast<const double2*>(b2l + (tt * C::NJ + jt) * 64);
        }
        dmma_8x8x4(o[0][0], acc[0][jt][0], f0.x);
        dmma_8x8x4(o[0][1], acc[1][jt][0], f0.x);
        if (h1) {
          dmma_8x8x4(o[0][0], acc[0][jt][1], f0.y);
          dmma_8x8x4(o[0][1], acc[1][jt][1], f0.y);
        }
        if (two) {
          double2 f1;
          if constexpr (C::SC) {
            const double* blk = ub + ((tt + 1) * C::NJ + jt) * 64;
            f1 = make_double2(blk[l20], blk[l21]);
          } else {
            f1 = *reinterpret_cast<const double2*>(b2l + ((tt + 1) * C::NJ + jt) * 64);
          }
          dmma_8x8x4(o[1][0], acc[0][jt][0], f1.x);
          dmma_8x8x4(o[1][1], acc[1][jt][0], f1.x);
          if (h1) {
            dmma_8x8x4(o[1][0], acc[0][jt][1], f1.y);
            dmma_8x8x4(o[1][1], acc[1][jt][1], f1.y);
          }
        }
      }
      // store: o[u][ms][h] = Z[t' = 8(tt+u) + 2c + h][s0 + ms]
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        if (u == 1 && !two) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int t = 8 * (tt + u) + 2 * c + h;
          if (t >= nt || s0 >= ncols) continue;
          double* dst = zp + size_t(t) * ld;
          if (C::VEC) {
            *reinterpret_cast<double2*>(dst) = make_double2(o[u][0][h], o[u][1][h]);
          } else {
            dst[0] = o[u][0][h];
            if (s0 + 1 < ncols) dst[1] = o[u][1][h];
          }
        }
      }
    }
    if (C::TAIL) {  // output rows J0 + w: Z^T[s][J0 + w] = sum_j Y^T[s][j] U_t[J0 + w][j]
      double pz[2][C::TV > 0 ? C::TV : 1];
#pragma unroll
      for (int w = 0; w < C::TV; ++w) pz[0][w] = pz[1][w] = 0.0;
#pragma unroll
      for (int jt = 0; jt < C::NJD; ++jt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int w = 0; w < C::TV; w += 2) {
            const double2 uw = *reinterpret_cast<const double2*>(uo + C::TV * (8 * jt + 4 * h + c) + w);
#pragma unroll
            for (int ms = 0; ms < 2; ++ms) {
              pz[ms][w] = fma(acc[ms][jt][h], uw.x, pz[ms][w]);
              pz[ms][w + 1] = fma(acc[ms][jt][h], uw.y, pz[ms][w + 1]);
            }
          }
      if (c == 0) {  // the tail-tail block (quad-uniform py): once per quad
#pragma unroll
        for (int v = 0; v < C::TV; ++v)
#pragma unroll
          for (int w = 0; w < C::TV; w += 2) {
            const double2 uw = *reinterpret_cast<const double2*>(uo + C::TV * (J0 + v) + w);
#pragma unroll
            for (int ms = 0; ms < 2; ++ms) {
              pz[ms][w] = fma(py[ms][v], uw.x, pz[ms][w]);
              pz[ms][w + 1] = fma(py[ms][v], uw.y, pz[ms][w + 1]);
            }
          }
      }
#pragma unroll
      for (int ms = 0; ms < 2; ++ms)
#pragma unroll
        for (int w = 0; w < C::TV; ++w) {
          pz[ms][w] += __shfl_xor_sync(0xffffffffu, pz[ms][w], 1);
          pz[ms][w] += __shfl_xor_sync(0xffffffffu, pz[ms][w], 2);
        }
#pragma unroll
      for (int w = 0; w < C::TV; ++w) {
        const int t = J0 + w;
        if (c != w || t >= nt || s0 >= ncols) continue;  // lane c = w of each quad stores row J0 + w
        double* dst = zp + size_t(t) * ld;
        if (C::VEC) {
          *reinterpret_cast<double2*>(dst) = make_double2(pz[0][w], pz[1][w]);
        } else {
          dst[0] = pz[0][w];
          if (s0 + 1 < ncols) dst[1] = pz[1][w];
        }
      }
    }
  }
}

}  // namespace ls
