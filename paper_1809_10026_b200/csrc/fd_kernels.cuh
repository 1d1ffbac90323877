// FD mode-k product kernel (Algorithm 1 steps 2-4, PAPER.md 959-962) for sm_100a.
//
// A d+1-mode tensor in colex layout is viewed, for the mode being applied, as
// X[P][n][Q] (row-major; n = the mode's extent, Q = product of the faster
// extents, P = product of the slower ones).  The mode-k product with a dense
// n x n matrix W is, for every column c = (p, q) of the (n x P*Q) unfolding,
//     Y[p][a][q] = sum_i W[a][i] X[p][i][q],
// i.e. a GEMM  Y_(k) = W X_(k)  with M = n, K = n, N = P*Q (mode-k unfolding;
// eq:kron_vec, PAPER.md 646).
//
// FP64 on B200 has no tcgen05 kind, so the contraction runs on
// the FP64 tensor path: mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4.  Measured
// (profiles/peaks_fp64_r01.json, tools/fp64_mix.cu): 37.0 TF/s chip peak,
// DMMA and DFMA share the FP64 datapath, one warp with >= 2 independent
// accumulators saturates its SM sub-partition (dependent latency ~27 cycles,
// issue interval 16 cycles).  Design ("v2", balanced per sub-partition):
//   * 8 warps per CTA (two per SMSP, so one warp's LDS / epilogue / loader
//     instructions overlap the other's DMMAs), persistent CTAs (one per SM).
//   * W (U^T or U, <= 136 x 136) lives in shared memory in m8n8k4 A-fragment
//     order (32 consecutive doubles per (m-tile, k-step): conflict-free LDS.64).
//   * Warp w owns the NT n-tiles (8 columns each) of group w%4 and the m-tile
//     half w/4 ([0, ceil(MT/2)) or [ceil(MT/2), MT)); the two warps of an SMSP
//     (w, w+4) together cover all m-tiles of one n-tile group, so every SMSP
//     does exactly the same number of DMMAs per tile (n = 132/133 has 17
//     m-tiles: a split of rows over 4 sub-partitions cannot balance).
//   * The streamed operand X is staged tile by tile (BN columns x Kp rows)
//     with cp.async (16-byte when aligned, else 8-byte) in an NSTAGE ring.
//     Row strides are = 4 (mod 16) doubles: the B-fragment reads
//     (lane -> k = lane%4, column = lane/4) are bank-conflict free.
//   * A/B fragments are double-buffered in registers one k-step ahead.
//   * Ragged extents: K padded to Kp = 4*ceil(n/4) (zero rows in smem, zero
//     columns in W), M to 8*ceil(n/8) (zero W rows; never stored), tail
//     columns skipped at the store.
//   * Optional epilogue (time mode, the last forward mode): Algorithm 1 step 3,
//     Y[a][c] /= (lambda_t[a] + Lambda_s[c]) (reading c3), reciprocal by
//     rcp.approx + 2 Newton steps (relative error ~1e-16).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pdl.cuh"

#include "plan.hpp"

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
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// 1/d for d > 0 (the FD divisor lambda_t + Lambda_s >= 2.4): FP32 MUFU.RCP seed (relative
// error <= 2^-22) and ONE Newton step in FP64, which squares the error to <= 2^-44 ~ 6e-14
// (c13: rounding-level, far below the 1e-9 parity bar).  Each FP64 op here competes with
// the DMMAs for the FP64 pipe, so the second Newton step (and the MUFU.RCP64H seed) are
// not taken.
__device__ __forceinline__ double fast_rcp(double d) {
  float xf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(xf) : "f"(__double2float_rn(d)));
  const double x = double(xf);
  return fma(x, fma(-d, x, 1.0), x);
}

constexpr int pad4mod16(int v) {  // smallest s >= v with s % 16 == 4
  return v + ((4 - v % 16) + 16) % 16;
}

template <int KS_, int NT_, bool MODE1_, bool SCALE_, int NSTAGE_>
struct ModeCfg {
  static constexpr int KS = KS_, NT = NT_, NSTAGE = NSTAGE_;
  static constexpr bool MODE1 = MODE1_, SCALE = SCALE_;
  static constexpr int NWARPS = 8;
  static constexpr int THREADS = 32 * NWARPS;
  static constexpr int MTILES = (KS + 1) / 2;   // ceil(n/8) for n in (4KS-4, 4KS]
  static constexpr int MTH = (MTILES + 1) / 2;  // m-tiles per warp (low half; high half may be one less)
  static constexpr int BN = 8 * NT * 4;         // columns per tile (4 n-tile groups)
  static constexpr int KP = 4 * KS;             // padded K
  static constexpr int SN = pad4mod16(BN);      // non-MODE1 tile [KP][SN]
  static constexpr int SK = pad4mod16(KP);      // MODE1 tile [BN][SK]
  static constexpr int TILE = MODE1 ? BN * SK : KP * SN;  // doubles
  static constexpr int KSP = (KS + 1) / 2;                 // k-step pairs
  static constexpr int WFRAG = MTILES * KSP * 64;         // doubles (A fragments, k-step pairs)
  static constexpr size_t SMEM = size_t(WFRAG + TILE * NSTAGE) * sizeof(double);
  static_assert(MODE1 || THREADS % (BN / 2) == 0, "loader: THREADS % (BN/2) == 0");
  static_assert(MODE1 || (BN / 2) <= THREADS, "loader: one column pair per thread");
  static_assert(SMEM <= 232448, "shared memory budget");
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
  bool y16;         // Y is 16-byte aligned (vector stores allowed)
  // fused all-to-all epilogue (register-direct kernel only): 0 = store to Y;
  // 1 = forward (this launch is the last forward spatial mode of a time slab: element
  //     (t_local, a, q) -> spatial s = a*Q + q -> peer chunk buffer, plan.hpp a2a_fwd_dest);
  // 2 = backward (this launch is the backward time mode of a spatial chunk: element
  //     (t = a, q) -> peer slab buffer, a2a_bwd_dest)
  int remote;
  double* const* peer;  // device table [world] of destination buffers
  int world, me;
  int64_t nt_g, Ns_g;   // global n_t, N_s
};

// One warp's share of one tile: MC m-tiles (compile time: no predicates, so no
// re-convergence around mma.sync) x NT n-tiles, all k-steps.  A fragments come
// two k-steps per LDS.128 and are double-buffered one k-step pair ahead.
template <class C, int MC, int MA>
__device__ __forceinline__ void compute_tile(double (&acc)[MA][C::NT][2], const double* wl,
                                             const double* t, int grp, int lane) {
#pragma unroll
  for (int mt = 0; mt < MA; ++mt)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
  if (MC == 0) return;
  const int col0 = grp * C::NT * 8 + (lane >> 2);
  const double* tb = C::MODE1 ? (t + col0 * C::SK + (lane & 3)) : (t + (lane & 3) * C::SN + col0);
  auto bfrag = [&](int ks, int nt) -> double {
    return C::MODE1 ? tb[nt * 8 * C::SK + ks * 4] : tb[ks * 4 * C::SN + nt * 8];
  };
  auto apair = [&](int mt, int ksp) -> double2 {
    return *reinterpret_cast<const double2*>(wl + (mt * C::KSP + ksp) * 64);
  };
  double2 af[2][MC > 0 ? MC : 1];
  double bf[2][2][C::NT];
#pragma unroll
  for (int mt = 0; mt < MC; ++mt) af[0][mt] = apair(mt, 0);
#pragma unroll
  for (int nt = 0; nt < C::NT; ++nt) {
    bf[0][0][nt] = bfrag(0, nt);
    bf[0][1][nt] = (1 < C::KS) ? bfrag(1, nt) : 0.0;
  }
#pragma unroll
  for (int ksp = 0; ksp < C::KSP; ++ksp) {
    const int cur = ksp & 1, nxt = cur ^ 1;
    if (ksp + 1 < C::KSP) {
#pragma unroll
      for (int mt = 0; mt < MC; ++mt) af[nxt][mt] = apair(mt, ksp + 1);
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        bf[nxt][0][nt] = bfrag(2 * ksp + 2, nt);
        bf[nxt][1][nt] = (2 * ksp + 3 < C::KS) ? bfrag(2 * ksp + 3, nt) : 0.0;
      }
    }
#pragma unroll
    for (int mt = 0; mt < MC; ++mt)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) dmma_8x8x4(acc[mt][nt], af[cur][mt].x, bf[cur][0][nt]);
    if (2 * ksp + 1 < C::KS) {
#pragma unroll
      for (int mt = 0; mt < MC; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) dmma_8x8x4(acc[mt][nt], af[cur][mt].y, bf[cur][1][nt]);
    }
  }
}

// compute_tile with the last m-tile replaced by DFMAs for its TAIL (1 or 2) valid rows:
// when n = 8 (MTILES - 1) + TAIL, that m-tile's DMMAs would be 7/8 or 3/4 padding.  Lane
// (row r = lane/4, k = lane%4) holds B[4 ks + k][col r (+8 nt)]; it accumulates
// sum_ks W[8 MC + t][4 ks + k] B[4 ks + k][col] for t < TAIL, and the four lanes of a quad
// are summed by two shuffles: tacc[t][nt] = D[8 MC + t][col0 + 8 nt] in every lane of the quad.
template <class C, int MC, int TAIL>
__device__ __forceinline__ void compute_tile_tail(double (&acc)[C::MTILES][C::NT][2], double (&tacc)[2][C::NT],
                                                  const double* wsm, const double* t, int grp, int lane) {
#pragma unroll
  for (int mt = 0; mt < C::MTILES; ++mt)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
#pragma unroll
  for (int r = 0; r < 2; ++r)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) tacc[r][nt] = 0.0;
  const double* wl = wsm + lane * 2;
  const int col0 = grp * C::NT * 8 + (lane >> 2);
  const double* tb = C::MODE1 ? (t + col0 * C::SK + (lane & 3)) : (t + (lane & 3) * C::SN + col0);
  auto bfrag = [&](int ks, int nt) -> double {
    return C::MODE1 ? tb[nt * 8 * C::SK + ks * 4] : tb[ks * 4 * C::SN + nt * 8];
  };
  auto apair = [&](int mt, int ksp) -> double2 {
    return *reinterpret_cast<const double2*>(wl + (mt * C::KSP + ksp) * 64);
  };
  auto tpair = [&](int r, int ksp) -> double2 {  // W[8 MC + r][4 (2 ksp) + k], W[..][4 (2 ksp + 1) + k]
    return *reinterpret_cast<const double2*>(wsm + ((MC * C::KSP + ksp) * 32 + r * 4 + (lane & 3)) * 2);
  };
  double2 af[2][MC];
  double2 tw[2][TAIL];
  double bf[2][2][C::NT];
#pragma unroll
  for (int mt = 0; mt < MC; ++mt) af[0][mt] = apair(mt, 0);
#pragma unroll
  for (int r = 0; r < TAIL; ++r) tw[0][r] = tpair(r, 0);
#pragma unroll
  for (int nt = 0; nt < C::NT; ++nt) {
    bf[0][0][nt] = bfrag(0, nt);
    bf[0][1][nt] = (1 < C::KS) ? bfrag(1, nt) : 0.0;
  }
#pragma unroll
  for (int ksp = 0; ksp < C::KSP; ++ksp) {
    const int cur = ksp & 1, nxt = cur ^ 1;
    if (ksp + 1 < C::KSP) {
#pragma unroll
      for (int mt = 0; mt < MC; ++mt) af[nxt][mt] = apair(mt, ksp + 1);
#pragma unroll
      for (int r = 0; r < TAIL; ++r) tw[nxt][r] = tpair(r, ksp + 1);
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        bf[nxt][0][nt] = bfrag(2 * ksp + 2, nt);
        bf[nxt][1][nt] = (2 * ksp + 3 < C::KS) ? bfrag(2 * ksp + 3, nt) : 0.0;
      }
    }
    if (ksp == C::KSP - 1 && (C::KS & 1)) {
      // the last k-step holds TAIL (= n - 4 (KS - 1)) valid columns of W: a rank-1 / rank-2
      // DFMA update of this lane's D entries instead of a 3/4- or 1/2-padded DMMA k-step
      const int kb = 4 * (C::KS - 1);
#pragma unroll
      for (int kv = 0; kv < TAIL; ++kv) {
        double xv[C::NT][2];
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int col = grp * C::NT * 8 + nt * 8 + 2 * (lane & 3) + h;
            xv[nt][h] = C::MODE1 ? t[col * C::SK + kb + kv] : t[(kb + kv) * C::SN + col];
          }
#pragma unroll
        for (int mt = 0; mt < MC; ++mt) {
          const double w = wsm[((mt * C::KSP + ksp) * 32 + (lane >> 2) * 4 + kv) * 2];
#pragma unroll
          for (int nt = 0; nt < C::NT; ++nt) {
            acc[mt][nt][0] = fma(w, xv[nt][0], acc[mt][nt][0]);
            acc[mt][nt][1] = fma(w, xv[nt][1], acc[mt][nt][1]);
          }
        }
      }
    } else {
#pragma unroll
      for (int mt = 0; mt < MC; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) dmma_8x8x4(acc[mt][nt], af[cur][mt].x, bf[cur][0][nt]);
    }
#pragma unroll
    for (int r = 0; r < TAIL; ++r)
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) tacc[r][nt] = fma(tw[cur][r].x, bf[cur][0][nt], tacc[r][nt]);
    if (2 * ksp + 1 < C::KS) {
#pragma unroll
      for (int mt = 0; mt < MC; ++mt)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) dmma_8x8x4(acc[mt][nt], af[cur][mt].y, bf[cur][1][nt]);
#pragma unroll
      for (int r = 0; r < TAIL; ++r)
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) tacc[r][nt] = fma(tw[cur][r].y, bf[cur][1][nt], tacc[r][nt]);
    }
  }
#pragma unroll
  for (int r = 0; r < TAIL; ++r)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      tacc[r][nt] += __shfl_xor_sync(0xffffffffu, tacc[r][nt], 1);
      tacc[r][nt] += __shfl_xor_sync(0xffffffffu, tacc[r][nt], 2);
    }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) fd_mode_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* wsm = smem;                 // W fragments
  double* tiles = smem + C::WFRAG;    // NSTAGE x TILE
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int grp = warp & 3;                       // n-tile group (= SMSP)
  const int mbase = (warp >> 2) ? C::MTH : 0;     // m-tile half
  const int mcount = (warp >> 2) ? (C::MTILES - C::MTH) : C::MTH;
  const int n = args.n;
  const uint32_t Q = args.Q;
  const uint32_t ncols = args.ncols;

  // ---- W -> shared memory in A-fragment order, two k-steps per lane-slot so one
  //      LDS.128 fetches both: wsm[((mt*KSP + ks/2)*32 + lane)*2 + ks%2]
  for (int e = tid; e < C::WFRAG; e += C::THREADS) {
    const int h = e & 1, l = (e >> 1) & 31, ksp = (e >> 6) % C::KSP, mt = (e >> 6) / C::KSP;
    const int ks = 2 * ksp + h;
    const int a = mt * 8 + (l >> 2), i = ks * 4 + (l & 3);
    wsm[e] = (a < n && i < n && ks < C::KS) ? __ldg(args.W + size_t(a) * n + i) : 0.0;
  }
  // ---- zero the K padding of every stage once (never written by the loader)
  for (int s = 0; s < C::NSTAGE; ++s) {
    double* t = tiles + s * C::TILE;
    if (C::MODE1) {
      const int padw = C::SK - n;
      for (int e = tid; e < C::BN * padw; e += C::THREADS) t[(e / padw) * C::SK + n + e % padw] = 0.0;
    } else {
      for (int e = tid; e < (C::KP - n) * C::SN; e += C::THREADS) t[n * C::SN + e] = 0.0;
    }
  }

  // ---- loader: tile -> stage (cp.async; 16 B where both sides are aligned)
  auto load_tile = [&](uint32_t tile, int stage) {
    double* t = tiles + stage * C::TILE;
    const uint32_t c0 = tile * C::BN;
    if (C::MODE1) {
      // the tile is the contiguous chunk X[c0*n, (c0+BN)*n): element e -> (c = e/n, i = e%n)
      const uint32_t cend = min(c0 + (uint32_t)C::BN, ncols);
      const uint32_t total = (cend - c0) * (uint32_t)n;
      const double* src = args.X + size_t(c0) * n;
      if ((n & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
        // even n: pairs (e, e+1) with e even never straddle a row; 16-byte copies
        const uint32_t half = total >> 1, hn = n >> 1;
        for (uint32_t h = tid; h < half; h += C::THREADS) {
          const uint32_t cc = h / hn, i = 2 * (h - cc * hn);
          cp_async16(t + cc * C::SK + i, src + 2 * h);
        }
      } else {
        uint32_t cc = tid / n, i = tid % n;
        const uint32_t dq = C::THREADS / n, dr = C::THREADS % n;
        for (uint32_t e = tid; e < total; e += C::THREADS) {
          cp_async8(t + cc * C::SK + i, src + e);
          cc += dq;
          i += dr;
          if (i >= (uint32_t)n) { i -= n; ++cc; }
        }
      }
    } else {
      // column pairs (cc, cc+1): one 16-byte copy when adjacent and aligned
      constexpr int PAIRS = C::BN / 2;
      const int pr = tid % PAIRS;
      const int cc = 2 * pr;
      const uint32_t c = c0 + cc;
      if (c < ncols) {
        const uint32_t p = c / Q, q = c - p * Q;
        const double* src = args.X + (size_t(p) * n) * Q + q;
        const bool second = (c + 1 < ncols);
        const bool vec = second && (q + 1 < Q) && ((Q & 1) == 0) &&
                         ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
        const double* src2 = nullptr;
        if (second && !vec) {
          const uint32_t c2 = c + 1, p2 = c2 / Q, q2 = c2 - p2 * Q;
          src2 = args.X + (size_t(p2) * n) * Q + q2;
        }
        for (int i = tid / PAIRS; i < n; i += C::THREADS / PAIRS) {
          double* dst = t + i * C::SN + cc;
          if (vec) {
            cp_async16(dst, src + size_t(i) * Q);
          } else {
            cp_async8(dst, src + size_t(i) * Q);
            if (second) cp_async8(dst + 1, src2 + size_t(i) * Q);
          }
        }
      }
    }
  };

  const uint32_t stride = gridDim.x;
  uint32_t tile = blockIdx.x;
  pdl_wait();  // X is the previous kernel's output
#pragma unroll 1
  for (int s = 0; s < C::NSTAGE - 1; ++s) {
    uint32_t tt = tile + s * stride;
    if (tt < args.ntiles) load_tile(tt, s);
    cp_async_commit();
  }

  // SCALE: this lane's output rows' lambda_t, loaded once
  double lam_row[C::SCALE ? C::MTH : 1];
#pragma unroll
  for (int mt = 0; mt < (C::SCALE ? C::MTH : 1); ++mt) {
    const int a = (mbase + mt) * 8 + (lane >> 2);
    lam_row[mt] = (C::SCALE && mt < mcount && a < n) ? __ldg(args.lam_a + a) : 0.0;
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
    const double* t = tiles + (j % C::NSTAGE) * C::TILE;
    const uint32_t c0 = tile * C::BN;
    // SCALE: this lane's columns' Lambda_s, prefetched before the k-loop
    double lam_col[C::SCALE ? C::NT : 1][2];
    if (C::SCALE) {
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        const uint32_t c = c0 + grp * C::NT * 8 + nt * 8 + 2 * (lane & 3);
        lam_col[nt][0] = c < ncols ? __ldg(args.lam_c + c) : 0.0;
        lam_col[nt][1] = c + 1 < ncols ? __ldg(args.lam_c + c + 1) : 0.0;
      }
    }

    double acc[C::MTH][C::NT][2];
    if (warp >> 2)
      compute_tile<C, C::MTILES - C::MTH, C::MTH>(acc, wsm + (C::MTH * C::KSP * 32 + lane) * 2, t, grp, lane);
    else
      compute_tile<C, C::MTH, C::MTH>(acc, wsm + lane * 2, t, grp, lane);

    // ---- epilogue: registers -> global (optionally scaled, Alg. 1 step 3)
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      const uint32_t c = c0 + grp * C::NT * 8 + nt * 8 + 2 * (lane & 3);  // even; lane owns c, c+1
      if (c >= ncols) continue;
      const bool two = (c + 1 < ncols);
      size_t base, base2 = 0;
      bool vec = false;
      if (C::MODE1) {
        base = size_t(c) * n;
        base2 = base + n;
      } else {
        const uint32_t p = c / Q, q = c - p * Q;
        base = size_t(p) * n * Q + q;
        vec = args.y16 && two && (q + 1 < Q) && ((Q & 1) == 0) && ((base & 1) == 0);
        if (two && !vec) {
          const uint32_t c2 = c + 1, p2 = c2 / Q, q2 = c2 - p2 * Q;
          base2 = size_t(p2) * n * Q + q2;
        }
      }
#pragma unroll
      for (int mt = 0; mt < C::MTH; ++mt) {
        const int a = (mbase + mt) * 8 + (lane >> 2);
        if (mt < mcount && a < n) {
          double v0 = acc[mt][nt][0], v1 = acc[mt][nt][1];
          if (C::SCALE) {
            v0 *= fast_rcp(lam_row[C::SCALE ? mt : 0] + lam_col[C::SCALE ? nt : 0][0]);
            v1 *= fast_rcp(lam_row[C::SCALE ? mt : 0] + lam_col[C::SCALE ? nt : 0][1]);
          }
          const size_t off = C::MODE1 ? size_t(a) : size_t(a) * Q;
          if (vec) {
            *reinterpret_cast<double2*>(args.Y + base + off) = make_double2(v0, v1);
          } else {
            args.Y[base + off] = v0;
            if (two) args.Y[base2 + off] = v1;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

// =====================================================================================
// Ping-pong variant (the production kernel).  Two warp sets of 4 warps (one warp per
// SMSP each) work on alternate tiles of the CTA's tile sequence; their DMMA phases are
// serialised by a pair of named barriers (set 0 MMA -> set 1 MMA -> set 0 MMA ...), so
// while one set runs its k-loop at the full DMMA rate of every SMSP the other set
// stores its previous tile and loads its next one.  Each warp owns all m-tiles of NT
// n-tiles (acc[MTILES][NT]); a set's 4 warps cover the tile's 4 n-tile groups.
// Stage s of the ring belongs to set s % 2 (SPS stages per set).
// =====================================================================================
template <int KS_, int NT_, bool MODE1_, bool SCALE_, int SPS_, int TAIL_ = 0>
struct PPCfg {
  static constexpr int KS = KS_, NT = NT_, SPS = SPS_;
  static constexpr int TAIL = TAIL_;  // 0, or the 1-2 rows of the last m-tile done by DFMAs
  static constexpr bool MODE1 = MODE1_, SCALE = SCALE_;
  static constexpr int THREADS = 256, SET_THREADS = 128;
  static constexpr int NSTAGE = 2 * SPS;
  static constexpr int MTILES = (KS + 1) / 2;
  static constexpr int MTH = MTILES;
  static constexpr int BN = 8 * NT * 4;
  static constexpr int KP = 4 * KS;
  static constexpr int SN = pad4mod16(BN);
  static constexpr int SK = pad4mod16(KP);
  static constexpr int TILE = MODE1 ? BN * SK : KP * SN;
  static constexpr int KSP = (KS + 1) / 2;
  static constexpr int WFRAG = MTILES * KSP * 64;
  static constexpr size_t SMEM = size_t(WFRAG + TILE * NSTAGE) * sizeof(double);
  static_assert(MODE1 || SET_THREADS % (BN / 2) == 0, "loader: SET_THREADS % (BN/2) == 0");
  static_assert(SMEM <= 232448, "shared memory budget");
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// cp.async loader of one tile by LT threads (thread index lt)
template <class C, int LT>
__device__ __forceinline__ void load_tile_dev(const ModeArgs& args, double* t, uint32_t tile, int lt) {
  const int n = args.n;
  const uint32_t Q = args.Q, ncols = args.ncols;
  const uint32_t c0 = tile * C::BN;
  if (C::MODE1) {
    const uint32_t cend = min(c0 + (uint32_t)C::BN, ncols);
    const uint32_t total = (cend - c0) * (uint32_t)n;
    const double* src = args.X + size_t(c0) * n;
    if ((n & 1) == 0 && ((reinterpret_cast<uintptr_t>(src) & 15) == 0)) {
      const uint32_t half = total >> 1, hn = n >> 1;
      for (uint32_t h = lt; h < half; h += LT) {
        const uint32_t cc = h / hn, i = 2 * (h - cc * hn);
        cp_async16(t + cc * C::SK + i, src + 2 * h);
      }
    } else {
      uint32_t cc = lt / n, i = lt % n;
      const uint32_t dq = LT / n, dr = LT % n;
      for (uint32_t e = lt; e < total; e += LT) {
        cp_async8(t + cc * C::SK + i, src + e);
        cc += dq;
        i += dr;
        if (i >= (uint32_t)n) { i -= n; ++cc; }
      }
    }
  } else {
    constexpr int PAIRS = C::BN / 2;
    const int cc = 2 * (lt % PAIRS);
    const uint32_t c = c0 + cc;
    if (c < ncols) {
      const uint32_t p = c / Q, q = c - p * Q;
      const double* src = args.X + (size_t(p) * n) * Q + q;
      const bool second = (c + 1 < ncols);
      const bool vec = second && (q + 1 < Q) && ((Q & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
      const double* src2 = src;
      if (second && !vec) {
        const uint32_t c2 = c + 1, p2 = c2 / Q, q2 = c2 - p2 * Q;
        src2 = args.X + (size_t(p2) * n) * Q + q2;
      }
      const size_t rstep = size_t(LT / PAIRS) * Q;
      int i = lt / PAIRS;
      const double* s1 = src + size_t(i) * Q;
      const double* s2 = src2 + size_t(i) * Q;
      double* dst = t + i * C::SN + cc;
      for (; i < n; i += LT / PAIRS) {
        if (vec) {
          cp_async16(dst, s1);
        } else {
          cp_async8(dst, s1);
          if (second) cp_async8(dst + 1, s2);
        }
        s1 += rstep;
        s2 += rstep;
        dst += (LT / PAIRS) * C::SN;
      }
    }
  }
}

template <class C>
__global__ void __launch_bounds__(256, 1) fd_mode_pp_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* wsm = smem;
  double* tiles = smem + C::WFRAG;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int set = warp >> 2;       // warp set (ping / pong)
  const int grp = warp & 3;        // n-tile group (= SMSP)
  const int stid = tid & 127;      // thread index within the set
  const int n = args.n;
  const uint32_t Q = args.Q;
  const uint32_t ncols = args.ncols;

  for (int e = tid; e < C::WFRAG; e += C::THREADS) {
    const int h = e & 1, l = (e >> 1) & 31, ksp = (e >> 6) % C::KSP, mt = (e >> 6) / C::KSP;
    const int ks = 2 * ksp + h;
    const int a = mt * 8 + (l >> 2), i = ks * 4 + (l & 3);
    wsm[e] = (a < n && i < n && ks < C::KS) ? __ldg(args.W + size_t(a) * n + i) : 0.0;
  }
  for (int s = 0; s < C::NSTAGE; ++s) {
    double* t = tiles + s * C::TILE;
    if (C::MODE1) {
      const int padw = C::SK - n;
      for (int e = tid; e < C::BN * padw; e += C::THREADS) t[(e / padw) * C::SK + n + e % padw] = 0.0;
    } else {
      for (int e = tid; e < (C::KP - n) * C::SN; e += C::THREADS) t[n * C::SN + e] = 0.0;
    }
  }
  double lam_row[C::SCALE ? C::MTILES : 1];
#pragma unroll
  for (int mt = 0; mt < (C::SCALE ? C::MTILES : 1); ++mt) {
    const int a = mt * 8 + (lane >> 2);
    lam_row[mt] = (C::SCALE && a < n) ? __ldg(args.lam_a + a) : 0.0;
  }
  __syncthreads();
  pdl_wait();  // X is the previous kernel's output

  // CTA tile sequence: local k -> blockIdx.x + k*gridDim.x; set s takes k = s, s+2, ...
  const uint32_t stride = gridDim.x;
  const uint32_t my_tiles = (args.ntiles > blockIdx.x) ? (args.ntiles - blockIdx.x + stride - 1) / stride : 0;
  const uint32_t n0 = (my_tiles + 1) / 2, n1 = my_tiles / 2;  // tiles of set 0 / set 1
  const uint32_t mine = set ? n1 : n0, other = set ? n0 : n1;
  auto tile_of = [&](uint32_t j) { return blockIdx.x + (set + 2 * j) * stride; };
  auto stage_of = [&](uint32_t j) { return set + 2 * int(j % C::SPS); };
#pragma unroll 1
  for (int j = 0; j < C::SPS; ++j) {
    if (uint32_t(j) < mine) load_tile_dev<C, 128>(args, tiles + stage_of(j) * C::TILE, tile_of(j), stid);
    cp_async_commit();
  }
  const int BAR_SET = 1 + set;                       // set-local barrier
  const int BAR_MY_TURN = 3 + set, BAR_OTHER_TURN = 3 + (set ^ 1);

#pragma unroll 1
  for (uint32_t j = 0; j < mine; ++j) {
    cp_async_wait<C::SPS - 1>();
    named_sync(BAR_SET, 128);                        // my stage is loaded for all 128 threads
    // DMMA phase, serialised with the other set: set 0 starts, then alternate
    if (set == 1 || j > 0) named_sync(BAR_MY_TURN, 256);
    const double* t = tiles + stage_of(j) * C::TILE;
    // SCALE: this lane's Lambda_s columns, loaded before the k-loop (latency hidden)
    double lcp[C::SCALE ? C::NT : 1][2];
    if (C::SCALE) {
      const uint32_t cb = tile_of(j) * C::BN + grp * C::NT * 8 + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < C::NT; ++nt) {
        const uint32_t c = cb + nt * 8;
        lcp[nt][0] = c < ncols ? __ldg(args.lam_c + c) : 0.0;
        lcp[nt][1] = c + 1 < ncols ? __ldg(args.lam_c + c + 1) : 0.0;
      }
    }
    double acc[C::MTILES][C::NT][2];
    double tacc[2][C::NT];
    constexpr int MCD = C::MTILES - (C::TAIL ? 1 : 0);  // m-tiles on the tensor pipe
    if constexpr (C::TAIL > 0)
      compute_tile_tail<C, MCD, C::TAIL>(acc, tacc, wsm, t, grp, lane);
    else
      compute_tile<C, C::MTILES, C::MTILES>(acc, wsm + lane * 2, t, grp, lane);
    // hand the tensor pipes to the other set if it has a tile for this turn
    if ((set == 0 && j < other) || (set == 1 && j + 1 < other)) named_arrive(BAR_OTHER_TURN, 256);
    named_sync(BAR_SET, 128);                        // all 4 warps done reading the stage
    {
      const uint32_t jn = j + C::SPS;
      if (jn < mine) load_tile_dev<C, 128>(args, tiles + stage_of(jn) * C::TILE, tile_of(jn), stid);
      cp_async_commit();
    }
    // ---- epilogue (overlaps the other set's DMMA phase)
    const uint32_t c0 = tile_of(j) * C::BN;
#pragma unroll
    for (int nt = 0; nt < C::NT; ++nt) {
      const uint32_t c = c0 + grp * C::NT * 8 + nt * 8 + 2 * (lane & 3);
      if (c >= ncols) continue;
      const bool two = (c + 1 < ncols);
      size_t base, base2 = 0;
      bool vec = false;
      if (C::MODE1) {
        base = size_t(c) * n;
        base2 = base + n;
      } else {
        const uint32_t p = c / Q, q = c - p * Q;
        base = size_t(p) * n * Q + q;
        vec = args.y16 && two && (q + 1 < Q) && ((Q & 1) == 0) && ((base & 1) == 0);
        if (two && !vec) {
          const uint32_t c2 = c + 1, p2 = c2 / Q, q2 = c2 - p2 * Q;
          base2 = size_t(p2) * n * Q + q2;
        }
      }
      double lc0 = 0.0, lc1 = 0.0;
      if (C::SCALE) {
        lc0 = lcp[C::SCALE ? nt : 0][0];
        lc1 = lcp[C::SCALE ? nt : 0][1];
      }
#pragma unroll
      for (int mt = 0; mt < MCD; ++mt) {
        const int a = mt * 8 + (lane >> 2);
        if (a < n) {
          double v0 = acc[mt][nt][0], v1 = acc[mt][nt][1];
          if (C::SCALE) {
            v0 *= fast_rcp(lam_row[C::SCALE ? mt : 0] + lc0);
            v1 *= fast_rcp(lam_row[C::SCALE ? mt : 0] + lc1);
          }
          const size_t off = C::MODE1 ? size_t(a) : size_t(a) * Q;
          if (vec) {
            *reinterpret_cast<double2*>(args.Y + base + off) = make_double2(v0, v1);
          } else {
            args.Y[base + off] = v0;
            if (two) args.Y[base2 + off] = v1;
          }
        }
      }
    }
    if constexpr (C::TAIL > 0) {  // rows 8 MCD .. 8 MCD + TAIL - 1: lane k = lane % 4 < TAIL stores row 8 MCD + k
      const int r = lane & 3;
      if (r < C::TAIL) {
        const int a = 8 * MCD + r;
#pragma unroll
        for (int nt = 0; nt < C::NT; ++nt) {
          const uint32_t c = c0 + grp * C::NT * 8 + nt * 8 + (lane >> 2);
          if (c >= ncols || a >= n) continue;
          double v = (r == 0) ? tacc[0][nt] : tacc[C::TAIL > 1 ? 1 : 0][nt];
          if (C::SCALE) v *= fast_rcp(__ldg(args.lam_a + a) + __ldg(args.lam_c + c));
          if (C::MODE1) {
            args.Y[size_t(c) * n + a] = v;
          } else {
            const uint32_t p = c / Q, q = c - p * Q;
            args.Y[size_t(p) * n * Q + size_t(a) * Q + q] = v;
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

} // namespace ls
