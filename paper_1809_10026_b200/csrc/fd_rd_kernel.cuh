// FD mode-k product, "register-direct" variant (Algorithm 1 steps 2-4,
// PAPER.md 959-962): Y_(k) = W X_(k) with W = U^T or U (n x n), the same GEMM
// view as fd_kernels.cuh (X viewed as [P][n][Q], columns c = (p, q)).
//
// Why a second design (profiles/r01, ncu source page of fd_mode_kernel at
// n = 132): the smem-staged kernel spent ~20% of its DMMA issue slots in
// __syncthreads waits, in the A-fragment LDS latency right before the DMMA
// that consumes it, and in the loader's index arithmetic.  Here
//   * W stays in shared memory in m8n8k4 A-fragment order (two k-steps per
//     LDS.128, conflict-free), loaded once per CTA;
//   * the streamed operand X never touches shared memory: every warp loads its
//     own B fragments straight from global memory into a rolling register
//     window D k-steps ahead (crossing into the warp's next tile), so there is
//     no block-level barrier after the prologue and the two warps of each SM
//     sub-partition run fully independently;
//   * each warp owns a tile of 8*NT columns and ALL m-tiles: acc[MT][NT] in
//     registers, every A fragment feeds 2*NT DMMAs;
//   * column permutation: lane l (B-fragment column n = l/4) holds the NT
//     physical columns NT*n .. NT*n+NT-1 of the tile, so its B loads are NT
//     contiguous doubles (LDG.128) for strided modes, and its accumulators
//     (C-fragment columns 2(l%4), 2(l%4)+1 of every n-tile) are the 2*NT
//     contiguous physical columns 2*NT*(l%4) .. +2*NT-1 (vector stores);
//   * K padding: rows >= n are never loaded (predicated to 0: a bucket's KS can exceed
//     ceil(n/4), and those rows would lie past the end of the column), W's padded
//     columns are 0; M padding rows are never stored;
//   * SCALE (forward time mode): Algorithm 1 step 3 in the epilogue,
//     Y[a][c] /= (lambda_t[a] + Lambda_s[c]) (reading c3).
// FAST = strided mode with Q % (2*NT) == 0 and 16-byte aligned X, Y: every
// NT-column group lies in one p-slice (vector loads/stores); otherwise every
// column is addressed on its own.
//
// CS (centrosymmetric split, spatial modes).  With uniform open knots and Dirichlet
// conditions at both ends (PAPER.md 266-267, 1111-1112) the space pencil (J, M) is
// centrosymmetric: R J R = J, R M R = M for the exchange matrix R (b_i(1-x) = b_{n+1-i}(x)).
// Its eigenvectors then split into he = ceil(n/2) even ones (u = R u) and ho = floor(n/2)
// odd ones (u = -R u), each fixed by its first half a (setup: reduced pencils
// Q^T J Q, Q^T M Q, api.cu cs_eig).  So U^T x = [A_e^T (x + R x)_half ; A_o^T (x - R x)_half]
// and U y = [p + q ; R (p - q)] with p = A_e y_e, q = A_o y_o: two half-size products
// instead of one n x n product, half the DMMA work (z = P^{-1} r is unchanged: any
// eigenbasis of the same pencil gives it; the eigen index order is [even | odd]).
// Fold (forward): the lane loads x[k] and x[n-1-k] and forms the sum / difference when
// the k-step is consumed; unfold (backward): two B rows (k and he + k) and the butterfly in
// the epilogue.  W = [W_e (he x he) | W_o (ho x ho)].
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"

namespace ls {

template <int KS_, int NT_, bool MODE1_, bool SCALE_, bool FAST_, int D_, int REMOTE_ = 0, int CS_ = 0, int MINB_ = 1,
          int TR_ = 0>
struct RDCfg {
  static constexpr int KS = KS_, NT = NT_, D = D_;
  // TR: DFMA tail rows (split kernels, odd KS).  When the half extents are 8(MT - 1) + 1 or + 2
  // (he = 66 at config 4, 33 at configs 2 / 3, 49 at config 5 p = 4) the last m-tile is 3/4 or
  // 7/8 padding: its TR = 2 rows are computed by DFMAs on the B fragments the lane already
  // holds (W rows from the same shared-memory fragments, a quad shuffle reduction at the end
  // of the tile) and the DMMA m-tiles stop at MT - 1.
  static constexpr int TR = TR_;
  static constexpr int MINB = MINB_;  // CTAs per SM the register budget is sized for
  static constexpr int REMOTE = REMOTE_;  // fused all-to-all epilogue (ModeArgs::remote)
  // CS: centrosymmetric split (see the header of this file): 0 = plain n x n product,
  // 1 = fold (forward: even/odd halves of the input, outputs [even | odd]),
  // 2 = unfold (backward: inputs [even | odd], outputs p + q and R(p - q))
  static constexpr int CS = CS_;
  static constexpr int NH = CS ? 2 : 1;    // half-products per tile
#ifndef LS_RD_PF64_MINKS
#define LS_RD_PF64_MINKS 17
#endif
  static constexpr bool PF64 = CS && KS >= LS_RD_PF64_MINKS;  // .L2::64B streaming loads (see ldg_stream)
  static constexpr bool MODE1 = MODE1_, SCALE = SCALE_, FAST = FAST_;
  static constexpr int MT = (KS + 1) / 2;  // ceil(n/8) for n in (4KS-4, 4KS] (CS: n -> ceil(n/2))
  static constexpr int MTD = TR ? MT - 1 : MT;  // m-tiles computed by DMMAs
  static constexpr int KSP = (KS + 1) / 2;  // k-step pairs
  static constexpr int KSE = ((KS + D - 1) / D) * D;  // k-steps rounded up to the window
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  static constexpr int TW = 8 * NT;  // columns per warp tile
  static constexpr int WFRAG1 = MT * KSP * 64;  // one half's A fragments
  static constexpr int WFRAG = NH * WFRAG1;
  static constexpr int LAMA = SCALE ? 8 * MT : 0;  // lambda_t per output row (SCALE)
  static constexpr size_t SMEM = size_t(WFRAG + LAMA) * sizeof(double);
  static_assert(!(MODE1 && FAST), "FAST is a strided-mode path");
  static_assert(REMOTE == 0 || (FAST && !SCALE), "fused all-to-all epilogues: unscaled FAST launches");
  static_assert(CS == 0 || !SCALE, "the scaled (time) mode is not centrosymmetric");
  static_assert(CS != 2 || REMOTE == 0, "unfold: local stores only");
  static_assert(NT == 1 || NT % 2 == 0, "NT = 1 or even (LDG.128 pairs)");
  static_assert(TR == 0 || (TR == 2 && CS != 0 && REMOTE == 0 && KS % 2 == 1), "tail rows: local split kernels, odd KS");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// one lane's B source for one warp tile: element offsets (< 2^32: N <= ~3.2e8 on
// one GPU) of its NT columns at row kq; FAST and MODE1 keep only off[0] live
template <int NT>
struct RDIn {
  uint32_t off[NT];
  uint32_t mask;  // bit j: column j valid
};

template <class C>
__device__ __forceinline__ RDIn<C::NT> rd_make_in(const ModeArgs& a, uint32_t tile, int lane) {
  RDIn<C::NT> r;
  r.mask = 0;
  const int kq = lane & 3, nq = lane >> 2;
  const uint32_t c0 = tile * C::TW + C::NT * nq;
  const uint32_t Q = a.Q;
#pragma unroll
  for (int j = 0; j < C::NT; ++j) r.off[j] = 0;
  if (C::FAST) {
    // NT columns in one p-slice (Q % 2NT == 0, ncols = P*Q): valid together
    const uint32_t p = c0 / Q, q = c0 - p * Q;
    r.off[0] = (p * uint32_t(a.n) + kq) * Q + q;
    r.mask = (c0 < a.ncols) ? ((1u << C::NT) - 1) : 0u;
  } else if (C::MODE1) {  // column j at off[0] + j*n
    r.off[0] = c0 * uint32_t(a.n) + kq;
#pragma unroll
    for (int j = 0; j < C::NT; ++j)
      if (c0 + j < a.ncols) r.mask |= 1u << j;
  } else {
#pragma unroll
    for (int j = 0; j < C::NT; ++j) {
      const uint32_t c = c0 + j;
      if (c < a.ncols) {
        r.mask |= 1u << j;
        const uint32_t p = c / Q, q = c - p * Q;
        r.off[j] = (p * uint32_t(a.n) + kq) * Q + q;
      }
    }
  }
  return r;
}

// streaming loads kept in program order at the NVVM level (volatile): the compiler
// otherwise hoists a whole tile of B loads ahead of the DMMAs and spills
#ifndef LS_LDG_L2PF
#define LS_LDG_L2PF ""  // L2 prefetch-size qualifier of the streaming loads (e.g. ".L2::128B")
#endif
// PF64: the .L2::64B prefetch-size hint (an L2 miss fills 64 bytes).  Measured (A/B of whole
// builds): config 4 fd_apply 14.795 -> 14.728 ms with it on every streaming load, but config 3
// +0.4 % and config 5 p = 8 +1.2 %; .L2::128B neutral, .L2::256B +1.1 % at config 4.  So it is
// used by the config-4-sized split kernels only (RDCfg::PF64).
template <bool PF64 = false>
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  if constexpr (PF64) asm volatile("ld.global.nc.L1::no_allocate.L2::64B.f64 %0, [%1];" : "=d"(v) : "l"(p));
  else asm volatile("ld.global.nc.L1::no_allocate" LS_LDG_L2PF ".f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
template <bool PF64 = false>
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 v;
  if constexpr (PF64)
    asm volatile("ld.global.nc.L1::no_allocate.L2::64B.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate" LS_LDG_L2PF ".v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// B fragments of one k-step (rows 4kk + lane%4 of the lane's NT columns; CS: the two half
// rows) from running pointers: lp[] at the half-0 row, lm[] at the half-1 row (fold: the
// mirror row n-1-k, moving backwards; unfold: row he + k).  NP pointers: one for FAST / MODE1
// (columns at +j or +j*n), one per column otherwise.  Advancing pointers instead of
// recomputing base + kk * kstep keeps the unrolled k-loop from holding one 64-bit address per
// k-step in registers.
template <class C>
struct RDPtr {
  static constexpr int NP = (C::FAST || C::MODE1) ? 1 : C::NT;
  const double* lp[NP];
  const double* lm[NP];
};

// LS_RD_PFA > 0 (experiment knob, split kernels): with every k-step's loads, an L2 prefetch of the
// rows LS_RD_PFA k-steps further down the same columns.  Why: ptxas sinks the window's loads
// towards their uses (255 registers: the SASS of the KS = 17 fold kernel issues a k-step pair's
// LDGs about 45 DMMAs before the DADDs that read them, not the 6 k-steps = 216 DMMAs of the
// source), and ncu attributes a quarter of the warp-stall samples to those DADDs' long
// scoreboard; a prefetch has no destination registers, so it stays where it is written.
#ifndef LS_RD_PFA
#define LS_RD_PFA 0
#endif
__device__ __forceinline__ void prefetch_l2(const double* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

template <class C>
__device__ __forceinline__ void rd_load(double (&dst)[C::NH][C::NT], RDPtr<C>& q, uint32_t mask, bool ok0,
                                        bool ok1, size_t kstep, int n, bool pf0 = false, bool pf1 = false) {
  if constexpr (LS_RD_PFA > 0 && C::CS != 0) {
    // FAST: the lane's NT columns are contiguous (one address); MODE1: column j at + j n
    const int64_t ahead = int64_t(LS_RD_PFA) * int64_t(kstep);
#pragma unroll
    for (int j = 0; j < ((C::FAST) ? 1 : C::NT); ++j) {
      const bool cm = C::FAST ? mask != 0 : ((mask >> j) & 1u);
      const double* p0 = C::MODE1 ? q.lp[0] + size_t(j) * n : q.lp[(C::MODE1 || C::FAST) ? 0 : j];
      const double* p1 = C::MODE1 ? q.lm[0] + size_t(j) * n : q.lm[(C::MODE1 || C::FAST) ? 0 : j];
      if (pf0 && cm) prefetch_l2(p0 + ahead);
      if (pf1 && cm) prefetch_l2(C::CS == 1 ? p1 - ahead : p1 + ahead);
    }
  }
  if (C::FAST) {
    const bool m = mask != 0;
    if constexpr (C::NT == 1) {
      dst[0][0] = (ok0 && m) ? ldg_stream<C::PF64>(q.lp[0]) : 0.0;
      if (C::CS) dst[C::NH - 1][0] = (ok1 && m) ? ldg_stream<C::PF64>(q.lm[0]) : 0.0;
    } else {
#pragma unroll
      for (int j = 0; j < C::NT; j += 2) {
        double2 v0 = make_double2(0.0, 0.0), v1 = make_double2(0.0, 0.0);
        if (ok0 && m) v0 = ldg_stream2<C::PF64>(q.lp[0] + j);
        if (C::CS && ok1 && m) v1 = ldg_stream2<C::PF64>(q.lm[0] + j);
        dst[0][j] = v0.x;
        dst[0][j + 1] = v0.y;
        if (C::CS) {
          dst[C::NH - 1][j] = v1.x;
          dst[C::NH - 1][j + 1] = v1.y;
        }
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < C::NT; ++j) {
      const bool cm = (mask >> j) & 1u;
      const double* p0 = C::MODE1 ? q.lp[0] + size_t(j) * n : q.lp[C::MODE1 ? 0 : j];
      dst[0][j] = (ok0 && cm) ? ldg_stream<C::PF64>(p0) : 0.0;
      if (C::CS) {
        const double* p1 = C::MODE1 ? q.lm[0] + size_t(j) * n : q.lm[C::MODE1 ? 0 : j];
        dst[C::NH - 1][j] = (ok1 && cm) ? ldg_stream<C::PF64>(p1) : 0.0;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < RDPtr<C>::NP; ++i) {
    q.lp[i] += kstep;
    if (C::CS == 1) q.lm[i] -= kstep;
    if (C::CS == 2) q.lm[i] += kstep;
  }
}

template <class C>
__global__ void __launch_bounds__(256, C::MINB) fd_mode_rd_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* wsm = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, nq = lane >> 2;
  const int n = args.n;
  const int he = C::CS ? (n + 1) / 2 : n, ho = C::CS ? n / 2 : 0;  // half sizes (CS)
  const uint32_t Q = args.Q, ncols = args.ncols;

  // W -> shared memory, A-fragment order, two k-steps per lane slot:
  // wsm[hf*WFRAG1 + ((mt*KSP + ks/2)*32 + l)*2 + ks%2] = W_hf[mt*8 + l/4][ks*4 + l%4]
  // (CS: W = [W_0 (he x he) | W_1 (ho x ho)], both row-major)
  for (int e = tid; e < C::WFRAG; e += C::THREADS) {
    const int hf = e / C::WFRAG1, e1 = e - hf * C::WFRAG1;
    const int h = e1 & 1, l = (e1 >> 1) & 31, ksp = (e1 >> 6) % C::KSP, mt = (e1 >> 6) / C::KSP;
    const int ks = 2 * ksp + h;
    const int a = mt * 8 + (l >> 2), i = ks * 4 + (l & 3);
    const int nh = C::CS ? (hf ? ho : he) : n;
    const double* Wh = args.W + (hf ? size_t(he) * he : 0);
    wsm[e] = (a < nh && i < nh && ks < C::KS) ? __ldg(Wh + size_t(a) * nh + i) : 0.0;
  }
  double* lam_a_s = wsm + C::WFRAG;  // SCALE: lambda_t of the output rows, staged once
  if (C::SCALE)
    for (int e = tid; e < C::LAMA; e += C::THREADS) lam_a_s[e] = e < n ? __ldg(args.lam_a + e) : 0.0;
  __syncthreads();

  const uint32_t ntw = (ncols + C::TW - 1) / C::TW;
  const uint32_t wstride = gridDim.x * C::WARPS;
  uint32_t tile = blockIdx.x * C::WARPS + warp;
  if (tile >= ntw) return;
  const size_t rstride = C::MODE1 ? size_t(1) : size_t(Q);
  const size_t kstep = 4 * rstride;
  // rows 4*kk + kq >= n (CS: >= he / ho) are never loaded (zero B fragment): the bucket's
  // KS may exceed ceil(n/4), and those rows lie past the end of the column
  auto row_ok = [&](int kk) { return 4 * kk + kq < he; };
  auto row_ok1 = [&](int kk) { return 4 * kk + kq < ho; };
  const int64_t off1 = C::CS == 1 ? int64_t(n - 1 - 2 * kq) * int64_t(rstride) : int64_t(he) * int64_t(rstride);
  const double* wl = wsm + lane * 2;

  pdl_wait();  // X is the previous kernel's output (fd_kernels.cuh)
  RDIn<C::NT> cur = rd_make_in<C>(args, tile, lane);
  double bw[C::D][C::NH][C::NT];
  RDPtr<C> q;
  auto set_ptrs = [&](const RDIn<C::NT>& in) {
#pragma unroll
    for (int i = 0; i < RDPtr<C>::NP; ++i) {
      q.lp[i] = args.X + in.off[i];
      q.lm[i] = q.lp[i] + off1;
    }
  };
  // loads run strictly in order: k-steps 0 .. KS-1 of a tile, then 0 .. of the next one
  auto load = [&](double (&dst)[C::NH][C::NT], const RDIn<C::NT>& in, int kk) {
    rd_load<C>(dst, q, in.mask, row_ok(kk), row_ok1(kk), kstep, n, kk + LS_RD_PFA < C::KS && row_ok(kk + LS_RD_PFA),
               kk + LS_RD_PFA < C::KS && row_ok1(kk + LS_RD_PFA));
  };
  set_ptrs(cur);
#pragma unroll
  for (int s = 0; s < C::D; ++s)
    if (s < C::KS) load(bw[s], cur, s);

#pragma unroll 1
  for (; tile < ntw; tile += wstride) {
    const RDIn<C::NT> nxt = rd_make_in<C>(args, tile + wstride, lane);
    // SCALE: this lane's Lambda_s columns, loaded before the k-loop (latency hidden)
    const uint32_t cg = tile * C::TW + 2 * C::NT * kq;
    double lc[C::SCALE ? 2 * C::NT : 1];
    if (C::SCALE) {
#pragma unroll
      for (int e = 0; e < 2 * C::NT; ++e) lc[e] = (cg + e < ncols) ? __ldg(args.lam_c + cg + e) : 0.0;
    }
    double acc[C::NH][C::MTD][C::NT][2];
#pragma unroll
    for (int hf = 0; hf < C::NH; ++hf)
#pragma unroll
      for (int mt = 0; mt < C::MTD; ++mt)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) acc[hf][mt][j][0] = acc[hf][mt][j][1] = 0.0;
    // tail rows 8 MTD + i: this lane's partial sums over its k = 4 ks + kq
    double tl[C::NH][C::TR ? C::TR : 1][C::NT];
#pragma unroll
    for (int hf = 0; hf < C::NH; ++hf)
#pragma unroll
      for (int i = 0; i < (C::TR ? C::TR : 1); ++i)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) tl[hf][i][j] = 0.0;

    // k-loop in pairs; phantom steps (KS <= ks < KSE) only refill the window
#pragma unroll
    for (int ksp = 0; ksp < C::KSE / 2 + (C::KSE & 1); ++ksp) {
      const int k0 = 2 * ksp, k1 = 2 * ksp + 1;
      if (k0 < C::KS) {
        // the B operands of both k-steps (fold: even half x + Rx, odd half x - Rx)
        double b[2][C::NH][C::NT];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < C::NT; ++j) {
            const int s = (k0 + h) % C::D;
            if (C::CS == 1) {
              b[h][0][j] = bw[s][0][j] + bw[s][C::NH - 1][j];
              b[h][C::NH - 1][j] = bw[s][0][j] - bw[s][C::NH - 1][j];
            } else {
#pragma unroll
              for (int hf = 0; hf < C::NH; ++hf) b[h][hf][j] = bw[s][hf][j];
            }
          }
        if constexpr (C::TR > 0) {
          // W_hf[8 MTD + i][4 k + kq] of both k-steps: the A-fragment slot of lane 4 i + kq
#pragma unroll
          for (int hf = 0; hf < C::NH; ++hf)
#pragma unroll
            for (int i = 0; i < C::TR; ++i) {
              const double2 wt = *reinterpret_cast<const double2*>(
                  wsm + hf * C::WFRAG1 + (C::MTD * C::KSP + ksp) * 64 + (4 * i + kq) * 2);
#pragma unroll
              for (int j = 0; j < C::NT; ++j) {
                tl[hf][i][j] = fma(wt.x, b[0][hf][j], tl[hf][i][j]);
                if (k1 < C::KS) tl[hf][i][j] = fma(wt.y, b[1][hf][j], tl[hf][i][j]);
              }
            }
        }
#pragma unroll
        for (int mt = 0; mt < C::MTD; ++mt) {
#pragma unroll
          for (int hf = 0; hf < C::NH; ++hf) {
            const double2 af = *reinterpret_cast<const double2*>(wl + hf * C::WFRAG1 + (mt * C::KSP + ksp) * 64);
#pragma unroll
            for (int j = 0; j < C::NT; ++j) dmma_8x8x4(acc[hf][mt][j], af.x, b[0][hf][j]);
            if (k1 < C::KS) {
#pragma unroll
              for (int j = 0; j < C::NT; ++j) dmma_8x8x4(acc[hf][mt][j], af.y, b[1][hf][j]);
            }
          }
        }
      }
      // refill the consumed slots with k-steps k + D (this tile) or k + D - KSE (next tile)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = k0 + h;
        if (k >= C::KSE) continue;
        const int kk = k + C::D;
        if (kk < C::KS) {
          load(bw[k % C::D], cur, kk);
        } else if (kk >= C::KSE) {
          const int s = kk - C::KSE;  // next tile's k-step, same slot (KSE % D == 0)
          if (s == 0) set_ptrs(nxt);
          if (s < C::KS) load(bw[k % C::D], nxt, s);
        }
      }
    }

    // ---- epilogue: lane's columns cg .. cg + 2NT - 1 (v[e] = column cg + e) at output row a
    constexpr bool ONEBASE = C::MODE1 || C::FAST || C::REMOTE;
    uint32_t fp = 0, fq = 0;
    if (cg < ncols) {
      fp = cg / Q;
      fq = cg - fp * Q;
    }
    size_t base[ONEBASE ? 1 : 2 * C::NT];
    if (C::MODE1) {
      base[0] = size_t(cg) * n;
    } else if (!ONEBASE) {
#pragma unroll
      for (int e = 0; e < (ONEBASE ? 1 : 2 * C::NT); ++e) {
        const uint32_t c = cg + e;
        const uint32_t p = c / Q, q = c - p * Q;
        base[e] = size_t(p) * n * Q + q;
      }
    }
    auto emit = [&](int a, const double (&v)[2 * C::NT]) {
      if (C::REMOTE) {
        // fused all-to-all: every output element goes straight to its owner's receive buffer
        // (peer memory over NVLink in a multi-GPU run); pairs that stay contiguous and
        // 16-byte aligned in the destination are stored as one double2
        if (cg >= ncols) return;
#pragma unroll
        for (int e = 0; e < 2 * C::NT; e += 2) {
          if (cg + e >= ncols) continue;
          int r0, r1;
          int64_t o0, o1;
          if (C::REMOTE == 1) {
            const int64_t s0 = int64_t(a) * Q + fq + e;
            a2a_fwd_dest(int64_t(fp), s0, args.nt_g, args.Ns_g, args.world, args.me, &r0, &o0);
            a2a_fwd_dest(int64_t(fp), s0 + 1, args.nt_g, args.Ns_g, args.world, args.me, &r1, &o1);
          } else {
            a2a_bwd_dest(int64_t(a), int64_t(fq) + e, args.nt_g, args.Ns_g, args.world, args.me, &r0, &o0);
            a2a_bwd_dest(int64_t(a), int64_t(fq) + e + 1, args.nt_g, args.Ns_g, args.world, args.me, &r1, &o1);
          }
          const bool second = cg + e + 1 < ncols;
          double* d0 = args.peer[r0] + o0;
          if (second && r1 == r0 && o1 == o0 + 1 && ((reinterpret_cast<uintptr_t>(d0) & 15) == 0)) {
            *reinterpret_cast<double2*>(d0) = make_double2(v[e], v[e + 1]);
          } else {
            *d0 = v[e];
            if (second) args.peer[r1][o1] = v[e + 1];
          }
        }
      } else if (C::FAST) {
        if (cg >= ncols) return;
        double* o = args.Y + size_t(fp) * n * Q + fq + size_t(a) * Q;
#pragma unroll
        for (int e = 0; e < 2 * C::NT; e += 2) *reinterpret_cast<double2*>(o + e) = make_double2(v[e], v[e + 1]);
      } else {
#pragma unroll
        for (int e = 0; e < 2 * C::NT; ++e) {
          if (cg + e < ncols) {
            if (C::MODE1) args.Y[base[0] + size_t(e) * n + a] = v[e];
            else args.Y[base[ONEBASE ? 0 : e] + size_t(a) * rstride] = v[e];
          }
        }
      }
    };
#pragma unroll
    for (int mt = 0; mt < C::MTD; ++mt) {
      const int a = mt * 8 + nq;
      double v[C::NH][2 * C::NT];
#pragma unroll
      for (int hf = 0; hf < C::NH; ++hf)
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int j = 0; j < C::NT; ++j) v[hf][h * C::NT + j] = acc[hf][mt][j][h];
      if (C::CS == 0) {
        if (a < n) {
          if (C::SCALE) {
            const double la = lam_a_s[a];
#pragma unroll
            for (int e = 0; e < 2 * C::NT; ++e) v[0][e] *= fast_rcp(la + lc[C::SCALE ? e : 0]);
          }
          emit(a, v[0]);
        }
      } else if (C::CS == 1) {  // outputs in eigen order [even (he) | odd (ho)]
        if (a < he) emit(a, v[0]);
        if (a < ho) emit(he + a, v[C::NH - 1]);
      } else {  // z[a] = p + q, z[n-1-a] = p - q (a < ho); z[h] = p (middle row, n odd)
        if (a < ho) {
          double s[2 * C::NT], t[2 * C::NT];
#pragma unroll
          for (int e = 0; e < 2 * C::NT; ++e) {
            s[e] = v[0][e] + v[C::NH - 1][e];
            t[e] = v[0][e] - v[C::NH - 1][e];
          }
          emit(a, s);
          emit(n - 1 - a, t);
        } else if (a < he) {
          emit(a, v[0]);
        }
      }
    }
    if constexpr (C::TR > 0) {
      // quad reduction over kq: every lane of quad nq then holds rows 8 MTD + {0, 1} of both
      // halves at the quad's NT columns c0 .. c0 + NT - 1 (the B-fragment columns); lane kq
      // stores one (half / sign th, row ti) combination
#pragma unroll
      for (int hf = 0; hf < C::NH; ++hf)
#pragma unroll
        for (int i = 0; i < C::TR; ++i)
#pragma unroll
          for (int j = 0; j < C::NT; ++j) {
            double t = tl[hf][i][j];
            t += __shfl_xor_sync(0xffffffffu, t, 1);
            t += __shfl_xor_sync(0xffffffffu, t, 2);
            tl[hf][i][j] = t;
          }
      const int ti = kq & 1, th = kq >> 1;
      const int a = 8 * C::MTD + ti;
      double tv[C::NT];
      int row = a;
      bool ok;
      if (C::CS == 1) {  // [even (he) | odd (ho)]
#pragma unroll
        for (int j = 0; j < C::NT; ++j)
          tv[j] = th ? (ti ? tl[C::NH - 1][1][j] : tl[C::NH - 1][0][j]) : (ti ? tl[0][1][j] : tl[0][0][j]);
        row = th ? he + a : a;
        ok = a < (th ? ho : he);
      } else {  // z[a] = p + q, z[n-1-a] = p - q (a < ho); z[a] = p (middle row, n odd)
#pragma unroll
        for (int j = 0; j < C::NT; ++j) {
          const double pv = ti ? tl[0][1][j] : tl[0][0][j];
          const double qv = ti ? tl[C::NH - 1][1][j] : tl[C::NH - 1][0][j];
          tv[j] = th ? pv - qv : pv + qv;
        }
        row = th ? n - 1 - a : a;
        ok = a < ho || (a < he && th == 0);
      }
      const uint32_t c0 = tile * C::TW + C::NT * nq;
      if (ok) {
        if (C::MODE1) {
#pragma unroll
          for (int j = 0; j < C::NT; ++j)
            if (c0 + j < ncols) args.Y[size_t(c0 + j) * n + row] = tv[j];
        } else if (C::FAST) {
          if (c0 < ncols) {
            const uint32_t p = c0 / Q, qq = c0 - p * Q;
            double* o = args.Y + (size_t(p) * n + row) * Q + qq;
            if constexpr (C::NT == 1) {
              o[0] = tv[0];
            } else {
#pragma unroll
              for (int j = 0; j < C::NT; j += 2)
                *reinterpret_cast<double2*>(o + j) = make_double2(tv[j], tv[j + 1 < C::NT ? j + 1 : j]);
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < C::NT; ++j) {
            const uint32_t c = c0 + j;
            if (c < ncols) {
              const uint32_t p = c / Q, qq = c - p * Q;
              args.Y[(size_t(p) * n + row) * Q + qq] = tv[j];
            }
          }
        }
      }
    }
    cur = nxt;
  }
}

}  // namespace ls
