// Matrix-free y = A x (eq:A_kron, PAPER.md 686-703), v3: the banded univariate
// products on the FP64 tensor pipe (DMMA.8x8x4), one streaming pass per direction.
//
// Order of the passes (the triple recursion of matvec2_kernels.cuh):
//     time:         Kx = K_t x,  Mx = M_t x
//     direction d:  A = M Kx + J Mx (+ K xT),  B = M Mx,  C = 2K Mx (+ M xT)
//                   (xT = x on the last time slice: the W_t = e e^T term)
//     directions d-1 .. 2:  A <- M A + J B + K C,  B <- M B,  C <- 2K B + M C
//     direction 1:  y = M A + J B + K C
// (d = 1: the direction-d pass writes y = A.)
//
// Band product as DMMA.  A pass computes Y = W X along its direction for band
// matrices W of half-bandwidth P: the 8 output rows of m-tile mt need input rows
// [8mt + S0 - P, 8mt + S0 + 7 + P] (S0 = (P mod 4) - 8 or 0 aligns that band on a
// k-step), i.e. the NKB = 2 + ceil(P/2) k-steps 2mt - OFF .. 2mt - OFF + NKB - 1.  The band blocks are
// precomputed on the host in m8n8k4 A-fragment order ([mat][mt][j][lane]) and
// staged in shared memory once per CTA.  A warp owns a strip of 8*NT columns and
// sweeps it top to bottom: B fragments (4 rows x 8 columns per k-step) come from
// global memory into a register ring of RING = NKB + 4 k-steps, refilled two
// m-tiles ahead (the m-tile loop is unrolled by RING/2 so ring slots are static);
// each m-tile's accumulators are complete after its NKB k-steps and are stored
// at once, so only one m-tile of accumulators is live.  Column permutation as in
// fd_rd_kernel.cuh: lane l holds columns NT*(l/4) .. +NT-1 for its B loads
// (LDG.128 when FAST) and columns 2NT*(l%4) .. +2NT-1 for its stores.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"  // dmma_8x8x4

namespace ls {

enum MV3Kind { MV3_TIME = 0, MV3_DIR = 1, MV3_DIR_A = 2, MV3_MID = 3, MV3_LAST = 4, MV3_D3 = 5, MV3_T2 = 6 };
// v4 order (mv4_kernels.cuh: the plane pass of directions 1 + 2 comes first):
//   MV3_D3 (direction 3): in (P_M, P_K, P_J) -> v1 = M P_M, v2 = J P_M + M P_J + 2K P_K, and on
//                         the last time slice v3 = K P_M + M P_K (one slice, into a.v3)
//   MV3_T2 (time):        in (v1, v2) -> y = K_t v1 + M_t v2 (+ v3 on the last time row: W_t)
template <int KIND>
struct MV3IsTime {
  static constexpr bool v = KIND == MV3_TIME || KIND == MV3_T2;
};

struct MV3Args {
  const double* frag;  // [nmat][MT][NKB][32] band A-fragments of this pass' direction
  const double* in[3];
  double* out[3];
  const double* xT;    // MV3_DIR*: x of the last time slice, same [n][Q] layout as one slice
  int n;               // extent of the pass direction (band rows)
  int mt;              // m-tiles = ceil(n / 8)
  int nmat;
  uint32_t Q;          // row stride (product of the faster extents; 1 = contiguous mode)
  uint32_t ncols;      // columns = P_slow * Q
  int tT;              // MV3_DIR*: index of the last time slice among the P_slow slices (or -1)
  // time pass with a halo-extended input: input rows [s_first, s_first + s_rows) of the
  // band, output rows [t_first, t_first + nout)
  int s_first, s_rows, t_first, nout;
  int mt0, mt1;        // m-tile range swept (time pass: the tiles covering the output rows)
  // layouts: the intermediates use rows of n1p >= n1 doubles (n1p % 8 == 0: 64-byte rows)
  uint32_t Qout;       // output row stride of strided passes (0: = Q)
  int map_n1, map_n1p; // time pass: padded column c' -> input column (c'/n1p)*n1 + c'%n1p (0: identity)
  int in_fiber, out_fiber;  // contiguous (MODE1) passes: fibre strides of input / output
  double* v3;          // MV3_D3: output slice of the last time slice's v3 ([n][Q]); MV3_T2: input v3 ([Q])
  // MV3_T2 only: fused PCG scalar p.q (SURVEY 3 pcg_solve) -- when dotp != nullptr every stored
  // y element is multiplied by dotp at the same offset and the CTA's sum is written to
  // dot_part[blockIdx.x] (fixed grid: deterministic)
  const double* dotp;
  double* dot_part;
};

template <int KIND>
struct MV3IO {
  // ring inputs (the xT input of the direction-d pass is loaded without the ring: only
  // the warps holding last-slice columns need it)
  static constexpr int NIN = (KIND == MV3_TIME) ? 1 : (KIND == MV3_DIR || KIND == MV3_DIR_A || KIND == MV3_T2) ? 2 : 3;
  static constexpr int NOUT = (KIND == MV3_TIME || KIND == MV3_D3) ? 2 : (KIND == MV3_DIR || KIND == MV3_MID) ? 3 : 1;
  static constexpr int NMAT = (KIND == MV3_TIME || KIND == MV3_T2) ? 2 : (KIND == MV3_LAST) ? 3 : 4;
};

template <int P, int KIND>
struct MV3Geom {
  // m-tile mt covers output rows [8mt + S0, 8mt + S0 + 8) with S0 = (P mod 4) - 8 (or 0):
  // its input band [8mt + S0 - P, 8mt + S0 + 7 + P] then starts on a k-step boundary, so
  // it spans NKB = 2 + ceil(P/2) k-steps (p = 6: 5 instead of 6 for tiles at 8mt)
  static constexpr int S0 = (P % 4) ? (P % 4) - 8 : 0;
  static constexpr int OFF = (P - S0) / 4;  // first k-step of m-tile mt: 2mt - OFF
  static constexpr int NKB = 2 + (P + 1) / 2;
  // prefetch depth (m-tiles ahead) by register budget: 4 for 1 ring input, 2 for 2 (the
  // 2-input pass runs 2 CTAs per SM within 128 registers), 3 for 3 inputs up to p = 6 and
  // 2 above (tools/mv3_ab.sh: config 4 11.96 -> 11.87 ms, config 5 p = 4 3.43 -> 3.34 ms;
  // p = 8 is 0.8 % slower at depth 3)
#ifndef MV3_AHEAD1
#define MV3_AHEAD1 4
#endif
#ifndef MV3_AHEAD2
#define MV3_AHEAD2 1
#endif
#ifndef MV3_AHEAD3
#define MV3_AHEAD3 4
#endif
#ifndef MV3_AHEAD3_HI
#define MV3_AHEAD3_HI 2
#endif
// v4 time pass (two ring inputs, 2 CTAs per SM): depth 2 (r02 end, tools/ab_mv.py, two A/B
// pairs: config 4 matvec 10.18 -> 10.08 ms, config 5 p = 8 3.742 -> 3.701 ms against depth 3,
// which spilled 48 B at 128 registers; 4 / 5 spill more; one CTA with depth 6 / 9: 10.57 /
// 10.59 ms)
#ifndef MV3_AHEAD_T2
#define MV3_AHEAD_T2 2
#endif
  static constexpr int AHEAD = KIND == MV3_T2 ? MV3_AHEAD_T2
                               : MV3IO<KIND>::NIN == 1 ? MV3_AHEAD1
                               : MV3IO<KIND>::NIN == 2 ? MV3_AHEAD2
                               : (P <= 6 ? MV3_AHEAD3 : MV3_AHEAD3_HI);
  static constexpr int RING = NKB + 2 * AHEAD + (NKB & 1);  // even: static slots per RING/2 m-tiles
  static constexpr int G = RING / 2;  // m-tiles per unrolled group
};

#ifndef LS_MV3_L2PF
#define LS_MV3_L2PF ""  // L2 prefetch-size qualifier of the band-pass loads (experiment knob)
#endif
__device__ __forceinline__ double mv3_ld(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate" LS_MV3_L2PF ".f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 mv3_ld2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate" LS_MV3_L2PF ".v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// two CTAs per SM for the one- and two-input passes (latency hiding; <= 128 registers)
template <int KIND>
struct MV3Occ {
#ifndef MV3_DIR_CTAS
#define MV3_DIR_CTAS 2
#endif
#ifndef MV3_TIME_CTAS
#define MV3_TIME_CTAS 2
#endif
#ifndef MV3_MID_CTAS
#define MV3_MID_CTAS 1
#endif
  static constexpr int CTAS = (KIND == MV3_TIME) ? MV3_TIME_CTAS
                              : (KIND == MV3_DIR || KIND == MV3_DIR_A || KIND == MV3_T2) ? MV3_DIR_CTAS
                                                                                         : MV3_MID_CTAS;
};

// independent accumulator chains (MV3_SPLIT): the direction-3 pass' v2 = J P_M + M P_J + 2K P_K
// and the time pass' y = K_t v1 + M_t v2 accumulate one product per chain, summed in a fixed
// order before the store, instead of one dependent DMMA chain of 3 NKB / 2 NKB links
#ifndef MV3_SPLIT
#define MV3_SPLIT 0
#endif
template <int KIND>
struct MV3Extra {
  static constexpr int NX = !MV3_SPLIT ? 0 : KIND == MV3_D3 ? 2 : (KIND == MV3_T2 && MV3_SPLIT == 1) ? 1 : 0;
};

template <int P, int NT, int KIND, bool MODE1, bool FAST>
__global__ void __launch_bounds__(256, MV3Occ<KIND>::CTAS) mv3_band_kernel(const __grid_constant__ MV3Args a) {
  pdl_wait();
  using Gm = MV3Geom<P, KIND>;
  using IO = MV3IO<KIND>;
  constexpr int NKB = Gm::NKB, OFF = Gm::OFF, RING = Gm::RING, G = Gm::G;
  constexpr int NIN = IO::NIN, NOUT = IO::NOUT;
  constexpr int TW = 8 * NT;
  extern __shared__ __align__(16) double fsm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, nq = lane >> 2;
  const int MT = a.mt;
  const int nfrag = IO::NMAT * MT * NKB * 32;
  for (int e = tid; e < nfrag; e += 256) fsm[e] = __ldg(a.frag + e);
  __syncthreads();
  const int n = a.n;
  const uint32_t Q = a.Q, ncols = a.ncols;
  const uint32_t Qo = a.Qout ? a.Qout : a.Q;
  const uint32_t nstrips = (ncols + TW - 1) / TW;
  // time pass: band row of stored input row 0 / of output row 0
  constexpr bool TPASS = MV3IsTime<KIND>::v;
  const int gin0 = TPASS ? a.s_first : 0;
  const int in_rows = TPASS ? a.s_rows : n;
  const int gout0 = TPASS ? a.t_first : 0;
  const int nout = TPASS ? a.nout : n;
  const size_t rstride = MODE1 ? 1 : size_t(Q);

  double dacc = 0.0;  // MV3_T2: fused p.q of this thread
  for (uint32_t strip = blockIdx.x * 8 + warp; strip < nstrips; strip += gridDim.x * 8) {
    // ---- this lane's B columns (NT) and store columns (2NT)
    const uint32_t cb = strip * TW + NT * nq;  // first B column
    uint32_t boff[NT];  // element offset of (row 0, column) per B column
    uint32_t bmask = 0;
    bool is_last = false;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const uint32_t c = cb + j;
      boff[j] = 0;
      if (c < ncols) {
        bmask |= 1u << j;
        // the time pass has one column per (padded) spatial index: no slow index
        const uint32_t pt = TPASS ? 0u : c / Q, q = c - pt * Q;
        if (MODE1) {
          boff[j] = c * uint32_t(a.in_fiber);
        } else if (KIND == MV3_TIME && a.map_n1) {  // padded column -> unpadded input column
          const uint32_t r = q % uint32_t(a.map_n1p);
          boff[j] = (q / uint32_t(a.map_n1p)) * uint32_t(a.map_n1) + r;
          if (r >= uint32_t(a.map_n1)) bmask &= ~(1u << j);
        } else {
          boff[j] = pt * uint32_t(in_rows) * Q + q;
        }
        if (KIND == MV3_DIR || KIND == MV3_DIR_A || KIND == MV3_D3) is_last |= int(pt) == a.tT;
      }
    }
    // W_t term: only warps holding a column of the last time slice do the xT products
    const bool warp_last = (KIND == MV3_DIR || KIND == MV3_DIR_A || KIND == MV3_D3) && __any_sync(0xffffffffu, is_last);
    // B fragment of input m, k-step ks (rows 4ks + kq) -> v[NT]
    auto loadB = [&](double (&v)[NT], int m, int ks) {
      const int row = 4 * ks + kq;           // band row
      const int sr = row - gin0;              // stored row
      const bool rok = row >= 0 && row < n && sr >= 0 && sr < in_rows;
      const double* src = (m == 2 && (KIND == MV3_DIR || KIND == MV3_DIR_A)) ? a.xT : a.in[m];
      if (FAST) {
        const bool ok = rok && bmask && (m != 2 || (KIND != MV3_DIR && KIND != MV3_DIR_A) || is_last);
        const size_t off = (m == 2 && (KIND == MV3_DIR || KIND == MV3_DIR_A))
                               ? size_t(boff[0] % Q)  // xT is one slice: (row, q)
                               : size_t(boff[0]);
        if (NT == 1) {
          v[0] = ok ? mv3_ld(src + off + size_t(sr) * rstride) : 0.0;
        } else {
#pragma unroll
          for (int j = 0; j + 1 < NT; j += 2) {
            double2 t = make_double2(0.0, 0.0);
            if (ok) t = mv3_ld2(src + off + size_t(sr) * rstride + j);
            v[j] = t.x;
            v[j + 1] = t.y;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          bool ok = rok && ((bmask >> j) & 1u);
          size_t off = boff[j];
          if (m == 2 && (KIND == MV3_DIR || KIND == MV3_DIR_A)) {
            const uint32_t c = cb + j;
            const uint32_t pt = c / Q;
            ok = ok && int(pt) == a.tT;
            off = c - pt * Q;
          }
          v[j] = ok ? mv3_ld(src + off + size_t(sr) * rstride) : 0.0;
        }
      }
    };
    double ring[NIN][RING][NT];
    // prologue: k-steps 2 mt0 - OFF + s into slots s = 0 .. RING-1
    const int mt0 = a.mt0, mt1 = a.mt1;
#pragma unroll
    for (int m = 0; m < NIN; ++m)
#pragma unroll
      for (int s = 0; s < RING; ++s) loadB(ring[m][s], m, 2 * mt0 - OFF + s);

    const uint32_t cs = strip * TW + 2 * NT * kq;  // first store column
    for (int g0 = mt0; g0 < mt1; g0 += G) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int mt = g0 + u;
        if (mt < mt1) {
          // MV3_T2 with the fused p.q: this m-tile's p values, loaded before its DMMAs so that
          // their latency overlaps them (as plain loads after the y stores they were exposed:
          // the time pass ran 2.5 instead of 1.6 ms at config 4)
          double pv[(KIND == MV3_T2 && FAST) ? 2 * NT : 1];
          if (KIND == MV3_T2 && FAST && a.dotp) {
            const int brow = 8 * mt + Gm::S0 + nq, lrow = brow - gout0;
            const bool ok = brow < n && lrow >= 0 && lrow < nout && cs < ncols;
            const uint32_t pt = cs / Qo, q = cs - pt * Qo;
            const double* src = a.dotp + (size_t(pt) * nout + (ok ? lrow : 0)) * Qo + q;
#pragma unroll
            for (int e = 0; e < 2 * NT; e += 2) {
              double2 t = make_double2(0.0, 0.0);
              if (ok) t = __ldg(reinterpret_cast<const double2*>(src + e));
              pv[e] = t.x;
              pv[e + 1] = t.y;
            }
          }
          constexpr int NX = MV3Extra<KIND>::NX;
          double acc[NOUT + NX][NT][2];
#pragma unroll
          for (int o = 0; o < NOUT + NX; ++o)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[o][j][0] = acc[o][j][1] = 0.0;
          double acc3[KIND == MV3_D3 ? NT : 1][2];  // MV3_D3: v3 of the last time slice
#pragma unroll
          for (int j = 0; j < (KIND == MV3_D3 ? NT : 1); ++j) acc3[j][0] = acc3[j][1] = 0.0;
          // sum over the NKB band k-steps: acc[o] += W_mat * ring[in]
#pragma unroll
          for (int jk = 0; jk < NKB; ++jk) {
            const int slot = (2 * u + jk) % RING;
            auto fr = [&](int mat) { return fsm[((mat * MT + mt) * NKB + jk) * 32 + lane]; };
            auto mma = [&](int o, int mat, int in) {
#pragma unroll
              for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[o][j], fr(mat), ring[in][slot][j]);
            };
            if (KIND == MV3_TIME) {          // mats: 0 K_t, 1 M_t
              mma(0, 0, 0);
              mma(1, 1, 0);
            } else if (KIND == MV3_DIR || KIND == MV3_DIR_A) {  // mats: 0 M, 1 J, 2 K, 3 2K; in: Kx, Mx
              mma(0, 0, 0);
              mma(0, 1, 1);
              if (KIND == MV3_DIR) {
                mma(1, 0, 1);
                mma(2, 3, 1);
              }
              if (warp_last) {  // W_t term: xT fragments loaded directly (rare warps)
                double xv[NT];
                loadB(xv, 2, 2 * mt - OFF + jk);
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[0][j], fr(2), xv[j]);
                if (KIND == MV3_DIR) {
#pragma unroll
                  for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[2][j], fr(0), xv[j]);
                }
              }
            } else if (KIND == MV3_D3) {     // mats: 0 M, 1 J, 2 K, 3 2K; in: P_M, P_K, P_J
              mma(0, 0, 0);
              mma(1, 1, 0);
              mma(NX ? NOUT : 1, 0, 2);
              mma(NX ? NOUT + 1 : 1, 3, 1);
              if (warp_last) {
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                  dmma_8x8x4(acc3[j], fr(2), ring[0][slot][j]);
                  dmma_8x8x4(acc3[j], fr(0), ring[1][slot][j]);
                }
              }
            } else if (KIND == MV3_T2) {     // mats: 0 K_t, 1 M_t; in: v1, v2
              mma(0, 0, 0);
              mma(NX ? NOUT : 0, 1, 1);
            } else if (KIND == MV3_MID) {    // mats: 0 M, 1 J, 2 K, 3 2K; in: A, B, C
              mma(0, 0, 0);
              mma(0, 1, 1);
              mma(0, 2, 2);
              mma(1, 0, 1);
              mma(2, 3, 1);
              mma(2, 0, 2);
            } else {                         // MV3_LAST, mats: 0 M, 1 J, 2 K
              mma(0, 0, 0);
              mma(0, 1, 1);
              mma(0, 2, 2);
            }
          }
          if (NX) {  // fold the extra chains: v2 = (J P_M + M P_J) + 2K P_K, y = K_t v1 + M_t v2
            constexpr int o0 = KIND == MV3_D3 ? 1 : 0;
#pragma unroll
            for (int j = 0; j < NT; ++j)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                acc[o0][j][h] += acc[NOUT][j][h];
                if (NX > 1) acc[o0][j][h] += acc[NOUT + (NX > 1 ? 1 : 0)][j][h];
              }
          }
          // refill the two consumed slots with k-steps two m-tiles ahead
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int slot = (2 * u + h) % RING;
            const int ks = 2 * (mt - mt0) - OFF + h + RING + 2 * mt0;
#pragma unroll
            for (int m = 0; m < NIN; ++m) loadB(ring[m][slot], m, ks);
          }
          // ---- store m-tile mt: rows 8mt + nq, columns cs .. cs + 2NT - 1
          const int brow = 8 * mt + Gm::S0 + nq;  // band row
          const int lrow = brow - gout0;          // local output row (time pass: slab rows)
          if (brow < n && lrow >= 0 && lrow < nout) {
            if (KIND == MV3_T2 && brow == n - 1) {  // W_t = e e^T: y_T += v3 (one slice, [Q])
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                  const uint32_t c = cs + NT * h + j;
                  if (c < ncols) acc[0][j][h] += a.v3[c];
                }
            }
            if (KIND == MV3_D3 && warp_last) {
#pragma unroll
              for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int j = 0; j < NT; ++j) {
                  const uint32_t c = cs + NT * h + j;
                  const uint32_t pt = c / Q;
                  if (c < ncols && int(pt) == a.tT) a.v3[size_t(lrow) * Q + (c - pt * Q)] = acc3[j][h];
                }
            }
#pragma unroll
            for (int o = 0; o < NOUT; ++o) {
              double* Y = a.out[o];
              if (FAST) {
                if (cs < ncols) {
                  const uint32_t pt = cs / Qo, q = cs - pt * Qo;
                  double* dst = Y + (size_t(pt) * nout + lrow) * Qo + q;
                  // accumulator column 2kq + h of n-tile j = physical column cs + NT*h + j
                  if (NT == 1) {  // physical columns cs, cs + 1 = accumulator columns 2kq, 2kq + 1
                    *reinterpret_cast<double2*>(dst) = make_double2(acc[o][0][0], acc[o][0][1]);
                    if (KIND == MV3_T2 && a.dotp) dacc = fma(acc[o][0][0], pv[0], fma(acc[o][0][1], pv[1], dacc));
                  } else {
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                      for (int j = 0; j + 1 < NT; j += 2) {
                        *reinterpret_cast<double2*>(dst + NT * h + j) = make_double2(acc[o][j][h], acc[o][j + 1][h]);
                        if (KIND == MV3_T2 && a.dotp)
                          dacc = fma(acc[o][j][h], pv[NT * h + j], fma(acc[o][j + 1][h], pv[NT * h + j + 1], dacc));
                      }
                  }
                }
              } else {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                  for (int j = 0; j < NT; ++j) {
                    const uint32_t c = cs + NT * h + j;
                    if (c < ncols) {
                      size_t o_off;
                      if (MODE1) {
                        o_off = size_t(c) * a.out_fiber + lrow;
                      } else {
                        const uint32_t pt = c / Qo, q = c - pt * Qo;
                        o_off = (size_t(pt) * nout + lrow) * Qo + q;
                      }
                      Y[o_off] = acc[o][j][h];
                      if (KIND == MV3_T2 && a.dotp) dacc = fma(acc[o][j][h], a.dotp[o_off], dacc);
                    }
                  }
              }
            }
          }
        }
      }
    }
  }
  if (KIND == MV3_T2 && a.dotp) {  // CTA sum of the fused p.q in a fixed order
    __shared__ double red[8];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) red[warp] = dacc;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) t += red[w];
      a.dot_part[blockIdx.x] = t;
    }
  }
}

// host-side launch (mv3.cu)
struct MV3Pass {
  MV3Args args;
  int kind;
  bool mode1;
  int p;  // degree of this pass' direction (time pass: p_t)
  unsigned grid = 0;  // set by mv3_run: the grid launched (number of dot_part entries)
};
// p: spline degree; returns the CUDA error; *launches += kernels launched
cudaError_t mv3_run(MV3Pass* passes, int npass, int num_sms, cudaStream_t s, int64_t* launches);
// dst[c'] = src[(c'/n1p)*n1 + c'%n1p] (0 in the padding) for one slice of Nsp padded columns
cudaError_t mv3_pad_slice(const double* src, double* dst, int64_t nsp, int n1, int n1p, cudaStream_t s,
                          int64_t* launches);
size_t mv3_frag_count(int p, int n, int nmat);  // doubles of one direction's fragment array
int mv3_nkb(int p);
int mv3_off(int p);
int mv3_s0(int p);          // band row of the first m-tile's row 0 (<= 0)
int mv3_mt(int p, int n);   // m-tiles covering [0, n)

// v4 plane pass (mv4_kernels.cuh / mv4.cu)
struct MV4PlaneArgs;
cudaError_t mv4_plane_run(const MV4PlaneArgs& a, int p, int num_sms, cudaStream_t s);
size_t mv4_plane_smem(int p, int mt2);

}  // namespace ls
