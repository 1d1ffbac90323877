// Matrix-free y = A x (eq:A_kron, PAPER.md 686-703), v4: the plane pass first.
//
// Order (d >= 2; directions 1 + 2 fused in one kernel, then direction 3 and time as
// single-direction DMMA band passes of matvec3_kernels.cuh, kinds MV3_D3 / MV3_T2):
//     plane (this file):  u_M = M_1 x, u_K = K_1 x, u_J = J_1 x                (direction 1)
//                         P_M = M_2 u_M, P_K = K_2 u_M + M_2 u_K,
//                         P_J = J_2 u_M + M_2 u_J + 2 K_2 u_K                    (direction 2)
//     direction 3:        v1 = M_3 P_M, v2 = J_3 P_M + M_3 P_J + 2 K_3 P_K, v3 = K_3 P_M + M_3 P_K
//     time:               y = K_t v1 + M_t v2 + W_t v3
// so that M_s = M_3 M_2 M_1 (v1), J_s = sum_k J_k(..) + 2 sum_{k<l} K_k K_l (v2), L_s = sum_k
// K_k(..) (v3); for d = 2 the time pass reads (P_M, P_J, P_K) directly.  HBM traffic: 8 + 24
// (plane) + 24 + 16 (direction 3) + 16 + 8 (time) = 96 B/DOF at d = 3 (v3: 144).
//
// Plane kernel.  A warp owns one column tile ct of direction 1 (output i_1 in [8ct + S0,
// 8ct + S0 + 8), the band geometry of matvec3_kernels.cuh) in one plane (t, i_3) and sweeps the
// direction-2 rows j in tiles of 8:
//   1. direction-1 DMMAs: u_X(i_1, j) = sum_l W1_X(i_1, l) x(j, l), A = the warp's band blocks of
//      M_1, K_1, J_1 (registers for the whole task), B = x rows (4 l x 8 j per k-step, global);
//      D fragments hold u_X(i_1 = lane/4, j = 2(lane%4) + {0,1});
//   2. quad shuffles turn them into direction-2 B fragments u_X(j = 4 ks + lane%4, i_1 = lane/4)
//      for the two k-steps of the tile, kept in a register ring;
//   3. once an output m-tile of direction 2 has all NKB k-steps in the ring, 6 DMMAs per k-step
//      (A = band blocks of M_2, K_2, J_2, 2K_2 staged in shared memory) give P_M, P_K, P_J,
//      stored at once.
// u never leaves the registers; x is read once from HBM (neighbouring column tiles re-read it
// from L1 / L2); P_* are written once.
//
// Packed direction 2 (LS_MV4_PACK): an 8-row band tile spans NKB k-steps, a 4-row one NKB - 1,
// so two matrices on the SAME 4 output rows share one DMMA tile with one k-step less per row
// (p = 6: 4 k-steps for 2 x 4 rows instead of 5 for 8).  With a = the tile's first output row,
// b = a + 4, and "X_a" the rows a .. a+3 of X, the six chains per output m-tile are
//     T1a = [M_a ; K_a] u_M    T2a = [2K_a ; M_a] u_K     (k-steps 0 .. NKB-2)
//     T1b = [K_b ; M_b] u_M    T2b = [M_b ; 2K_b] u_K     (k-steps 1 .. NKB-1)
//     Jt  = J u_M,  Mt = M u_J (plain 8-row tiles)
// and a lane of row r (D rows 0-3: lanes 0-15, rows 4-7: lanes 16-31) finds its outputs in the
// same registers in both halves: P_M(a + r) = T1a | T1b, P_J(a + r) = (T2a | T2b) + Jt + Mt,
// P_K(a + r + 4 | a + r - 4) = T1b + T2b | T1a + T2a.  26 instead of 30 DMMAs per m-tile at
// p = 6 (4 (NKB - 1) + 2 NKB vs 6 NKB).  The packed fragments are assembled in the prologue
// from the plain ones (same lane for the matrix in its own half, lane -+ 16 for the other).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"  // dmma_8x8x4
#include "pdl.cuh"

namespace ls {

struct MV4PlaneArgs {
  const double* x;      // [nplanes][n2][n1]
  double* out[3];       // P_M, P_K, P_J (same layout)
  const double* frag1;  // direction-1 band A-fragments [4: M, J, K, 2K][mt1][NKB][32]
  const double* frag2;  // direction-2 band A-fragments [4: M, J, K, 2K][mt2][NKB][32]
  int n1, n2, mt1, mt2;
  int64_t nplanes;
};

template <int P>
struct MV4Geom {
  static constexpr int S0 = (P % 4) ? (P % 4) - 8 : 0;
  static constexpr int OFF = (P - S0) / 4;
  static constexpr int NKB = 2 + (P + 1) / 2;
  // output m-tile mt2 = jt - LAG is complete after source row tile jt (k-steps 2jt, 2jt+1); the
  // kernel emits it one row tile later (software pipelining, see the loop)
  static constexpr int LAG0 = NKB - OFF - 2;
  static constexpr int LAG = LAG0 > 0 ? (LAG0 + 1) / 2 : 0;
  static constexpr int SPAN = 2 * LAG + OFF + 2;  // live k-steps
  static constexpr int G = (SPAN + 1) / 2;        // row tiles per unrolled group
  static constexpr int RING = 2 * G;
  static constexpr int JT0 = -((OFF + 1) / 2);    // first source row tile (k-step 2 JT0 <= -OFF)
};

#ifndef LS_MV4_PACK
#define LS_MV4_PACK 0
#endif
// shared memory of the plane kernel (doubles): plain [M, J, K, 2K] fragments, or packed:
// [M, J] plain + [T1a, T2a, T1b, T2b] x (NKB - 1) k-steps
template <int P, bool PACK>
constexpr size_t mv4_smem_doubles(int mt2) {
  return PACK ? size_t(mt2) * 32 * (2 * MV4Geom<P>::NKB + 4 * (MV4Geom<P>::NKB - 1))
              : size_t(4) * mt2 * MV4Geom<P>::NKB * 32;
}

#ifndef LS_MV4_L2PF
#define LS_MV4_L2PF ""  // L2 prefetch-size qualifier of the plane-pass loads (experiment knob)
#endif
__device__ __forceinline__ double mv4_ld(const double* p) {
  double v;
  asm volatile("ld.global.nc" LS_MV4_L2PF ".f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// CTAS = CTAs per SM the register budget is sized for (1: <= 255 registers, 2: <= 128)
// WARPS per CTA: 8, or 16 for the packed kernel in place of 2 CTAs of 8 (one shared copy of the
// fragments, which no longer fit twice per SM at p = 6, n = 132)
template <int P, int CTAS, bool PACK = false, int WARPS = 8>
__global__ void __launch_bounds__(32 * WARPS, CTAS) mv4_plane_kernel(const __grid_constant__ MV4PlaneArgs a) {
  using Gm = MV4Geom<P>;
  constexpr int NKB = Gm::NKB, OFF = Gm::OFF, S0 = Gm::S0, LAG = Gm::LAG, G = Gm::G, RING = Gm::RING;
  constexpr int JT0 = Gm::JT0;
  constexpr int KP = NKB - 1;  // k-steps of a packed 4-row tile
  extern __shared__ __align__(16) double fsm[];  // frag2: 4 plain matrices, or 2 plain + 4 packed
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = lane & 3, r = lane >> 2;
  const int MT1 = a.mt1, MT2 = a.mt2, n1 = a.n1, n2 = a.n2;
  if (!PACK) {
    const int nf = 4 * MT2 * NKB * 32;
    for (int e = tid; e < nf; e += 32 * WARPS) fsm[e] = __ldg(a.frag2 + e);
  } else {
    // plain M (mat 0) and J (mat 1) as they are, then the packed tiles [4][MT2][KP][32]
    const int nf = 2 * MT2 * NKB * 32;
    for (int e = tid; e < nf; e += 32 * WARPS) fsm[e] = __ldg(a.frag2 + e);
    const int mstride = MT2 * NKB * 32;  // frag2 matrices: 0 M, 1 J, 2 K, 3 2K
    const int np = 4 * MT2 * KP * 32;
    for (int e = tid; e < np; e += 32 * WARPS) {
      const int l = e & 31, jp = (e >> 5) % KP, mt = (e >> 5) / KP % MT2, t = (e >> 5) / (KP * MT2);
      const bool top = l < 16;  // D rows 0-3 of the packed tile
      int mat, src_l, jk;
      switch (t) {
        case 0: mat = top ? 0 : 2; src_l = top ? l : l - 16; jk = jp; break;      // T1a = [M_a ; K_a]
        case 1: mat = top ? 3 : 0; src_l = top ? l : l - 16; jk = jp; break;      // T2a = [2K_a ; M_a]
        case 2: mat = top ? 2 : 0; src_l = top ? l + 16 : l; jk = jp + 1; break;  // T1b = [K_b ; M_b]
        default: mat = top ? 0 : 3; src_l = top ? l + 16 : l; jk = jp + 1; break; // T2b = [M_b ; 2K_b]
      }
      fsm[nf + e] = __ldg(a.frag2 + mat * mstride + (mt * NKB + jk) * 32 + src_l);
    }
  }
  __syncthreads();
  pdl_wait();
  const int64_t ntasks = a.nplanes * MT1;
  const int64_t plane_sz = int64_t(n1) * n2;
  const int sh_lo = (lane & ~3) | (q >> 1), sh_hi = (lane & ~3) | (2 + (q >> 1));
  const bool odd = q & 1;
  for (int64_t task = int64_t(blockIdx.x) * WARPS + warp; task < ntasks; task += int64_t(gridDim.x) * WARPS) {
    const int64_t plane = task / MT1;
    const int ct = int(task - plane * MT1);
    const double* X = a.x + plane * plane_sz;
    // direction-1 band blocks of the warp's column tile: M, K, J (frag mats 0, 2, 1)
    double A1[3][NKB];
#pragma unroll
    for (int jk = 0; jk < NKB; ++jk) {
      A1[0][jk] = __ldg(a.frag1 + ((0 * MT1 + ct) * NKB + jk) * 32 + lane);
      A1[1][jk] = __ldg(a.frag1 + ((2 * MT1 + ct) * NKB + jk) * 32 + lane);
      A1[2][jk] = __ldg(a.frag1 + ((1 * MT1 + ct) * NKB + jk) * 32 + lane);
    }
    // this lane's source columns l = 4 (2 ct - OFF + jk) + q and their validity
    int lcol[NKB];
    unsigned lmask = 0;
#pragma unroll
    for (int jk = 0; jk < NKB; ++jk) {
      lcol[jk] = 4 * (2 * ct - OFF + jk) + q;
      if (lcol[jk] >= 0 && lcol[jk] < n1) lmask |= 1u << jk;
    }
    auto loadx = [&](double (&v)[NKB], int jt) {
      const int j = 8 * jt + r;
      const bool rok = j >= 0 && j < n2;
#pragma unroll
      for (int jk = 0; jk < NKB; ++jk)
        v[jk] = (rok && ((lmask >> jk) & 1u)) ? mv4_ld(X + int64_t(j) * n1 + lcol[jk]) : 0.0;
    };
    double ring[3][RING];
#pragma unroll
    for (int m = 0; m < 3; ++m)
#pragma unroll
      for (int s = 0; s < RING; ++s) ring[m][s] = 0.0;
    double xb[NKB];
    loadx(xb, JT0);
    const int JT1 = MT2 + LAG + 1;  // source row tiles JT0 .. JT1 - 1
    const int i1 = 8 * ct + S0 + 2 * q;  // store columns i1, i1 + 1
    for (int g0 = JT0; g0 < JT1; g0 += G) {
#pragma unroll
      for (int u = 0; u < G; ++u) {
        const int jt = g0 + u;
        if (jt < JT1) {
          double xn[NKB];
          loadx(xn, jt + 1);  // prefetch the next row tile
          double uu[3][2];
#pragma unroll
          for (int m = 0; m < 3; ++m) uu[m][0] = uu[m][1] = 0.0;
          if (jt >= 0 && 8 * jt < n2) {  // row tiles outside the plane contribute zeros
#pragma unroll
            for (int jk = 0; jk < NKB; ++jk)
#pragma unroll
              for (int m = 0; m < 3; ++m) dmma_8x8x4(uu[m], A1[m][jk], xb[jk]);
          }
          // output m-tile of the PREVIOUS row tile (one extra step of lag): its DMMAs are
          // independent of this tile's direction-1 DMMAs, which stay in flight meanwhile
          const int mt2 = jt - 1 - LAG;
          if (PACK && mt2 >= 0) {
            double t1a[2] = {0.0, 0.0}, t2a[2] = {0.0, 0.0}, t1b[2] = {0.0, 0.0}, t2b[2] = {0.0, 0.0};
            double jt_[2] = {0.0, 0.0}, mt_[2] = {0.0, 0.0};
            const double* fp = fsm + 2 * MT2 * NKB * 32 + mt2 * KP * 32 + lane;  // packed tile 0
            constexpr int PS = 0;  // (packed tile stride MT2 * KP * 32 is run-time)
            const int pst = MT2 * KP * 32;
#pragma unroll
            for (int jk = 0; jk < NKB; ++jk) {
              constexpr int base = RING * 8;
              const int slot = (base + 2 * u - 2 - 2 * LAG - OFF + jk) % RING;
              const double* f = fsm + (mt2 * NKB + jk) * 32 + lane;
              const double fM = f[0], fJ = f[MT2 * NKB * 32];
              const double bM = ring[0][slot], bK = ring[1][slot], bJ = ring[2][slot];
              dmma_8x8x4(jt_, fJ, bM);
              dmma_8x8x4(mt_, fM, bJ);
              if (jk < KP) {
                dmma_8x8x4(t1a, fp[PS + jk * 32], bM);
                dmma_8x8x4(t2a, fp[pst + jk * 32], bK);
              }
              if (jk >= 1) {
                dmma_8x8x4(t1b, fp[2 * pst + (jk - 1) * 32], bM);
                dmma_8x8x4(t2b, fp[3 * pst + (jk - 1) * 32], bK);
              }
            }
            const bool lo = lane < 16;
            const int i2 = 8 * mt2 + S0 + r;               // P_M, P_J row
            const int i2k = lo ? i2 + 4 : i2 - 4;          // P_K row
            double pm[2], pk[2], pj[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              pm[h] = lo ? t1a[h] : t1b[h];
              pk[h] = lo ? t1b[h] + t2b[h] : t1a[h] + t2a[h];
              pj[h] = (lo ? t2a[h] : t2b[h]) + jt_[h] + mt_[h];
            }
            const int64_t ob = plane * plane_sz + i1;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (i1 + h >= 0 && i1 + h < n1) {
                if (i2 >= 0 && i2 < n2) {
                  a.out[0][ob + int64_t(i2) * n1 + h] = pm[h];
                  a.out[2][ob + int64_t(i2) * n1 + h] = pj[h];
                }
                if (i2k >= 0 && i2k < n2) a.out[1][ob + int64_t(i2k) * n1 + h] = pk[h];
              }
            }
          }
          if (!PACK && mt2 >= 0) {
            // six independent accumulator chains (P_K, P_J summed at the end)
            double pm[2] = {0.0, 0.0}, pk[2] = {0.0, 0.0}, pj[2] = {0.0, 0.0};
            double pk1[2] = {0.0, 0.0}, pj1[2] = {0.0, 0.0}, pj2[2] = {0.0, 0.0};
#pragma unroll
            for (int jk = 0; jk < NKB; ++jk) {
              constexpr int base = RING * 8;  // keep the slot index non-negative
              const int slot = (base + 2 * u - 2 - 2 * LAG - OFF + jk) % RING;
              const double* f = fsm + (mt2 * NKB + jk) * 32 + lane;
              const double fM = f[0], fJ = f[MT2 * NKB * 32], fK = f[2 * MT2 * NKB * 32],
                           f2K = f[3 * MT2 * NKB * 32];
              const double bM = ring[0][slot], bK = ring[1][slot], bJ = ring[2][slot];
              dmma_8x8x4(pm, fM, bM);
              dmma_8x8x4(pk, fK, bM);
              dmma_8x8x4(pj, fJ, bM);
              dmma_8x8x4(pk1, fM, bK);
              dmma_8x8x4(pj1, fM, bJ);
              dmma_8x8x4(pj2, f2K, bK);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              pk[h] += pk1[h];
              pj[h] += pj1[h] + pj2[h];
            }
            const int i2 = 8 * mt2 + S0 + r;
            if (i2 >= 0 && i2 < n2) {
              const int64_t o = plane * plane_sz + int64_t(i2) * n1 + i1;
              if (i1 >= 0 && i1 < n1) {
                a.out[0][o] = pm[0];
                a.out[1][o] = pk[0];
                a.out[2][o] = pj[0];
              }
              if (i1 + 1 >= 0 && i1 + 1 < n1) {
                a.out[0][o + 1] = pm[1];
                a.out[1][o + 1] = pk[1];
                a.out[2][o + 1] = pj[1];
              }
            }
          }
          // D (i1 = r, j = 2q + {0,1}) -> B fragments of k-steps 2jt (j = q) and 2jt + 1 (j = 4 + q)
#pragma unroll
          for (int m = 0; m < 3; ++m) {
            const double a0 = __shfl_sync(0xffffffffu, uu[m][0], sh_lo);
            const double a1 = __shfl_sync(0xffffffffu, uu[m][1], sh_lo);
            const double c0 = __shfl_sync(0xffffffffu, uu[m][0], sh_hi);
            const double c1 = __shfl_sync(0xffffffffu, uu[m][1], sh_hi);
            ring[m][(2 * u) % RING] = odd ? a1 : a0;
            ring[m][(2 * u + 1) % RING] = odd ? c1 : c0;
          }
#pragma unroll
          for (int jk = 0; jk < NKB; ++jk) xb[jk] = xn[jk];
        }
      }
    }
  }
}

}  // namespace ls
