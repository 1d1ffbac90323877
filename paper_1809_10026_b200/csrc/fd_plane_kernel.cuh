// Spatial mode products of directions 1 AND 2 in one kernel (Algorithm 1 steps 2 and 4,
// PAPER.md 959-962), centrosymmetric split (fd_rd_kernel.cuh "CS", reading c25), for a
// square plane n1 = n2 = n with the same eigenbasis A = [A_e | A_o] in both directions:
//   forward  (FWD):  Y[k2][k1] = sum_{i2,i1} U^T[k2][i2] U^T[k1][i1] X[i2][i1]
//   backward (!FWD): Z[i2][i1] = sum_{j2,j1} U[i2][j2]  U[i1][j1]  Y[j2][j1]
// on every plane (i2, i1) of the tensor (planes = the slower indices (i3, .., t)).  The
// intermediate of the two mode products never leaves the registers, so the pair costs one
// HBM round trip (16 B/DOF) instead of two.
//
// Work: one CTA per plane (persistent over planes), warp w = one (even, odd) pair of 8-row
// m-tiles of the FIRST product, which contracts direction 2 (the plane's rows):
//   C1[hf][m][c] = sum_k W_hf[m][k] B_hf[k][c],  m = output index of direction 2 (half hf),
//   columns c = direction-1 indices (all of them, NT n-tiles per warp).
// The rows stream through a shared-memory ring of 16-row blocks (cp.async, zero-filled where
// a row does not exist; row stride S = 4 mod 16 doubles: conflict-free B-fragment reads);
// the W fragments of both products sit in shared memory.  Forward: the fold of direction 2
// happens at the B read (rows k and n-1-k of a block: x + Rx, x - Rx); backward: the even
// and odd input rows (j2 < he, he + j2) are read directly.
// SECOND product (direction 1), straight from the registers: a C fragment of the first
// product (lane (r, c): row m = r, columns 2c, 2c+1 of an n-tile) IS a B fragment of the
// second (B[k = c][n = r] of k-step h = column 2c + h), so the second product contracts the
// columns with A = W1 fragments whose k order is j = 8q + 2c + h.  Forward: the fold of
// direction 1 is a register add / subtract of an n-tile and its mirror n-tile (the first
// product's columns are laid out as [i1 = 8q + r | i1 = n-1-(8q + r) | middle]); backward:
// the columns are [even j1 | odd j1], the unfold butterflies of both directions happen at
// the stores (z[a] = p + q, z[n-1-a] = p - q).
// Sizes: he = ceil(n/2) <= 4 KS, ho = floor(n/2) <= 8 NTH, MID = n odd.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_rd_kernel.cuh"  // dmma_8x8x4, pdl_wait

namespace ls {

struct PLArgs {
  const double* X;
  double* Y;
  const double* W2;  // first product (direction 2): forward [A_e^T | A_o^T], backward [A_e | A_o] (row-major halves)
  const double* W1;  // second product (direction 1): same matrices (isotropic plane)
  int n;
  uint32_t planes;
};

template <int KS_, int NTH_, int MID_, bool FWD_, int MINB_, int KB_ = 4>
struct PLCfg {
  static constexpr int KS = KS_, NTH = NTH_, MID = MID_, MINB = MINB_, KB = KB_;
  static constexpr bool FWD = FWD_;
  static constexpr int MT = (KS + 1) / 2;   // m-tile pairs of the first product = warps
  static constexpr int KSP = (KS + 1) / 2;  // k-step pairs (W2 fragments)
  static constexpr int NB = (KS + KB - 1) / KB;  // ring blocks per plane (KB k-steps each)
  static constexpr int NT = 2 * NTH + MID;  // first-product n-tiles (direction-1 columns)
  static constexpr int NQE = NTH + MID;     // second product: k-step pairs, even half
  static constexpr int NQ = NTH + MID;      // (odd half: NTH)
  static constexpr int WARPS = MT, THREADS = 32 * MT;
  static constexpr int NSTAGE = 3;
  static constexpr int NMAX = (8 * KS < 16 * NTH + MID) ? 8 * KS : 16 * NTH + MID;  // largest n of the bucket
  static constexpr int S = pad4mod16(NMAX);  // ring row stride (doubles)
  static constexpr int HR = 4 * KB;          // half-rows per ring block
  static constexpr int W2H = MT * KSP * 64;  // one half, rd A-fragment order
  static constexpr int W1H = MT * NQ * 64;   // one half, [mt][q][lane][h]
  static constexpr int WN = 2 * W2H + 2 * W1H;
  static constexpr size_t SMEM = size_t(WN + NSTAGE * 2 * HR * S) * sizeof(double);
  static_assert(KB % 2 == 0 && THREADS % HR == 0, "ring block shape");
  static_assert(SMEM <= 232448, "shared memory budget");
};

// cp.async with zero fill (src-size 0 when !ok: the slot row of a missing half-row is zero)
__device__ __forceinline__ void cp_async8z(void* smem, const void* gmem, bool ok) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, bool ok) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 16 : 0));
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB) fd_plane_kernel(PLArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* w2 = smem;               // [hf][mt][ksp][lane][2]
  double* w1 = smem + 2 * C::W2H;  // [hf][mt1][q][lane][2]
  double* ring = w1 + 2 * C::W1H;  // [NSTAGE][2 HR][S]
  const int tid = threadIdx.x, lane = tid & 31, mt = tid >> 5;
  const int c = lane & 3, r = lane >> 2;
  const int n = a.n, he = (n + 1) / 2, ho = n / 2;
  constexpr int S = C::S;

  // ---- W fragments -> shared memory
  for (int e = tid; e < 2 * C::W2H; e += C::THREADS) {
    const int hf = e / C::W2H, e1 = e - hf * C::W2H;
    const int h = e1 & 1, l = (e1 >> 1) & 31, ksp = (e1 >> 6) % C::KSP, m = (e1 >> 6) / C::KSP;
    const int row = m * 8 + (l >> 2), col = (2 * ksp + h) * 4 + (l & 3);
    const int nh = hf ? ho : he;
    const double* Wh = a.W2 + (hf ? size_t(he) * he : 0);
    w2[e] = (row < nh && col < nh) ? __ldg(Wh + size_t(row) * nh + col) : 0.0;
  }
  for (int e = tid; e < 2 * C::W1H; e += C::THREADS) {
    const int hf = e / C::W1H, e1 = e - hf * C::W1H;
    const int h = e1 & 1, l = (e1 >> 1) & 31, q = (e1 >> 6) % C::NQ, m = (e1 >> 6) / C::NQ;
    const int row = m * 8 + (l >> 2);
    const int nh = hf ? ho : he;
    int col = 8 * q + 2 * (l & 3) + h;
    bool ok = col < nh;
    if (C::FWD) {  // k-steps (q, h) <-> fold index 8q + 2c + h < ho; the middle (n odd) at q = NTH, c = h = 0
      ok = q < C::NTH ? col < ho : (hf == 0 && (l & 3) == 0 && h == 0);
      if (q >= C::NTH) col = ho;
    }
    const double* Wh = a.W1 + (hf ? size_t(he) * he : 0);
    w1[e] = (ok && row < nh) ? __ldg(Wh + size_t(row) * nh + col) : 0.0;
  }
  __syncthreads();

  const uint32_t P = a.planes;
  if (blockIdx.x >= P) return;
  const size_t plane_sz = size_t(n) * n;
  pdl_wait();  // X is the previous kernel's output

  // ---- ring loader (cp.async, zero-filled where a row does not exist): block g (plane
  // iteration g / NB, k-step group g % NB) holds HR = 4 KB half-rows: slot row i < HR is the
  // even / direct half-row k = HR b + i, slot row HR + i the odd / mirror one (forward: row
  // n-1-k, folded at the B read; backward: row he + k).  Thread tid owns half-row li = tid / TPR
  // and the columns (or 16-byte column pairs, n even) lj + TPR m: no per-element index math.
  constexpr int TPR = C::THREADS / C::HR;
  constexpr int EPT = (C::NMAX + TPR - 1) / TPR;
  constexpr int EPT2 = (C::NMAX / 2 + TPR - 1) / TPR;
  const int li = tid / TPR, lj = tid - li * TPR;
  const bool v16 = (n % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
  auto issue = [&](uint32_t g) {
    const uint32_t it = g / C::NB, b = g - it * C::NB;
    const uint32_t plane = blockIdx.x + it * gridDim.x;
    if (plane < P) {
      const int k = C::HR * int(b) + li;
      const bool oka = k < he, okb = k < ho;
      const double* src = a.X + size_t(plane) * plane_sz;
      const double* pa = src + size_t(oka ? k : 0) * n;
      const double* pb = src + size_t(okb ? (C::FWD ? n - 1 - k : he + k) : 0) * n;
      double* dst = ring + (g % C::NSTAGE) * (2 * C::HR * S) + li * S;
      if (v16) {
#pragma unroll
        for (int m = 0; m < EPT2; ++m) {
          const int j = 2 * (lj + TPR * m);
          if (j < n) {
            cp_async16z(dst + j, pa + j, oka);
            cp_async16z(dst + C::HR * S + j, pb + j, okb);
          }
        }
      } else {
#pragma unroll
        for (int m = 0; m < EPT; ++m) {
          const int j = lj + TPR * m;
          if (j < n) {
            cp_async8z(dst + j, pa + j, oka);
            cp_async8z(dst + C::HR * S + j, pb + j, okb);
          }
        }
      }
    }
    cp_async_commit();
  };

  // first-product columns of the lane (B column n = r of n-tile t): a per-lane base plus a
  // compile-time step per tile (no per-tile registers)
  //   forward:  t < NTH: 8t + r | t < 2 NTH: n-1-r - 8(t-NTH) | middle: ho (lane r = 0)
  //   backward: t < NQE: 8t + r | else: he + r + 8(t-NQE)
  const int cb0 = r, cb1 = C::FWD ? n - 1 - r : he + r;
  auto colof = [&](int t) -> int {
    if (C::FWD) {
      if (t < C::NTH) return cb0 + 8 * t;
      if (t < 2 * C::NTH) return cb1 - 8 * (t - C::NTH);
      return ho;
    }
    return t < C::NQE ? cb0 + 8 * t : cb1 + 8 * (t - C::NQE);
  };
  auto okof = [&](int t) -> bool {
    if (C::FWD) return t < 2 * C::NTH ? r < ho - 8 * (t % C::NTH) : r == 0;
    return t < C::NQE ? r < he - 8 * t : r < ho - 8 * (t - C::NQE);
  };
  const double* w2l = w2 + mt * C::KSP * 64 + 2 * lane;
  const double* w1l = w1 + 2 * lane;

#pragma unroll
  for (int st = 0; st < C::NSTAGE - 1; ++st) issue(st);
  uint32_t g = 0;
#pragma unroll 1
  for (uint32_t plane = blockIdx.x; plane < P; plane += gridDim.x) {
    double acc[2][C::NT][2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int t = 0; t < C::NT; ++t) acc[hf][t][0] = acc[hf][t][1] = 0.0;

    // ---- first product (direction 2), KB k-steps per ring block; block g + NSTAGE - 1 is
    // issued into the slot every warp finished reading before this iteration's barrier
#pragma unroll 1
    for (int b = 0; b < C::NB; ++b, ++g) {
      cp_async_wait<C::NSTAGE - 2>();
      __syncthreads();
      issue(g + C::NSTAGE - 1);
      const double* slot = ring + (g % C::NSTAGE) * (2 * C::HR * S);
#pragma unroll
      for (int kp = 0; kp < C::KB / 2; ++kp) {
        const int ksp = (C::KB / 2) * b + kp;
        if (2 * ksp >= C::KS) break;
        const double2 ae = *reinterpret_cast<const double2*>(w2l + ksp * 64);
        const double2 ao = *reinterpret_cast<const double2*>(w2l + C::W2H + ksp * 64);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (2 * ksp + h >= C::KS) break;
          const double* r0 = slot + (8 * kp + 4 * h + c) * S;
          const double* r1 = r0 + C::HR * S;
          const double fe = h ? ae.y : ae.x, fo = h ? ao.y : ao.x;
#pragma unroll
          for (int t = 0; t < C::NT; ++t) {
            const bool ok = okof(t);
            const double x0 = ok ? r0[colof(t)] : 0.0;
            const double x1 = ok ? r1[colof(t)] : 0.0;
            if (C::FWD) {  // fold of direction 2: x_k + x_{n-1-k}, x_k - x_{n-1-k}
              dmma_8x8x4(acc[0][t], fe, x0 + x1);
              dmma_8x8x4(acc[1][t], fo, x0 - x1);
            } else {
              dmma_8x8x4(acc[0][t], fe, x0);
              dmma_8x8x4(acc[1][t], fo, x1);
            }
          }
        }
      }
    }

    double* out = a.Y + size_t(plane) * plane_sz;
    if (C::FWD) {
      // ---- fold of direction 1 in registers: tile q <- even (x + Rx), tile NTH + q <- odd
#pragma unroll
      for (int hf = 0; hf < 2; ++hf)
#pragma unroll
        for (int q = 0; q < C::NTH; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double u = acc[hf][q][h], v = acc[hf][C::NTH + q][h];
            acc[hf][q][h] = u + v;
            acc[hf][C::NTH + q][h] = u - v;
          }
      // ---- second product (direction 1): out[hf1][hf2] rows k1 = 8 m1 + r, columns k2 = 8 mt + 2c + h
#pragma unroll 1
      for (int m1 = 0; m1 < C::MT; ++m1) {
        double o[2][2][2];
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) o[i][j][0] = o[i][j][1] = 0.0;
#pragma unroll
        for (int q = 0; q < C::NQE; ++q) {
          const double2 fe = *reinterpret_cast<const double2*>(w1l + (m1 * C::NQ + q) * 64);
          const int te = q < C::NTH ? q : 2 * C::NTH;  // even k-steps: folded tiles, then the middle
#pragma unroll
          for (int hf2 = 0; hf2 < 2; ++hf2) {
            dmma_8x8x4(o[0][hf2], fe.x, acc[hf2][te][0]);
            if (q < C::NTH) dmma_8x8x4(o[0][hf2], fe.y, acc[hf2][te][1]);
          }
          if (q < C::NTH) {
            const double2 fo = *reinterpret_cast<const double2*>(w1l + C::W1H + (m1 * C::NQ + q) * 64);
#pragma unroll
            for (int hf2 = 0; hf2 < 2; ++hf2) {
              dmma_8x8x4(o[1][hf2], fo.x, acc[hf2][C::NTH + q][0]);
              dmma_8x8x4(o[1][hf2], fo.y, acc[hf2][C::NTH + q][1]);
            }
          }
        }
        const int k1 = 8 * m1 + r;
#pragma unroll
        for (int hf1 = 0; hf1 < 2; ++hf1) {
          if (k1 >= (hf1 ? ho : he)) continue;
          const int k1g = hf1 * he + k1;
#pragma unroll
          for (int hf2 = 0; hf2 < 2; ++hf2)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int k2 = 8 * mt + 2 * c + h;
              if (k2 < (hf2 ? ho : he)) out[size_t(hf2 * he + k2) * n + k1g] = o[hf1][hf2][h];
            }
        }
      }
    } else {
      // ---- second product (direction 1) and both unfolds at the stores
#pragma unroll 1
      for (int m1 = 0; m1 < C::MT; ++m1) {
        double o[2][2][2];  // [hf1: e/o output half][hf2: p/q tile][h]
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
          for (int j = 0; j < 2; ++j) o[i][j][0] = o[i][j][1] = 0.0;
#pragma unroll
        for (int q = 0; q < C::NQE; ++q) {
          const double2 fe = *reinterpret_cast<const double2*>(w1l + (m1 * C::NQ + q) * 64);
#pragma unroll
          for (int hf2 = 0; hf2 < 2; ++hf2) {
            dmma_8x8x4(o[0][hf2], fe.x, acc[hf2][q][0]);
            dmma_8x8x4(o[0][hf2], fe.y, acc[hf2][q][1]);
          }
          if (q < C::NTH) {
            const double2 fo = *reinterpret_cast<const double2*>(w1l + C::W1H + (m1 * C::NQ + q) * 64);
#pragma unroll
            for (int hf2 = 0; hf2 < 2; ++hf2) {
              dmma_8x8x4(o[1][hf2], fo.x, acc[hf2][C::NQE + q][0]);
              dmma_8x8x4(o[1][hf2], fo.y, acc[hf2][C::NQE + q][1]);
            }
          }
        }
        const int i1 = 8 * m1 + r;  // direction-1 output index (even-part row)
        if (i1 < he) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int i2 = 8 * mt + 2 * c + h;  // direction-2 output index
            if (i2 >= he) continue;
            // direction 1: z1 = [e + o ; R(e - o)] per direction-2 half (p, q)
            double z1[2][2];  // [hf2][0: column i1, 1: column n-1-i1]
#pragma unroll
            for (int hf2 = 0; hf2 < 2; ++hf2) {
              const double e = o[0][hf2][h], od = i1 < ho ? o[1][hf2][h] : 0.0;
              z1[hf2][0] = e + od;
              z1[hf2][1] = e - od;
            }
            const bool m2 = i2 < ho, m1v = i1 < ho;
            double* row0 = out + size_t(i2) * n;
            double* row1 = out + size_t(n - 1 - i2) * n;
            const double q0 = m2 ? z1[1][0] : 0.0, q1 = m2 ? z1[1][1] : 0.0;
            row0[i1] = z1[0][0] + q0;
            if (m1v) row0[n - 1 - i1] = z1[0][1] + q1;
            if (m2) {
              row1[i1] = z1[0][0] - q0;
              if (m1v) row1[n - 1 - i1] = z1[0][1] - q1;
            }
          }
        }
      }
    }
  }
}

}  // namespace ls
