// FD mode product with the centrosymmetric split (fd_rd_kernel.cuh, CS = 1 fold / 2 unfold),
// "staged" variant: the streamed operand arrives by cp.async in a per-warp shared-memory ring
// instead of a register window.
//
// Why (profiles/r02, ncu of the register-direct split kernels at config 4): the split halves the
// DMMA work per loaded byte, so the register window that hides the load latency must double
// for the same lead time; with 2 n-tiles per warp, two accumulator sets and the window the kernel
// sits at 255 registers and 8 warps per SM, and the B loads show up as long-scoreboard stalls
// (77 % DMMA pipe against 88-94 % for the unsplit kernel).  Here a warp owns 8 columns (NT = 1:
// 2 x 9 m-tiles of accumulators at he = 66), its B data for the next D - 1 k-steps sit in shared
// memory (no registers), so 2 CTAs of 8 warps fit per SM (<= 128 registers) and every warp
// keeps D - 1 k-steps of loads in flight.  No block barriers: each warp stages and reads only its
// own ring (cp.async groups + __syncwarp).
//
// Scope: n even (he = ho = n/2), FAST strided modes (Q even, 16-byte aligned X / Y: a 16-byte
// chunk is two columns of one row) and the contiguous mode 1 (two 8-byte copies per lane: rows
// 2j, 2j+1 of one column); other launches keep the register-direct kernel.
//   fold (forward):  stage[0] = rows k = 4kk + r, stage[1] = mirror rows n-1-k;  B_even = s0 + s1,
//                    B_odd = s0 - s1 (k < he, zero-filled beyond);
//   unfold (backward): stage[0] = rows k, stage[1] = rows he + k;  epilogue p + q, R(p - q).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"

namespace ls {

template <int KS_, bool MODE1_, int CS_, int D_>
struct RDSCfg {
  static constexpr int KS = KS_, D = D_, CS = CS_;
  static constexpr bool MODE1 = MODE1_;
  static constexpr int WARPS = 8, THREADS = 256, TW = 8;
  static constexpr int MT = (KS + 1) / 2, KSP = (KS + 1) / 2;
  static constexpr int WFRAG1 = MT * KSP * 64, WFRAG = 2 * WFRAG1;
  static constexpr int STAGE = 64;  // doubles per k-step per warp: [2 halves][32]
  static constexpr size_t SMEM = size_t(WFRAG + WARPS * D * STAGE) * sizeof(double);
  static_assert(CS == 1 || CS == 2, "split kernels only");
  static_assert(D >= 2, "ring of at least 2 stages");
};

__device__ __forceinline__ void rds_cp16(double* dst, const double* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void rds_cp8(double* dst, const double* src, int bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(bytes));
}

template <class C>
__global__ void __launch_bounds__(256, 2) fd_mode_rds_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* wsm = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, nq = lane >> 2;
  const int n = args.n;
  const int he = n / 2;  // = ho (n even)
  const uint32_t Q = args.Q, ncols = args.ncols;
  // W -> shared memory in A-fragment order (as fd_rd_kernel.cuh, two halves)
  for (int e = tid; e < C::WFRAG; e += C::THREADS) {
    const int hf = e / C::WFRAG1, e1 = e - hf * C::WFRAG1;
    const int h = e1 & 1, l = (e1 >> 1) & 31, ksp = (e1 >> 6) % C::KSP, mt = (e1 >> 6) / C::KSP;
    const int ks = 2 * ksp + h;
    const int a = mt * 8 + (l >> 2), i = ks * 4 + (l & 3);
    const double* Wh = args.W + (hf ? size_t(he) * he : 0);
    wsm[e] = (a < he && i < he && ks < C::KS) ? __ldg(Wh + size_t(a) * he + i) : 0.0;
  }
  __syncthreads();
  double* ring = smem + C::WFRAG + warp * (C::D * C::STAGE);
  const uint32_t ntw = (ncols + C::TW - 1) / C::TW;
  const uint32_t wstride = gridDim.x * C::WARPS;
  const uint32_t tile0 = blockIdx.x * C::WARPS + warp;
  const double* wl = wsm + lane * 2;
  const double* X = args.X;
  pdl_wait();  // X is the previous kernel's output

  // cp.async of k-step kk of tile t into ring stage s (one commit group per call, empty past the
  // warp's last tile so that the group count stays uniform)
  auto issue = [&](uint32_t t, int kk, int s) {
    double* st = ring + s * C::STAGE;
    const bool tv = t < ntw;
    if (C::MODE1) {
      // lane: half h, column j of the tile, rows 2pr, 2pr + 1 of the k-step (two 8-byte copies)
      const int h = lane >> 4, j = (lane >> 1) & 7, pr = lane & 1;
      const uint32_t c = t * C::TW + j;
      const bool cv = tv && c < ncols;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 2 * pr + u, k = 4 * kk + r;
        const bool rv = cv && k < he;
        int row = k;
        if (h == 1) row = (C::CS == 1) ? n - 1 - k : he + k;
        const double* src = rv ? X + size_t(c) * n + row : X;
        rds_cp8(st + h * 32 + j * 4 + r, src, rv ? 8 : 0);
      }
    } else {
      // lane: half h, row r of the k-step, 16-byte chunk q4 (columns 2q4, 2q4 + 1)
      const int h = lane >> 4, r = (lane >> 2) & 3, q4 = lane & 3;
      const int k = 4 * kk + r;
      const uint32_t c = t * C::TW + 2 * q4;
      int bytes = 0;
      const double* src = X;
      if (tv && k < he && c < ncols) {
        const int row = (h == 0) ? k : ((C::CS == 1) ? n - 1 - k : he + k);
        const uint32_t p = c / Q, q = c - p * Q;
        src = X + (size_t(p) * n + row) * Q + q;
        bytes = (c + 1 < ncols) ? 16 : 8;
      }
      rds_cp16(st + h * 32 + r * 8 + 2 * q4, src, bytes);
    }
    cp_async_commit();
  };
  // the warp's k-step sequence: (tile0 + (g / KS) wstride, g % KS), g = 0, 1, ...
  auto issue_seq = [&](uint32_t g) {
    issue(tile0 + (g / C::KS) * wstride, int(g % C::KS), int(g % C::D));
  };
#pragma unroll
  for (int s = 0; s < C::D - 1; ++s) issue_seq(uint32_t(s));

  uint32_t g = 0;  // sequence index of the next k-step consumed
  for (uint32_t tile = tile0; tile < ntw; tile += wstride) {
    double acc[2][C::MT][2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) acc[hf][mt][0] = acc[hf][mt][1] = 0.0;
#pragma unroll
    for (int ksp = 0; ksp < C::KSP; ++ksp) {
      double b[2][2];  // [k-step of the pair][half]
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        b[u][0] = b[u][1] = 0.0;
        if (2 * ksp + u < C::KS) {
          cp_async_wait<C::D - 2>();
          __syncwarp();
          const double* st = ring + (g % C::D) * C::STAGE;
          const int ix = C::MODE1 ? nq * 4 + kq : kq * 8 + nq;
          const double s0 = st[ix], s1 = st[32 + ix];
          if (C::CS == 1) {
            b[u][0] = s0 + s1;
            b[u][1] = s0 - s1;
          } else {
            b[u][0] = s0;
            b[u][1] = s1;
          }
          issue_seq(g + C::D - 1);  // refills the stage every lane finished reading last step
          ++g;
        }
      }
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const double2 af = *reinterpret_cast<const double2*>(wl + hf * C::WFRAG1 + (mt * C::KSP + ksp) * 64);
          dmma_8x8x4(acc[hf][mt], af.x, b[0][hf]);
          if (2 * ksp + 1 < C::KS) dmma_8x8x4(acc[hf][mt], af.y, b[1][hf]);
        }
    }
    // ---- epilogue: the lane's columns cg, cg + 1 at rows a (fold: [even | odd]; unfold: p + q, R(p - q))
    const uint32_t cg = tile * C::TW + 2 * kq;
    if (cg < ncols) {
      const bool two = cg + 1 < ncols;
      auto emit = [&](int a, double v0, double v1) {
        if (C::MODE1) {
          args.Y[size_t(cg) * n + a] = v0;
          if (two) args.Y[size_t(cg + 1) * n + a] = v1;
        } else {
          const uint32_t p = cg / Q, q = cg - p * Q;
          double* o = args.Y + (size_t(p) * n + a) * Q + q;
          *reinterpret_cast<double2*>(o) = make_double2(v0, v1);  // Q even, cg even: one row, aligned
        }
      };
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        const int a = mt * 8 + nq;
        if (a < he) {
          if (C::CS == 1) {
            emit(a, acc[0][mt][0], acc[0][mt][1]);
            emit(he + a, acc[1][mt][0], acc[1][mt][1]);
          } else {
            emit(a, acc[0][mt][0] + acc[1][mt][0], acc[0][mt][1] + acc[1][mt][1]);
            emit(n - 1 - a, acc[0][mt][0] - acc[1][mt][0], acc[0][mt][1] - acc[1][mt][1]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

}  // namespace ls
