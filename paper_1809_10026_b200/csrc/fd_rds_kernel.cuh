// FD mode product with the centrosymmetric split (fd_rd_kernel.cuh, CS = 1 fold / 2 unfold),
// "staged" variant: the streamed operand arrives by cp.async in a per-warp shared-memory ring
// instead of a register window.
//
// Why (profiles/r02, ncu of the register-direct split kernels at config 4): the split halves the
// DMMA work per loaded byte, so the register window that hides the load latency must double for
// the same lead time; with two accumulator sets and the window the kernel sits at 255 registers
// and the B loads show up as long-scoreboard stalls (77 % DMMA pipe against 88-94 % for the
// unsplit kernel).  Here a warp's B data for the next D - 1 k-steps sit in shared memory (no
// registers held in flight).  No block barriers: each warp stages and reads only its own ring
// (cp.async groups + __syncwarp).  NT n-tiles per warp (column permutation of fd_rd_kernel.cuh:
// lane l's B columns are NT (l/4) .. + NT - 1 of the tile, its accumulator columns 2 NT (l%4) ..
// + 2 NT - 1), MINB CTAs per SM.
//
// Scope: n even (he = ho = n/2), FAST strided modes (Q even, 16-byte aligned X / Y: a 16-byte
// chunk is two columns of one row) and the contiguous mode 1 (8-byte copies); other launches
// keep the register-direct kernel.
//   fold (forward):  stage[0] = rows k = 4kk + r, stage[1] = mirror rows n-1-k;  B_even = s0 + s1,
//                    B_odd = s0 - s1 (k < he, zero-filled beyond);
//   unfold (backward): stage[0] = rows k, stage[1] = rows he + k;  epilogue p + q, R(p - q).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"

namespace ls {

template <int KS_, bool MODE1_, int CS_, int D_, int NT_ = 1, int MINB_ = 2>
struct RDSCfg {
  static constexpr int KS = KS_, D = D_, CS = CS_, NT = NT_, MINB = MINB_;
  static constexpr bool MODE1 = MODE1_;
  static constexpr int WARPS = 8, THREADS = 256, TW = 8 * NT;
  static constexpr int MT = (KS + 1) / 2, KSP = (KS + 1) / 2;
  static constexpr int WFRAG1 = MT * KSP * 64, WFRAG = 2 * WFRAG1;
  static constexpr int HSTAGE = 4 * TW;      // doubles per half per k-step: 4 rows x TW columns
  static constexpr int STAGE = 2 * HSTAGE;   // doubles per k-step per warp
  static constexpr size_t SMEM = size_t(WFRAG + WARPS * D * STAGE) * sizeof(double);
  static_assert(CS == 1 || CS == 2, "split kernels only");
  static_assert(D >= 2, "ring of at least 2 stages");
  static_assert(NT == 1 || NT == 2, "1 or 2 n-tiles per warp");
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
__global__ void __launch_bounds__(256, C::MINB) fd_mode_rds_kernel(ModeArgs args) {
  constexpr int NT = C::NT, TW = C::TW;
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
  const uint32_t ntw = (ncols + TW - 1) / TW;
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
      // element e = (half h, column j, row r): layout [h][j][r]; 8-byte copies, 2 NT per lane
#pragma unroll
      for (int u = 0; u < 2 * NT; ++u) {
        const int e = lane + 32 * u;
        const int h = e / (4 * TW), j = (e / 4) % TW, r = e % 4;
        const uint32_t c = t * TW + j;
        const int k = 4 * kk + r;
        const bool v = tv && c < ncols && k < he;
        const int row = (h == 0) ? k : ((C::CS == 1) ? n - 1 - k : he + k);
        rds_cp8(st + e, v ? X + size_t(c) * n + row : X, v ? 8 : 0);
      }
    } else {
      // chunk e = (half h, row r, 16-byte part q4 of TW columns): layout [h][r][TW]
#pragma unroll
      for (int u = 0; u < NT; ++u) {
        const int e = lane + 32 * u;
        const int h = e / (2 * TW), r = (e / (TW / 2)) % 4, q4 = e % (TW / 2);
        const int k = 4 * kk + r;
        const uint32_t c = t * TW + 2 * q4;
        int bytes = 0;
        const double* src = X;
        if (tv && k < he && c < ncols) {
          const int row = (h == 0) ? k : ((C::CS == 1) ? n - 1 - k : he + k);
          const uint32_t p = c / Q, q = c - p * Q;
          src = X + (size_t(p) * n + row) * Q + q;
          bytes = (c + 1 < ncols) ? 16 : 8;
        }
        rds_cp16(st + h * C::HSTAGE + r * TW + 2 * q4, src, bytes);
      }
    }
    cp_async_commit();
  };
  // the warp's k-step sequence: (tile0 + (g / KS) wstride, g % KS), g = 0, 1, ...
  auto issue_seq = [&](uint32_t g) { issue(tile0 + (g / C::KS) * wstride, int(g % C::KS), int(g % C::D)); };
#pragma unroll
  for (int s = 0; s < C::D - 1; ++s) issue_seq(uint32_t(s));

  uint32_t g = 0;  // sequence index of the next k-step consumed
  for (uint32_t tile = tile0; tile < ntw; tile += wstride) {
    double acc[2][C::MT][NT][2];
#pragma unroll
    for (int hf = 0; hf < 2; ++hf)
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[hf][mt][j][0] = acc[hf][mt][j][1] = 0.0;
#pragma unroll
    for (int ksp = 0; ksp < C::KSP; ++ksp) {
      double b[2][2][NT];  // [k-step of the pair][half][n-tile]
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int j = 0; j < NT; ++j) b[u][0][j] = b[u][1][j] = 0.0;
        if (2 * ksp + u < C::KS) {
          cp_async_wait<C::D - 2>();
          __syncwarp();
          const double* st = ring + (g % C::D) * C::STAGE;
          double s0[NT], s1[NT];
          if (C::MODE1) {
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              s0[j] = st[(NT * nq + j) * 4 + kq];
              s1[j] = st[C::HSTAGE + (NT * nq + j) * 4 + kq];
            }
          } else if (NT == 2) {
            const double2 a0 = *reinterpret_cast<const double2*>(st + kq * TW + NT * nq);
            const double2 a1 = *reinterpret_cast<const double2*>(st + C::HSTAGE + kq * TW + NT * nq);
            s0[0] = a0.x;
            s0[NT - 1] = a0.y;
            s1[0] = a1.x;
            s1[NT - 1] = a1.y;
          } else {
            s0[0] = st[kq * TW + nq];
            s1[0] = st[C::HSTAGE + kq * TW + nq];
          }
#pragma unroll
          for (int j = 0; j < NT; ++j) {
            if (C::CS == 1) {
              b[u][0][j] = s0[j] + s1[j];
              b[u][1][j] = s0[j] - s1[j];
            } else {
              b[u][0][j] = s0[j];
              b[u][1][j] = s1[j];
            }
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
#pragma unroll
          for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[hf][mt][j], af.x, b[0][hf][j]);
          if (2 * ksp + 1 < C::KS) {
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma_8x8x4(acc[hf][mt][j], af.y, b[1][hf][j]);
          }
        }
    }
    // ---- epilogue: the lane's columns cg .. cg + 2NT - 1 (v[e] = column cg + e) at rows a
    //      (fold: [even | odd]; unfold: p + q, R(p - q))
    const uint32_t cg = tile * TW + 2 * NT * kq;
    if (cg < ncols) {
      auto emit = [&](int a, const double (&v)[2 * NT]) {
        if (C::MODE1) {
#pragma unroll
          for (int e = 0; e < 2 * NT; ++e)
            if (cg + e < ncols) args.Y[size_t(cg + e) * n + a] = v[e];
        } else {
          // Q even, cg even: pairs stay in one row and 16-byte aligned
#pragma unroll
          for (int e = 0; e < 2 * NT; e += 2) {
            const uint32_t c = cg + e;
            if (c < ncols) {
              const uint32_t p = c / Q, q = c - p * Q;
              *reinterpret_cast<double2*>(args.Y + (size_t(p) * n + a) * Q + q) = make_double2(v[e], v[e + 1]);
            }
          }
        }
      };
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        const int a = mt * 8 + nq;
        if (a < he) {
          double v0[2 * NT], v1[2 * NT];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < NT; ++j) {
              v0[h * NT + j] = acc[0][mt][j][h];
              v1[h * NT + j] = acc[1][mt][j][h];
            }
          if (C::CS == 1) {
            emit(a, v0);
            emit(he + a, v1);
          } else {
            double s[2 * NT], t[2 * NT];
#pragma unroll
            for (int e = 0; e < 2 * NT; ++e) {
              s[e] = v0[e] + v1[e];
              t[e] = v0[e] - v1[e];
            }
            emit(a, s);
            emit(n - 1 - a, t);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

}  // namespace ls
