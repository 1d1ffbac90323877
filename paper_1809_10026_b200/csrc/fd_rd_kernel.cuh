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
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"

namespace ls {

template <int KS_, int NT_, bool MODE1_, bool SCALE_, bool FAST_, int D_, int REMOTE_ = 0>
struct RDCfg {
  static constexpr int KS = KS_, NT = NT_, D = D_;
  static constexpr int REMOTE = REMOTE_;  // fused all-to-all epilogue (ModeArgs::remote)
  static constexpr bool MODE1 = MODE1_, SCALE = SCALE_, FAST = FAST_;
  static constexpr int MT = (KS + 1) / 2;  // ceil(n/8) for n in (4KS-4, 4KS]
  static constexpr int KSP = (KS + 1) / 2;  // k-step pairs
  static constexpr int KSE = ((KS + D - 1) / D) * D;  // k-steps rounded up to the window
  static constexpr int WARPS = 8, THREADS = 32 * WARPS;
  static constexpr int TW = 8 * NT;  // columns per warp tile
  static constexpr int WFRAG = MT * KSP * 64;
  static constexpr int LAMA = SCALE ? 8 * MT : 0;  // lambda_t per output row (SCALE)
  static constexpr size_t SMEM = size_t(WFRAG + LAMA) * sizeof(double);
  static_assert(!(MODE1 && FAST), "FAST is a strided-mode path");
  static_assert(REMOTE == 0 || (FAST && !SCALE), "fused all-to-all epilogues: unscaled FAST launches");
  static_assert(NT % 2 == 0, "NT even (LDG.128 pairs)");
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
__device__ __forceinline__ double ldg_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// B fragments of k-step kk (rows 4kk + lane%4) of the lane's NT columns
template <class C>
__device__ __forceinline__ void rd_load(double (&dst)[C::NT], const double* __restrict__ X, const RDIn<C::NT>& in,
                                        int kk, size_t kstep, bool kok, int n) {
  if (C::FAST) {
    const bool ok = kok && in.mask;
    const double* src = X + in.off[0] + kk * kstep;
#pragma unroll
    for (int j = 0; j < C::NT; j += 2) {
      double2 v = make_double2(0.0, 0.0);
      if (ok) v = ldg_stream2(src + j);
      dst[j] = v.x;
      dst[j + 1] = v.y;
    }
  } else if (C::MODE1) {
    const double* src = X + in.off[0] + kk * kstep;
#pragma unroll
    for (int j = 0; j < C::NT; ++j) dst[j] = (kok && ((in.mask >> j) & 1u)) ? ldg_stream(src + size_t(j) * n) : 0.0;
  } else {
#pragma unroll
    for (int j = 0; j < C::NT; ++j)
      dst[j] = (kok && ((in.mask >> j) & 1u)) ? ldg_stream(X + in.off[j] + kk * kstep) : 0.0;
  }
}

template <class C>
__global__ void __launch_bounds__(256, 1) fd_mode_rd_kernel(ModeArgs args) {
  extern __shared__ __align__(16) double smem[];
  double* wsm = smem;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, nq = lane >> 2;
  const int n = args.n;
  const uint32_t Q = args.Q, ncols = args.ncols;

  // W -> shared memory, A-fragment order, two k-steps per lane slot:
  // wsm[((mt*KSP + ks/2)*32 + l)*2 + ks%2] = W[mt*8 + l/4][ks*4 + l%4]
  for (int e = tid; e < C::WFRAG; e += C::THREADS) {
    const int h = e & 1, l = (e >> 1) & 31, ksp = (e >> 6) % C::KSP, mt = (e >> 6) / C::KSP;
    const int ks = 2 * ksp + h;
    const int a = mt * 8 + (l >> 2), i = ks * 4 + (l & 3);
    wsm[e] = (a < n && i < n && ks < C::KS) ? __ldg(args.W + size_t(a) * n + i) : 0.0;
  }
  double* lam_a_s = wsm + C::WFRAG;  // SCALE: lambda_t of the output rows, staged once
  if (C::SCALE)
    for (int e = tid; e < C::LAMA; e += C::THREADS) lam_a_s[e] = e < n ? __ldg(args.lam_a + e) : 0.0;
  __syncthreads();

  const uint32_t ntw = (ncols + C::TW - 1) / C::TW;
  const uint32_t wstride = gridDim.x * C::WARPS;
  uint32_t tile = blockIdx.x * C::WARPS + warp;
  if (tile >= ntw) return;
  const size_t kstep = C::MODE1 ? size_t(4) : size_t(4) * Q;
  // rows 4*kk + kq >= n are never loaded (zero B fragment): the bucket's KS may exceed
  // ceil(n/4) by a few k-steps, and those rows lie past the end of the column
  // (the k-step buckets exceed ceil(n/4) by at most 5, so only the last 6 k-steps test)
  auto row_ok = [&](int kk) { return 4 * kk + kq < n; };
  const double* wl = wsm + lane * 2;

  pdl_wait();  // X is the previous kernel's output (fd_kernels.cuh)
  RDIn<C::NT> cur = rd_make_in<C>(args, tile, lane);
  double bw[C::D][C::NT];
#pragma unroll
  for (int s = 0; s < C::D; ++s)
    if (s < C::KS) rd_load<C>(bw[s], args.X, cur, s, kstep, row_ok(s), n);

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
    double acc[C::MT][C::NT][2];
#pragma unroll
    for (int mt = 0; mt < C::MT; ++mt)
#pragma unroll
      for (int j = 0; j < C::NT; ++j) acc[mt][j][0] = acc[mt][j][1] = 0.0;

    // k-loop in pairs; phantom steps (KS <= ks < KSE) only refill the window
#pragma unroll
    for (int ksp = 0; ksp < C::KSE / 2 + (C::KSE & 1); ++ksp) {
      const int k0 = 2 * ksp, k1 = 2 * ksp + 1;
      if (k0 < C::KS) {
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const double2 af = *reinterpret_cast<const double2*>(wl + (mt * C::KSP + ksp) * 64);
#pragma unroll
          for (int j = 0; j < C::NT; ++j) dmma_8x8x4(acc[mt][j], af.x, bw[k0 % C::D][j]);
          if (k1 < C::KS) {
#pragma unroll
            for (int j = 0; j < C::NT; ++j) dmma_8x8x4(acc[mt][j], af.y, bw[k1 % C::D][j]);
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
          rd_load<C>(bw[k % C::D], args.X, cur, kk, kstep, row_ok(kk), n);
        } else if (kk >= C::KSE) {
          const int s = kk - C::KSE;  // next tile's k-step, same slot (KSE % D == 0)
          if (s < C::KS) rd_load<C>(bw[k % C::D], args.X, nxt, s, kstep, row_ok(s), n);
        }
      }
    }

    // ---- epilogue: lane's columns cg .. cg + 2NT - 1, rows mt*8 + nq
    if (C::REMOTE) {
      // fused all-to-all: every output element goes straight to its owner's receive buffer
      // (peer memory over NVLink in a multi-GPU run); pairs that stay contiguous and
      // 16-byte aligned in the destination are stored as one double2
      if (cg < ncols) {
        const uint32_t p = cg / Q, q = cg - p * Q;
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const int a = mt * 8 + nq;
          if (a < n) {
#pragma unroll
            for (int e = 0; e < 2 * C::NT; e += 2) {
              if (cg + e >= ncols) continue;
              const double v0 = acc[mt][e % C::NT][e / C::NT];
              const double v1 = acc[mt][(e + 1) % C::NT][(e + 1) / C::NT];
              int r0, r1;
              int64_t o0, o1;
              if (C::REMOTE == 1) {
                const int64_t s0 = int64_t(a) * Q + q + e;
                a2a_fwd_dest(int64_t(p), s0, args.nt_g, args.Ns_g, args.world, args.me, &r0, &o0);
                a2a_fwd_dest(int64_t(p), s0 + 1, args.nt_g, args.Ns_g, args.world, args.me, &r1, &o1);
              } else {
                a2a_bwd_dest(int64_t(a), int64_t(q) + e, args.nt_g, args.Ns_g, args.world, args.me, &r0, &o0);
                a2a_bwd_dest(int64_t(a), int64_t(q) + e + 1, args.nt_g, args.Ns_g, args.world, args.me, &r1, &o1);
              }
              const bool second = cg + e + 1 < ncols;
              double* d0 = args.peer[r0] + o0;
              if (second && r1 == r0 && o1 == o0 + 1 && ((reinterpret_cast<uintptr_t>(d0) & 15) == 0)) {
                *reinterpret_cast<double2*>(d0) = make_double2(v0, v1);
              } else {
                *d0 = v0;
                if (second) args.peer[r1][o1] = v1;
              }
            }
          }
        }
      }
    } else if (C::FAST) {
      if (cg < ncols) {
        const uint32_t p = cg / Q, q = cg - p * Q;
        double* ob = args.Y + size_t(p) * n * Q + q;
#pragma unroll
        for (int mt = 0; mt < C::MT; ++mt) {
          const int a = mt * 8 + nq;
          if (a < n) {
            double v[2 * C::NT];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
              for (int j = 0; j < C::NT; ++j) v[h * C::NT + j] = acc[mt][j][h];
            if (C::SCALE) {
              const double la = lam_a_s[a];
#pragma unroll
              for (int e = 0; e < 2 * C::NT; ++e) v[e] *= fast_rcp(la + lc[C::SCALE ? e : 0]);
            }
            double* o = ob + size_t(a) * Q;
#pragma unroll
            for (int e = 0; e < 2 * C::NT; e += 2) *reinterpret_cast<double2*>(o + e) = make_double2(v[e], v[e + 1]);
          }
        }
      }
    } else {
      size_t base[C::MODE1 ? 1 : 2 * C::NT];
      if (C::MODE1) {
        base[0] = size_t(cg) * n;
      } else {
#pragma unroll
        for (int e = 0; e < (C::MODE1 ? 1 : 2 * C::NT); ++e) {
          const uint32_t c = cg + e;
          const uint32_t p = c / Q, q = c - p * Q;
          base[e] = size_t(p) * n * Q + q;
        }
      }
      const size_t rstride = C::MODE1 ? size_t(1) : size_t(Q);
#pragma unroll
      for (int mt = 0; mt < C::MT; ++mt) {
        const int a = mt * 8 + nq;
        if (a < n) {
          double la = 0.0;
          if (C::SCALE) la = lam_a_s[a];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int j = 0; j < C::NT; ++j) {
              const int e = h * C::NT + j;
              if (cg + e < ncols) {
                double v = acc[mt][j][h];
                if (C::SCALE) v *= fast_rcp(la + lc[C::SCALE ? e : 0]);
                if (C::MODE1) args.Y[base[0] + size_t(e) * n + a] = v;
                else args.Y[base[C::MODE1 ? 0 : e] + size_t(a) * rstride] = v;
              }
            }
        }
      }
    }
    cur = nxt;
  }
}

}  // namespace ls
