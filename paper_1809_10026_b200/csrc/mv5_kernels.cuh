// Matrix-free y = A x (eq:A_kron, PAPER.md 686-703), v5: the direction-3 and time passes of
// v4 (matvec3_kernels.cuh MV3_D3 + MV3_T2) fused into one kernel, so v1 = M_3 P_M and
// v2 = J_3 P_M + M_3 P_J + 2 K_3 P_K never go to HBM (16 B/DOF written and read back in v4):
//     y = K_t v1 + M_t v2 + W_t v3,   v3 = K_3 P_M + M_3 P_K on the last time slice only.
// HBM per DOF: P_M, P_K, P_J read (24 B) + y written (8 B).
//
// Work unit = (strip of 8 spatial columns c of Q = n_1 n_2, direction-3 m-tile mt of 8 rows i_3).
// A warp sweeps the input time slices t' of its unit in order:
//   1. the band rows of P_M, P_K, P_J at slice t' (4 NKB rows x 8 c each) arrive in the warp's
//      shared-memory ring by cp.async, DEPTH - 1 slices ahead (no registers held in flight);
//   2. direction-3 DMMAs: v1, v2 (8 i_3 x 8 c, D fragments: lane holds i_3 = lane/4,
//      c = 2(lane%4) + h) from the band A-fragments of M_3, J_3, 2K_3 (registers for the unit)
//      and B fragments read from the ring;
//   3. the time product as a scatter with DFMAs, without padding waste or a transposition:
//      every output row t in [t' - p_t, t' + p_t] gets K_t[t][t'] v1 + M_t[t][t'] v2 in a
//      register ring of 2 p_t + 1 partial rows per element; row t' - p_t is then complete and
//      stored (+ v3 on row n_t - 1: W_t = e e^T).  The column band of K_t, M_t at t' is a
//      broadcast read from shared memory.  The slice loop is unrolled by the ring period, so
//      ring slots are static.
// Band blocks and geometry of direction 3 as matvec3_kernels.cuh (S0, OFF, NKB).  Neighbouring
// m-tiles of a strip re-read 2p rows of P_*: units are numbered m-tile fastest, so the warps of a
// CTA mostly share the strip and those rows come from L2.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "fd_kernels.cuh"  // dmma_8x8x4, cp_async_commit / cp_async_wait
#include "pdl.cuh"

namespace ls {

struct MV5Args {
  const double* in[3];   // P_M, P_K, P_J: [rows][n3][Q] (the plane pass' outputs)
  double* y;             // output rows [t_first, t_first + nout): [nout][n3][Q]
  const double* frag3;   // direction-3 band A-fragments [4: M, J, K, 2K][mt3][NKB][32]
  const double* tcol;    // time column bands [nt][40]: K_t[t' - p_t + k][t'] at k, M_t[..][t'] at 20 + k
  int n3, mt3;           // direction-3 extent and m-tiles
  int nt;                // global time extent
  uint32_t Q;            // n_1 n_2 (columns per (t, i_3) row)
  int s_first, rows;     // input slab: global time rows [s_first, s_first + rows)
  int t_first, nout;     // output rows (global)
  int vec16;             // 16-byte cp.async (Q even, inputs 16-byte aligned), else 8-byte
  // fused PCG scalar p.q (as MV3_T2): every stored y element times dotp at the same offset,
  // CTA sums to dot_part[blockIdx.x] (fixed grid: deterministic)
  const double* dotp;
  double* dot_part;
};

template <int P>
struct MV5Geo {
  static constexpr int S0 = (P % 4) ? (P % 4) - 8 : 0;
  static constexpr int OFF = (P - S0) / 4;
  static constexpr int NKB = 2 + (P + 1) / 2;
};

template <int P, int PT>
struct MV5Cfg {
  static constexpr int WARPS = 8;
  static constexpr int RB = 4 * MV5Geo<P>::NKB;      // band rows per input
  static constexpr int RS = 12;                      // ring row stride (doubles): conflict-free B reads
  static constexpr int DEPTH = RB >= 24 ? 3 : 4;     // slices in the cp.async ring (shared memory)
  static constexpr int SLICE = 3 * RB * RS;          // doubles per slice
  static constexpr int WARP_SMEM = DEPTH * SLICE;
  static constexpr int R = 2 * PT + 1;               // partial output rows per element
  static constexpr int TCOL = 40;                    // doubles per time slice in tcol (2 x 20)
  static size_t smem(int nt) { return (size_t(WARPS) * WARP_SMEM + size_t(nt) * TCOL) * sizeof(double); }
};

__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, int src_bytes) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}

template <int P, int PT>
__global__ void __launch_bounds__(256, 1) mv5_d3t_kernel(const __grid_constant__ MV5Args a) {
  using G3 = MV5Geo<P>;
  using Cf = MV5Cfg<P, PT>;
  constexpr int NKB = G3::NKB, RB = Cf::RB, RS = Cf::RS, DEPTH = Cf::DEPTH, R = Cf::R;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kq = lane & 3, nq = lane >> 2;
  double* ring = smem + warp * Cf::WARP_SMEM;
  double* tcs = smem + Cf::WARPS * Cf::WARP_SMEM;  // [nt][TCOL]
  const uint32_t Q = a.Q;
  const int n3 = a.n3, MT3 = a.mt3, nt = a.nt;
  const int64_t plane = int64_t(n3) * Q;  // one time slice
  const uint32_t nstrips = (Q + 7) / 8;
  const int64_t units = int64_t(nstrips) * MT3;
  const int t_end = a.s_first + a.rows;  // one past the last input slice (global)
  const int o_lo = a.t_first, o_hi = a.t_first + a.nout;  // own output rows
  for (int e = tid; e < nt * Cf::TCOL; e += 256) tcs[e] = __ldg(a.tcol + e);
  __syncthreads();
  double dacc = 0.0;
  pdl_wait();

  for (int64_t u = int64_t(blockIdx.x) * Cf::WARPS + warp; u < units; u += int64_t(gridDim.x) * Cf::WARPS) {
    const int mt = int(u % MT3);
    const uint32_t strip = uint32_t(u / MT3);
    const int row0 = 4 * (2 * mt - G3::OFF);  // first band row of direction 3
    // direction-3 band blocks of m-tile mt: M, J, K, 2K
    double A3[4][NKB];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
      for (int j = 0; j < NKB; ++j) A3[m][j] = __ldg(a.frag3 + ((m * MT3 + mt) * NKB + j) * 32 + lane);
    // cp.async of one slice's band rows into ring slot (slice - s_first) mod DEPTH: chunk e ->
    // (input m, row r, 16-byte part h) (vec16) or (m, r, column) (8-byte); rows outside [0, n3),
    // columns >= Q and slices past the slab are zero-filled
    int tload = a.s_first;
    auto issue = [&]() {
      double* dst = ring + ((tload - a.s_first) % DEPTH) * Cf::SLICE;
      const bool tok = tload < t_end;
      const int64_t toff = int64_t(tload - a.s_first) * plane;
      if (a.vec16) {
        for (int e = lane; e < 3 * RB * 4; e += 32) {
          const int m = e / (RB * 4), r = (e / 4) % RB, h = e % 4;
          const int row = row0 + r;
          const uint32_t c = strip * 8 + 2 * h;
          int bytes = 0;
          if (tok && row >= 0 && row < n3 && c < Q) bytes = (c + 1 < Q) ? 16 : 8;
          const double* src = a.in[m] + (bytes ? toff + int64_t(row) * Q + c : 0);
          cp_async16_zfill(dst + (m * RB + r) * RS + 2 * h, src, bytes);
        }
      } else {
        for (int e = lane; e < 3 * RB * 8; e += 32) {
          const int m = e / (RB * 8), r = (e / 8) % RB, h = e % 8;
          const int row = row0 + r;
          const uint32_t c = strip * 8 + h;
          const int bytes = (tok && row >= 0 && row < n3 && c < Q) ? 8 : 0;
          const double* src = a.in[m] + (bytes ? toff + int64_t(row) * Q + c : 0);
          cp_async8_zfill(dst + (m * RB + r) * RS + h, src, bytes);
        }
      }
      cp_async_commit();
      ++tload;
    };
#pragma unroll
    for (int s = 0; s < DEPTH - 1; ++s) issue();
    // partial output rows: yr[k] holds row t with t mod R == k (2 elements: c = 2kq + h)
    double yr[R][2];
#pragma unroll
    for (int k = 0; k < R; ++k) yr[k][0] = yr[k][1] = 0.0;
    double w3[2] = {0.0, 0.0};  // v3 (last time slice)
    const int i3 = 8 * mt + G3::S0 + nq;     // this lane's output row of direction 3
    const uint32_t cy = strip * 8 + 2 * kq;  // its output columns cy, cy + 1
    const bool lane_ok = i3 >= 0 && i3 < n3 && cy < Q;
    const bool two = cy + 1 < Q;
    // p of the row emitted at this slice (fused p.q), loaded before the slice's DMMAs
    auto pload = [&](int t, double (&pv)[2]) {
      pv[0] = pv[1] = 0.0;
      if (a.dotp && t >= o_lo && t < o_hi && t < nt && lane_ok) {
        const double* pp = a.dotp + int64_t(t - o_lo) * plane + int64_t(i3) * Q + cy;
        pv[0] = __ldg(pp);
        if (two) pv[1] = __ldg(pp + 1);
      }
    };
    // store row t (global) from a ring slot, then clear the slot
    auto emit = [&](double (&yk)[2], int t, const double (&pv)[2]) {
      if (t >= o_lo && t < o_hi && t < nt && lane_ok) {
        double y0 = yk[0], y1 = yk[1];
        if (t == nt - 1) {
          y0 += w3[0];
          y1 += w3[1];
        }
        double* o = a.y + int64_t(t - o_lo) * plane + int64_t(i3) * Q + cy;
        if (two && ((reinterpret_cast<uintptr_t>(o) & 15) == 0)) {
          *reinterpret_cast<double2*>(o) = make_double2(y0, y1);
        } else {
          o[0] = y0;
          if (two) o[1] = y1;
        }
        if (a.dotp) dacc = fma(y0, pv[0], fma(y1, pv[1], dacc));  // pv[1] = 0 when !two
      }
      yk[0] = yk[1] = 0.0;
    };
    // slices in order; the body is unrolled by R so that the rows touched at slice t' = t0 + s
    // sit in static ring slots: t0 is kept a multiple of R
    const int tb = a.s_first - ((a.s_first % R) + R) % R;  // first multiple of R <= s_first
    for (int t0 = tb; t0 < t_end; t0 += R) {
#pragma unroll
      for (int s = 0; s < R; ++s) {
        const int tp = t0 + s;  // global slice
        if (tp >= a.s_first && tp < t_end) {
          double pv[2];
          pload(tp - PT, pv);
          issue();  // slice tp + DEPTH - 1
          cp_async_wait<DEPTH - 1>();
          __syncwarp();
          const double* sl = ring + ((tp - a.s_first) % DEPTH) * Cf::SLICE;
          // 1. direction 3: v1 = M P_M; v2 = J P_M + M P_J + 2K P_K (four independent chains)
          double v1[2] = {0.0, 0.0}, v2a[2] = {0.0, 0.0}, v2b[2] = {0.0, 0.0}, v2c[2] = {0.0, 0.0};
#pragma unroll
          for (int j = 0; j < NKB; ++j) {
            const double* br = sl + (4 * j + kq) * RS + nq;
            const double bM = br[0], bK = br[RB * RS], bJ = br[2 * RB * RS];
            dmma_8x8x4(v1, A3[0][j], bM);
            dmma_8x8x4(v2a, A3[1][j], bM);
            dmma_8x8x4(v2b, A3[0][j], bJ);
            dmma_8x8x4(v2c, A3[3][j], bK);
          }
          if (tp == nt - 1) {  // W_t term: v3 = K P_M + M P_K on the last time slice
#pragma unroll
            for (int j = 0; j < NKB; ++j) {
              const double* br = sl + (4 * j + kq) * RS + nq;
              dmma_8x8x4(w3, A3[2][j], br[0]);
              dmma_8x8x4(w3, A3[0][j], br[RB * RS]);
            }
          }
          __syncwarp();  // every lane has read the slot before the next issue() refills it
          const double v2[2] = {v2a[0] + v2b[0] + v2c[0], v2a[1] + v2b[1] + v2c[1]};
          // 2. time scatter: row t = tp - PT + k gets K_t[t][tp] v1 + M_t[t][tp] v2 (zero bands
          //    outside [0, nt)); its ring slot is t mod R = (s + k - PT) mod R
          const double* tc = tcs + tp * Cf::TCOL;
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const double kt = tc[k], mtc = tc[20 + k];
            double(&yk)[2] = yr[(s + k - PT + 2 * R) % R];
            yk[0] = fma(kt, v1[0], fma(mtc, v2[0], yk[0]));
            yk[1] = fma(kt, v1[1], fma(mtc, v2[1], yk[1]));
          }
          // 3. row tp - PT is complete
          emit(yr[(s - PT + 2 * R) % R], tp - PT, pv);
        }
      }
    }
    // the rows still open after the last slice: t_end - PT .. t_end - 1 (rows past them get
    // nothing more from this slab and are not its own rows)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const int te = t_end - PT;
      const int t = te + ((k - te) % R + R) % R;  // the row in slot k among [te, te + R)
      if (t < t_end) {
        double pv[2];
        pload(t, pv);
        emit(yr[k], t, pv);
      }
    }
    cp_async_wait<0>();
    __syncwarp();  // the ring is reused by the warp's next unit
  }
  if (a.dotp) {  // CTA sum of the fused p.q in a fixed order
    __shared__ double red[Cf::WARPS];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dacc += __shfl_xor_sync(0xffffffffu, dacc, o);
    if (lane == 0) red[warp] = dacc;
    __syncthreads();
    if (tid == 0) {
      double s = 0.0;
#pragma unroll
      for (int w = 0; w < Cf::WARPS; ++w) s += red[w];
      a.dot_part[blockIdx.x] = s;
    }
  }
}

// host side (mv5.cu): launches the fused pass; *grid_out = the grid (dot partials)
cudaError_t mv5_run(const MV5Args& a, int p, int pt, int num_sms, cudaStream_t s, unsigned* grid_out);
bool mv5_supported(int p, int pt);

}  // namespace ls
