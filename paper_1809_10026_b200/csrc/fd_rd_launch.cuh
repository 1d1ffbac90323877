// Launcher of fd_mode_rd_kernel for one k-step bucket KS (explicitly
// instantiated per bucket in rd_ks*.cu so the buckets compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "fd_rd_kernel.cuh"
#include "fd_rds_kernel.cuh"

namespace ls {

#define LS_RD_CS_MAXKS 17  // largest k-step bucket of the centrosymmetric split (n <= 136)
extern int g_rd_staged;  // ls_tune LS_TUNE_FD_STAGED (process-wide), api.cu
extern int g_rd_tail;    // ls_tune LS_TUNE_FD_TAIL (process-wide for the split kernels), api.cu
// tuning of the split kernels (variant builds: tools/rd_variant_libs.sh): n-tiles per warp,
// CTAs per SM, prefetch window (0 = the per-bucket rule in rd_launch_cs)
#ifndef LS_RD_CS_NT
#define LS_RD_CS_NT 0
#endif
#ifndef LS_RD_CS_MINB
#define LS_RD_CS_MINB 0
#endif
#ifndef LS_RD_CS_D
#define LS_RD_CS_D 0
#endif

// NT (n-tiles per warp) and the prefetch window D per k-step bucket.
template <int KS, int NH = 1>
struct RDBucket {
  static constexpr int MT = (KS + 1) / 2;
  static constexpr int NT = 2;
  // prefetch window (k-steps): a tile's DMMA time per k-step is NH * MT m-tiles, so small
  // extents need a deeper window to keep enough bytes in flight
  static constexpr int D = NH * MT >= 15 ? 4 : NH * MT >= 10 ? 8 : 12;
};

template <class C>
static cudaError_t rd_launch_cfg(const ModeArgs& a, cudaStream_t s, int num_sms) {
  static bool ready = false;
  if (!ready) {
    cudaError_t e = cudaFuncSetAttribute(fd_mode_rd_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(C::SMEM));
    if (e != cudaSuccess) return e;
    ready = true;
  }
  const uint32_t ntw = (a.ncols + C::TW - 1) / C::TW;
  if (ntw == 0) return cudaSuccess;
  const unsigned grid = std::min<unsigned>((ntw + C::WARPS - 1) / C::WARPS, unsigned(num_sms * C::MINB));
  const cudaError_t e = launch_pdl(fd_mode_rd_kernel<C>, grid, C::THREADS, C::SMEM, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// staged split kernel (fd_rds_kernel.cuh): n even, FAST or contiguous, local stores
template <class C>
static cudaError_t rds_launch_cfg(const ModeArgs& a, cudaStream_t s, int num_sms) {
  static bool ready = false;
  if (!ready) {
    cudaError_t e = cudaFuncSetAttribute(fd_mode_rds_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(C::SMEM));
    if (e != cudaSuccess) return e;
    ready = true;
  }
  const uint32_t ntw = (a.ncols + C::TW - 1) / C::TW;
  if (ntw == 0) return cudaSuccess;
  const unsigned grid = std::min<unsigned>((ntw + C::WARPS - 1) / C::WARPS, unsigned(num_sms * C::MINB));
  const cudaError_t e = launch_pdl(fd_mode_rds_kernel<C>, grid, C::THREADS, C::SMEM, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#ifndef LS_RDS_NT
#define LS_RDS_NT 1  // staged split kernel: n-tiles per warp (1: 2 CTAs per SM; 2: 1 CTA per SM, measured slower)
#endif
#ifndef LS_RDS_D
#define LS_RDS_D 0   // staged split kernel: ring depth (0: 12 at NT = 2, 6 / 8 at NT = 1)
#endif
#ifndef LS_RD_STAGED
#define LS_RD_STAGED 1  // the staged split kernel where it applies (n even, FAST / contiguous)
#endif

// centrosymmetric split (cs = 1 fold / 2 unfold; KS = k-steps of the half extent ceil(n/2))
template <int KS>
cudaError_t rd_launch_cs(const ModeArgs& a, bool mode1, int cs, cudaStream_t s, int num_sms) {
  if constexpr (KS > LS_RD_CS_MAXKS) {
    return cudaErrorInvalidValue;
  } else {
    if (LS_RD_STAGED && g_rd_staged && a.n % 2 == 0 && !a.remote) {
      const bool fast16 = !mode1 && (a.Q % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                          ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0);
      // NT n-tiles per warp, MINB CTAs per SM, ring depth DS (within 227 KB of shared memory)
      constexpr int NTS = LS_RDS_NT, MBS = NTS == 2 ? 1 : 2;
      constexpr int DS = LS_RDS_D > 0 ? LS_RDS_D : (NTS == 2 ? 12 : (KS >= 16 ? 6 : 8));
      if (mode1) {
        if (cs == 1) return rds_launch_cfg<RDSCfg<KS, true, 1, DS, NTS, MBS>>(a, s, num_sms);
        return rds_launch_cfg<RDSCfg<KS, true, 2, DS, NTS, MBS>>(a, s, num_sms);
      }
      if (fast16 && a.Q % (2 * NTS) == 0) {
        if (cs == 1) return rds_launch_cfg<RDSCfg<KS, false, 1, DS, NTS, MBS>>(a, s, num_sms);
        return rds_launch_cfg<RDSCfg<KS, false, 2, DS, NTS, MBS>>(a, s, num_sms);
      }
    }
    // measured (tools/rd_variant_libs.sh + tools/ab_fd.py): half extents up to 52
    // (configs 3, 5) run 1 n-tile per warp, 2 CTAs per SM, (window 4 until r02); above (config 4, he = 66) 2
    // n-tiles per warp, 1 CTA per SM; window 6 for both
    constexpr bool SMALL = KS <= 13;
    constexpr int NT = LS_RD_CS_NT > 0 ? LS_RD_CS_NT : (SMALL ? 1 : 2);
    constexpr int MB = LS_RD_CS_MINB > 0 ? LS_RD_CS_MINB : (SMALL ? 2 : 1);
    constexpr int D = LS_RD_CS_D > 0 ? LS_RD_CS_D : 6;  // r02: window 6 also for SMALL (4 -> 6: config 3 -0.6 %, config 5 -0.2..-0.9 %)
    const bool fast = !mode1 && (a.Q % (2 * NT) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                      ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0);
    // DFMA tail rows (RDCfg::TR): half extents 8(MT - 1) + 1 or + 2 in an odd k-step bucket
    // (he = 66: config 4; 33: configs 2, 3; 49: config 5 p = 4), local stores
    if constexpr (KS % 2 == 1 && KS >= 5) {
      const int he = (a.n + 1) / 2;
      if (g_rd_tail && !a.remote && he - 8 * ((KS + 1) / 2 - 1) <= 2 && he > 8 * ((KS + 1) / 2 - 1)) {
        if (cs == 1) {
          if (mode1) return rd_launch_cfg<RDCfg<KS, NT, true, false, false, D, 0, 1, MB, 2>>(a, s, num_sms);
          if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 0, 1, MB, 2>>(a, s, num_sms);
          return rd_launch_cfg<RDCfg<KS, NT, false, false, false, D, 0, 1, MB, 2>>(a, s, num_sms);
        }
        if (mode1) return rd_launch_cfg<RDCfg<KS, NT, true, false, false, D, 0, 2, MB, 2>>(a, s, num_sms);
        if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 0, 2, MB, 2>>(a, s, num_sms);
        return rd_launch_cfg<RDCfg<KS, NT, false, false, false, D, 0, 2, MB, 2>>(a, s, num_sms);
      }
    }
    if (cs == 1) {
      if (a.remote == 1) {
        if (!fast) return cudaErrorInvalidValue;
        return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 1, 1, MB>>(a, s, num_sms);
      }
      if (a.remote) return cudaErrorInvalidValue;
      if (mode1) return rd_launch_cfg<RDCfg<KS, NT, true, false, false, D, 0, 1, MB>>(a, s, num_sms);
      if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 0, 1, MB>>(a, s, num_sms);
      return rd_launch_cfg<RDCfg<KS, NT, false, false, false, D, 0, 1, MB>>(a, s, num_sms);
    }
    if (a.remote) return cudaErrorInvalidValue;
    if (mode1) return rd_launch_cfg<RDCfg<KS, NT, true, false, false, D, 0, 2, MB>>(a, s, num_sms);
    if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 0, 2, MB>>(a, s, num_sms);
    return rd_launch_cfg<RDCfg<KS, NT, false, false, false, D, 0, 2, MB>>(a, s, num_sms);
  }
}

// mode1: contiguous mode (Q == 1); scale: fused Algorithm-1 step 3 (time mode, P == 1)
template <int KS>
cudaError_t rd_launch(const ModeArgs& a, bool mode1, bool scale, int cs, cudaStream_t s, int num_sms) {
  if (cs) return scale ? cudaErrorInvalidValue : rd_launch_cs<KS>(a, mode1, cs, s, num_sms);
  using B = RDBucket<KS>;
  constexpr int NT = B::NT, D = B::D;
  if (mode1) return a.remote ? cudaErrorInvalidValue : rd_launch_cfg<RDCfg<KS, NT, true, false, false, D>>(a, s, num_sms);
  const bool fast = (a.Q % (2 * NT) == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0);
  if (a.remote) {  // fused all-to-all epilogues exist for unscaled FAST launches only
    if (!fast || scale) return cudaErrorInvalidValue;
    if (a.remote == 1) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 1>>(a, s, num_sms);
    return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D, 2>>(a, s, num_sms);
  }
  if (scale) {
    if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, true, true, D>>(a, s, num_sms);
    return rd_launch_cfg<RDCfg<KS, NT, false, true, false, D>>(a, s, num_sms);
  }
  if (fast) return rd_launch_cfg<RDCfg<KS, NT, false, false, true, D>>(a, s, num_sms);
  return rd_launch_cfg<RDCfg<KS, NT, false, false, false, D>>(a, s, num_sms);
}

// k-step buckets (the CS half extents ceil(n/2) <= 68 use the buckets up to 17; 9 and 13 are
// there for them: n = 65..72 and 97..104)
#define LS_RD_BUCKETS(X) X(2) X(4) X(5) X(8) X(9) X(12) X(13) X(16) X(17) X(18) X(24) X(25) X(26) X(30) X(33) X(34)
#define LS_RD_DECL(K) extern template cudaError_t rd_launch<K>(const ModeArgs&, bool, bool, int, cudaStream_t, int);
LS_RD_BUCKETS(LS_RD_DECL)
#undef LS_RD_DECL

}  // namespace ls
