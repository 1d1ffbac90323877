// Launcher of fd_mode_rd_kernel for one k-step bucket KS (explicitly
// instantiated per bucket in rd_ks*.cu so the buckets compile in parallel).
#pragma once
#include <cuda_runtime.h>

#include "fd_rd_kernel.cuh"

namespace ls {

// NT (n-tiles per warp) and the prefetch window D per k-step bucket.
template <int KS>
struct RDBucket {
  static constexpr int MT = (KS + 1) / 2;
  static constexpr int NT = 2;
  // prefetch window (k-steps): a tile's DMMA time shrinks with MT, so small extents need a
  // deeper window to keep enough bytes in flight
  static constexpr int D = MT >= 15 ? 4 : MT >= 10 ? 8 : 12;
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
  const unsigned grid = std::min<unsigned>((ntw + C::WARPS - 1) / C::WARPS, unsigned(num_sms));
  const cudaError_t e = launch_pdl(fd_mode_rd_kernel<C>, grid, C::THREADS, C::SMEM, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// mode1: contiguous mode (Q == 1); scale: fused Algorithm-1 step 3 (time mode, P == 1)
template <int KS>
cudaError_t rd_launch(const ModeArgs& a, bool mode1, bool scale, cudaStream_t s, int num_sms) {
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

#define LS_RD_BUCKETS(X) X(2) X(4) X(5) X(8) X(12) X(16) X(17) X(18) X(24) X(25) X(26) X(30) X(33) X(34)
#define LS_RD_DECL(K) extern template cudaError_t rd_launch<K>(const ModeArgs&, bool, bool, cudaStream_t, int);
LS_RD_BUCKETS(LS_RD_DECL)
#undef LS_RD_DECL

}  // namespace ls
