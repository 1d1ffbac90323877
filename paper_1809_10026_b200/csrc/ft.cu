// Instantiations and launcher of the fused time-mode kernel (fd_time_kernel.cuh).
#include <algorithm>

#include "fd_time_kernel.cuh"
#include "ft.hpp"

namespace ls {

template <class C>
static cudaError_t ft_launch_cfg(const FTArgs& a, cudaStream_t s, int num_sms) {
  static bool ready = false;
  if (!ready) {
    cudaError_t e = cudaFuncSetAttribute(fd_time_fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(C::SMEM));
    if (e != cudaSuccess) return e;
    ready = true;
  }
  const uint32_t ntw = (a.ncols + C::TW - 1) / C::TW;
  if (ntw == 0) return cudaSuccess;
  const unsigned grid = std::min<unsigned>((ntw + C::WARPS - 1) / C::WARPS, unsigned(num_sms * C::MINB));
  const cudaError_t e = launch_pdl(fd_time_fused_kernel<C>, grid, C::THREADS, C::SMEM, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

#ifndef LS_FT_D
#define LS_FT_D 6  // prefetch window (k-steps)
#endif
#ifndef LS_FT_D_SC
#define LS_FT_D_SC 8  // prefetch window of the single-copy buckets (config 4: 6 -> 8: 14.85 -> 14.79 ms)
#endif
#ifndef LS_FT_TAIL
#define LS_FT_TAIL 1  // DFMA tail tiles (FTCfg TAIL) where they apply
#endif
#ifndef LS_FT_TAIL_MAXV
#define LS_FT_TAIL_MAXV 4  // largest number of valid indices in a DFMA tail tile
#endif
#ifndef LS_FT_MINB2_MAXKS
#define LS_FT_MINB2_MAXKS 18  // buckets up to this KS run 2 CTAs per SM (<= 128 registers)
#endif

template <int KS>
static cudaError_t ft_launch_ks(const FTArgs& a, bool vec, cudaStream_t s, int num_sms) {
  if constexpr (KS > 26) {  // n_t > 104: the single swizzled copy of U_t (FTCfg SC), 1 CTA per SM
    if (vec) return ft_launch_cfg<FTCfg<KS, true, LS_FT_D_SC, 1, 0, true>>(a, s, num_sms);
    return ft_launch_cfg<FTCfg<KS, false, LS_FT_D_SC, 1, 0, true>>(a, s, num_sms);
  } else {
  // two CTAs per SM while both fragment sets and the accumulators fit (n_t <= 72)
  constexpr int MINB = KS <= LS_FT_MINB2_MAXKS ? 2 : 1;
  // DFMA tail when the last 8-wide tile of j / t' holds at most 4 valid indices
  constexpr int J0 = 8 * ((KS + 1) / 2 - 1);
  const int tv = a.nt - J0;  // valid indices in the last tile
  if (LS_FT_TAIL && J0 > 0 && tv >= 1 && tv <= LS_FT_TAIL_MAXV) {
    // the tail accumulators do not fit 128 registers above n_t = 36: 1 CTA per SM there
    constexpr int MINBT = KS <= 9 ? 2 : 1;
    if (tv <= 2) {
      if (vec) return ft_launch_cfg<FTCfg<KS, true, LS_FT_D, MINBT, 2>>(a, s, num_sms);
      return ft_launch_cfg<FTCfg<KS, false, LS_FT_D, MINBT, 2>>(a, s, num_sms);
    }
    if constexpr (LS_FT_TAIL_MAXV >= 3) {
      if (vec) return ft_launch_cfg<FTCfg<KS, true, LS_FT_D, MINBT, 4>>(a, s, num_sms);
      return ft_launch_cfg<FTCfg<KS, false, LS_FT_D, MINBT, 4>>(a, s, num_sms);
    }
  }
  if (vec) return ft_launch_cfg<FTCfg<KS, true, LS_FT_D, MINB>>(a, s, num_sms);
  return ft_launch_cfg<FTCfg<KS, false, LS_FT_D, MINB>>(a, s, num_sms);
  }
}

int ft_bucket(int nt) {
  static const int list[] = {LS_FT_BUCKETS};
  const int ks = (nt + 3) / 4;
  for (int v : list)
    if (ks <= v) return v;
  return -1;
}

cudaError_t ft_launch(const FTArgs& a, cudaStream_t s, int num_sms) {
  const bool vec = (a.ld % 2 == 0) && (a.ncols % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.Z) & 15) == 0);
  switch (ft_bucket(a.nt)) {
    case 3: return ft_launch_ks<3>(a, vec, s, num_sms);
    case 5: return ft_launch_ks<5>(a, vec, s, num_sms);
    case 9: return ft_launch_ks<9>(a, vec, s, num_sms);
    case 13: return ft_launch_ks<13>(a, vec, s, num_sms);
    case 17: return ft_launch_ks<17>(a, vec, s, num_sms);
    case 21: return ft_launch_ks<21>(a, vec, s, num_sms);
    case 25: return ft_launch_ks<25>(a, vec, s, num_sms);
    case 26: return ft_launch_ks<26>(a, vec, s, num_sms);
    case 30: return ft_launch_ks<30>(a, vec, s, num_sms);
    case 33: return ft_launch_ks<33>(a, vec, s, num_sms);
    case 34: return ft_launch_ks<34>(a, vec, s, num_sms);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ls
