// Instantiations and launcher of the plane kernel (fd_plane_kernel.cuh): spatial modes 1 + 2
// of fd_apply in one launch (centrosymmetric split, n1 = n2).
#include <algorithm>

#include "fd_plane_kernel.cuh"
#include "pl.hpp"

namespace ls {

template <class C>
static cudaError_t pl_launch_cfg(const PLArgs& a0, cudaStream_t s, int num_sms) {
  const PLArgs& a = a0;
  const size_t smem = C::SMEM;
  static size_t ready = 0;
  if (ready < smem) {
    cudaError_t e = cudaFuncSetAttribute(fd_plane_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    ready = smem;
  }
  if (a.planes == 0) return cudaSuccess;
  int occ = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fd_plane_kernel<C>, C::THREADS, smem);
  if (e != cudaSuccess) return e;
  occ = std::max(occ, 1);
  const unsigned grid = std::min<unsigned>(a.planes, unsigned(num_sms * occ));
  e = launch_pdl(fd_plane_kernel<C>, grid, C::THREADS, smem, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// buckets (KS, NTH, MID): he = ceil(n/2) <= 4 KS, ho = floor(n/2) <= 8 NTH, MID = n odd
#define LS_PL_BUCKETS(X) \
  X(3, 1, 1) X(5, 2, 1) X(9, 4, 1) X(13, 6, 1) X(13, 7, 1) \
  X(2, 1, 0) X(4, 2, 0) X(8, 4, 0) X(12, 6, 0) X(13, 7, 0)

int pl_supported(int n) {
  const int he = (n + 1) / 2, ho = n / 2, mid = n & 1;
  const int ks = (he + 3) / 4, nth = (ho + 7) / 8;
#define LS_PL_FIND(K, T, M) \
  if (M == mid && ks <= K && nth <= T) return 1;
  LS_PL_BUCKETS(LS_PL_FIND)
#undef LS_PL_FIND
  return 0;
}

cudaError_t pl_launch(const PLArgs& a, bool fwd, cudaStream_t s, int num_sms) {
  const int n = a.n, he = (n + 1) / 2, ho = n / 2, mid = n & 1;
  const int ks = (he + 3) / 4, nth = (ho + 7) / 8;
#define LS_PL_GO(K, T, M)                                                                                  \
  if (M == mid && ks <= K && nth <= T) {                                                                   \
    constexpr int MINB = K <= 9 ? 2 : 1; /* two CTAs per SM while both fit (n <= 72) */      \
    return fwd ? pl_launch_cfg<PLCfg<K, T, M, true, MINB>>(a, s, num_sms)                                  \
               : pl_launch_cfg<PLCfg<K, T, M, false, MINB>>(a, s, num_sms);                                \
  }
  LS_PL_BUCKETS(LS_PL_GO)
#undef LS_PL_GO
  return cudaErrorInvalidValue;
}

}  // namespace ls
