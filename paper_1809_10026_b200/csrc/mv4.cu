// ls_matvec v4 plane-pass launches (mv4_kernels.cuh), one translation unit of their own.
#include "mv4_kernels.cuh"

#include <algorithm>

namespace ls {

extern int g_mv4_ctas;

constexpr bool kPack = LS_MV4_PACK != 0;

template <int P, int CTAS>
static cudaError_t plane_c(const MV4PlaneArgs& a, int num_sms, cudaStream_t s) {
  // packed: one CTA of 16 warps in place of two of 8 (see mv4_kernels.cuh)
  constexpr int W = (kPack && CTAS == 2) ? 16 : 8;
  constexpr int C = (kPack && CTAS == 2) ? 1 : CTAS;
  const size_t smem = mv4_smem_doubles<P, kPack>(a.mt2) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(mv4_plane_kernel<P, C, kPack, W>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024 / C);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int ctas = C;
  // shared memory bounds the residency (228 KB per SM, 1 KB of it reserved per CTA)
  if (C > 1 && (smem + 1024) * C > 228 * 1024) ctas = 1;
  if (smem > 227 * 1024 / size_t(C)) return cudaErrorInvalidValue;
  const int64_t warps = a.nplanes * a.mt1;
  const unsigned grid = unsigned(std::min<int64_t>((warps + W - 1) / W, int64_t(num_sms) * ctas));
  if (grid == 0) return cudaSuccess;
  const cudaError_t e = launch_pdl(mv4_plane_kernel<P, C, kPack, W>, grid, 32 * W, smem, s, a);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int P>
static cudaError_t plane(const MV4PlaneArgs& a, int num_sms, cudaStream_t s) {
  return g_mv4_ctas == 2 ? plane_c<P, 2>(a, num_sms, s) : plane_c<P, 1>(a, num_sms, s);
}

int g_mv4_ctas = 2;

size_t mv4_plane_smem(int p, int mt2) {
  const size_t nkb = 2 + (p + 1) / 2;
  return (kPack ? mt2 * 32 * (2 * nkb + 4 * (nkb - 1)) : 4 * mt2 * nkb * 32) * sizeof(double);
}

cudaError_t mv4_plane_run(const MV4PlaneArgs& a, int p, int num_sms, cudaStream_t s) {
  switch (p) {
    case 2: return plane<2>(a, num_sms, s);
    case 3: return plane<3>(a, num_sms, s);
    case 4: return plane<4>(a, num_sms, s);
    case 5: return plane<5>(a, num_sms, s);
    case 6: return plane<6>(a, num_sms, s);
    case 7: return plane<7>(a, num_sms, s);
    case 8: return plane<8>(a, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ls
