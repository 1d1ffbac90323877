// ls_matvec v5 launches (mv5_kernels.cuh): the fused direction-3 + time pass, one translation unit.
#include "mv5_kernels.cuh"

#include <algorithm>

namespace ls {

template <int P>
static cudaError_t run(const MV5Args& a, int num_sms, cudaStream_t s, unsigned* grid_out) {
  using Cf = MV5Cfg<P, P>;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(mv5_d3t_kernel<P, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t smem = Cf::smem(a.nt);
  if (smem > 226 * 1024) return cudaErrorInvalidValue;
  const int64_t units = int64_t((a.Q + 7) / 8) * a.mt3;
  const unsigned grid = unsigned(std::min<int64_t>((units + Cf::WARPS - 1) / Cf::WARPS, num_sms));
  *grid_out = grid;
  if (grid == 0) return cudaSuccess;
  MV5Args b = a;
  b.vec16 = (a.Q % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.in[0]) | reinterpret_cast<uintptr_t>(a.in[1]) |
                                reinterpret_cast<uintptr_t>(a.in[2])) % 16 == 0);
  const cudaError_t e = launch_pdl(mv5_d3t_kernel<P, P>, grid, 256, smem, s, b);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool mv5_supported(int p, int pt) { return p == pt && p >= 2 && p <= 8; }

cudaError_t mv5_run(const MV5Args& a, int p, int pt, int num_sms, cudaStream_t s, unsigned* grid_out) {
  if (!mv5_supported(p, pt)) return cudaErrorInvalidValue;
  switch (p) {
    case 2: return run<2>(a, num_sms, s, grid_out);
    case 3: return run<3>(a, num_sms, s, grid_out);
    case 4: return run<4>(a, num_sms, s, grid_out);
    case 5: return run<5>(a, num_sms, s, grid_out);
    case 6: return run<6>(a, num_sms, s, grid_out);
    case 7: return run<7>(a, num_sms, s, grid_out);
    case 8: return run<8>(a, num_sms, s, grid_out);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ls
