// ls_matvec v2 launches (matvec2_kernels.cuh), one translation unit of their own.
#include "matvec2_kernels.cuh"

#include <algorithm>

namespace ls {

#ifndef LS_MV2_SWEEP_D
#define LS_MV2_SWEEP_D 2  // rows loaded ahead by the sweep plane pass (A/B: 2 best of 2, 4, 6)
#endif

template <int P>
static cudaError_t run_time(const MV2Plan& pl, int64_t* launches) {
  constexpr int R = 8;
  if (pl.grid_time) {
    const cudaError_t e0 = launch_pdl(mv_time_kernel<P, R>, dim3(pl.grid_time, (pl.time.nout + R * MV_CY - 1) / (R * MV_CY)),
                                      dim3(32, MV_CY), 0, pl.stream, pl.time);
    if (e0 != cudaSuccess) return e0;
    ++*launches;
    return cudaGetLastError();
  }
  return cudaSuccess;
}

template <int P>
static cudaError_t run_p(const MV2Plan& pl, int64_t* launches) {
  constexpr int R = 8;
  cudaError_t e;
  if (pl.grid_dir) {
    const dim3 g(pl.grid_dir, (pl.dir.n + R * MV_CY - 1) / (R * MV_CY));
    e = (pl.d == 1) ? launch_pdl(mv_dir_kernel<P, R, true>, g, dim3(32, MV_CY), 0, pl.stream, pl.dir)
                    : launch_pdl(mv_dir_kernel<P, R, false>, g, dim3(32, MV_CY), 0, pl.stream, pl.dir);
    if (e != cudaSuccess) return e;
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (pl.d == 3 && pl.sweep_cw > 0 && pl.grid_plane) {
    e = cudaErrorInvalidValue;
    if constexpr (P == 2) {
      switch (pl.sweep_cw) {
        case 2: e = launch_pdl(mv_sweep_kernel<P, 2, LS_MV2_SWEEP_D>, pl.grid_plane, 256, 0, pl.stream, pl.plane); break;
        case 3: e = launch_pdl(mv_sweep_kernel<P, 3, LS_MV2_SWEEP_D>, pl.grid_plane, 256, 0, pl.stream, pl.plane); break;
        case 4: e = launch_pdl(mv_sweep_kernel<P, 4, LS_MV2_SWEEP_D>, pl.grid_plane, 256, 0, pl.stream, pl.plane); break;
        default: break;
      }
    }
    if (e != cudaSuccess) return e;
    ++*launches;
    return cudaGetLastError();
  }
  if (pl.d >= 2 && pl.grid_plane) {
    static bool attr[2] = {false, false};
    const int ph = pl.d == 3;
    if (!attr[ph]) {
      e = ph ? cudaFuncSetAttribute(mv_plane_kernel<P, R, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024)
             : cudaFuncSetAttribute(mv_plane_kernel<P, R, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      if (e != cudaSuccess) return e;
      attr[ph] = true;
    }
    e = ph ? launch_pdl(mv_plane_kernel<P, R, true>, pl.grid_plane, MV_PLANE_THREADS, pl.smem_plane, pl.stream, pl.plane)
           : launch_pdl(mv_plane_kernel<P, R, false>, pl.grid_plane, MV_PLANE_THREADS, pl.smem_plane, pl.stream, pl.plane);
    if (e != cudaSuccess) return e;
    ++*launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#ifndef LS_MV4_SWEEP_D
#define LS_MV4_SWEEP_D 2  // rows of x loaded ahead by the v4 sweep plane pass
#endif

template <int P, int CW>
static cudaError_t sweep4(const MVArgs& a, int num_sms, cudaStream_t s) {
  if (a.ncols == 0) return cudaSuccess;
  const unsigned grid = unsigned(std::min<uint64_t>((uint64_t(a.ncols) + 7) / 8, uint64_t(num_sms)));
  const cudaError_t e = launch_pdl(mv4_sweep_kernel<P, CW, LS_MV4_SWEEP_D>, grid, 256, 0, s, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t mv4_sweep_run(const MVArgs& a, int p, int cw, int num_sms, cudaStream_t s) {
  if (p == 3 && cw == 3) return sweep4<3, 3>(a, num_sms, s);
  if (p == 3 && cw == 4) return sweep4<3, 4>(a, num_sms, s);
  if (p == 4 && cw == 4) return sweep4<4, 4>(a, num_sms, s);
  return cudaErrorInvalidValue;
}

cudaError_t mv2_run(int p, int pt, const MV2Plan& plan, int64_t* launches) {
  cudaError_t e;
  switch (pt) {  // time pass: the time degree
    case 2: e = run_time<2>(plan, launches); break;
    case 3: e = run_time<3>(plan, launches); break;
    case 4: e = run_time<4>(plan, launches); break;
    case 5: e = run_time<5>(plan, launches); break;
    case 6: e = run_time<6>(plan, launches); break;
    case 7: e = run_time<7>(plan, launches); break;
    case 8: e = run_time<8>(plan, launches); break;
    default: return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  switch (p) {  // spatial passes: the space degree
    case 2: return run_p<2>(plan, launches);
    case 3: return run_p<3>(plan, launches);
    case 4: return run_p<4>(plan, launches);
    case 5: return run_p<5>(plan, launches);
    case 6: return run_p<6>(plan, launches);
    case 7: return run_p<7>(plan, launches);
    case 8: return run_p<8>(plan, launches);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ls
