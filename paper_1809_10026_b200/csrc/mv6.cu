// ls_matvec v6 launches (matvec6_kernels.cuh): DFMA stencil direction-3 and time passes.
#include <algorithm>

#include "matvec6_kernels.cuh"

namespace ls {

#ifndef LS_MV6_RD3
#define LS_MV6_RD3 12  // rows per warp item, direction-3 pass
#endif
#ifndef LS_MV6_RT
#define LS_MV6_RT 16  // rows per warp item, time pass
#endif

template <class K>
static unsigned persistent_grid(K k, uint64_t warps_needed, int num_sms, unsigned cap) {
  int occ = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, MV6_THREADS, 0) != cudaSuccess || occ < 1) occ = 1;
  const uint64_t want = (warps_needed + MV6_WARPS - 1) / MV6_WARPS;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>({want, uint64_t(num_sms) * occ, uint64_t(cap)})));
}

template <int P>
static cudaError_t run_d3(const MV6Args& a, int num_sms, cudaStream_t s) {
  constexpr int R = LS_MV6_RD3;
  const uint64_t items = uint64_t(a.rows) * ((a.Q + 31) / 32) * ((a.m.n + R - 1) / R);
  if (items == 0) return cudaSuccess;
  const unsigned g = persistent_grid(mv6_d3_kernel<P, R>, items, num_sms, 1u << 30);
  const cudaError_t e = launch_pdl(mv6_d3_kernel<P, R>, g, MV6_THREADS, 0, s, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <int P>
static cudaError_t run_time(const MV6Args& a, int num_sms, cudaStream_t s, unsigned* grid) {
  constexpr int R = LS_MV6_RT;
  const uint64_t items = uint64_t((a.Q + 31) / 32) * ((a.m.nout + R - 1) / R);
  *grid = 0;
  if (items == 0) return cudaSuccess;
  const unsigned g = persistent_grid(mv6_time_kernel<P, R>, items, num_sms, MV6_MAX_DOT_GRID);
  *grid = g;
  const cudaError_t e = launch_pdl(mv6_time_kernel<P, R>, g, MV6_THREADS, 0, s, a);
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t mv6_run_d3(const MV6Args& a, int p, int num_sms, cudaStream_t s) {
  switch (p) {
    case 2: return run_d3<2>(a, num_sms, s);
    case 3: return run_d3<3>(a, num_sms, s);
    case 4: return run_d3<4>(a, num_sms, s);
    case 5: return run_d3<5>(a, num_sms, s);
    case 6: return run_d3<6>(a, num_sms, s);
    case 7: return run_d3<7>(a, num_sms, s);
    case 8: return run_d3<8>(a, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t mv6_run_time(const MV6Args& a, int pt, int num_sms, cudaStream_t s, unsigned* grid) {
  switch (pt) {
    case 2: return run_time<2>(a, num_sms, s, grid);
    case 3: return run_time<3>(a, num_sms, s, grid);
    case 4: return run_time<4>(a, num_sms, s, grid);
    case 5: return run_time<5>(a, num_sms, s, grid);
    case 6: return run_time<6>(a, num_sms, s, grid);
    case 7: return run_time<7>(a, num_sms, s, grid);
    case 8: return run_time<8>(a, num_sms, s, grid);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ls
