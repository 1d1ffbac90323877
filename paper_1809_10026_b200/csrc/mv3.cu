// ls_matvec v3 launches (matvec3_kernels.cuh), one translation unit of their own.
#include "matvec3_kernels.cuh"

#include <algorithm>

namespace ls {

int mv3_s0(int p) { return (p % 4) ? (p % 4) - 8 : 0; }
int mv3_nkb(int p) { return 2 + (p + 1) / 2; }
int mv3_off(int p) { return (p - mv3_s0(p)) / 4; }
int mv3_mt(int p, int n) { return (n - mv3_s0(p) + 7) / 8; }
size_t mv3_frag_count(int p, int n, int nmat) { return size_t(nmat) * mv3_mt(p, n) * mv3_nkb(p) * 32; }

template <int P, int KIND, bool MODE1, bool FAST>
static cudaError_t launch(const MV3Args& a, int num_sms, cudaStream_t s, unsigned* grid_out) {
#ifndef MV3_NT
#define MV3_NT 2
#endif
  constexpr int NT = MV3_NT;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mv3_band_kernel<P, NT, KIND, MODE1, FAST>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);  // + static (fused dot)
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t smem = size_t(MV3IO<KIND>::NMAT) * a.mt * MV3Geom<P, KIND>::NKB * 32 * sizeof(double);
  const uint32_t nstrips = (a.ncols + 8 * NT - 1) / (8 * NT);
  const unsigned grid = std::min<unsigned>((nstrips + 7) / 8, unsigned(num_sms * MV3Occ<KIND>::CTAS));
  *grid_out = (a.mt1 <= a.mt0) ? 0u : grid;
  if (grid == 0 || a.mt1 <= a.mt0) return cudaSuccess;
  {
    const cudaError_t e = launch_pdl(mv3_band_kernel<P, NT, KIND, MODE1, FAST>, grid, 256, smem, s, a);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

template <int P>
static cudaError_t run_pass(MV3Pass& ps, int num_sms, cudaStream_t s) {
  const MV3Args& a = ps.args;
  unsigned* g = &ps.grid;
  // NT = 2: 2-column loads / 4-column stores stay inside one row and 16-byte aligned
  const uint32_t qo = a.Qout ? a.Qout : a.Q;
  const bool fast = !ps.mode1 && (a.Q % (2 * MV3_NT) == 0) && (qo % (2 * MV3_NT) == 0) &&
                    (a.map_n1 == 0 || (a.map_n1 % 2 == 0 && a.map_n1p % 4 == 0));
  switch (ps.kind) {
    case MV3_TIME: return fast ? launch<P, MV3_TIME, false, true>(a, num_sms, s, g) : launch<P, MV3_TIME, false, false>(a, num_sms, s, g);
    case MV3_DIR: return fast ? launch<P, MV3_DIR, false, true>(a, num_sms, s, g) : launch<P, MV3_DIR, false, false>(a, num_sms, s, g);
    case MV3_DIR_A: return launch<P, MV3_DIR_A, true, false>(a, num_sms, s, g);
    case MV3_MID: return fast ? launch<P, MV3_MID, false, true>(a, num_sms, s, g) : launch<P, MV3_MID, false, false>(a, num_sms, s, g);
    case MV3_LAST: return launch<P, MV3_LAST, true, false>(a, num_sms, s, g);
    case MV3_D3: return fast ? launch<P, MV3_D3, false, true>(a, num_sms, s, g) : launch<P, MV3_D3, false, false>(a, num_sms, s, g);
    case MV3_T2: return fast ? launch<P, MV3_T2, false, true>(a, num_sms, s, g) : launch<P, MV3_T2, false, false>(a, num_sms, s, g);
    default: return cudaErrorInvalidValue;
  }
}

__global__ void mv3_pad_slice_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t nsp,
                                     int n1, int n1p) {
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < nsp; e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = e / n1p, r = e - row * n1p;
    dst[e] = r < n1 ? src[row * n1 + r] : 0.0;
  }
}

cudaError_t mv3_pad_slice(const double* src, double* dst, int64_t nsp, int n1, int n1p, cudaStream_t s,
                          int64_t* launches) {
  mv3_pad_slice_kernel<<<unsigned(std::min<int64_t>((nsp + 255) / 256, 148 * 8)), 256, 0, s>>>(src, dst, nsp, n1, n1p);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t mv3_run(MV3Pass* passes, int npass, int num_sms, cudaStream_t s, int64_t* launches) {
  for (int i = 0; i < npass; ++i) {
    cudaError_t e;
    switch (passes[i].p) {
      case 2: e = run_pass<2>(passes[i], num_sms, s); break;
      case 3: e = run_pass<3>(passes[i], num_sms, s); break;
      case 4: e = run_pass<4>(passes[i], num_sms, s); break;
      case 5: e = run_pass<5>(passes[i], num_sms, s); break;
      case 6: e = run_pass<6>(passes[i], num_sms, s); break;
      case 7: e = run_pass<7>(passes[i], num_sms, s); break;
      case 8: e = run_pass<8>(passes[i], num_sms, s); break;
      default: return cudaErrorInvalidValue;
    }
    if (e != cudaSuccess) return e;
    ++*launches;
  }
  return cudaSuccess;
}

}  // namespace ls
