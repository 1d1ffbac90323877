// ls_matvec v3 launches (matvec3_kernels.cuh), one translation unit of their own.
#include "matvec3_kernels.cuh"

#include <algorithm>

namespace ls {

int mv3_nkb(int p) { return p <= 4 ? 4 : 6; }
int mv3_off(int p) { return p <= 4 ? 1 : 2; }
size_t mv3_frag_count(int p, int n, int nmat) { return size_t(nmat) * ((n + 7) / 8) * mv3_nkb(p) * 32; }

template <int P, int KIND, bool MODE1, bool FAST>
static cudaError_t launch(const MV3Args& a, int num_sms, cudaStream_t s) {
  constexpr int NT = 2;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(mv3_band_kernel<P, NT, KIND, MODE1, FAST>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const size_t smem = size_t(MV3IO<KIND>::NMAT) * a.mt * MV3Geom<P, KIND>::NKB * 32 * sizeof(double);
  const uint32_t nstrips = (a.ncols + 8 * NT - 1) / (8 * NT);
  const unsigned grid = std::min<unsigned>((nstrips + 7) / 8, unsigned(num_sms));
  if (grid == 0 || a.mt1 <= a.mt0) return cudaSuccess;
  mv3_band_kernel<P, NT, KIND, MODE1, FAST><<<grid, 256, smem, s>>>(a);
  return cudaGetLastError();
}

template <int P>
static cudaError_t run_pass(const MV3Pass& ps, int num_sms, cudaStream_t s) {
  const MV3Args& a = ps.args;
  const bool fast = !ps.mode1 && (a.Q % 4 == 0);  // NT = 2: Q % 2NT
  switch (ps.kind) {
    case MV3_TIME: return fast ? launch<P, MV3_TIME, false, true>(a, num_sms, s) : launch<P, MV3_TIME, false, false>(a, num_sms, s);
    case MV3_DIR: return fast ? launch<P, MV3_DIR, false, true>(a, num_sms, s) : launch<P, MV3_DIR, false, false>(a, num_sms, s);
    case MV3_DIR_A: return launch<P, MV3_DIR_A, true, false>(a, num_sms, s);
    case MV3_MID: return fast ? launch<P, MV3_MID, false, true>(a, num_sms, s) : launch<P, MV3_MID, false, false>(a, num_sms, s);
    case MV3_LAST: return launch<P, MV3_LAST, true, false>(a, num_sms, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t mv3_run(int p, const MV3Pass* passes, int npass, int num_sms, cudaStream_t s, int64_t* launches) {
  for (int i = 0; i < npass; ++i) {
    cudaError_t e;
    switch (p) {
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
