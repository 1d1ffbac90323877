// Discretisation-error norms: see err.cu and ls_error_norms in ls_api.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "ls_api.h"

namespace ls {

struct GeoMap;

struct ErrSetup {
  int d = 0, ps = 0, pt = 0, kind = 0, nt = 0;
  int64_t n_el[4] = {0, 0, 0, 0};  // directions 1..d, then time
  const GeoMap* gmap = nullptr;    // mapped domain, or nullptr for the cube
};

// out8 (host): the eight space-time integrals of err.cu's header for u_h = sum_i x_i B_i
// (x: device [n_t][N_s]).  Synchronous on stream s.  LS_ENOTSUP for kinds / dimensions
// without a built-in exact solution.
int error_norms(const ErrSetup& es, const double* x, cudaStream_t s, int64_t* launches, double* out8);

}  // namespace ls
