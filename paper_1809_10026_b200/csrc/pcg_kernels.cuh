// PCG vector kernels (PAPER.md 710-712, 1109; textbook Hestenes-Stiefel).
// Scalars live on the device; alpha and beta are formed inside the update
// kernels from the reduced dot products, so an iteration needs one 8-byte
// device->host read (the stopping test).  Reductions are two-stage with a fixed
// grid, hence deterministic run to run.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pdl.cuh"

namespace ls {

constexpr int RED_THREADS = 256;
constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs; fixed for determinism

// scalar slots
enum { S_RHO0 = 0, S_RHO1 = 1, S_PQ = 2, S_RR = 3, S_BB = 4, S_ALPHA = 5, S_BETA = 6, S_AUX = 7, S_K = 8, S_STAT = 9,
       S_NSLOT = 10 };

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double sh[RED_THREADS / 32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  v = 0;
  if (threadIdx.x < 32) {
    v = threadIdx.x < RED_THREADS / 32 ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

// partials[blockIdx] = sum a*b over this block's grid-stride share
__global__ void __launch_bounds__(RED_THREADS) dot_partial_kernel(const double* __restrict__ a,
                                                                  const double* __restrict__ b,
                                                                  uint64_t n, double* partials) {
  pdl_wait();
  double s = 0;
  for (uint64_t i = blockIdx.x * uint64_t(RED_THREADS) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * RED_THREADS)
    s = fma(__ldg(a + i), __ldg(b + i), s);
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// scal[slot] = sum partials (single block, fixed order)
__global__ void __launch_bounds__(RED_THREADS) reduce_final_kernel(const double* partials, int np,
                                                                   double* scal, int slot) {
  pdl_wait();
  double s = 0;
  for (int i = threadIdx.x; i < np; i += RED_THREADS) s += partials[i];
  s = block_sum(s);
  if (threadIdx.x == 0) scal[slot] = s;
}

// alpha = rho/pq ; x += alpha p ; r -= alpha q ; partials <- r.r
__global__ void __launch_bounds__(RED_THREADS) update_xr_kernel(double* __restrict__ x, double* __restrict__ r,
                                                                const double* __restrict__ p,
                                                                const double* __restrict__ q, uint64_t n,
                                                                double* scal, int rho_slot,
                                                                double* partials) {
  pdl_wait();
  const double alpha = scal[rho_slot] / scal[S_PQ];
  if (blockIdx.x == 0 && threadIdx.x == 0) scal[S_ALPHA] = alpha;
  double s = 0;
  for (uint64_t i = blockIdx.x * uint64_t(RED_THREADS) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * RED_THREADS) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    s = fma(ri, ri, s);
  }
  s = block_sum(s);
  if (threadIdx.x == 0) partials[blockIdx.x] = s;
}

// beta = rho_new/rho_old ; p = z + beta p
__global__ void __launch_bounds__(RED_THREADS) update_p_kernel(double* __restrict__ p, const double* __restrict__ z,
                                                               uint64_t n, double* scal, int new_slot,
                                                               int old_slot) {
  pdl_wait();
  const double beta = scal[new_slot] / scal[old_slot];
  if (blockIdx.x == 0 && threadIdx.x == 0) scal[S_BETA] = beta;
  for (uint64_t i = blockIdx.x * uint64_t(RED_THREADS) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * RED_THREADS)
    p[i] = fma(beta, p[i], z[i]);
}

// graph-resident PCG (pcg_solve, one GPU): scal[S_RHO0] = scal[S_RHO1] after update_p, so
// the captured loop body uses fixed slots
__global__ void copy_slot_kernel(double* scal, int dst, int src) {
  pdl_wait(); scal[dst] = scal[src]; }

// end of a graph-resident iteration: k += 1 and the stopping test of the host loop
// (reading c7: ||r_k|| / ||b|| <= tol; NaN/Inf -> LS_ENUMERIC; k = max_iter -> LS_ENOCONV),
// written to scal[S_K], scal[S_STAT]; the WHILE node continues while the test fails
__global__ void pcg_check_kernel(double* scal, double tol, int max_iter, cudaGraphConditionalHandle h) {
  pdl_wait();
  const double k = scal[S_K] + 1.0;
  scal[S_K] = k;
  const double rr = scal[S_RR], alpha = scal[S_ALPHA];
  unsigned cont = 0;
  double stat;
  if (!isfinite(rr) || !isfinite(alpha)) {
    stat = 4.0;  // LS_ENUMERIC
  } else if (sqrt(rr) / sqrt(scal[S_BB]) <= tol) {
    stat = 0.0;  // LS_OK
  } else if (k >= double(max_iter)) {
    stat = 3.0;  // LS_ENOCONV
  } else {
    stat = 3.0;
    cont = 1;
  }
  scal[S_STAT] = stat;
  cudaGraphSetConditional(h, cont);
}

// y = a - b
__global__ void __launch_bounds__(RED_THREADS) sub_kernel(double* __restrict__ y, const double* __restrict__ a,
                                                          const double* __restrict__ b, uint64_t n) {
  pdl_wait();
  for (uint64_t i = blockIdx.x * uint64_t(RED_THREADS) + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * RED_THREADS)
    y[i] = a[i] - b[i];
}

// Lambda_s[s] = sum_k lambda_k[i_k(s)] for every spatial index s (colex), reading c3.
__global__ void lambda_s_kernel(double* out, const double* l1, const double* l2, const double* l3,
                                int n1, int n2, int d, uint64_t Ns) {
  for (uint64_t s = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; s < Ns;
       s += uint64_t(gridDim.x) * blockDim.x) {
    const int i1 = int(s % n1);
    double v = l1[i1];
    if (d >= 2) v += l2[int((s / n1) % n2)];
    if (d >= 3) v += l3[int(s / (uint64_t(n1) * n2))];
    out[s] = v;
  }
}

// b[t][s] = G1[t] S0(s) - G0[t] sum_k S0..S2_(k)..S0 (separable RHS, PAPER.md 409)
__global__ void rhs_outer_kernel(double* b, const double* G0, const double* G1, const double* S0,
                                 const double* S2, int d, int n1, int n2, int n3, uint64_t Ns,
                                 uint64_t total, uint64_t t0) {
  // S0/S2 are stacked per direction: S0 + k*nmax
  for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < total;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t t = e / Ns + t0;
    const uint64_t s = e % Ns;
    int idx[3] = {int(s % n1), d >= 2 ? int((s / n1) % n2) : 0,
                  d >= 3 ? int(s / (uint64_t(n1) * n2)) : 0};
    const int nn[3] = {n1, n2, n3};
    (void)nn;
    const int nmax = 256;
    double prod0 = 1.0;
    for (int k = 0; k < d; ++k) prod0 *= S0[k * nmax + idx[k]];
    double lap = 0.0;
    for (int k = 0; k < d; ++k) {
      double pr = S2[k * nmax + idx[k]];
      for (int l = 0; l < d; ++l)
        if (l != k) pr *= S0[l * nmax + idx[l]];
      lap += pr;
    }
    b[e] = G1[t] * prod0 - G0[t] * lap;
  }
}

} // namespace ls
