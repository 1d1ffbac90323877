// Mapped spatial domains: the NURBS geometry map F,
// the physical spatial factors M_s, L_s, J_s of eq:A_kron (PAPER.md 686-703) assembled
// on the device in a per-row stencil layout, the stencil matvec, and the host setup of the
// geometry-aware preconditioner P^G (PAPER.md 969-1045).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "ls_api.h"

namespace ls {

// Host copy of the map (reading c19: tensor-product NURBS of its own degrees and knots).
struct GeoMap {
  int d = 0;
  int q[3] = {0, 0, 0};
  int m[3] = {1, 1, 1};
  std::vector<double> knots[3];
  std::vector<double> ctrl;  // [prod m][d], colex (direction 1 fastest)
  std::vector<double> w;     // [prod m], all 1 for a polynomial spline map
};

// Validates and copies the caller's description; LS_EINVAL on any inconsistency.
int geo_copy(const ls_geometry* g, int d, GeoMap& out);

// F(eta) and Jac[m][j] = dF_m / deta_j at one parametric point (host, 80-bit, rounded once).
void geo_eval(const GeoMap& g, const double* eta, double* x, double* jac);

// P^G univariate factors (readings c20-c22): midpoint coefficients c_tau, c_k, least-squares
// fit of their logarithms by alternating (Gauss-Seidel) sweeps, per-element mu_k, omega_k.
int pg_weights(const GeoMap& g, const int64_t* n_el, std::vector<double> mu[3], std::vector<double> om[3],
               double* fit_rel_res);

// Weighted constrained (i = 2..m-1) factors [M^G]_ij = int mu b_i b_j,
// [J^G]_ij = int omega b_i'' b_j'' (p+1 Gauss points per element, factors interpolated
// piecewise linearly between element midpoints; 80-bit sums rounded once).
void weighted_space_factors(int n_el, int p, const std::vector<double>& mu, const std::vector<double>& om,
                            std::vector<double>& M, std::vector<double>& J);

// Device data of the mapped-domain matvec.
struct GeoDev {
  int d = 0, p = 0, pt = 0;
  int n[3] = {1, 1, 1};       // constrained sizes n_1..n_d
  int nel[3] = {1, 1, 1};
  int64_t Ns = 0;
  int S = 0;                  // stencil width (2p+1)^d
  double* st = nullptr;       // [3][S][Ns]: M_s, J_s, L_s rows in stencil layout
  double* diag[3] = {nullptr, nullptr, nullptr};  // views of the centre entries
  int variant = 0;            // 0: DMMA band tiles (default), 1: DFMA stencil kernel
  double* lv = nullptr;        // ls_rhs kinds 2, 3: [4][N_s] spatial load integrals (geo_load)
  int lv_kind = 0;
  double fint[2] = {0.0, 0.0};  // int_Omega s_1^2, int_Omega s_2^2
  std::vector<void*> allocs;
  ~GeoDev();
};

// Assemble M_s, J_s, L_s on the device (one CTA per element, (p+1)^d launches over the
// element colour classes so that the stencil-row updates never collide: deterministic).  launches is incremented by the kernels launched.
int geo_assemble(GeoDev& gd, const GeoMap& g, int d, int p, const int64_t* n_el, cudaStream_t s,
                 int64_t* launches);

// Rows [t_first, t_first + nout) of y = (K_t (x) M_s + M_t (x) J_s + W_t (x) L_s) x,
// W_t = e_{n_t} e_{n_t}^T (T = 1), from the global rows [s_first, ...) of x held in x (a time
// slab with its halo; the whole vector with s_first = t_first = 0, nout = n_t on one GPU):
// banded time products into t1, t2 (nout * N_s each), then the stencil pass.
int geo_matvec(const GeoDev& gd, const double* bKt, const double* bMt, int nt_global, const double* x,
               int s_first, int t_first, int nout, double* y, double* t1, double* t2, cudaStream_t s,
               int64_t* launches);

// Spatial load integrals of the mapped-domain benchmarks (PAPER.md 1128-1129, 1219-1221):
// kind 2 (d = 2): u = P sin(pi t), s_1 = P, s_2 = -Lap P; kind 3 (d = 3): f = (P - Lap P) sin z.
// int s_m phi_i, int s_m Lap phi_i on Omega with p+5 Gauss points per element (reading c16)
// and int s_m^2; computed once per kind and cached in gd.  LS_ENOTSUP for another d.
int geo_load(GeoDev& gd, const GeoMap& g, const int64_t* n_el, int kind, cudaStream_t s, int64_t* launches);

// b on the slab rows [t0, t0 + nrows) from gd.lv and the time integrals G (device,
// [G0_1 | G1_1 | G0_2 | G1_2] x n_t): the load vector F(B_i) of PAPER.md 409.
int geo_rhs(const GeoDev& gd, const double* G, double* b, int t0, int nrows, int nt, cudaStream_t s,
            int64_t* launches);

// D^{-1/2} of P^G = D^{1/2} Pbar^G D^{1/2}, D_ii = A_ii / Pbar_ii, as an N-vector
// (diag(A) from the stencil centres and the banded time diagonals).
// for the slab rows [t0, t0 + nrows) of the global time axis
int pg_scaling(const GeoDev& gd, const double* bKt, const double* bMt, int nt, const double* pdiag_t,
               const double* pdiag_s, double* dm12, int t0, int nrows, cudaStream_t s, int64_t* launches);

// Host tables of one direction for qpe Gauss points per element (uniform open knots, 80-bit,
// rounded once): points xq and weights wq [n_el * qpe], and the p + 1 local B-splines' values,
// 1st and 2nd derivatives bt [n_el][qpe][p + 1][3] (full, unconstrained local numbering).
void dir_tables(int n_el, int p, int qpe, std::vector<double>& xq, std::vector<double>& wq,
                std::vector<double>& bt);

// Map data at the tensor Gauss points of the uniform meshes n_el (qpe per element and
// direction; device, allocations appended to `allocs`): qd = [16][NQ] with |det J| w_q,
// J^{-1}[3][3] (row j = grad eta_j), the Laplacian's first-order coefficients b[3], x[3].
int geo_point_data(const GeoMap& g, int d, int p, const int64_t* n_el, int qpe, std::vector<void*>& allocs,
                   cudaStream_t s, double** qd, int64_t* NQ, int64_t* launches);

// y = s * x elementwise (the D^{-1/2} pre / post scaling of the P^G application)
int scale_vec(const double* s_, const double* x, double* y, int64_t n, cudaStream_t s, int64_t* launches);

}  // namespace ls
