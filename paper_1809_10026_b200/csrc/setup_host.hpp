// Host-side univariate setup: knots, Gauss-Legendre,
// B-spline evaluation and dense assembly of the univariate factor matrices.
// Everything here is O(n^2 p) per direction and runs once in ls_setup.
#pragma once
#include <cstdint>
#include <vector>

namespace ls {

// Open uniform knot vector on [0,1] with n_el elements (PAPER.md 144-147, 1111-1112).
std::vector<double> open_uniform_knots(int n_el, int p);
std::vector<long double> open_uniform_knots_ld(int n_el, int p);

// q-point Gauss-Legendre nodes/weights on [-1,1] (Newton on the Legendre recurrence),
// in 80-bit extended precision.
void gauss_legendre(int q, std::vector<long double>& x, std::vector<long double>& w);

// Values and first/second derivatives of all m = len(knots)-p-1 B-splines at x
// (Cox-de Boor, PAPER.md 148-166; derivative recursion of de Boor), extended precision.
void bspline_eval(const std::vector<long double>& knots, int p, long double x, long double* v0,
                  long double* v1, long double* v2);
void bspline_eval(const std::vector<double>& knots, int p, long double x, long double* v0,
                  long double* v1, long double* v2);

struct Factors {
  int n = 0;                   // constrained size
  std::vector<double> M, K, J; // dense n x n row-major; J empty for time
};

// Space pencil on the Dirichlet-constrained basis (i = 2..m-1): M, K (= int b'b'), J.
Factors space_factors(int n_el, int p);
// Time matrices on the initial-condition-constrained basis (i = 2..m): M_t^, K_t^.
Factors time_factors(int n_el, int p);

// Univariate load integrals for a separable forcing with q = p + 5 Gauss points
// per element (reading c16).  fn: 0 = sin(pi x), 1 = e^t, 2 = cos t + c sin t, 3 = cos(pi x), 4 = 1.
// Returns int fn b_i, int fn b_i', int fn b_i'' over the constrained basis.
void load_integrals(int n_el, int p, bool space, int fn, double c, std::vector<double>& i0,
                    std::vector<double>& i1, std::vector<double>& i2);

// K U = M U Lambda with U^T M U = I, lambda ascending (extended-precision Cholesky +
// cyclic Jacobi).  U row-major, column j = eigenvector j.  Returns 1 if M is not SPD.
int generalized_eig(const std::vector<double>& K, const std::vector<double>& M, int n,
                    std::vector<double>& lam, std::vector<double>& U);
// the same for a pencil given in extended precision (the centrosymmetric reductions of
// api.cu, formed in 80-bit from the fp64 matrices)
int generalized_eig(const std::vector<long double>& K, const std::vector<long double>& M, int n,
                    std::vector<double>& lam, std::vector<double>& U);

} // namespace ls
