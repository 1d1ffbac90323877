/*
 * ls_api.h -- C-ABI of the B200-native hot path of the space-time
 * least-squares isogeometric method for the heat equation
 * (Montardini, Negri, Sangalli, Tani, arXiv 1809.10026; PAPER.md = the paper).
 *
 * Problem (PAPER.md 343-353, eq:heat_eq): d_t u - Lap u = f on the
 * identity-mapped unit hypercube [0,1]^d x [0,T], T = 1 (reading c9), or on a
 * mapped domain Omega = F([0,1]^d) (ls_setup_geo), homogeneous Dirichlet and
 * initial data.  Discretisation: tensor B-splines of
 * degree p, C^{p-1}, n_el uniform elements per direction (PAPER.md 144-213,
 * 1111-1112); space basis i_k = 2..m_k-1, time basis i_t = 2..m_t
 * (eq:basis_par, PAPER.md 266-267), so n_k = n_el,k + p - 2 and
 * n_t = n_el,t + p - 1 (reading c1).
 *
 * VECTOR LAYOUT (all entry points): a vector of N = n_t * n_d * ... * n_1
 * fp64 values in the colexicographic DOF order of PAPER.md 271-285, i.e. the
 * row-major tensor [n_t][n_d]...[n_1] with direction 1 contiguous and time
 * slowest.  Flat index = i_1 + n_1 (i_2 + n_2 (... + n_d i_t)).
 * For a distributed context (ls_setup_dist) each rank holds the contiguous
 * time slab [t0, t0 + nt_local) of that tensor (see ls_layout).
 *
 * OWNERSHIP: vectors passed to fd_apply / ls_matvec / ls_rhs / pcg_solve are
 * caller-owned DEVICE memory (cudaMalloc / torch CUDA tensors), 8-byte
 * aligned, not overlapping partially.  The *_host variants take caller-owned
 * HOST memory (pinned recommended).  The library owns everything else
 * (eigenvectors, eigenvalues, banded factors, workspaces); all allocation
 * happens in ls_setup*, none in the hot calls.
 *
 * STREAMS: every device call is enqueued on the stream set by ls_set_stream
 * (default: the legacy default stream).  fd_apply / ls_matvec / ls_rhs are
 * asynchronous; pcg_solve and the *_host calls are synchronous.
 *
 * ERRORS: every int-returning call returns LS_OK (0) or one of the codes
 * below; ls_strerror maps a code to a static string.  A failed call leaves
 * the output unspecified and the context usable unless LS_ECUDA is returned.
 * Not thread-safe per context; one context per device, and one device per process (the
 * kernels' shared-memory attributes are set once per process, on the first launch; the
 * multi-GPU path runs one process per GPU).
 */
#ifndef LS_API_H
#define LS_API_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LS_OK 0
#define LS_EINVAL 1     /* bad argument: d not in {1,2,3}, p < 2, n_el < 1, null/misaligned ptr */
#define LS_ENOTSPD 2    /* Cholesky failure of a mass matrix in the generalized eigensolver */
#define LS_ENOCONV 3    /* PCG did not reach tol within max_iter (stats still filled) */
#define LS_ENUMERIC 4   /* NaN/Inf in a PCG scalar (alpha, beta) */
#define LS_ENOMEM 5     /* estimated device memory exceeds the free HBM; refused up front */
#define LS_ECUDA 6      /* CUDA runtime error */
#define LS_ENCCL 7      /* NCCL error (distributed contexts) */
#define LS_ENOTSUP 8    /* operation not supported for this context */

typedef struct ls_ctx ls_ctx; /* opaque, library-owned */

typedef struct {
  int iters;           /* number of A-products performed (reading c7) */
  double rel_res;      /* final recurrence residual ||r_k|| / ||b|| */
  double true_rel_res; /* ||b - A x|| / ||b|| recomputed after the loop */
  int status;          /* LS_OK, LS_ENOCONV or LS_ENUMERIC */
} ls_pcg_stats;

/*
 * ls_setup -- build the method's univariate data on the current CUDA device.
 *   d        : number of space dimensions, 1..3 (PAPER.md 175-178).
 *   p        : spline degree p_s = p_t >= 2 (Assumption 2, PAPER.md 218-223).
 *   n_elems  : host array of d+1 element counts; n_elems[k-1] = direction k,
 *              n_elems[d] = time (PAPER.md 179-180 orders p = (p_s, p_t)).
 *   out      : receives the new context.
 * Work (untimed setup): open uniform knots,
 * Gauss-Legendre assembly of M_k, K_k, J_k (space) and M_t, K_t, W_t (time)
 * on the host in 80-bit extended precision, rounded once to fp64 (PAPER.md
 * 686-703, 738-757; reading c17); generalized eigendecompositions
 * J_k U_k = M_k U_k Lambda_k, K_t U_t = M_t U_t Lambda_t with U^T M U = I
 * (eq:eig_dec, PAPER.md 939-945) by extended-precision Cholesky + cyclic Jacobi
 * on the host (O(n^3), n <= 136); upload of U, U^T, Lambda; workspace
 * allocation.  Extents: every n_k and n_t must be <= 136.
 * Errors: LS_EINVAL, LS_ENOTSPD, LS_ENOMEM, LS_ECUDA.
 */
int ls_setup(int d, int p, const int64_t* n_elems, ls_ctx** out);

/*
 * ls_setup_deg -- as ls_setup with separate degrees in space and time, p = (p_s, p_t)
 * (PAPER.md 179-180; e.g. p_s = p_t + 1 as in Fig. 2b, PAPER.md 1132): p_s >= 2
 * (Assumption 2), 1 <= p_t; n_k = n_el,k + p_s - 2, n_t = n_el,t + p_t - 1.  ls_matvec
 * supports p_s, p_t <= 8.  ls_setup(d, p, ...) is ls_setup_deg(d, p, p, ...).
 */
int ls_setup_deg(int d, int p_s, int p_t, const int64_t* n_elems, ls_ctx** out);

/*
 * ls_setup_dist -- as ls_setup, for rank `rank` of `world` processes (one
 * GPU each).  The time axis is split into contiguous slabs (uneven allowed);
 * fd_apply reshards slab <-> spatial chunk with two NCCL all-to-alls for the
 * time mode, ls_matvec exchanges p halo time slices with the neighbour ranks,
 * pcg_solve all-reduces its scalars.  nccl_unique_id: 128 bytes produced by
 * ls_get_unique_id on rank 0 and broadcast by the caller.
 * Errors: as ls_setup plus LS_ENCCL.
 */
int ls_setup_dist(int d, int p, const int64_t* n_elems, int rank, int world,
                  const void* nccl_unique_id, ls_ctx** out);
int ls_setup_dist_deg(int d, int p_s, int p_t, const int64_t* n_elems, int rank, int world,
                      const void* nccl_unique_id, ls_ctx** out);
int ls_get_unique_id(void* out128);

/*
 * ls_layout -- sizes: n_t, n_s[0..d-1] (= n_1..n_d), and this rank's time slab
 * [t0, t0 + nt_local) (t0 = 0, nt_local = n_t for ls_setup).  Any output
 * pointer may be NULL.
 */
int ls_layout(const ls_ctx* ctx, int64_t* n_t, int64_t* n_s, int64_t* t0, int64_t* nt_local);

/* ls_set_stream -- enqueue subsequent work on `cuda_stream` (a cudaStream_t). */
int ls_set_stream(ls_ctx* ctx, void* cuda_stream);

/*
 * fd_apply -- z = P^{-1} r, Algorithm 1 steps 2-4 (PAPER.md 955-964):
 *   s~ = (U_t (x) U_s)^T r ; q~ = (Lambda_t (x) I + I (x) Lambda_s)^{-1} s~ ;
 *   z = (U_t (x) U_s) q~,
 * with P = K_t^ (x) M_s^ + M_t^ (x) J_s~ (eq:preconditioner, PAPER.md 733).
 * r, z: device vectors of this rank's slab (layout above).  z == r (in place)
 * is allowed.  Asynchronous on the context stream.
 */
int fd_apply(ls_ctx* ctx, const double* r, double* z);

/*
 * fd_apply_stage -- one stage of fd_apply on a caller-chosen piece, i.e. what every rank
 * of ls_setup_dist runs between its all-to-alls (for custom decompositions):
 *   stage 0: forward spatial modes  X x_1 U_1^T .. x_d U_d^T  on a = #time slices of
 *            in/out ([a][N_s], 1 <= a <= slab length);  stage 2: backward (U_d .. U_1);
 *   stage 1: time mode of a spatial chunk [n_t][b] whose first spatial index is a:
 *            U_t^T, divide by lambda_t[i_t] + Lambda_s[a + j] (Alg. 1 step 3), U_t.
 * in and out must not overlap.  Asynchronous.  Errors: LS_EINVAL.
 */
int fd_apply_stage(ls_ctx* ctx, int stage, const double* in, double* out, int64_t a, int64_t b);

/*
 * fd_apply_scatter -- the two fused-all-to-all stages of the distributed fd_apply for rank
 * `me` of `world`, with caller-given destination buffers (dst_host: host array of `world`
 * device pointers; the same stores a multi-GPU run makes into peer memory):
 *   stage 0: forward spatial modes of rank me's slab `in` ([a][N_s], a = its slab length
 *            under ls_partition(n_t, world)); the last mode writes element (t, s) into
 *            dst[h][(t0_me + t) * ld_h + s - c0_h], h = owner of s, ld_h = 4*ceil(len_h/4);
 *   stage 1: time mode of rank me's chunk `in` ([n_t][ld_me], a = c0_me, b = len_me under
 *            ls_partition(N_s, world)); the backward time mode writes element (t, j) into
 *            dst[g][(t - t0_g) * N_s + c0_me + j], g = owner of t.
 * Asynchronous.  Errors: LS_EINVAL (geometry), LS_ENOTSUP (d = 1 or a mode stride not a
 * multiple of 4).
 */
int fd_apply_scatter(ls_ctx* ctx, int stage, const double* in, int64_t a, int64_t b, int world, int me,
                     double* const* dst_host);

/*
 * ls_matvec -- y = A x, A = K_t (x) M_s + M_t (x) J_s + W_t (x) L_s
 * (eq:A_kron, PAPER.md 686-703), matrix-free and sum-factorised on the banded
 * univariate factors (identity map).  x, y: device vectors, y != x.
 * Asynchronous on the context stream.
 */
int ls_matvec(ls_ctx* ctx, const double* x, double* y);

/*
 * ls_matvec_slab -- the slab-local kernel of ls_matvec (the part every rank runs after
 * its halo exchange), exposed so a caller can drive its own time decomposition:
 * y = rows [t_first, t_first + nout) of A x, given the rows [s_first, s_first + s_rows)
 * of x in x_ext ([s_rows][N_s], device).  The stored rows must include the time band
 * of the outputs, [max(0, t_first - p), min(n_t, t_first + nout + p)); nout must not
 * exceed this context's slab length and s_rows its slab length + 2p.  y: [nout][N_s]
 * device.  Asynchronous.  Errors: LS_EINVAL (geometry), LS_ENOTSUP (p > 8).
 */
int ls_matvec_slab(ls_ctx* ctx, const double* x_ext, int64_t s_first, int64_t s_rows, double* y,
                   int64_t t_first, int64_t nout);
/*
 * ls_matvec_slab3 -- ls_matvec_slab with the stored rows in three separate device buffers, as
 * the distributed ls_matvec holds them (no copy of x into a halo-extended buffer): rows
 * [s_first, s_first + lo) in x_lo ([lo][N_s]), the next `own` rows in x_own, the last `hi` rows
 * in x_hi; s_rows = lo + own + hi, same requirements and outputs as ls_matvec_slab.  The v4
 * path (d >= 2, 3 <= p <= 8) reads the three buffers directly (own rows first: in the
 * distributed ls_matvec the halo exchange overlaps that plane pass); other paths gather the
 * rows into a workspace first.  A buffer may be null when its row count is 0.
 */
int ls_matvec_slab3(ls_ctx* ctx, const double* x_lo, int64_t lo, const double* x_own, int64_t own,
                    const double* x_hi, int64_t hi, int64_t s_first, double* y, int64_t t_first, int64_t nout);

/*
 * ls_rhs -- b_i = F(B_i) = int int f (d_t B_i - Lap B_i) (PAPER.md 409) for a
 * built-in separable forcing (reading c11):
 *   kind 0: f = e^t prod_k sin(pi x_k)                        (BASELINE config 2)
 *   kind 1: f = prod_k sin(pi x_k) (cos t + d pi^2 sin t)     (cube, PAPER.md 1166)
 *   kind 2: mapped 2D domains only (ls_setup_geo, d = 2): f = (d_t - Lap) u for
 *           u = -(x^2+y^2-1)(x^2+y^2-4) x y^2 sin(pi t) (quarter annulus, PAPER.md 1129)
 *   kind 3: mapped 3D domains only (d = 3): f = -Lap u for the time-independent
 *           u = -(x^2+y^2-1)(x^2+y^2-4) x y^2 sin(z) of the rotated quarter annulus
 *           (PAPER.md 1221), with homogeneous boundary / initial data (DESIGN.md c23)
 * b: device vector (this rank's slab).  Errors: LS_EINVAL for an unknown kind,
 * LS_ENOTSUP for a kind the context does not support.
 */
int ls_rhs(ls_ctx* ctx, int kind, double* b);

/*
 * pcg_solve -- preconditioned CG for A x = b with P (PAPER.md 710-712, 1109):
 * x0 = 0, stop when ||r_k||_2 <= tol ||b||_2 (recurrence residual, reading c7)
 * or after max_iter A-products.  x is overwritten (x must not alias b: LS_EINVAL).
 * b == 0 returns x = 0 with
 * 0 iterations.  Synchronous.  Returns LS_OK, LS_ENOCONV or LS_ENUMERIC (st
 * filled in all three cases; st may be NULL).  On one GPU the solve after the b.b test is
 * one CUDA-graph launch (LS_TUNE_PCG_GRAPH; cached per (b, x, tol, max_iter), dropped by
 * ls_tune).
 */
int pcg_solve(ls_ctx* ctx, const double* b, double* x, double tol, int max_iter,
              ls_pcg_stats* st);

/*
 * ls_energy_error -- the least-squares functional at u_h = sum_i x_i B_i (PAPER.md
 * 392-410): out4[0] = J = ||f - (d_t - Lap) u_h||^2_{L2(Q)} = ||f||^2 - 2 F(u_h) + A(u_h, u_h),
 * out4[1] = ||f||^2 (closed form), out4[2] = F(u_h) = b.x, out4[3] = A(u_h, u_h) = x.A x,
 * for the built-in forcing `kind` (ls_rhs).  With f = (d_t - Lap) u (kind 1, the cube's
 * manufactured u), sqrt(J) is the error ||(d_t - Lap)(u - u_h)||, equivalent to the V_0 norm
 * of Thm teo:a-priori (PAPER.md 600-610).  J is a difference of O(||f||^2) terms: it is
 * resolved down to ~1e-13 ||f||^2.  x: device vector (this rank's slab).  Synchronous.
 */
int ls_energy_error(ls_ctx* ctx, int kind, const double* x, double* out4);

/*
 * ls_error_norms -- discretisation error of u_h = sum_i x_i B_i against the exact solution
 * of a built-in benchmark, by direct space-time Gauss quadrature (p_s + 3 points per element
 * and space direction, p_t + 3 in time; reading c24), T = 1:
 *   kind 1: the cube, u = prod_k sin(pi x_k) sin t (PAPER.md 1166; ls_rhs kind 1), any d;
 *   kind 2: the quarter annulus of ls_setup_geo (d = 2), u = -(x^2+y^2-1)(x^2+y^2-4) x y^2
 *           sin(pi t) (PAPER.md 1128-1129; ls_rhs kind 2).
 * out8 (host): [0] ||e||^2_L2(Q), [1] ||d_t e||^2, [2] ||grad_x e||^2, [3] ||Lap e||^2, and
 * [4..7] the same four integrals of u (e = u - u_h, Q = Omega x (0, 1)).  Hence
 * ||e||_V0^2 = [1] + [3] (the norm of PAPER.md 318-323, Thm teo:a-priori), ||e||_L2^2 = [0],
 * and the space-time ||e||_H1^2 = [0] + [1] + [2] (Fig. 2, PAPER.md 1131-1139).  Every term
 * is a sum of non-negative quadrature contributions (no cancellation).
 * x: device vector (the whole [n_t][N_s] tensor; single-GPU contexts only).  Synchronous.
 * Errors: LS_EINVAL (null / misaligned), LS_ENOTSUP (kind without an exact solution for this
 * context: kind 1 on a mapped domain, kind 2 on the cube or d != 2, a distributed context,
 * shared-memory footprint above 200 KB, e.g. d = 3 with p_s > 7), LS_ENOMEM, LS_ECUDA.
 */
int ls_error_norms(ls_ctx* ctx, int kind, const double* x, double* out8);

/*
 * ls_geometry -- a mapped spatial domain Omega = F([0,1]^d) (PAPER.md 226-250,
 * Assumption 1; reading c19: a tensor-product NURBS map, rational when `weights`
 * is given, e.g. the exact quarter annulus / revolved quarter annulus of Sec. 5,
 * PAPER.md 1219).  Per direction k = 1..d (index k-1): degree[k-1] >= 1 and an
 * open knot vector knots[k-1] on [0,1] of n_knots[k-1] entries, so
 * m_k = n_knots - degree - 1 functions.  ctrl: host [m_1 m_2 .. m_d][d] control
 * points in colex order (direction 1 fastest); weights: host [m_1 .. m_d], all
 * > 0, or NULL for a polynomial spline map.  Copied by ls_setup_geo (caller keeps
 * ownership).  The discrete space is the push-forward of the constrained B-spline
 * basis (eq:disc_space, PAPER.md 291-300) on the uniform meshes of n_elems.
 */
typedef struct {
  int degree[3];
  int64_t n_knots[3];
  const double* knots[3];
  const double* ctrl;
  const double* weights;
} ls_geometry;

#define LS_PRECOND_P 0  /* P of eq:preconditioner (parametric, PAPER.md 733) */
#define LS_PRECOND_PG 1 /* P^G = D^{1/2} Pbar^G D^{1/2} of Sec. 4.4 (PAPER.md 969-1045) */

/*
 * ls_setup_geo -- single-GPU context on a mapped domain, T = 1.
 *   ls_matvec: y = A x with A = K_t (x) M_s + M_t (x) J_s + W_t (x) L_s (eq:A_kron,
 *     PAPER.md 686-703) and the PHYSICAL spatial factors [M_s]_ij = int_Omega B_i B_j,
 *     [L_s]_ij = int grad B_i . grad B_j, [J_s]_ij = int Lap B_i Lap B_j, assembled on the
 *     device at setup (chain rule of PAPER.md 986-990; p_s + 1 Gauss points per element
 *     and direction, reading c6) and stored per row in a (2 p_s + 1)^d stencil layout
 *     (3 (2 p_s + 1)^d N_s doubles).
 *   fd_apply: z = P^{-1} r with precond = LS_PRECOND_P (the parametric P of the cube),
 *     or z = (P^G)^{-1} r = D^{-1/2} Pbar^{-1} D^{-1/2} r with precond = LS_PRECOND_PG:
 *     c_tau, c_k at the element midpoints, separable least-squares fit of their
 *     logarithms (reading c21), factors interpolated piecewise linearly (reading c22),
 *     weighted univariate matrices, Algorithm 1 for Pbar^G, D_ii = A_ii / Pbar^G_ii.
 *   pcg_solve works unchanged; ls_matvec_slab applies slab rows (as for the cube);
 *     ls_rhs / ls_energy_error support kinds 2 (d = 2) and 3 (d = 3) only: the forcings of
 *     the paper's quarter-annulus benchmarks (PAPER.md 1128-1129, 1219-1221; see ls_rhs;
 *     spatial integrals with p_s + 5 Gauss points per element on Omega, reading c16), other
 *     kinds LS_ENOTSUP (the caller supplies b); fd_apply_stage / fd_apply_scatter LS_ENOTSUP.
 * Limits: (p_s + 1)^d <= 343 local functions per element (d = 3: p_s <= 6).
 * Errors: as ls_setup; LS_EINVAL also for an invalid map description, or a Jacobian
 * determinant that vanishes, is not finite or changes sign at a quadrature point
 * (Assumption 4, PAPER.md 238-240: F^{-1} with bounded derivatives).
 */
int ls_setup_geo(int d, int p_s, int p_t, const int64_t* n_elems, const ls_geometry* geo, int precond,
                 ls_ctx** out);

/*
 * ls_setup_geo_dist -- ls_setup_geo for rank `rank` of `world` processes (one GPU each), with
 * the time-slab layout of ls_setup_dist: every rank assembles the (spatial)
 * physical factors, ls_matvec exchanges p_t halo slices and applies the slab rows
 * (ls_matvec_slab likewise), fd_apply = D^{-1/2} (slab-local) around the distributed
 * Algorithm 1, pcg_solve all-reduces its scalars.  ls_setup_geo(...) is ls_setup_geo_dist
 * with rank 0 of 1.  Errors: as ls_setup_geo plus LS_ENCCL.
 */
int ls_setup_geo_dist(int d, int p_s, int p_t, const int64_t* n_elems, const ls_geometry* geo, int precond,
                      int rank, int world, const void* nccl_unique_id, ls_ctx** out);

/*
 * ls_pg_factors -- host only (no device work): the P^G setup of ls_setup_geo for a map and
 * spatial mesh, for inspection and CPU tests.  mu, omega: per-element univariate factors,
 * directions concatenated (sum_k n_elems[k] values each; defined up to the gauge
 * mu_j -> a_j mu_j, omega_k -> omega_k a_k / prod_j a_j of reading c21, which leaves every
 * product and Pbar^G unchanged); Mw, Jw: the weighted constrained factors M^G_k, J^G_k
 * (row-major n_k x n_k, n_k = n_elems[k] + p_s - 2, concatenated); fit_rel_res as
 * ls_geo_info.  Errors: LS_EINVAL (arguments, invalid or singular map).
 */
int ls_pg_factors(const ls_geometry* geo, int d, int p_s, const int64_t* n_elems, double* mu, double* omega,
                  double* Mw, double* Jw, double* fit_rel_res);

/*
 * ls_geo_info -- out2[0] = max relative residual of the separable fit of c_tau, c_k at
 * the element midpoints (0 for LS_PRECOND_P or an exactly separable map), out2[1] =
 * number of stencil entries per spatial row ((2 p_s + 1)^d).  Errors: LS_EINVAL,
 * LS_ENOTSUP (not a mapped-domain context).
 */
int ls_geo_info(const ls_ctx* ctx, double* out2);

/*
 * fd_apply_host -- fd_apply with HOST vectors: copies r host->device, runs
 * fd_apply, copies z device->host, synchronises.  The end-to-end entry point
 * of the public API (bench.py "e2e").  Single-GPU contexts pipeline the copies
 * over 8 time-slice chunks on a second stream (the copies overlap the spatial
 * modes); pinned host memory is needed for the overlap.
 */
int fd_apply_host(ls_ctx* ctx, const double* r_host, double* z_host);

/*
 * fd_apply_host_batch -- z_k = P^{-1} r_k (Algorithm 1, PAPER.md 955-964) for count HOST vector
 * pairs (r_host[k], z_host[k]; each the rank's local slab, pinned host memory recommended),
 * pipelined across the vectors: the host->device copy of r_{k+1} and the device->host copy of
 * z_{k-1} overlap the application to r_k (two device buffer pairs, allocated on the first call:
 * + 2 N doubles; separate copy streams).  Synchronous: returns when every z_k is on the host.
 * r_host[k] may alias r_host[j]; z_host[k] must not alias any r_host[j].
 * Errors: LS_EINVAL (null table or entry, count < 0), LS_ENOMEM, LS_ECUDA.
 */
int fd_apply_host_batch(ls_ctx* ctx, const double* const* r_host, double* const* z_host, int64_t count);

/*
 * ls_get_factor -- copy a setup quantity to host memory (introspection for
 * tests).  which: 0 = M_k, 1 = K_k, 2 = J_k (dense n_k x n_k, row-major; dir
 * = k in 1..d), 3 = M_t^ , 4 = K_t^ (n_t x n_t, dir ignored), 5 = lambda_k
 * (n_k), 6 = lambda_t (n_t), 7 = U_k (n_k x n_k row-major, column j = j-th
 * eigenvector), 8 = U_t.  Synchronous.
 */
int ls_get_factor(const ls_ctx* ctx, int which, int dir, double* host_out);

/*
 * Host-only plan queries of the time-slab decomposition; no GPU
 * and no context needed.  They are the exact functions the NCCL plumbing uses,
 * exported so the multi-rank logic can be tested on CPU.
 * ls_partition -- even split of `total` items over `world` parts (first
 *   total % world parts one larger): part `part` is [*off, *off + *len).
 *   Time slabs: total = n_t; spatial chunks of the time mode: total = N_s.
 * ls_a2a_plan -- slab -> chunk all-to-all of `rank` (counts in doubles), arrays
 *   of length world indexed by peer h: send [send_off[h], +send_cnt[h]) of the
 *   packed send buffer; receive [recv_off[h], +recv_cnt[h]) of the [n_t][chunk]
 *   tensor.  chunk -> slab is the transpose (send<->recv).
 * ls_pack_map -- pos[e] = packed send-buffer position of element e of an
 *   [ntl][N_s] slab (pos must hold ntl*N_s entries).
 * ls_halo_plan -- ls_matvec halo of `rank`: slab [*t0, *t0 + *ntl), halo rows
 *   *lo below (from rank-1) and *hi above (from rank+1), each = p or 0.
 *   LS_EINVAL if a slab is thinner than p.
 */
int ls_partition(int64_t total, int world, int part, int64_t* off, int64_t* len);
int ls_a2a_plan(int64_t n_t, int64_t N_s, int world, int rank, int64_t* send_off,
                int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt);
int ls_pack_map(int64_t ntl, int64_t N_s, int world, int64_t* pos);
/* ls_a2a_piece_plan -- piece `piece` of the pipelined slab -> chunk all-to-all of `rank`
 * (the default NCCL path of the distributed fd_apply: every slab is cut into *pieces =
 * min(4, floor(n_t / world)) runs of consecutive time slices; the spatial modes of piece c + 1
 * run while piece c is exchanged).  Arrays of length world as ls_a2a_plan; the union over the
 * pieces is ls_a2a_plan's exchange.  piece < 0 only returns *pieces. */
int ls_a2a_piece_plan(int64_t n_t, int64_t N_s, int world, int rank, int piece, int* pieces, int64_t* send_off,
                      int64_t* send_cnt, int64_t* recv_off, int64_t* recv_cnt);
int ls_halo_plan(int64_t n_t, int world, int rank, int p, int64_t* t0, int64_t* ntl,
                 int64_t* lo, int64_t* hi);
/* ls_a2a_dest -- destination of one element in the fused all-to-all (the addressing of
 * the peer-memory epilogues, LS_TUNE_A2A / fd_apply_scatter): dir 0 (slab -> chunk):
 * element (i = local time slice, j = spatial index) of rank `rank`'s slab; dir 1 (chunk ->
 * slab): element (i = time slice, j = local spatial index) of its chunk.  Returns the
 * destination rank and element offset in that rank's receive buffer ([n_t][4*ceil(len/4)]
 * chunk, resp. [ntl][N_s] slab). */
int ls_a2a_dest(int64_t n_t, int64_t N_s, int world, int rank, int dir, int64_t i, int64_t j, int* peer,
                int64_t* off);

/* ls_kernel_launches -- number of kernels the library has launched so far. */
int64_t ls_kernel_launches(const ls_ctx* ctx);

/*
 * ls_profile -- enable (1) / disable (0) per-launch CUDA-event timing of the
 * FD mode-product kernel (the dominant kernel of fd_apply).  Events are
 * recorded on the context stream around each launch.
 * ls_profile_read -- synchronise, return the summed device time [ms], the
 * summed ALGORITHMIC flops (2 n^2 per column per mode product, padding not
 * counted) and the number of launches recorded since the last read; resets.
 */
int ls_profile(ls_ctx* ctx, int enable);
int ls_profile_read(ls_ctx* ctx, double* total_ms, double* total_flops, int64_t* launches);

/*
 * ls_tune -- select among equivalent implementations (same results up to
 * rounding order, c13); for benchmarking.  Knobs:
 *   LS_TUNE_FD_KERNEL: 0 = automatic per mode extent (default),
 *                      1 = shared-memory-staged DMMA mode kernels,
 *                      2 = register-direct DMMA mode kernel.
 *   LS_TUNE_MATVEC:    0 = automatic per degree (default),
 *                      1 = four banded passes, 152 B/DOF,
 *                      2 = three fused banded passes (Toeplitz stencils), 96 B/DOF,
 *                      3 = four banded passes on the FP64 tensor pipe (DMMA),
 *                      4 = plane pass (directions 1 + 2 fused, DMMA) + direction-3 and time
 *                          DMMA passes, 96 B/DOF (d >= 2, 2 <= p_s, p_t <= 8; else LS_ENOTSUP).
 * Errors: LS_EINVAL for an unknown knob or value.
 */
#define LS_TUNE_FD_KERNEL 1
#define LS_TUNE_MATVEC 2
#define LS_TUNE_MV3_PAD 3  /* v3 matvec: direction-1 row granularity of its intermediates: 1, 8, 16 */
/* LS_TUNE_A2A (distributed contexts, d >= 2, N_1*..*N_{d-1} % 4 == 0): 0 = NCCL all-to-all
 * (default), 1 = fused all-to-all: the last forward spatial mode and the backward time mode
 * store their outputs straight into the owners' receive buffers in peer memory (CUDA IPC
 * over NVLink), each followed by a cross-GPU flag barrier.  Enabling is collective (every
 * rank calls it).  Not yet validated on a multi-GPU box. */
#define LS_TUNE_A2A 4
/* LS_TUNE_PCG_GRAPH: 1 = pcg_solve runs as one CUDA-graph launch (first iteration, a WHILE
 * conditional node around the captured iteration, true residual; no per-iteration host
 * round trip; default on one GPU), 0 = host-driven loop.  Same kernels in the same order. */
#define LS_TUNE_PCG_GRAPH 5
/* LS_TUNE_PDL (process-wide): 1 = the FD mode kernels use programmatic dependent launch
 * (their shared-memory staging of U / lambda overlaps the previous kernel's tail; default),
 * 0 = plain stream order. */
#define LS_TUNE_PDL 6
/* LS_TUNE_FD_TAIL: 1 = when n = 8 m + 1 or 8 m + 2 in an odd k-step bucket (e.g. n = 65, 66),
 * the shared-memory FD kernel computes the last one or two output rows with DFMAs instead of
 * a 7/8- or 3/4-padded DMMA m-tile (default), 0 = all rows on DMMAs, 2 = as 1 and also in the
 * centrosymmetric split kernels (process-wide; half extents 8 m + 1 or 8 m + 2: n = 65, 66, 97,
 * 98, 129 .. 132; opt-in: measured slower at config 4, 14.72 -> 16.25 ms). */
#define LS_TUNE_FD_TAIL 7
/* LS_TUNE_MV4_CTAS: process-wide; the v4 plane pass' register budget, 1 or 2 CTAs of 256
 * threads per SM (<= 255 / <= 128 registers per thread); default 2. */
#define LS_TUNE_MV4_CTAS 8
/* LS_TUNE_FD_CS: 1 = the spatial mode products of fd_apply use the centrosymmetric split
 * (default): with uniform open knots and Dirichlet conditions at both ends (PAPER.md 266-267,
 * 1111-1112) the space pencil (J_k, M_k) commutes with the index reversal R, so U_k is built
 * from even and odd eigenvectors (eq:eig_dec, PAPER.md 939-945, solved as two half-size
 * pencils at setup) and every spatial mode product is two half-size products (half the
 * flops; z = P^{-1} r is unchanged).  0 = n x n products with the same U_k.  Directions
 * whose pencil is not centrosymmetric (P^G's weighted pencils) always use n x n products.
 * The eigen index order of such a direction is [even | odd] (ls_get_factor 5 / 7). */
#define LS_TUNE_FD_CS 9
/* LS_TUNE_MV5: 1 = the v4 matvec (LS_TUNE_MATVEC 4, the automatic choice for d >= 2, p >= 3)
 * runs its direction-3 and time passes as ONE kernel (d = 3, p_s = p_t): the direction-3 results
 * stay on chip and the time band product is a register scatter; 0 = two DMMA passes through
 * HBM; 2 = automatic (default): the fused pass for p <= 4, where it measured faster. */
#define LS_TUNE_MV5 10
/* LS_TUNE_FD_STAGED (process-wide): 1 = the split spatial mode products with an even extent
 * (FAST strided or contiguous modes) run the cp.async-staged kernel (B operand ring in shared
 * memory, 1 n-tile per warp, 2 CTAs per SM), 0 = the register-window kernel (default: the
 * staged one measured 5 % slower at configs 4 and 5 p = 2, 2 % faster at p = 8). */
#define LS_TUNE_FD_STAGED 11
/* LS_TUNE_PQ_FUSE: 1 = pcg_solve forms p.q in the epilogue of ls_matvec's last pass (v4 / v5
 * paths; default), 0 = a separate dot pass. */
#define LS_TUNE_PQ_FUSE 12
/* LS_TUNE_FD_TIME: 1 = fd_apply's time mode (U_t^T, the division by lambda_t + Lambda_s of
 * Algorithm 1 step 3, U_t; PAPER.md 947-962) runs as ONE kernel whose intermediate stays in
 * registers (default; every supported n_t <= 136); 0 = two launches (the scaled forward product
 * into a workspace, then the backward product). */
#define LS_TUNE_FD_TIME 13
/* LS_TUNE_FD_PLANE: 1 = fd_apply's spatial mode products of directions 1 and 2 run as ONE
 * kernel per (i_3, .., t) plane whose intermediate stays in registers, where both directions
 * use the centrosymmetric split (LS_TUNE_FD_CS) with n_1 = n_2 <= 104; 0 = one launch per
 * direction (default: the plane kernel measured 5-10 % slower at BASELINE configs 3 and 5). */
#define LS_TUNE_FD_PLANE 14
/* LS_TUNE_MV6: the v4 matvec's direction-3 and time passes (after its DMMA plane pass) as
 * streaming DFMA Toeplitz-stencil passes (exactly 2p + 1 multiply-adds per banded output, no
 * band-tile padding) instead of DMMA band tiles: 0 = off (default: latency-bound, measured
 * slower at configs 4 and 5), 1 = on (the v5 fused pass, where it applies, takes precedence). */
#define LS_TUNE_MV6 15
/* LS_TUNE_MV2_SWEEP: the v2 matvec's (p_s = 2) d = 3 plane pass of directions 2 + 1 as a
 * register sweep (one warp per plane, no shared memory or barriers; n_1 <= 128; default 1) or
 * as the shared-memory two-phase kernel (0). */
#define LS_TUNE_MV2_SWEEP 16
/* LS_TUNE_MV4_SWEEP: the v4 matvec's plane pass (directions 1 + 2) as a DFMA register sweep
 * (one warp per plane, Toeplitz stencils; d = 3, p_s = 3 or 4, n_1 <= 128) (1) or as the DMMA
 * band-tile kernel (0, default: the sweep measured 2.2x slower at config 5 p = 4). */
#define LS_TUNE_MV4_SWEEP 17
int ls_tune(ls_ctx* ctx, int knob, int value);

void ls_destroy(ls_ctx* ctx);
const char* ls_strerror(int code);

#ifdef __cplusplus
}
#endif

#endif /* LS_API_H */
